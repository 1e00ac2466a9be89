// ASan/UBSan run: the reference (shimmed) and the oracle restatement on cfg1.
#include "lg.h"
#include <cstdio>
#include <cstring>
struct ref_inputs; struct ref_result; struct orc_result;
extern "C" {
int ref_prepare(const char*, const char*, const char*, const char*, const char*, long long, int, int, ref_inputs**);
int ref_params(const ref_inputs*, lg_run_params*);
int ref_hand_desc(const ref_inputs*, lg_hand_desc*);
int ref_patches_desc(const ref_inputs*, lg_patches_desc*);
int ref_raw_samples(const ref_inputs*, const double**, int*);
int ref_run_batch(const ref_inputs*, ref_result**);
long long ref_result_num_grasps(const ref_result*);
const lg_grasp* ref_result_grasps(const ref_result*);
int orc_run_batch(const lg_hand_desc*, const lg_patches_desc*, const double*, int, const lg_run_params*, int, orc_result**);
long long orc_result_num_grasps(const orc_result*);
const lg_grasp* orc_result_grasps(const orc_result*);
}
int main(int argc, char** argv) {
  const char* A = "/root/repo/assets";
  char cfg[256], hand[256], obj[256];
  snprintf(cfg, 256, "%s/configs/%s", A, argv[1]); snprintf(hand, 256, "%s/hands/%s", A, argv[2]); snprintf(obj, 256, "%s/objects/%s", A, argv[3]);
  ref_inputs* in = nullptr;
  if (ref_prepare(cfg, "passes = 2", hand, obj, "/tmp/san_out", -1, 48, 4, &in)) return 2;
  lg_run_params p; lg_hand_desc h; lg_patches_desc pd; const double* raw; int n;
  ref_params(in, &p); ref_hand_desc(in, &h); ref_patches_desc(in, &pd); ref_raw_samples(in, &raw, &n);
  ref_result* rr = nullptr; ref_run_batch(in, &rr);
  orc_result* orr = nullptr; if (orc_run_batch(&h, &pd, raw, n, &p, 4, &orr)) return 3;
  long long a = ref_result_num_grasps(rr), b = orc_result_num_grasps(orr);
  int same = a == b;
  for (long long i = 0; same && i < a; ++i) same = !memcmp(ref_result_grasps(rr)[i].q, orc_result_grasps(orr)[i].q, sizeof(double) * 32);
  printf("%s: ref %lld grasps, oracle %lld grasps, identical=%d\n", argv[2], a, b, same);
  return same ? 0 : 1;
}
