// dev_patches.cuh — decompose_patches (reference contact_field.cpp:26-99) on
// the GPU, the host bottleneck of build_field for dense hands (SURVEY 8(f)
// rank 3).
//
// The greedy cover is sequential in its decisions (each patch's seed is the
// pick-th still-uncovered sample, drawn from stream 'patc'), so one CTA owns
// one link and runs the reference's loop; what is parallel is the work inside
// an iteration: the distance test of every uncovered sample and the stable
// split of the uncovered list into members / rest (one block-wide scan per
// 1024 samples), which keeps both lists in ascending sample order exactly as
// the reference's std::vector walk does.  Field-point subsets (stream 'subs',
// keyed by the global patch id) run afterwards, thread per patch.
#pragma once

#include "dev_geom.cuh"

namespace lgd {

constexpr int kCoverThreads = 1024;

// seg b covers samples [off[b], off[b+1]) of one link.  Outputs per segment:
// members[off[b] ..] = sample ids (segment-local) in patch order (seed first,
// then ascending), pstart[off[b] + k] = start of patch k in that list,
// npatch[b] = patch count.
__global__ void __launch_bounds__(kCoverThreads)
k_patch_cover(int nseg, const int* seg_link, const long long* off, const double* pos,
              double gather, uint64_t seed, int* unc_a, int* unc_b, int* members, int* pstart,
              int* npatch) {
  typedef cub::BlockScan<int, kCoverThreads> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_sid, s_tot;
  __shared__ double s_c[3];
  const int b = blockIdx.x;
  if (b >= nseg) return;
  const long long base = off[b];
  const int N = (int)(off[b + 1] - base);
  const double* P = pos + 3 * base;
  int* A = unc_a + base;
  int* B = unc_b + base;
  for (int i = threadIdx.x; i < N; i += blockDim.x) A[i] = i;
  DRng rng;
  if (threadIdx.x == 0) rng.seed(mix_seed(seed, 0x70617463ull, (uint64_t)seg_link[b]));  // 'patc'
  __syncthreads();
  int U = N, w = 0, k = 0;
  while (U > 0) {
    if (threadIdx.x == 0) {
      int sid = A[rng.index((uint64_t)U)];
      s_sid = sid;
      s_c[0] = P[3 * sid];
      s_c[1] = P[3 * sid + 1];
      s_c[2] = P[3 * sid + 2];
      pstart[base + k] = w;
      members[base + w] = sid;
    }
    __syncthreads();
    const int sid = s_sid;
    const V3 c = v3(s_c[0], s_c[1], s_c[2]);
    int mcount = 1, rcount = 0;
    for (int c0 = 0; c0 < U; c0 += blockDim.x) {
      const int i = c0 + threadIdx.x;
      int id = i < U ? A[i] : -1;
      int flag = 0;
      if (id >= 0 && id != sid) {
        V3 p = v3(P[3 * id], P[3 * id + 1], P[3 * id + 2]);
        flag = norm(sub(p, c)) <= gather ? 1 : (1 << 16);  // member : rest
      }
      int pos_, tot;
      Scan(tmp).ExclusiveSum(flag, pos_, tot);
      if (flag == 1) members[base + w + mcount + (pos_ & 0xffff)] = id;
      else if (flag) B[rcount + (pos_ >> 16)] = id;
      mcount += tot & 0xffff;
      rcount += tot >> 16;
      __syncthreads();  // TempStorage reuse
    }
    w += mcount;
    ++k;
    U = rcount;
    int* t = A;
    A = B;
    B = t;
    __syncthreads();
  }
  if (threadIdx.x == 0) npatch[b] = k;
}

// Field points of patch t (global id gid[t], m members): all when m <= cap,
// else member 0 plus cap - 1 draws of a partial Fisher-Yates over 1..m-1
// (stream 'subs', contact_field.cpp:80-93), sorted.  The pool is virtual:
// only the <= cap - 1 swapped slots are stored.
__global__ void k_patch_fields(int np, const int* gid, const int* msize, const int* fp_off, int cap,
                               uint64_t seed, int* fps) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= np) return;
  const int m = msize[t];
  int* out = fps + fp_off[t];
  if (m <= cap) {
    for (int i = 0; i < m; ++i) out[i] = i;
    return;
  }
  int key[16], val[16], nk = 0;  // pool[key] = val for swapped slots
  auto get = [&](int s) {
    for (int q = 0; q < nk; ++q)
      if (key[q] == s) return val[q];
    return s + 1;  // pool[i] = i + 1 initially
  };
  auto put = [&](int s, int v) {
    for (int q = 0; q < nk; ++q)
      if (key[q] == s) {
        val[q] = v;
        return;
      }
    key[nk] = s;
    val[nk] = v;
    ++nk;
  };
  DRng sr;
  sr.seed(mix_seed(seed, 0x73756273ull, (uint64_t)gid[t]));  // 'subs'
  const int pool = m - 1;
  int cnt = 0;
  out[cnt++] = 0;
  for (int i = 0; i < cap - 1; ++i) {
    int j = i + (int)sr.index((uint64_t)(pool - i));
    int vi = get(i), vj = get(j);
    put(i, vj);
    put(j, vi);
    out[cnt++] = vj;
  }
  for (int a = 1; a < cnt; ++a)  // insertion sort (cap <= 16)
    for (int b2 = a; b2 > 0 && out[b2 - 1] > out[b2]; --b2) {
      int x = out[b2];
      out[b2] = out[b2 - 1];
      out[b2 - 1] = x;
    }
}

}  // namespace lgd
