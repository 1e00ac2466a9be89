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

// sample_surface (mesh.cpp:297-339) for many meshes at once.  Each sample
// takes exactly three draws (face, u, v) of its mesh's stream, so one thread
// per mesh writes the stream and one thread per sample builds the point:
// face by lower_bound on the cumulative areas, the same corner arithmetic.
struct SampleSeg {
  long long tri0, s0;  // first triangle (corners [t][9], normals [t][3], cum [t]) / sample
  int ntri, count;
  uint64_t seed;
};

__global__ void k_sample_draws(int nseg, const SampleSeg* seg, uint64_t* draws) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nseg) return;
  DRng rng;
  rng.seed(seg[b].seed);
  uint64_t* o = draws + 3 * seg[b].s0;
  for (long long i = 0; i < 3ll * seg[b].count; ++i) o[i] = rng.u64();
}

__global__ void k_sample_points(long long n, int nseg, const SampleSeg* seg, const long long* sample_seg_start,
                                const double* corners, const double* fnrm, const double* cum,
                                const uint64_t* draws, double* pos, double* nrm) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;  // segment of sample i
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (sample_seg_start[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const SampleSeg S = seg[lo];
    const uint64_t* d = draws + 3 * i;
    const double* c = cum + S.tri0;
    const double pick = u01(d[0]) * c[S.ntri - 1];
    int a = 0, z = S.ntri;  // lower_bound: first cum >= pick
    while (a < z) {
      int m = (a + z) >> 1;
      if (c[m] < pick) a = m + 1;
      else z = m;
    }
    const int t = a < S.ntri ? a : S.ntri - 1;
    double u = u01(d[1]), v = u01(d[2]);
    if (u + v > 1.0) {
      u = 1.0 - u;
      v = 1.0 - v;
    }
    const double* q = corners + 9 * (S.tri0 + t);
    V3 A = v3(q[0], q[1], q[2]), B = v3(q[3], q[4], q[5]), Cc = v3(q[6], q[7], q[8]);
    v3_store(pos + 3 * i, axpy(axpy(A, u, sub(B, A)), v, sub(Cc, A)));
    v3_store(nrm + 3 * i, v3_load(fnrm + 3 * (S.tri0 + t)));
  }
}

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
  __shared__ int s_sid;
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
  int key[32], val[32], nk = 0;  // pool[key] = val for swapped slots (<= 2 (cap - 1))
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
