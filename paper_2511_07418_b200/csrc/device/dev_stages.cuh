// dev_stages.cuh — the per-candidate stages of run_batch
// (reference pipeline.cpp:384-615) as batched sm_100a kernels.
#pragma once

#include <cub/cub.cuh>

#include "dev_field.cuh"
#include "dev_ikw.cuh"

namespace lgd {

// RNG stream tags (pipeline.cpp:19-25)
constexpr uint64_t kTagPlacement = 0x706c6163;
constexpr uint64_t kTagGroups = 0x67727073;
constexpr uint64_t kTagContactOpt = 0x636f7074;
constexpr uint64_t kTagReverse = 0x72657673;
constexpr uint64_t kTagUnused = 0x756e7573;

// Object samples as SoA (x, y, z, nx, ny, nz).
struct DSamples {
  int n;
  const double* x[6];
  __device__ __forceinline__ V3 p(int i) const { return v3(x[0][i], x[1][i], x[2][i]); }
  __device__ __forceinline__ V3 nrm(int i) const { return v3(x[3][i], x[4][i], x[5][i]); }
};

__device__ __forceinline__ Xf load_xf(const double* p) {
  Xf x;
  x.R = m3_load(p);
  x.t = v3_load(p + 9);
  return x;
}
__device__ __forceinline__ void store_xf(double* p, const Xf& x) {
  m3_store(p, x.R);
  v3_store(p + 9, x.t);
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = dmax(v, u);
  }
  return v;
}

// Block-wide max of a double (blockDim multiple of 32, <= 1024).
__device__ __forceinline__ double block_max(double v, double* scratch) {
  v = warp_max(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    int nw = (blockDim.x + 31) >> 5;
    v = l < nw ? scratch[l] : -kInf;
    v = warp_max(v);
    if (l == 0) scratch[0] = v;
  }
  __syncthreads();
  double r = scratch[0];
  __syncthreads();
  return r;
}

// Samples [n_src][6] (position, normal) -> SoA columns out[a][n], rows
// idx[t] (all rows when idx is null).
__global__ void k_soa_gather(int n, const double* rows, const int* idx, double* out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const size_t src = idx ? (size_t)idx[t] : (size_t)t;
#pragma unroll
    for (int a = 0; a < 6; ++a) out[(size_t)a * n + t] = rows[6 * src + a];
  }
}

// --------------------------------------------------- object sample grid
// Uniform grid over object-frame samples: cell width w from origin lo, the
// sample ids sorted by cell (ascending inside a cell), per-cell offsets and
// the samples in cell order (SoA).  It only decides which samples a test
// visits: a region test (an axis box in the object frame) visits every cell
// the box touches, widened by w 2^-20, far more than the rounding of any
// coordinate involved, so no sample that can pass is skipped; the test on a
// visited sample is the reference's, unchanged.  Cells along x are
// contiguous in the order, so each (y, z) row of a box is one sample range.
struct DGrid {
  int ok;
  double lo[3], w;
  int dim[3];
  const int* start;    // [cells + 1]
  const int* id;       // [n] sample id in cell order
  const double* x[6];  // samples in cell order (position, normal)
};

__device__ __forceinline__ int grid_cell(const DGrid& g, int a, double v) {
  const double f = floor((v - g.lo[a]) / g.w);
  if (!(f > 0.0)) return 0;  // below the grid, or NaN
  return f >= (double)(g.dim[a] - 1) ? g.dim[a] - 1 : (int)f;
}

__global__ void k_grid_keys(DSamples s, DGrid g, unsigned* keys, int* vals, int* cnt) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < s.n; j += gridDim.x * blockDim.x) {
    const V3 p = s.p(j);
    const unsigned c = (unsigned)((grid_cell(g, 2, p.z) * g.dim[1] + grid_cell(g, 1, p.y)) * g.dim[0] +
                                  grid_cell(g, 0, p.x));
    keys[j] = c;
    vals[j] = j;
    atomicAdd(cnt + c, 1);
  }
}

__global__ void k_grid_gather(DSamples s, const int* id, DGrid g) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < s.n; t += gridDim.x * blockDim.x) {
    const int j = id[t];
    for (int a = 0; a < 6; ++a) const_cast<double*>(g.x[a])[t] = s.x[a][j];
  }
}

// preprocess_object (pipeline.cpp:71-98) through the grid: the j loop visits
// the cells of the probe cube [c - h, c + h] only (any j outside it fails the
// reference's |d| > h test); blocked is an existential, so the visit order
// does not matter.
__global__ void k_preprocess_grid(DSamples s, DGrid g, double h, double d, uint8_t* keep) {
  // threads take the samples in cell order, so a warp's probe cubes overlap
  // and their row loads hit L1
  const int ti = blockIdx.x * blockDim.x + threadIdx.x;
  if (ti >= s.n) return;
  const int i = g.id[ti];
  const V3 ni = s.nrm(i);
  const V3 c = axpy(s.p(i), d, ni);
  const double m = g.w * 0x1p-20;
  const int x0 = grid_cell(g, 0, c.x - h - m), x1 = grid_cell(g, 0, c.x + h + m);
  const int y0 = grid_cell(g, 1, c.y - h - m), y1 = grid_cell(g, 1, c.y + h + m);
  const int z0 = grid_cell(g, 2, c.z - h - m), z1 = grid_cell(g, 2, c.z + h + m);
  bool blocked = false;
  for (int z = z0; z <= z1 && !blocked; ++z)
    for (int y = y0; y <= y1 && !blocked; ++y) {
      const int row = (z * g.dim[1] + y) * g.dim[0];
      const int t1 = g.start[row + x1 + 1];
      for (int t = g.start[row + x0]; t < t1; ++t) {
        if (g.id[t] == i) continue;
        const V3 dd = sub(v3(g.x[0][t], g.x[1][t], g.x[2][t]), c);
        if (dabs(dd.x) > h || dabs(dd.y) > h || dabs(dd.z) > h) continue;
        if (dot(v3(g.x[3][t], g.x[4][t], g.x[5][t]), ni) < 0.0) {
          blocked = true;
          break;
        }
      }
    }
  keep[i] = blocked ? 0 : 1;
}

// -------------------------------------------------------- preprocess_object
// pipeline.cpp:71-98: sample i is dropped when some j != i lies inside the
// axis cube of half width h around p_i + d n_i and n_j . n_i < 0.  The
// j loop is staged through shared memory one block-width tile at a time.
__global__ void k_preprocess(DSamples s, double h, double d, uint8_t* keep) {
  __shared__ double t[6][256];
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool active = i < s.n;
  V3 c = v3(0, 0, 0), ni = v3(0, 0, 0);
  if (active) {
    ni = s.nrm(i);
    c = axpy(s.p(i), d, ni);
  }
  bool blocked = false;
  for (int base = 0; base < s.n; base += blockDim.x) {
    int j = base + threadIdx.x;
    __syncthreads();
    if (j < s.n)
      for (int a = 0; a < 6; ++a) t[a][threadIdx.x] = s.x[a][j];
    __syncthreads();
    int m = min((int)blockDim.x, s.n - base);
    if (active && !blocked) {
      for (int jj = 0; jj < m; ++jj) {
        if (base + jj == i) continue;
        V3 dd = sub(v3(t[0][jj], t[1][jj], t[2][jj]), c);
        if (dabs(dd.x) > h || dabs(dd.y) > h || dabs(dd.z) > h) continue;
        if (dot(v3(t[3][jj], t[4][jj], t[5][jj]), ni) < 0.0) {
          blocked = true;
          break;
        }
      }
    }
  }
  if (active) keep[i] = blocked ? 0 : 1;
}

// ------------------------------------------------- collect_static_surface
// pipeline.cpp:100-120: FK at mid_config, static parts posed, static patch
// samples in base frame.
__global__ void k_statics(int n_pts, const int* pt_idx, const int* pt_link, const double* pts,
                          const double* nrm, int n_sp, const int* sp_link, double* ss_p,
                          double* ss_n, double* sp_pose) {
  __shared__ double fr[kMaxLinks * 12];
  if (threadIdx.x == 0) {
    Xf f[kMaxLinks];
    fk(c_hand.mid, f);
    for (int l = 0; l < c_hand.n_links; ++l) store_xf(fr + 12 * l, f[l]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_sp; i += blockDim.x)
    for (int a = 0; a < 12; ++a) sp_pose[12 * i + a] = fr[12 * sp_link[i] + a];
  for (int i = threadIdx.x; i < n_pts; i += blockDim.x) {
    Xf f = load_xf(fr + 12 * pt_link[i]);
    int p = pt_idx[i];
    v3_store(ss_p + 3 * i, xf_apply(f, v3_load(pts + 3 * p)));
    v3_store(ss_n + 3 * i, xf_rotate(f, v3_load(nrm + 3 * p)));
  }
}

// ------------------------------------------------------------ place_object
struct PlaceCfg {
  uint64_t seed;
  int c_lo, Bl, mode;
  double static_prob, margin;
  double center[3], half[3];
  int n_ss;
  const double* ss_p;
  const double* ss_n;
  const int* ss_link;
  int P;
  const int* patch_link;
  const int* point_off;
  const int* fp_off;
  const int* fps;
  const double* pts;
  const double* nrm;
};

// pipeline.cpp:122-172: the pose draw, one thread per candidate.
__global__ void k_place_pose(PlaceCfg C, DSamples fs, double* pose, int* n_static, int* st_link,
                             double* st_p, double* st_n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.Bl) return;
  int c = C.c_lo + i;
  DRng rng;
  rng.seed(mix_seed(C.seed, kTagPlacement, (uint64_t)c));
  bool want_static = rng.uniform() < C.static_prob;
  int oi = (int)rng.index((uint64_t)fs.n);
  V3 osp = fs.p(oi), osn = fs.nrm(oi);
  Xf x;
  n_static[i] = 0;
  st_link[i] = -1;
  if (want_static && C.n_ss > 0) {
    int si = (int)rng.index((uint64_t)C.n_ss);
    V3 sp = v3_load(C.ss_p + 3 * si), sn = v3_load(C.ss_n + 3 * si);
    double roll = rng.uniform(0.0, 2.0 * kPi);
    M3 r = mul(angle_axis(roll, sn), rotation_between(osn, neg(sn)));
    x.R = r;
    x.t = sub(sp, mul(r, osp));
    n_static[i] = 1;
    st_link[i] = C.ss_link[si];
    v3_store(st_p + 3 * i, sp);
    v3_store(st_n + 3 * i, sn);
  } else if (C.mode == 0) {
    int P = (int)rng.index((uint64_t)C.P);
    int nfp = C.fp_off[P + 1] - C.fp_off[P];
    int fp = C.fps[C.fp_off[P] + (int)rng.index((uint64_t)nfp)];
    double q[kMaxDof];
    for (int j = 0; j < c_hand.dof; ++j) q[j] = rng.uniform(c_hand.jlo[j], c_hand.jhi[j]);
    Xf fr[kMaxLinks];
    fk(q, fr);
    int link = C.patch_link[P];
    int pi = C.point_off[P] + fp;
    V3 xp = xf_apply(fr[link], v3_load(C.pts + 3 * pi));
    V3 m = xf_rotate(fr[link], v3_load(C.nrm + 3 * pi));
    double roll = rng.uniform(0.0, 2.0 * kPi);
    M3 r = mul(angle_axis(roll, m), rotation_between(osn, neg(m)));
    x.R = r;
    x.t = sub(xp, mul(r, osp));
  } else {
    double t[3] = {C.center[0], C.center[1], C.center[2]};
    for (int a = 0; a < 3; ++a) t[a] += rng.uniform(-C.half[a], C.half[a]);
    double w, qx, qy, qz;
    rng.quaternion(&w, &qx, &qy, &qz);
    x.R = quat_to_matrix(w, qx, qy, qz);
    x.t = v3(t[0], t[1], t[2]);
  }
  store_xf(pose + 12 * i, x);
}

// pipeline.cpp:174-182 + object_penetration (collision.cpp:209-228) against
// every static part: block per candidate, threads over samples, max-reduce
// (max is order independent, so the verdict and depth are exact).
__global__ void k_place_verdict(int Bl, DSamples fs, const double* pose, int n_sp,
                                const int* sp_part, const double* sp_pose, double margin,
                                int* accepted, double* penetration) {
  __shared__ double scratch[32];
  int i = blockIdx.x;
  if (i >= Bl) return;
  Xf x = load_xf(pose + 12 * i);
  double pen = 0.0;
  for (int s = 0; s < n_sp; ++s) {
    int part = sp_part[s];
    Xf inv = xf_inverse(load_xf(sp_pose + 12 * s));
    const double* b = c_hand.bounds + 6 * part;
    double mx = 0.0;
    for (int j = threadIdx.x; j < fs.n; j += blockDim.x) {
      V3 local = xf_apply(inv, xf_apply(x, fs.p(j)));
      if (!(local.x >= b[0] - 1e-9 && local.y >= b[1] - 1e-9 && local.z >= b[2] - 1e-9 &&
            local.x <= b[3] + 1e-9 && local.y <= b[4] + 1e-9 && local.z <= b[5] + 1e-9))
        continue;
      double depth = part_interior_depth(part, local);
      if (depth > margin) mx = dmax(mx, depth);
    }
    mx = block_max(mx, scratch);
    pen = dmax(pen, mx);
  }
  if (threadIdx.x == 0) {
    penetration[i] = pen;
    accepted[i] = pen <= margin ? 1 : 0;
  }
}

// ---------------------------------------------------------- query_domains
// contact_field.cpp:380-448 for accepted candidates: block per candidate,
// threads over field samples; writes the reachability mask (bit g: sample
// is an element of group g's domain) and the per-group domain sizes.
__global__ void k_query(int Bl, DField f, const int* group_of_patch, DSamples fs,
                        const double* pose, const int* accepted, double theta, int G,
                        int cb_in_smem, uint32_t* mask, int* dom_count) {
  extern __shared__ double s_cb[];
  __shared__ int s_cnt[LG_MAX_GROUPS];
  int i = blockIdx.x;
  if (i >= Bl) return;
  uint32_t* m = mask + (size_t)i * fs.n;
  if (!accepted[i]) {
    for (int j = threadIdx.x; j < fs.n; j += blockDim.x) m[j] = 0u;
    for (int g = threadIdx.x; g < G; g += blockDim.x) dom_count[i * G + g] = 0;
    return;
  }
  if (cb_in_smem)
    for (int a = threadIdx.x; a < 3 * f.C; a += blockDim.x) s_cb[a] = f.codebook[a];
  for (int g = threadIdx.x; g < LG_MAX_GROUPS; g += blockDim.x) s_cnt[g] = 0;
  __syncthreads();
  const double* cb = cb_in_smem ? s_cb : f.codebook;
  Xf x = load_xf(pose + 12 * i);
  for (int j = threadIdx.x; j < fs.n; j += blockDim.x) {
    V3 p = xf_apply(x, fs.p(j));
    V3 n = xf_rotate(x, fs.nrm(j));
    uint32_t bits = sample_mask(f, cb, group_of_patch, p, n, theta);
    m[j] = bits;
    while (bits) {
      int g = __ffs(bits) - 1;
      bits &= bits - 1;
      atomicAdd(&s_cnt[g], 1);
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) dom_count[i * G + g] = s_cnt[g];
}

// Load-balanced query over the dense cell grid: a warp takes 32 samples,
// prefix-sums their per-cell box counts and spreads the (sample, box) items
// evenly over its lanes; a hit ORs the box's group bit into the sample's
// mask (OR is order independent, so the mask equals the per-sample scan).
__global__ void __launch_bounds__(256)
k_query2(int Bl, DField f, DSamples fs, const double* pose, const int* accepted, double theta,
         int G, int cb_in_smem, uint32_t* mask, int* dom_count) {
  extern __shared__ double s_cb[];
  __shared__ int s_cnt[LG_MAX_GROUPS];
  __shared__ int s_ex[8][33];
  __shared__ int s_st[8][32];
  __shared__ double s_n[8][32][3];
  __shared__ unsigned s_bits[8][32];
  const int i = blockIdx.x;
  if (i >= Bl) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* m = mask + (size_t)i * fs.n;
  if (!accepted[i]) {
    for (int j = threadIdx.x; j < fs.n; j += blockDim.x) m[j] = 0u;
    for (int g = threadIdx.x; g < G; g += blockDim.x) dom_count[i * G + g] = 0;
    return;
  }
  if (cb_in_smem)
    for (int a = threadIdx.x; a < 3 * f.C; a += blockDim.x) s_cb[a] = f.codebook[a];
  for (int g = threadIdx.x; g < LG_MAX_GROUPS; g += blockDim.x) s_cnt[g] = 0;
  __syncthreads();
  const double* cb = cb_in_smem ? s_cb : f.codebook;
  const Xf x = load_xf(pose + 12 * i);
  for (int base = warp * 32; base < fs.n; base += nw * 32) {
    const int j = base + lane;
    int start = 0, count = 0;
    if (j < fs.n) {
      V3 p = xf_apply(x, fs.p(j));
      V3 n = xf_rotate(x, fs.nrm(j));
      s_n[warp][lane][0] = n.x;
      s_n[warp][lane][1] = n.y;
      s_n[warp][lane][2] = n.z;
      long long c[3];
      cell_of(p, f.w, c);
      long long cx = c[0] - f.gbase[0], cy = c[1] - f.gbase[1], cz = c[2] - f.gbase[2];
      if (cx >= 0 && cy >= 0 && cz >= 0 && cx < f.gdim[0] && cy < f.gdim[1] && cz < f.gdim[2]) {
        int2 se = f.grid[(cx * f.gdim[1] + cy) * f.gdim[2] + cz];
        start = se.x;
        count = se.y;
      }
    }
    int incl = count;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    s_ex[warp][lane] = incl - count;
    if (lane == 31) s_ex[warp][32] = incl;
    s_st[warp][lane] = start;
    s_bits[warp][lane] = 0u;
    __syncwarp();
    for (int it = lane; it < total; it += 32) {
      int lo = 0, hi = 31;  // owner = last lane with ex <= it
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (s_ex[warp][mid] <= it) lo = mid;
        else hi = mid - 1;
      }
      int4 r = f.rec[s_st[warp][lo] + (it - s_ex[warp][lo])];
      if (r.x < 0) continue;
      V3 n = v3(s_n[warp][lo][0], s_n[warp][lo][1], s_n[warp][lo][2]);
      for (int q = r.y; q < r.y + r.z; ++q) {
        int code = f.codes[q];
        if (-dot(v3(cb[3 * code], cb[3 * code + 1], cb[3 * code + 2]), n) >= theta) {
          atomicOr(&s_bits[warp][lo], 1u << r.x);
          break;
        }
      }
    }
    __syncwarp();
    if (j < fs.n) {
      uint32_t bits = s_bits[warp][lane];
      m[j] = bits;
      while (bits) {
        int g = __ffs(bits) - 1;
        bits &= bits - 1;
        atomicAdd(&s_cnt[g], 1);
      }
    }
    __syncwarp();
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) dom_count[i * G + g] = s_cnt[g];
}

// Code-major query (sample_mask_cm): block per candidate, thread per field
// sample; a sample costs one grid read plus ~10 code tests.
__global__ void __launch_bounds__(256)
k_query3(int Bl, DField f, DSamples fs, const double* pose, const int* accepted, double theta,
         int G, int cb_in_smem, uint32_t* mask, int* dom_count) {
  extern __shared__ double s_cb[];
  __shared__ int s_cnt[LG_MAX_GROUPS];
  const int i = blockIdx.x;
  if (i >= Bl) return;
  uint32_t* m = mask + (size_t)i * fs.n;
  if (!accepted[i]) {
    for (int j = threadIdx.x; j < fs.n; j += blockDim.x) m[j] = 0u;
    for (int g = threadIdx.x; g < G; g += blockDim.x) dom_count[i * G + g] = 0;
    return;
  }
  if (cb_in_smem)
    for (int a = threadIdx.x; a < 3 * f.C; a += blockDim.x) s_cb[a] = f.codebook[a];
  for (int g = threadIdx.x; g < LG_MAX_GROUPS; g += blockDim.x) s_cnt[g] = 0;
  __syncthreads();
  const Xf x = load_xf(pose + 12 * i);
  for (int j = threadIdx.x; j < fs.n; j += blockDim.x) {
    V3 p = xf_apply(x, fs.p(j));
    V3 n = xf_rotate(x, fs.nrm(j));
    uint32_t bits = cb_in_smem ? sample_mask_cm(f, s_cb, p, n, theta)
                               : sample_mask_cm(f, f.codebook, p, n, theta);
    m[j] = bits;
    while (bits) {
      int g = __ffs(bits) - 1;
      bits &= bits - 1;
      atomicAdd(&s_cnt[g], 1);
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) dom_count[i * G + g] = s_cnt[g];
}

// Element scores of query_domains (contact_field.cpp:412-445) for
// lg_query_domains_batch's optional output: per (pose, sample) the max over
// the sample's domain elements of their score = max over hit boxes of the
// box's best code score (0 without a hit).  Maxima are order independent.
__global__ void k_query_scores(int m, DField f, const int* group_of_patch, DSamples fs,
                               const double* pose, double theta, double* scores) {
  const int i = blockIdx.x;
  if (i >= m) return;
  const Xf x = load_xf(pose + 12 * i);
  for (int j = threadIdx.x; j < fs.n; j += blockDim.x) {
    V3 p = xf_apply(x, fs.p(j));
    V3 n = xf_rotate(x, fs.nrm(j));
    long long c[3];
    cell_of(p, f.w, c);
    int r = find_run(f, c);
    double sc = 0.0;
    if (r >= 0)
      for (int t = f.run_start[r]; t < f.run_start[r] + f.run_count[r]; ++t) {
        int b = f.cell_box[t];
        if (group_of_patch[f.box_patch[b]] < 0) continue;
        double best = -2.0;
        for (long long q = f.box_code_off[b]; q < f.box_code_off[b + 1]; ++q) {
          int code = f.codes[q];
          best = dmax(best, -dot(v3(f.codebook[3 * code], f.codebook[3 * code + 1],
                                    f.codebook[3 * code + 2]), n));
        }
        if (best >= theta) sc = dmax(sc, best);
      }
    scores[(size_t)i * fs.n + j] = sc;
  }
}

// Per-candidate world AABB of the raw object samples (the broad-phase
// object box of validate_grasp_collisions, collision.cpp:243-245).
__global__ void k_obj_aabb(int Bl, DSamples raw, const double* pose, const int* accepted,
                           double* aabb) {
  __shared__ double scratch[32];
  int i = blockIdx.x;
  if (i >= Bl || !accepted[i]) return;
  Xf x = load_xf(pose + 12 * i);
  double mn[3] = {kInf, kInf, kInf}, mx[3] = {-kInf, -kInf, -kInf};
  for (int j = threadIdx.x; j < raw.n; j += blockDim.x) {
    V3 w = xf_apply(x, raw.p(j));
    mn[0] = dmin(mn[0], w.x);
    mn[1] = dmin(mn[1], w.y);
    mn[2] = dmin(mn[2], w.z);
    mx[0] = dmax(mx[0], w.x);
    mx[1] = dmax(mx[1], w.y);
    mx[2] = dmax(mx[2], w.z);
  }
  for (int a = 0; a < 3; ++a) {
    double lo = -block_max(-mn[a], scratch);
    double hi = block_max(mx[a], scratch);
    if (threadIdx.x == 0) {
      aabb[6 * i + a] = lo;
      aabb[6 * i + 3 + a] = hi;
    }
  }
}

// ---------------------------------------------------------------- group pick
// pipeline.cpp:421-438.
__global__ void k_group_pick(int Bl, int c_lo, int B, int pass, uint64_t seed, int k, int G,
                             const int* accepted, const int* dom_count, int* alive,
                             int* chosen) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Bl) return;
  alive[i] = 0;
  if (!accepted[i]) return;
  int nonempty[LG_MAX_GROUPS];
  int n = 0;
  for (int g = 0; g < G; ++g)
    if (dom_count[i * G + g] > 0) nonempty[n++] = g;
  if (n < k) return;
  uint64_t gid = (uint64_t)pass * B + (uint64_t)(c_lo + i);
  DRng rng;
  rng.seed(mix_seed(seed, kTagGroups, gid));
  for (int pick = 0; pick < k; ++pick) {
    int j = pick + (int)rng.index((uint64_t)(n - pick));
    int t = nonempty[pick];
    nonempty[pick] = nonempty[j];
    nonempty[j] = t;
  }
  for (int q = 0; q < k; ++q) chosen[i * kMaxK + q] = nonempty[q];
  alive[i] = 1;
}

// Domain element data: the materialised arrays (p, n: [e][3]), or — for
// large domains, which skip them — recomputed from the element's sample id
// and the candidate's pose with k_domain_fill's own arithmetic (the same
// bits).  a = alive index of the element's candidate.
struct ElemSrc {
  const double* p;
  const double* n;
  const int* s;
  DSamples fs;
  const double* pose;
  const int* alive_idx;
  long long big_min;  // domains of at least this many elements are not materialised
  __device__ __forceinline__ bool big(long long count) const { return count >= big_min; }
  __device__ __forceinline__ V3 pos(long long e, int a, bool bg) const {
    if (!bg) return v3_load(p + 3 * e);
    return xf_apply(load_xf(pose + 12 * alive_idx[a]), fs.p(s[e]));
  }
  __device__ __forceinline__ V3 nrm(long long e, int a, bool bg) const {
    if (!bg) return v3_load(n + 3 * e);
    return xf_rotate(load_xf(pose + 12 * alive_idx[a]), fs.nrm(s[e]));
  }
};

// ------------------------------------------------- chosen domain elements
// Elements of domain (a, slot) in sample order.  Writes sample id, position
// and normal.
__global__ void k_domain_fill(int nA, int k, const int* alive_idx, const int* chosen,
                              const uint32_t* mask, DSamples fs, const double* pose,
                              const long long* el_off, int* el_s, double* el_p, double* el_n,
                              long long big_min) {
  // a warp per domain: ballots over 32 samples at a time give each member
  // its rank, no block-wide scans
  const int lane = threadIdx.x & 31;
  const long long seg = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (seg >= (long long)nA * k) return;  // warp-uniform
  const int a = (int)(seg / k), slot = (int)(seg % k);
  const int i = alive_idx[a];
  const int g = chosen[i * kMaxK + slot];
  const uint32_t* m = mask + (size_t)i * fs.n;
  const Xf x = load_xf(pose + 12 * i);
  const long long off = el_off[seg];
  // large domains keep the sample ids only (ElemSrc)
  const bool mat = el_off[seg + 1] - off < big_min;
  long long run = off;
  for (int base = 0; base < fs.n; base += 32) {
    const int j = base + lane;
    const bool flag = j < fs.n && ((m[j] >> g) & 1u);
    const unsigned b = __ballot_sync(0xffffffffu, flag);
    if (flag) {
      const long long e = run + __popc(b & ((1u << lane) - 1u));
      el_s[e] = j;
      if (mat) {
        V3 p = xf_apply(x, fs.p(j));
        V3 n = xf_rotate(x, fs.nrm(j));
        el_p[3 * e] = p.x;
        el_p[3 * e + 1] = p.y;
        el_p[3 * e + 2] = p.z;
        el_n[3 * e] = n.x;
        el_n[3 * e + 1] = n.y;
        el_n[3 * e + 2] = n.z;
      }
    }
    run += __popc(b);
  }
}

// --------------------------------------------------- copt stream draws
// Stream 'copt', g (contact_opt.cpp:61,84-109): per restart k index draws
// followed by one Box-Muller pair (2 u64) per mutation.  The count per
// restart is fixed, so every restart's draws are at a known offset and the
// restarts can run in parallel.  One thread per candidate walks the stream.
__global__ void k_copt_draws(int nA, const int* alive_idx, int c_lo, int B, int pass,
                             uint64_t seed, long long per_cand, uint64_t* out) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nA) return;
  int i = alive_idx[a];
  uint64_t gid = (uint64_t)pass * B + (uint64_t)(c_lo + i);
  Mt64 g;
  mt_seed(g, mix_seed(seed, kTagContactOpt, gid));
  uint64_t* o = out + (size_t)a * per_cand;
  for (long long d = 0; d < per_cand; ++d) o[d] = mt_next(g);
}

// The same stream with one warp per candidate: the MT19937-64 state lives in
// shared memory and each 312-draw block is produced by the block twist in
// two parallel halves (entries i < 156 read only old words; entries
// i >= 156 read old words and the new word i - 156, and entry 311 the new
// word 0: exactly what the element-by-element twist of mt_next reads), then
// tempered and written by all lanes.  The Box-Muller pairs of every restart
// are then turned into the tangent-plane offsets in the same launch (the
// candidate's draws are still in L2): k_copt_draws + k_copt_normals fused.
constexpr int kDrawWarps = 4;
__global__ void __launch_bounds__(32 * kDrawWarps)
k_copt_draws_warp(int nA, const int* alive_idx, int c_lo, int B, int pass, uint64_t seed,
                  long long per_cand, long long per_restart, int k, int prp, double sigma,
                  uint64_t* out) {
  __shared__ uint64_t s_mt[kDrawWarps][312];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int a = blockIdx.x * kDrawWarps + w;
  if (a >= nA) return;  // warp-uniform
  uint64_t* mt = s_mt[w];
  const int i = alive_idx[a];
  if (lane == 0) {
    const uint64_t gid = (uint64_t)pass * B + (uint64_t)(c_lo + i);
    mt[0] = mix_seed(seed, kTagContactOpt, gid);
    for (int t = 1; t < 312; ++t) mt[t] = 6364136223846793005ull * (mt[t - 1] ^ (mt[t - 1] >> 62)) + (uint64_t)t;
  }
  __syncwarp();
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, MA = 0xB5026F5AA96619E9ull;
  uint64_t* o = out + (size_t)a * per_cand;
  for (long long b0 = 0; b0 < per_cand; b0 += 312) {
    uint64_t nv[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {  // entries 0..155
      const int e = lane + 32 * t;
      if (e < 156) {
        const uint64_t y = (mt[e] & UM) | (mt[e + 1] & LM);
        nv[t] = mt[e + 156] ^ (y >> 1) ^ ((y & 1ull) ? MA : 0ull);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 5; ++t)
      if (lane + 32 * t < 156) mt[lane + 32 * t] = nv[t];
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 5; ++t) {  // entries 156..311
      const int e = 156 + lane + 32 * t;
      if (e < 312) {
        const uint64_t y = (mt[e] & UM) | (mt[e + 1 == 312 ? 0 : e + 1] & LM);
        nv[t] = mt[e - 156] ^ (y >> 1) ^ ((y & 1ull) ? MA : 0ull);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 5; ++t)
      if (156 + lane + 32 * t < 312) mt[156 + lane + 32 * t] = nv[t];
    __syncwarp();
    for (int e = lane; e < 312 && b0 + e < per_cand; e += 32) {
      uint64_t z = mt[e];
      z ^= (z >> 29) & 0x5555555555555555ull;
      z ^= (z << 17) & 0x71D67FFFEDA60000ull;
      z ^= (z << 37) & 0xFFF7EEE000000000ull;
      z ^= (z >> 43);
      o[b0 + e] = z;
    }
  }
  __syncwarp();
  const long long np = (per_cand / per_restart) * (long long)prp;
  for (long long t = lane; t < np; t += 32) {
    const long long r = t / prp;
    const int j = (int)(t - r * prp);
    uint64_t* d2 = o + r * per_restart + k + 2 * j;
    double z1, z2;
    box_muller(d2[0], d2[1], &z1, &z2);
    d2[0] = (uint64_t)__double_as_longlong(sigma * z1);
    d2[1] = (uint64_t)__double_as_longlong(sigma * z2);
  }
}

// The mutation draws of every restart as the tangent-plane offsets the
// search consumes: each (u64, u64) pair becomes (sigma * z1, sigma * z2) with
// (z1, z2) the Box-Muller pair of rng.hpp:47-61 — u = sigma * normal(),
// v = sigma * normal() of contact_opt.cpp:108-109 (the second normal() call
// returns the cached spare).  In place, bit-cast into the u64 buffer; one
// thread per pair, so the transcendentals stay out of the search kernel.
__global__ void k_copt_normals(long long n_pairs, int per_restart_pairs, int k,
                               long long per_restart, double sigma, uint64_t* draws) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_pairs;
       t += (long long)gridDim.x * blockDim.x) {
    long long rr = t / per_restart_pairs;  // (candidate, restart) index
    int j = (int)(t - rr * per_restart_pairs);
    uint64_t* d2 = draws + rr * per_restart + k + 2 * j;
    double z1, z2;
    box_muller(d2[0], d2[1], &z1, &z2);
    d2[0] = (uint64_t)__double_as_longlong(sigma * z1);
    d2[1] = (uint64_t)__double_as_longlong(sigma * z2);
  }
}

// ------------------------------------------------------ optimize_contacts
struct CoptCfg {
  int k, n_outer, n_inner, restarts;
  double sigma, lambda, mu;
  WOpts o;
  long long per_restart, per_cand;
};

// ------------------------------------------------ validate_grasp_collisions
// collision.cpp:230-288, block per call.  Only clean() and the deepest
// penetration feed decisions; both are order independent (any / max).
struct CollCfg {
  double margin;
  DSamples raw;
  const int* part_link;
  DGrid grid;  // over raw (grid.ok == 0: sweep every sample)
};

// ------------------------------------------------------------ postprocess
// pipeline.cpp:553-603: contacts re-projected at the final q, force
// direction from the nearest preprocessed sample, statics appended, flags
// and the cold GSWO stability solve.
struct FinalCfg {
  int k;
  double contact_tol, lambda, mu, eps;
  WOpts o;
};

}  // namespace lgd
