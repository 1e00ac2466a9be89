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

// ------------------------------------------------- chosen domain elements
// Elements of domain (a, slot) in sample order: block per (a, slot), block
// scan over the mask row.  Writes sample id, position and normal (SoA).
__global__ void k_domain_fill(int nA, int k, const int* alive_idx, const int* chosen,
                              const uint32_t* mask, DSamples fs, const double* pose,
                              const long long* el_off, int* el_s, double* el_p, double* el_n) {
  typedef cub::BlockScan<int, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  int a = blockIdx.x / k, slot = blockIdx.x % k;
  if (a >= nA) return;
  int i = alive_idx[a];
  int g = chosen[i * kMaxK + slot];
  const uint32_t* m = mask + (size_t)i * fs.n;
  Xf x = load_xf(pose + 12 * i);
  long long off = el_off[a * k + slot];
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int base = 0; base < fs.n; base += 256) {
    int j = base + threadIdx.x;
    int flag = (j < fs.n && ((m[j] >> g) & 1u)) ? 1 : 0;
    int pos, total;
    Scan(tmp).ExclusiveSum(flag, pos, total);
    if (flag) {
      long long e = off + s_base + pos;
      el_s[e] = j;
      V3 p = xf_apply(x, fs.p(j));
      V3 n = xf_rotate(x, fs.nrm(j));
      el_p[3 * e] = p.x;
      el_p[3 * e + 1] = p.y;
      el_p[3 * e + 2] = p.z;
      el_n[3 * e] = n.x;
      el_n[3 * e + 1] = n.y;
      el_n[3 * e + 2] = n.z;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
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

// ------------------------------------------------------ optimize_contacts
struct CoptCfg {
  int k, n_outer, n_inner, restarts;
  double sigma, lambda, mu;
  WOpts o;
  long long per_restart, per_cand;
};

// contact_opt.cpp:45-142: block per candidate, one warp per restart, lanes
// over the n_inner mutations of a (outer, slot) step.  Every mutation is
// projected and warm-solved independently from the same incumbent; the
// winner is argmin (objective, m) among objectives strictly below the
// incumbent, identical to the sequential first-strict-improvement rule.
__global__ void k_contact_opt(int nA, const int* alive_idx, CoptCfg cfg, const int* n_static,
                              const double* st_p, const double* st_n, const long long* el_off,
                              const int* el_s, const double* el_p, const double* el_n,
                              const uint64_t* draws, int* out_ids, double* out_obj,
                              int* out_anchor, double* out_sol, double eps_stable, int* balanced) {
  extern __shared__ double s_res[];  // per warp: objective, ids[k], anchor, sol[3*6]
  const int a = blockIdx.x;
  if (a >= nA) return;
  const int i = alive_idx[a];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int k = cfg.k;
  const int s = n_static[i];
  const int n = k + s;
  const int stride = 2 + k + 3 * kMaxC;
  long long off[kMaxK], cnt[kMaxK];
  for (int q = 0; q < k; ++q) {
    off[q] = el_off[a * k + q];
    cnt[q] = el_off[a * k + q + 1] - off[q];
  }
  Ctr ctr = {0, 0, 0, 0, 0};
  for (int rbase = 0; rbase < cfg.restarts; rbase += nw) {
    const int r = rbase + warp;
    if (r < cfg.restarts) {
    const uint64_t* D = draws + (size_t)a * cfg.per_cand + (size_t)r * cfg.per_restart;
    WProb prob;
    prob.n = n;
    prob.lambda = cfg.lambda;
    prob.mu = cfg.mu;
    if (s) wprob_set(prob, k, v3_load(st_p + 3 * i), v3_load(st_n + 3 * i));
    int ids[kMaxK];
    for (int q = 0; q < k; ++q) {
      ids[q] = (int)(D[q] % (uint64_t)cnt[q]);
      long long e = off[q] + ids[q];
      wprob_set(prob, q, v3_load(el_p + 3 * e), neg(v3_load(el_n + 3 * e)));
    }
    // cold solve: lanes over anchors, best anchor by strict '<'
    WState sol;
    double obj;
    int anchor;
    {
      WState st;
      double val = kInf;
      if (lane < n) val = wsolve_anchor(prob, lane, prob.mu > 0.0, cfg.o, nullptr, st, ctr);
      if (!(val < kInf)) val = kInf;  // NaN / inf anchors never win (strict '<')
      double best = val;
      int bl = val < kInf ? lane : 99;
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (ov < best || (ov == best && ol < bl)) {
          best = ov;
          bl = ol;
        }
      }
      // anchors whose value is not < inf never win (reference: strict '<')
      anchor = (best < kInf) ? bl : -1;
      obj = best;
      int src = anchor >= 0 ? anchor : 0;
      for (int c = 0; c < kMaxC; ++c) {
        sol.a[c] = __shfl_sync(0xffffffffu, st.a[c], src);
        sol.bx[c] = __shfl_sync(0xffffffffu, st.bx[c], src);
        sol.by[c] = __shfl_sync(0xffffffffu, st.by[c], src);
      }
    }
    const uint64_t* M = D + k;
    for (int outer = 0; outer < cfg.n_outer; ++outer) {
      for (int q = 0; q < k; ++q) {
        long long ce = off[q] + ids[q];
        V3 cur_p = v3_load(el_p + 3 * ce);
        V3 tx, ty;
        tangent_basis(neg(v3_load(el_n + 3 * ce)), tx, ty);
        double best_obj = obj;
        int best_m = 0x7fffffff, best_id = -1;
        WState best_sol = sol;
        int best_anchor = -1;
        for (int mb = 0; mb < cfg.n_inner; mb += 32) {
          int m = mb + lane;
          double val = kInf;
          int cand = -1, an = -1;
          WState ws;
          if (m < cfg.n_inner) {
            const uint64_t* d2 = M + 2 * ((long long)(outer * k + q) * cfg.n_inner + m);
            double z1, z2;
            box_muller(d2[0], d2[1], &z1, &z2);
            double u = cfg.sigma * z1;
            double v = cfg.sigma * z2;
            V3 cp = axpy(axpy(cur_p, u, tx), v, ty);
            // project_to_domain (contact_opt.cpp:11-25)
            const double* P = el_p + 3 * off[q];
            double bd = sqnorm(sub(v3(P[0], P[1], P[2]), cp));
            int bi = 0;
            ctr.proj += (unsigned long long)cnt[q];
            for (long long e = 1; e < cnt[q]; ++e) {
              double d2v = sqnorm(sub(v3(P[3 * e], P[3 * e + 1], P[3 * e + 2]), cp));
              if (d2v < bd) {
                bd = d2v;
                bi = (int)e;
              }
            }
            cand = bi;
            WProb trial = prob;
            long long e = off[q] + bi;
            wprob_set(trial, q, v3_load(el_p + 3 * e), neg(v3_load(el_n + 3 * e)));
            val = wsolve(trial, cfg.o, anchor >= 0 ? &sol : nullptr, &an, ws, ctr);
          }
          // lowest (value, m) among value < best_obj
          double bv = (val < best_obj) ? val : kInf;
          int bm = (val < best_obj) ? m : 0x7fffffff;
          for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            int om = __shfl_xor_sync(0xffffffffu, bm, o);
            if (ov < bv || (ov == bv && om < bm)) {
              bv = ov;
              bm = om;
            }
          }
          if (bm != 0x7fffffff) {
            int src = bm - mb;
            best_obj = bv;
            best_m = bm;
            best_id = __shfl_sync(0xffffffffu, cand, src);
            best_anchor = __shfl_sync(0xffffffffu, an, src);
            for (int c = 0; c < kMaxC; ++c) {
              best_sol.a[c] = __shfl_sync(0xffffffffu, ws.a[c], src);
              best_sol.bx[c] = __shfl_sync(0xffffffffu, ws.bx[c], src);
              best_sol.by[c] = __shfl_sync(0xffffffffu, ws.by[c], src);
            }
          }
        }
        (void)best_m;
        if (best_id >= 0) {
          ids[q] = best_id;
          long long e = off[q] + best_id;
          wprob_set(prob, q, v3_load(el_p + 3 * e), neg(v3_load(el_n + 3 * e)));
          sol = best_sol;
          obj = best_obj;
          anchor = best_anchor;
        }
      }
    }
    if (lane == 0) {
      double* R = s_res + warp * stride;
      R[0] = obj;
      R[1] = (double)anchor;
      for (int q = 0; q < k; ++q) R[2 + q] = (double)ids[q];
      for (int c = 0; c < kMaxC; ++c) {
        R[2 + k + c] = sol.a[c];
        R[2 + k + kMaxC + c] = sol.bx[c];
        R[2 + k + 2 * kMaxC + c] = sol.by[c];
      }
    }
    }  // r < restarts
    // fold this round's restarts into the per-block result in restart order
    __syncthreads();
    if (threadIdx.x == 0) {
      double* best = s_res + nw * stride;
      for (int w = 0; w < nw && rbase + w < cfg.restarts; ++w) {
        double* R = s_res + w * stride;
        bool first = (rbase + w) == 0;
        if (first || R[0] < best[0])
          for (int t = 0; t < stride; ++t) best[t] = R[t];
        if (first && !(R[0] < kInf)) best[0] = kInf;
      }
    }
    __syncthreads();
  }
  ctr_flush(ctr);
  if (threadIdx.x == 0) {
    double* best = s_res + nw * stride;
    out_obj[a] = best[0];
    int an = (int)best[1];
    // result.solution stays default (anchor -1) unless a restart beat +inf
    if (!(best[0] < kInf)) an = -1;
    out_anchor[a] = an;
    for (int q = 0; q < k; ++q) out_ids[a * kMaxK + q] = (int)best[2 + q];
    for (int c = 0; c < 3 * kMaxC; ++c) out_sol[a * 3 * kMaxC + c] = best[2 + k + c];
    balanced[a] = (an >= 0 && best[0] < eps_stable) ? 1 : 0;
  }
}

// ------------------------------------------------ lookup-attempt targets
// reverse_lookup (contact_field.cpp:450-484) for every slot of the active
// candidates: the element's hit list is recomputed from (sample, group,
// pose) in patch order, one hit is drawn from stream 'revs', and the
// best-aligned code of that box gives the representative.
__global__ void k_targets(int nAct, const int* act, const int* alive_idx, int k, int attempt,
                          int c_lo, int B, int pass, uint64_t seed, DField f,
                          const int* group_of_patch, const double* patch_pts,
                          const double* patch_nrm, const int* patch_link, const int* chosen,
                          const int* opt_ids, const long long* el_off, const double* el_p,
                          const double* el_n, double theta, double* tgt, int* tgt_link,
                          int* err) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nAct * k) return;
  int ai = t / k, slot = t % k;
  int a = act[ai];
  int i = alive_idx[a];
  int g = chosen[i * kMaxK + slot];
  long long e = el_off[a * k + slot] + opt_ids[a * kMaxK + slot];
  V3 p = v3_load(el_p + 3 * e), n = v3_load(el_n + 3 * e);
  int nh = 0;
  sample_hits(f, f.codebook, p, n, theta, [&](int patch, int, double) {
    if (group_of_patch[patch] == g) ++nh;
  });
  if (nh == 0) {
    atomicExch(err, 1);
    return;
  }
  uint64_t gid = (uint64_t)pass * B + (uint64_t)(c_lo + i);
  DRng rng;
  rng.seed(mix_seed(seed, kTagReverse, (gid << 6) + ((uint64_t)attempt << 3) + (uint64_t)slot));
  int pick = (int)rng.index((uint64_t)nh);
  int box = -1, cnt = 0;
  sample_hits(f, f.codebook, p, n, theta, [&](int patch, int b, double) {
    if (group_of_patch[patch] == g) {
      if (cnt == pick) box = b;
      ++cnt;
    }
  });
  int best = -1;
  double best_dot = -2.0;
  long long q0 = f.box_code_off[box], q1 = f.box_code_off[box + 1];
  for (long long q = q0; q < q1; ++q) {
    int code = f.codes[q];
    double d = -dot(v3(f.codebook[3 * code], f.codebook[3 * code + 1], f.codebook[3 * code + 2]), n);
    if (d > best_dot) {
      best_dot = d;
      best = (int)(q - q0);
    }
  }
  const double* rp = f.rep_pn + 6 * (q0 + best);
  double* T = tgt + (size_t)(ai * k + slot) * 12;
  v3_store(T, p);
  v3_store(T + 3, neg(n));
  v3_store(T + 6, v3_load(rp));
  v3_store(T + 9, v3_load(rp + 3));
  tgt_link[ai * k + slot] = patch_link[f.box_patch[box]];
}

__device__ __forceinline__ void load_targets(const double* tgt, const int* tl, int k, Target* T) {
  for (int q = 0; q < k; ++q) {
    const double* s = tgt + 12 * q;
    T[q].op = v3_load(s);
    T[q].on = v3_load(s + 3);
    T[q].hp = v3_load(s + 6);
    T[q].hn = v3_load(s + 9);
    T[q].link = tl[q];
  }
}

// realize_grasp from mid_config, one thread per active candidate.
__global__ void k_realize(int nAct, int k, IkCfg P, int rounds, int fine_iters,
                          const double* tgt, const int* tgt_link, double* q_out, double* max_res,
                          int* finite, unsigned long long* used) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nAct) return;
  Target T[kMaxK];
  load_targets(tgt + (size_t)t * k * 12, tgt_link + t * k, k, T);
  double q[kMaxDof];
  for (int j = 0; j < c_hand.dof; ++j) q[j] = c_hand.mid[j];
  double mr;
  unsigned long long u;
  Ctr ctr = {0, 0, 0, 0, 0};
  bool fin = realize_grasp(q, T, k, P, rounds, fine_iters, &mr, &u, ctr);
  ctr_flush(ctr);
  for (int j = 0; j < c_hand.dof; ++j) q_out[(size_t)t * kMaxDof + j] = q[j];
  max_res[t] = mr;
  finite[t] = fin ? 1 : 0;
  used[t] = u;
}

// ------------------------------------------------ validate_grasp_collisions
// collision.cpp:230-288, block per call.  Only clean() and the deepest
// penetration feed decisions; both are order independent (any / max).
struct CollCfg {
  double margin;
  DSamples raw;
  const int* part_link;
};

__global__ void k_collision(int n_calls, CollCfg C, const int* call_cand, const int* call_on,
                            const double* q_all, const double* pose, const double* obj_aabb,
                            uint8_t* clean_out, double* maxpen_out) {
  __shared__ double s_fr[kMaxLinks * 12];
  __shared__ double s_box[64 * 6];
  __shared__ int s_pairs[2 * 2112];
  __shared__ int s_np;
  __shared__ int s_viol;
  __shared__ double scratch[32];
  int call = blockIdx.x;
  if (call >= n_calls) return;
  if (call_on && !call_on[call]) return;
  int i = call_cand[call];
  const int np = c_hand.n_parts;
  if (threadIdx.x == 0) {
    Xf f[kMaxLinks];
    fk(q_all + (size_t)call * kMaxDof, f);
    for (int l = 0; l < c_hand.n_links; ++l) store_xf(s_fr + 12 * l, f[l]);
    s_np = 0;
    s_viol = 0;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
    V3 mn, mx;
    world_bounds(p, load_xf(s_fr + 12 * C.part_link[p]), &mn, &mx);
    s_box[6 * p + 0] = mn.x - C.margin;
    s_box[6 * p + 1] = mn.y - C.margin;
    s_box[6 * p + 2] = mn.z - C.margin;
    s_box[6 * p + 3] = mx.x + C.margin;
    s_box[6 * p + 4] = mx.y + C.margin;
    s_box[6 * p + 5] = mx.z + C.margin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // broad_phase (collision.cpp:22-45), pair order kept
    const double* ob = obj_aabb + 6 * i;
    double oi[6] = {ob[0] - C.margin, ob[1] - C.margin, ob[2] - C.margin,
                    ob[3] + C.margin, ob[4] + C.margin, ob[5] + C.margin};
    bool have_obj = C.raw.n > 0;
    int cnt = 0;
    auto ovl = [](const double* a, const double* b) {
      return a[0] <= b[3] && a[1] <= b[4] && a[2] <= b[5] && a[3] >= b[0] && a[4] >= b[1] &&
             a[5] >= b[2];
    };
    for (int p = 0; p < np; ++p) {
      for (int q = p + 1; q < np; ++q)
        if (ovl(s_box + 6 * p, s_box + 6 * q) && cnt < 2112) {
          s_pairs[2 * cnt] = p;
          s_pairs[2 * cnt + 1] = q;
          ++cnt;
        }
      if (have_obj && ovl(s_box + 6 * p, oi) && cnt < 2112) {
        s_pairs[2 * cnt] = p;
        s_pairs[2 * cnt + 1] = -1;
        ++cnt;
      }
    }
    s_np = cnt;
  }
  __syncthreads();
  const int npairs = s_np;
  // narrow phase 1: GJK on link-link candidates, one pair per thread
  for (int e = threadIdx.x; e < npairs; e += blockDim.x) {
    int pa = s_pairs[2 * e], pb = s_pairs[2 * e + 1];
    if (pb < 0) continue;
    int la = C.part_link[pa], lb = C.part_link[pb];
    if (la == lb || c_hand.parent[la] == lb || c_hand.parent[lb] == la) continue;
    if (gjk_distance(pa, load_xf(s_fr + 12 * la), pb, load_xf(s_fr + 12 * lb)) == 0.0)
      atomicOr(&s_viol, 1);
  }
  // narrow phase 2: half-plane depth of the object samples per part
  Xf x = load_xf(pose + 12 * i);
  double maxpen = 0.0;
  for (int e = 0; e < npairs; ++e) {
    int pa = s_pairs[2 * e], pb = s_pairs[2 * e + 1];
    if (pb >= 0) continue;
    Xf inv = xf_inverse(load_xf(s_fr + 12 * C.part_link[pa]));
    const double* b = c_hand.bounds + 6 * pa;
    double mx = 0.0;
    bool off = false;
    for (int j = threadIdx.x; j < C.raw.n; j += blockDim.x) {
      V3 local = xf_apply(inv, xf_apply(x, C.raw.p(j)));
      if (!(local.x >= b[0] - 1e-9 && local.y >= b[1] - 1e-9 && local.z >= b[2] - 1e-9 &&
            local.x <= b[3] + 1e-9 && local.y <= b[4] + 1e-9 && local.z <= b[5] + 1e-9))
        continue;
      double depth = part_interior_depth(pa, local);
      if (depth > C.margin) {
        off = true;
        mx = dmax(mx, depth);
      }
    }
    if (off) atomicOr(&s_viol, 1);
    mx = block_max(mx, scratch);
    maxpen = dmax(maxpen, mx);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    clean_out[call] = s_viol ? 0 : 1;
    if (maxpen_out) maxpen_out[call] = maxpen;
  }
}

// ------------------------------------------------------ attempt bookkeeping
// pipeline.cpp:496-520: keep the best attempt (clear first, then lower
// residual); stop searching once a clear attempt is kept.
__global__ void k_attempt_update(int nAct, const int* act, int k, int attempt,
                                 const double* q_try, const double* res, const int* finite,
                                 const unsigned long long* used, const uint8_t* clean,
                                 const int* conv, const double* tgt, const int* tgt_link,
                                 double contact_tol, int* have, int* best_clear,
                                 double* best_res, double* best_q, unsigned long long* best_used,
                                 double* best_tgt, int* best_link, int* best_attempt,
                                 int* searching) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nAct) return;
  int a = act[t];
  if (!finite[t]) return;
  bool cv = res[t] <= contact_tol;
  bool clear = cv ? (clean[t] != 0) : false;
  (void)conv;
  bool better;
  if (!have[a]) better = true;
  else if (clear != (best_clear[a] != 0)) better = clear;
  else better = res[t] < best_res[a];
  if (better) {
    have[a] = 1;
    best_clear[a] = clear ? 1 : 0;
    best_res[a] = res[t];
    for (int j = 0; j < kMaxDof; ++j) best_q[(size_t)a * kMaxDof + j] = q_try[(size_t)t * kMaxDof + j];
    best_used[a] = used[t];
    for (int c = 0; c < 12 * k; ++c) best_tgt[(size_t)a * kMaxK * 12 + c] = tgt[(size_t)t * k * 12 + c];
    for (int q = 0; q < k; ++q) best_link[a * kMaxK + q] = tgt_link[t * k + q];
    best_attempt[a] = attempt;
  }
  if (best_clear[a]) searching[a] = 0;
}

// ------------------------------------------------------- unused joints
// pipeline.cpp:535-551: every attempt redraws each unused joint in ascending
// order from stream 'unus'; attempt j therefore starts at draw j * #unused.
__global__ void k_unused_q(int nAct, const int* act, const int* alive_idx, int attempt, int c_lo,
                           int B, int pass, uint64_t seed, const double* best_q,
                           const unsigned long long* best_used, double* q_out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nAct) return;
  int a = act[t];
  int i = alive_idx[a];
  uint64_t gid = (uint64_t)pass * B + (uint64_t)(c_lo + i);
  Mt64 g;
  mt_seed(g, mix_seed(seed, kTagUnused, gid));
  unsigned long long used = best_used[a];
  const int dof = c_hand.dof;
  int nu = 0;
  for (int j = 0; j < dof; ++j)
    if (!((used >> j) & 1ull)) ++nu;
  for (long long d = 0; d < (long long)attempt * nu; ++d) mt_next(g);
  double* q = q_out + (size_t)t * kMaxDof;
  for (int j = 0; j < dof; ++j) {
    q[j] = best_q[(size_t)a * kMaxDof + j];
    if ((used >> j) & 1ull) continue;
    q[j] = c_hand.jlo[j] + (c_hand.jhi[j] - c_hand.jlo[j]) * u01(mt_next(g));
  }
}

// ------------------------------------------------------------ postprocess
// pipeline.cpp:553-603: contacts re-projected at the final q, force
// direction from the nearest preprocessed sample, statics appended, flags
// and the cold GSWO stability solve.
struct FinalCfg {
  int k;
  double contact_tol, lambda, mu, eps;
  WOpts o;
};

__global__ void k_finalize(int nT, const int* act, const int* alive_idx, FinalCfg C, DSamples fs,
                           const double* pose, const int* n_static, const int* st_link,
                           const double* st_p, const double* st_n, const double* q_final,
                           const uint8_t* clean, const double* best_tgt, const int* best_link,
                           lg_grasp* out, int* valid, int* dropped) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nT) return;
  int a = act[t];
  int i = alive_idx[a];
  const int k = C.k;
  lg_grasp& g = out[a];
  valid[a] = 0;
  dropped[a] = 0;
  g.n_contacts = 0;
  g.penetration_free = 0;
  g.stable = 0;
  g.ik_converged = 0;
  g.objective = 0.0;
  const double* q = q_final + (size_t)a * kMaxDof;
  Xf fr[kMaxLinks];
  fk(q, fr);
  Xf x = load_xf(pose + 12 * i);
  double worst = 0.0;
  for (int s = 0; s < k; ++s) {
    const double* T = best_tgt + (size_t)a * kMaxK * 12 + 12 * s;
    int link = best_link[a * kMaxK + s];
    Xf inv = xf_inverse(fr[link]);
    V3 sp = v3(0, 0, 0), sn = v3(0, 0, 0);
    double d = closest_on_parts(link, xf_apply(inv, v3_load(T)), &sp, &sn);
    if (!is_finite(d)) {
      dropped[a] = 1;
      return;
    }
    worst = dmax(worst, d);
    V3 pw = xf_apply(fr[link], sp);
    int nearest = 0;
    double best_d2 = kInf;
    for (int j = 0; j < fs.n; ++j) {
      double d2 = sqnorm(sub(xf_apply(x, fs.p(j)), pw));
      if (d2 < best_d2) {
        best_d2 = d2;
        nearest = j;
      }
    }
    int ci = g.n_contacts++;
    v3_store(g.contact_p[ci], pw);
    v3_store(g.contact_n[ci], neg(xf_rotate(x, fs.nrm(nearest))));
    g.contact_link[ci] = link;
  }
  if (n_static[i]) {
    int ci = g.n_contacts++;
    v3_store(g.contact_p[ci], v3_load(st_p + 3 * i));
    v3_store(g.contact_n[ci], v3_load(st_n + 3 * i));
    g.contact_link[ci] = st_link[i];
  }
  g.ik_converged = worst <= C.contact_tol;
  g.penetration_free = clean[a] ? 1 : 0;
  WProb w;
  w.n = g.n_contacts;
  w.lambda = C.lambda;
  w.mu = C.mu;
  for (int c = 0; c < g.n_contacts; ++c) wprob_set(w, c, v3_load(g.contact_p[c]), v3_load(g.contact_n[c]));
  WState ws;
  int an;
  Ctr ctr = {0, 0, 0, 0, 0};
  double obj = wsolve(w, C.o, nullptr, &an, ws, ctr);
  ctr_flush(ctr);
  g.objective = obj;
  g.stable = obj < C.eps ? 1 : 0;
  g.g = 0;
  m3_store(g.pose_R, x.R);
  v3_store(g.pose_t, x.t);
  g.dof = c_hand.dof;
  for (int j = 0; j < c_hand.dof; ++j) g.q[j] = q[j];
  valid[a] = (g.penetration_free && g.stable && g.ik_converged) ? 1 : 0;
}

}  // namespace lgd
