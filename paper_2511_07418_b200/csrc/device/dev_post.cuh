// dev_post.cuh — realisation attempts and postprocess as whole-batch
// launches (reference pipeline.cpp:465-604).
//
// The reference runs lookup attempt a+1 only while no attempt so far is
// both converged and collision-free, and redraws the unused joints until a
// configuration is clean.  Both loops almost always run to exhaustion (most
// candidates never turn penetration-free), so every attempt is evaluated at
// once and the reference's in-order selection rule is applied on the device
// afterwards; the kept attempt, and everything derived from it, is identical.
#pragma once

#include "dev_stages.cuh"

namespace lgd {

// validate_grasp_collisions (collision.cpp:230-288), one warp per
// configuration (4 per CTA, no block barriers): the warp's FK, part boxes
// and object-overlap list, then the link-link GJK pairs and the object-sample
// sweep, lanes striding over each.  Each sample is moved to world once; a
// part is tested only when the world point lies in the part's world box (the
// transformed local box, so it contains every point the local AABB test
// accepts, widened by 1e-6), and then with the reference's exact local
// transform and depth.  clean() is an OR of violations and max_penetration a
// max, both order independent.  With clean_only (the pipeline consumes only
// clean()), work stops at the first violation.
constexpr int kCollWarps = 4;
constexpr int kCollGridMin = 20000;
struct CollWarpSmem {
  double q[kMaxDof];
  double fr[kMaxLinks * kFS];
  double inv[kMaxLinks * kFS];
  double box[64 * 6];
  int obj[64];
  int nobj, viol;
};

// GRID: the object-sample grid path is compiled in (objects of at least
// kCollGridMin samples); the plain instance keeps the smaller sweep-only body.
template <int MINB, bool GRID>
__global__ void __launch_bounds__(32 * kCollWarps, MINB)
k_collision3(int n_calls, CollCfg C, const int* call_cand, const int* call_on, const double* q_all,
             const double* pose, const double* obj_aabb, int clean_only, uint8_t* clean_out,
             double* maxpen_out) {
  __shared__ CollWarpSmem S[kCollWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int call = blockIdx.x * kCollWarps + wid;
  if (call >= n_calls) return;  // warp-uniform
  if (call_on && !call_on[call]) return;
  CollWarpSmem& W = S[wid];
  const int i = call_cand[call];
  const int np = c_hand.n_parts, nl = c_hand.n_links;
  if (lane < c_hand.dof) W.q[lane] = q_all[(size_t)call * kMaxDof + lane];
  if (lane == 0) {
    W.nobj = 0;
    W.viol = 0;
  }
  __syncwarp();
  wfk_s(W.q, W.fr, lane);
  if (lane < nl) st_xf(W.inv + kFS * lane, xf_inverse(ld_xf(W.fr + kFS * lane)));
  const double* ob = obj_aabb + 6 * i;
  const double oi[6] = {ob[0] - C.margin, ob[1] - C.margin, ob[2] - C.margin,
                        ob[3] + C.margin, ob[4] + C.margin, ob[5] + C.margin};
  auto ovl = [](const double* a, const double* b) {
    return a[0] <= b[3] && a[1] <= b[4] && a[2] <= b[5] && a[3] >= b[0] && a[4] >= b[1] &&
           a[5] >= b[2];
  };
  for (int p = lane; p < np; p += 32) {
    V3 mn, mx;
    world_bounds(p, ld_xf(W.fr + kFS * C.part_link[p]), &mn, &mx);
    double* bx = W.box + 6 * p;
    bx[0] = mn.x - C.margin;
    bx[1] = mn.y - C.margin;
    bx[2] = mn.z - C.margin;
    bx[3] = mx.x + C.margin;
    bx[4] = mx.y + C.margin;
    bx[5] = mx.z + C.margin;
    if (C.raw.n > 0 && ovl(bx, oi)) W.obj[atomicAdd(&W.nobj, 1)] = p;
  }
  __syncwarp();
  // broad phase (collision.cpp:22-45) + GJK narrow phase
  for (int e = lane; e < np * np; e += 32) {
    int pa = e / np, pb = e % np;
    if (pb <= pa || !ovl(W.box + 6 * pa, W.box + 6 * pb)) continue;
    int la = C.part_link[pa], lb = C.part_link[pb];
    if (la == lb || g_hand.parent[la] == lb || g_hand.parent[lb] == la) continue;
    if (clean_only && *(volatile int*)&W.viol) break;
    if (gjk_distance(pa, ld_xf(W.fr + kFS * la), pb, ld_xf(W.fr + kFS * lb)) == 0.0)
      atomicOr(&W.viol, 1);
  }
  // object samples (collision.cpp:260-284): world point once, world-box
  // prefilter (widened 1e-6), then the exact local test and depth
  double mx = 0.0;
  const int nobj = W.nobj;
  const Xf x = load_xf(pose + 12 * i);
  // Through the raw-sample grid: part by part, only the cells of the
  // object-frame box around the preimage of the part's widened world box.
  // For w = R p + t with R orthonormal, |p - c_o| <= |R|^T h componentwise,
  // so every sample whose world point passes the world-box test lies in it
  // (rounding ~1e-16 relative, covered by the grid's w 2^-20 widening).  A
  // pose whose R is not orthonormal to 1e-9 takes the full sweep, and so do
  // objects with few samples (a part's rows hold too few samples to keep
  // the lanes busy: the sweep, one world point per sample, is faster).
  bool use_grid = GRID && C.grid.ok && nobj > 0 && C.raw.n >= kCollGridMin;
  if (use_grid) {
    const M3 RtR = mul(transpose(x.R), x.R);
    for (int a = 0; a < 9; ++a)
      use_grid = use_grid && dabs(RtR.m[a] - ((a % 4) == 0 ? 1.0 : 0.0)) <= 1e-9;
  }
  if (GRID && use_grid) {
    const DGrid& g = C.grid;
    for (int o = 0; o < nobj; ++o) {
      if (clean_only && *(volatile int*)&W.viol) break;
      const int pa = W.obj[o];
      const double* bx = W.box + 6 * pa;
      const double cw[3] = {0.5 * (bx[0] + bx[3]) - x.t.x, 0.5 * (bx[1] + bx[4]) - x.t.y,
                            0.5 * (bx[2] + bx[5]) - x.t.z};
      const double hw[3] = {0.5 * (bx[3] - bx[0]) + 1e-6, 0.5 * (bx[4] - bx[1]) + 1e-6,
                            0.5 * (bx[5] - bx[2]) + 1e-6};
      int c0[3], c1[3];
      for (int a = 0; a < 3; ++a) {
        double co = 0.0, ho = 0.0;
        for (int b = 0; b < 3; ++b) {
          co += x.R.m[3 * b + a] * cw[b];
          ho += dabs(x.R.m[3 * b + a]) * hw[b];
        }
        const double m = g.w * 0x1p-20 + (dabs(co) + ho) * 0x1p-40;
        c0[a] = grid_cell(g, a, co - ho - m);
        c1[a] = grid_cell(g, a, co + ho + m);
      }
      const Xf li = ld_xf(W.inv + kFS * C.part_link[pa]);
      const double* b = c_hand.bounds + 6 * pa;
      bool hit = false;
      for (int z = c0[2]; z <= c1[2]; ++z)
        for (int y = c0[1]; y <= c1[1]; ++y) {
          const int row = (z * g.dim[1] + y) * g.dim[0];
          const int t1 = g.start[row + c1[0] + 1];
          for (int t = g.start[row + c0[0]] + lane; t < t1; t += 32) {
            if (clean_only && *(volatile int*)&W.viol) break;
            const V3 w = xf_apply(x, v3(g.x[0][t], g.x[1][t], g.x[2][t]));
            if (!(w.x >= bx[0] - 1e-6 && w.y >= bx[1] - 1e-6 && w.z >= bx[2] - 1e-6 &&
                  w.x <= bx[3] + 1e-6 && w.y <= bx[4] + 1e-6 && w.z <= bx[5] + 1e-6))
              continue;
            const V3 local = xf_apply(li, w);
            if (!(local.x >= b[0] - 1e-9 && local.y >= b[1] - 1e-9 && local.z >= b[2] - 1e-9 &&
                  local.x <= b[3] + 1e-9 && local.y <= b[4] + 1e-9 && local.z <= b[5] + 1e-9))
              continue;
            const double depth = part_interior_depth(pa, local);
            if (depth > C.margin) {
              hit = true;
              mx = dmax(mx, depth);
            }
          }
        }
      if (hit) atomicOr(&W.viol, 1);
    }
  } else if (nobj > 0) {
    for (int j = lane; j < C.raw.n; j += 32) {
      if (clean_only && *(volatile int*)&W.viol) break;
      V3 w = xf_apply(x, C.raw.p(j));
      bool hit = false;
      for (int o = 0; o < nobj; ++o) {
        const int pa = W.obj[o];
        const double* bx = W.box + 6 * pa;
        if (!(w.x >= bx[0] - 1e-6 && w.y >= bx[1] - 1e-6 && w.z >= bx[2] - 1e-6 &&
              w.x <= bx[3] + 1e-6 && w.y <= bx[4] + 1e-6 && w.z <= bx[5] + 1e-6))
          continue;
        V3 local = xf_apply(ld_xf(W.inv + kFS * C.part_link[pa]), w);
        const double* b = c_hand.bounds + 6 * pa;
        if (!(local.x >= b[0] - 1e-9 && local.y >= b[1] - 1e-9 && local.z >= b[2] - 1e-9 &&
              local.x <= b[3] + 1e-9 && local.y <= b[4] + 1e-9 && local.z <= b[5] + 1e-9))
          continue;
        double depth = part_interior_depth(pa, local);
        if (depth > C.margin) {
          hit = true;
          mx = dmax(mx, depth);
          if (clean_only) break;
        }
      }
      if (hit) atomicOr(&W.viol, 1);
    }
  }
  __syncwarp();
  if (maxpen_out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = dmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    clean_out[call] = W.viol ? 0 : 1;
    if (maxpen_out) maxpen_out[call] = mx;
  }
}

// Stable compaction of the kept grasp records (candidate order preserved):
// one CTA of 1024 threads ranks the flags (per 1024-flag tile each warp
// ballots, warp totals are scanned in shared memory), then a warp per kept
// record copies it with coalesced 8-byte lanes.  n_out receives the count.
__global__ void __launch_bounds__(1024) k_compact_rank(int n, const uint8_t* keep, int* dest,
                                                       int* n_out) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int tile = 0; tile < n; tile += 1024) {
    const int i = tile + threadIdx.x;
    const bool f = i < n && keep[i];
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_warp[wid] = __popc(b);
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the 32 warp counts
      const int c = s_warp[lane];
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      s_warp[lane] = incl - c;
    }
    __syncthreads();
    if (i < n) dest[i] = f ? s_base + s_warp[wid] + __popc(b & ((1u << lane) - 1u)) : -1;
    __syncthreads();
    if (threadIdx.x == 1023) s_base += s_warp[31] + __popc(b);
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = s_base;
}

__global__ void k_copy_grasps(int n, const lg_grasp* in, const int* dest, lg_grasp* out) {
  const int lane = threadIdx.x & 31;
  const int i = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  if (i >= n) return;
  const int d = dest[i];
  if (d < 0) return;  // warp-uniform
  static_assert(sizeof(lg_grasp) % 8 == 0, "lg_grasp copies as 8-byte words");
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(in + i);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(out + d);
  for (int w = lane; w < (int)(sizeof(lg_grasp) / 8); w += 32) dst[w] = src[w];
}

// Funnel counts over the realised candidates (records of the others are
// zero) and the kept-grasp flags (valid, not dropped) for the compaction.
__global__ void k_grasp_flags(int nA, const lg_grasp* g, const int* valid, const int* drop,
                              uint8_t* keep, int* counts) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nA) return;
  keep[a] = (valid[a] && !drop[a]) ? 1 : 0;
  if (drop[a]) return;
  if (g[a].penetration_free) atomicAdd(counts, 1);
  if (g[a].ik_converged) atomicAdd(counts + 1, 1);
  if (g[a].stable) atomicAdd(counts + 2, 1);
}

// Reverse lookup for (candidate b, attempt, slot) (contact_field.cpp:450-484).
__global__ void k_targets_all(int nB, const int* bal, const int* alive_idx, int k, int A, int c_lo,
                              int Bsz, int pass, uint64_t seed, DField f,
                              const int* group_of_patch, const double* patch_pts,
                              const double* patch_nrm, const int* patch_link, const int* chosen,
                              const int* opt_ids, const long long* el_off, ElemSrc el,
                              double theta, double* tgt, int* tgt_link,
                              int* err) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)nB * A * k) return;
  int slot = (int)(t % k);
  int attempt = (int)((t / k) % A);
  int b = (int)(t / ((long long)k * A));
  int a = bal[b];
  int i = alive_idx[a];
  int g = chosen[i * kMaxK + slot];
  long long e = el_off[a * k + slot] + opt_ids[a * kMaxK + slot];
  const bool bg = el.big(el_off[a * k + slot + 1] - el_off[a * k + slot]);
  V3 p = el.pos(e, a, bg), n = el.nrm(e, a, bg);
  int nh = 0;
  sample_hits(f, f.codebook, p, n, theta, [&](int patch, int, double) {
    if (group_of_patch[patch] == g) ++nh;
  });
  if (nh == 0) {
    atomicExch(err, 1);
    return;
  }
  uint64_t gid = (uint64_t)pass * Bsz + (uint64_t)(c_lo + i);
  DRng rng;
  rng.seed(mix_seed(seed, kTagReverse, (gid << 6) + ((uint64_t)attempt << 3) + (uint64_t)slot));
  int pick = (int)rng.index((uint64_t)nh);
  int box = -1, cnt = 0;
  sample_hits(f, f.codebook, p, n, theta, [&](int patch, int bx, double) {
    if (group_of_patch[patch] == g) {
      if (cnt == pick) box = bx;
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
  double* T = tgt + (size_t)t * 12;
  v3_store(T, p);
  v3_store(T + 3, neg(n));
  v3_store(T + 6, v3_load(rp));
  v3_store(T + 9, v3_load(rp + 3));
  tgt_link[t] = f.rep_link[q0 + best];
}

__global__ void k_conv_flags(int n, const int* finite, const double* res, double tol, int* on) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) on[t] = (finite[t] && res[t] <= tol) ? 1 : 0;
}

// pipeline.cpp:476-522: walk the attempts in order, keep the better one
// (clear first, then lower residual), stop at the first clear keeper.
__global__ void k_attempt_select(int nB, const int* bal, int k, int A, const double* q_try,
                                 const double* res, const int* finite,
                                 const unsigned long long* used, const uint8_t* clean,
                                 const double* tgt, const int* tgt_link, double contact_tol,
                                 int* have, int* best_clear, double* best_res, double* best_q,
                                 unsigned long long* best_used, double* best_tgt, int* best_link,
                                 int* best_attempt, int* attempts_run) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nB) return;
  int a = bal[b];
  bool hv = false, bc = false;
  double br = 0.0;
  int ba = -1, runs = 0;
  for (int att = 0; att < A; ++att) {
    ++runs;
    int p = b * A + att;
    if (!finite[p]) continue;
    bool conv = res[p] <= contact_tol;
    bool clear = conv ? (clean[p] != 0) : false;
    bool better;
    if (!hv) better = true;
    else if (clear != bc) better = clear;
    else better = res[p] < br;
    if (better) {
      hv = true;
      bc = clear;
      br = res[p];
      ba = att;
    }
    if (bc) break;
  }
  have[a] = hv;
  best_clear[a] = bc;
  best_attempt[a] = ba;
  attempts_run[a] = runs;
  if (!hv) return;
  int p = b * A + ba;
  best_res[a] = res[p];
  best_used[a] = used[p];
  for (int j = 0; j < kMaxDof; ++j) best_q[(size_t)a * kMaxDof + j] = q_try[(size_t)p * kMaxDof + j];
  for (int c = 0; c < 12 * k; ++c) best_tgt[(size_t)a * kMaxK * 12 + c] = tgt[(size_t)p * k * 12 + c];
  for (int q = 0; q < k; ++q) best_link[a * kMaxK + q] = tgt_link[p * k + q];
}

// pipeline.cpp:535-546: every unused-joint redraw of every attempt; attempt j
// consumes draws [j*nu, (j+1)*nu) of stream 'unus', g.
__global__ void k_unused_all(int nR, const int* real, const int* alive_idx, int U, int c_lo,
                             int Bsz, int pass, uint64_t seed, const double* best_q,
                             const unsigned long long* best_used, double* q_all) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nR) return;
  int a = real[r];
  int i = alive_idx[a];
  uint64_t gid = (uint64_t)pass * Bsz + (uint64_t)(c_lo + i);
  Mt64 g;
  mt_seed(g, mix_seed(seed, kTagUnused, gid));
  unsigned long long used = best_used[a];
  const int dof = c_hand.dof;
  for (int att = 0; att < U; ++att) {
    double* q = q_all + ((size_t)r * U + att) * kMaxDof;
    for (int j = 0; j < dof; ++j) {
      q[j] = best_q[(size_t)a * kMaxDof + j];
      if ((used >> j) & 1ull) continue;
      q[j] = c_hand.jlo[j] + (c_hand.jhi[j] - c_hand.jlo[j]) * u01(mt_next(g));
    }
  }
}

// First clean redraw, else the last one (pipeline.cpp:538-551).
__global__ void k_unused_select(int nR, const int* real, int U, const double* q_all,
                                const uint8_t* clean, double* final_q, uint8_t* final_clean,
                                int* uatt) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nR) return;
  int a = real[r];
  int sel = U - 1;
  for (int att = 0; att < U; ++att)
    if (clean[(size_t)r * U + att]) {
      sel = att;
      break;
    }
  uatt[a] = sel;
  final_clean[a] = clean[(size_t)r * U + sel];
  for (int j = 0; j < kMaxDof; ++j)
    final_q[(size_t)a * kMaxDof + j] = q_all[((size_t)r * U + sel) * kMaxDof + j];
}

// Postprocess (pipeline.cpp:553-603), one warp per candidate: lanes < k
// re-project the targets, all lanes split each nearest-sample scan (argmin
// with lowest index on ties), lanes < n run one anchor each of the cold
// stability solve.
__global__ void k_finalize_warp(int nT, const int* act, const int* alive_idx, FinalCfg C,
                                DSamples fs, const double* pose, const int* n_static,
                                const int* st_link, const double* st_p, const double* st_n,
                                const double* q_final, const uint8_t* clean,
                                const double* best_tgt, const int* best_link, lg_grasp* out,
                                int* valid, int* dropped) {
  __shared__ double s_q[4][kMaxDof];
  __shared__ double s_F[4][kFS * kMaxLinks];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * (blockDim.x >> 5) + w;
  if (t >= nT) return;
  const int a = act[t];
  const int i = alive_idx[a];
  const int k = C.k;
  if (lane < c_hand.dof) s_q[w][lane] = q_final[(size_t)a * kMaxDof + lane];
  __syncwarp();
  wfk_s(s_q[w], s_F[w], lane);
  Xf x = load_xf(pose + 12 * i);
  // re-projection at the final q: lane s < k
  int link = lane < k ? best_link[a * kMaxK + lane] : 0;
  double d = 0.0;
  V3 pw = v3(0, 0, 0);
  if (lane < k) {
    Xf F = ld_xf(s_F[w] + kFS * link);
    const double* T = best_tgt + (size_t)a * kMaxK * 12 + 12 * lane;
    Xf inv = xf_inverse(F);
    V3 sp = v3(0, 0, 0), sn = v3(0, 0, 0);
    d = closest_on_parts(link, xf_apply(inv, v3_load(T)), &sp, &sn);
    pw = xf_apply(F, sp);
  }
  // reference: the first non-finite distance (slot order) drops the candidate
  bool nonfin = lane < k && !is_finite(d);
  lg_grasp& g = out[a];
  if (__any_sync(kFull, nonfin)) {
    if (lane == 0) {
      dropped[a] = 1;
      valid[a] = 0;
    }
    return;
  }
  double worst = warp_max_d(lane < k ? d : 0.0);
  // nearest preprocessed sample of every contact in one sweep: each sample
  // is moved to world once and compared with all k contacts (per contact
  // the lane's comparisons stay in ascending sample order)
  V3 ps[kMaxK];
  double bd[kMaxK];
  int bi[kMaxK];
#pragma unroll
  for (int c = 0; c < kMaxK; ++c) {
    const int src = c < k ? c : 0;
    ps[c] = v3(__shfl_sync(kFull, pw.x, src), __shfl_sync(kFull, pw.y, src),
               __shfl_sync(kFull, pw.z, src));
    bd[c] = kInf;
    bi[c] = 0x7fffffff;
  }
  for (int j = lane; j < fs.n; j += 32) {
    const V3 w = xf_apply(x, fs.p(j));
#pragma unroll
    for (int c = 0; c < kMaxK; ++c) {
      if (c >= k) break;
      const double d2 = sqnorm(sub(w, ps[c]));
      if (d2 < bd[c]) {
        bd[c] = d2;
        bi[c] = j;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kMaxK; ++c) {
    if (c >= k) break;
    double b = bd[c];
    int ix = bi[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double od = __shfl_xor_sync(kFull, b, o);
      int oi = __shfl_xor_sync(kFull, ix, o);
      if (od < b || (od == b && oi < ix)) {
        b = od;
        ix = oi;
      }
    }
    int nearest = ix == 0x7fffffff ? 0 : ix;
    if (lane == 0) {
      v3_store(g.contact_p[c], ps[c]);
      v3_store(g.contact_n[c], neg(xf_rotate(x, fs.nrm(nearest))));
      g.contact_link[c] = best_link[a * kMaxK + c];
    }
  }
  int nc = k;
  if (n_static[i]) {
    if (lane == 0) {
      v3_store(g.contact_p[k], v3_load(st_p + 3 * i));
      v3_store(g.contact_n[k], v3_load(st_n + 3 * i));
      g.contact_link[k] = st_link[i];
    }
    nc = k + 1;
  }
  __syncwarp();
  // is_stable (wrench.cpp:260-267): cold GSWO, lanes over anchors
  WProb wp;
  wp.n = nc;
  wp.lambda = C.lambda;
  wp.mu = C.mu;
  for (int c = 0; c < nc; ++c) wprob_set(wp, c, v3_load(g.contact_p[c]), v3_load(g.contact_n[c]));
  Ctr ctr = {0, 0, 0, 0, 0};
  WState st;
  double val = kInf;
  if (lane < nc) val = wsolve_anchor(wp, lane, wp.mu > 0.0, C.o, nullptr, st, ctr);
  if (!(val < kInf)) val = kInf;
  double best = val;
  int bl = val < kInf ? lane : 99;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(kFull, best, o);
    int ol = __shfl_xor_sync(kFull, bl, o);
    if (ov < best || (ov == best && ol < bl)) {
      best = ov;
      bl = ol;
    }
  }
  ctr_flush(ctr);
  if (lane == 0) {
    g.n_contacts = nc;
    g.ik_converged = worst <= C.contact_tol;
    g.penetration_free = clean[a] ? 1 : 0;
    g.objective = best;
    g.stable = best < C.eps ? 1 : 0;
    g.g = 0;
    m3_store(g.pose_R, x.R);
    v3_store(g.pose_t, x.t);
    g.dof = c_hand.dof;
    for (int j = 0; j < c_hand.dof; ++j) g.q[j] = s_q[w][j];
    dropped[a] = 0;
    valid[a] = (g.penetration_free && g.stable && g.ik_converged) ? 1 : 0;
  }
}

}  // namespace lgd
