// dev_copt.cuh — optimize_contacts (reference contact_opt.cpp:45-142) with a
// register-lean wrench solver (wrench.cpp:124-226).
//
// Layout per warp (one warp = one restart), all in shared memory:
//   incumbent problem  k + s contacts x (p, n, tx, ty, p x n, p x tx, p x ty)
//                      = 21 doubles each;
//   each lane's trial slot (21 doubles) and solver state (alpha, beta_x,
//   beta_y); the incumbent solution (warm start) and the step's winner.
// The solver never stores the backtracking trial state or the gradient:
// projection is per contact, so trial_i = project_i(s_i - step g_i) is
// computed, projected and accumulated contact by contact, and recomputed
// with identical arithmetic when accepted.  In the frictionless descent the
// beta terms are exactly zero and are skipped: force/torque accumulators
// start at +0 and x + (+-0) == x, so every sum is unchanged bit for bit.
// Every other sum keeps the oracle's order (bit-identical results).
#pragma once

#include "dev_stages.cuh"

namespace lgd {

constexpr int kSlot = 21;

// Problem view: contacts from shared memory, slot `tq` from the lane's own
// trial record.
struct PV {
  const double* sp;
  const double* ts;
  int n, tq;
  double lambda, mu;
  __device__ __forceinline__ const double* slot(int i) const { return i == tq ? ts : sp + kSlot * i; }
};

__device__ __forceinline__ V3 ld3(const double* p) { return v3(p[0], p[1], p[2]); }

// write_slot (contact_opt.cpp:31-35) into a 21-double slot record.
__device__ __noinline__ void slot_make(double* o, V3 p, V3 n) {
  V3 tx, ty;
  tangent_basis(n, tx, ty);
  V3 cn = cross(p, n), cx = cross(p, tx), cy = cross(p, ty);
  v3_store(o, p);
  v3_store(o + 3, n);
  v3_store(o + 6, tx);
  v3_store(o + 9, ty);
  v3_store(o + 12, cn);
  v3_store(o + 15, cx);
  v3_store(o + 18, cy);
}

template <bool FR>
__device__ __forceinline__ void proj_one(bool is_anchor, double mu, double& a, double& bx,
                                         double& by) {
  if (is_anchor) a = 1.0;
  else if (a < 0.0) a = 0.0;
  if (!FR) {
    bx = 0.0;
    by = 0.0;
    return;
  }
  double cap = mu * a;
  double r;
  if (lgl::hypot_exceeds(bx, by, cap, &r)) {
    if (cap <= 0.0 || r <= 0.0) {
      bx = 0.0;
      by = 0.0;
    } else {
      double kk = cap / r;
      bx *= kk;
      by *= kk;
    }
  }
}

// force += a n + bx tx + by ty ; torque += a cn + bx cx + by cy
template <bool FR>
__device__ __forceinline__ void acc_contact(const double* s, double a, double bx, double by, V3& f,
                                            V3& t) {
  if (FR) {
    f = add(f, add(add(scale(a, ld3(s + 3)), scale(bx, ld3(s + 6))), scale(by, ld3(s + 9))));
    t = add(t, add(add(scale(a, ld3(s + 12)), scale(bx, ld3(s + 15))), scale(by, ld3(s + 18))));
  } else {
    f = add(f, scale(a, ld3(s + 3)));
    t = add(t, scale(a, ld3(s + 12)));
  }
}

// descend (wrench.cpp:124-177) on state (a, bx, by) in shared memory.  The
// trial state goes to the lane's shared scratch `tr` ([3][NC]) and is copied
// on acceptance instead of being recomputed from the gradient, and the
// accepted trial's force / torque sums serve as the next gradient's.
template <bool FR, int NC>
__device__ double pv_descend(const PV& w, int anchor, int iterations, double step0, int max_bt,
                             double* a, double* bx, double* by, double* tr, Ctr& ctr) {
  #pragma unroll 1
  for (int i = 0; i < w.n; ++i) proj_one<FR>(i == anchor, w.mu, a[i], bx[i], by[i]);
  V3 f = v3(0.0, 0.0, 0.0), t = v3(0.0, 0.0, 0.0);
  #pragma unroll 1
  for (int i = 0; i < w.n; ++i) acc_contact<FR>(w.slot(i), a[i], bx[i], by[i], f, t);
  double current = sqnorm(f) + w.lambda * sqnorm(t);
  ++ctr.weval;
  double* ta = tr;
  double* tbx = tr + NC;
  double* tby = tr + 2 * NC;
  for (int it = 0; it < iterations; ++it) {
    // the gradient's force / torque sums at the current state are exactly the
    // sums of its evaluation (same state, same operations, same order): the
    // initial one, then the accepted trial's
    V3 force = f;
    ++ctr.wgrad;
    V3 torque = v3(t.x * w.lambda, t.y * w.lambda, t.z * w.lambda);
    double step = step0;
    bool moved = false;
    for (int bt = 0; bt <= max_bt; ++bt) {
      V3 f2 = v3(0.0, 0.0, 0.0), t2 = v3(0.0, 0.0, 0.0);
      #pragma unroll 1
      for (int i = 0; i < w.n; ++i) {
        const double* s = w.slot(i);
        double xa = a[i] - step * (2.0 * (dot(force, ld3(s + 3)) + dot(torque, ld3(s + 12))));
        double xbx = 0.0, xby = 0.0;
        if (FR) {
          xbx = bx[i] - step * (2.0 * (dot(force, ld3(s + 6)) + dot(torque, ld3(s + 15))));
          xby = by[i] - step * (2.0 * (dot(force, ld3(s + 9)) + dot(torque, ld3(s + 18))));
        }
        proj_one<FR>(i == anchor, w.mu, xa, xbx, xby);
        acc_contact<FR>(s, xa, xbx, xby, f2, t2);
        ta[i] = xa;
        tbx[i] = xbx;
        tby[i] = xby;
      }
      double next = sqnorm(f2) + w.lambda * sqnorm(t2);
      ++ctr.weval;
      if (next <= current) {
        #pragma unroll 1
        for (int i = 0; i < w.n; ++i) {
          a[i] = ta[i];
          bx[i] = tbx[i];
          by[i] = tby[i];
        }
        f = f2;
        t = t2;
        current = next;
        moved = true;
        break;
      }
      step *= 0.5;
    }
    if (!moved) break;
  }
  return current;
}

// One anchor of run_solver (wrench.cpp:336-367): cold (warm == nullptr) or
// warm-started from `warm` ([3][kMaxC]); state st = [3][kMaxC].
template <int NC>
__device__ __forceinline__ double pv_anchor(const PV& w, int anchor, const WOpts& o,
                                            const double* warm, double* st, double* tr, Ctr& ctr) {
  const int iters = warm ? o.warm_iterations : o.iterations;
  double* a = st;
  double* bx = st + NC;
  double* by = st + 2 * NC;
  #pragma unroll 1
  for (int i = 0; i < w.n; ++i) {
    a[i] = warm ? warm[i] : 1.0;
    bx[i] = warm ? warm[NC + i] : 0.0;
    by[i] = warm ? warm[2 * NC + i] : 0.0;
  }
  if (w.mu > 0.0) {
    pv_descend<false, NC>(w, anchor, iters, o.step, o.max_bt, a, bx, by, tr, ctr);
    return pv_descend<true, NC>(w, anchor, iters, o.step, o.max_bt, a, bx, by, tr, ctr);
  }
  return pv_descend<false, NC>(w, anchor, iters, o.step, o.max_bt, a, bx, by, tr, ctr);
}

// Per-warp shared doubles for problems of at most NC contacts.
template <int NC>
// per-lane doubles: trial slot, state, best, trial state; odd so that the 32
// lanes' records fall in distinct banks (an even multiple of 16 serialises)
constexpr int copt_lane() { return (kSlot + 9 * NC) | 1; }
template <int NC>
constexpr int copt_per_warp() { return NC * kSlot + 6 * NC + 32 * copt_lane<NC>(); }

// Block per candidate, warp per restart, lanes over the n_inner mutations.
// NC = compile-time bound on k + statics (sizes the shared-memory layout).
template <int NC, int MINB>
__global__ void __launch_bounds__(128, MINB)
k_contact_opt2(int nA, const int* alive_idx, CoptCfg cfg, const int* n_static, const double* st_p,
               const double* st_n, const long long* el_off, const double* el_p, const double* el_n,
               const uint64_t* draws, int* out_ids, double* out_obj, int* out_anchor,
               double* out_sol, double eps_stable, int* balanced) {
  extern __shared__ __align__(16) double s_co[];
  const int a = blockIdx.x;
  if (a >= nA) return;
  const int i = alive_idx[a];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int k = cfg.k;
  const int s = n_static[i];
  const int n = k + s;
  double* W = s_co + warp * copt_per_warp<NC>();
  double* sp = W;                        // incumbent problem
  double* inc = W + NC * kSlot;       // incumbent solution (warm start)
  double* win = inc + 3 * NC;         // best mutation's solution of this step
  double* lane_base = win + 3 * NC;   // per lane: trial slot, working state, best state
  double* tslot = lane_base + lane * copt_lane<NC>();
  double* wst = tslot + kSlot;
  double* bst = wst + 3 * NC;
  double* tst = bst + 3 * NC;
  const int rstride = 2 + k + 3 * NC;
  double* res = s_co + nw * copt_per_warp<NC>();
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
      int ids[kMaxK];
      #pragma unroll 1
      for (int q = 0; q < k; ++q) ids[q] = (int)(D[q] % (uint64_t)cnt[q]);
      if (lane < k) {
        long long e = off[lane] + ids[lane];
        slot_make(sp + kSlot * lane, v3_load(el_p + 3 * e), neg(v3_load(el_n + 3 * e)));
      } else if (lane == k && s) {
        slot_make(sp + kSlot * k, v3_load(st_p + 3 * i), v3_load(st_n + 3 * i));
      }
      __syncwarp();
      PV w;
      w.sp = sp;
      w.ts = tslot;
      w.n = n;
      w.tq = -1;
      w.lambda = cfg.lambda;
      w.mu = cfg.mu;
      // cold solve: lanes over anchors, best anchor by strict '<'
      double val = kInf;
      if (lane < n) val = pv_anchor<NC>(w, lane, cfg.o, nullptr, wst, tst, ctr);
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
      int anchor = best < kInf ? bl : -1;
      double obj = best;
      __syncwarp();
      if (lane < 3 * NC)
        inc[lane] = anchor >= 0 ? lane_base[anchor * copt_lane<NC>() + kSlot + lane] : 0.0;
      __syncwarp();
      const uint64_t* M = D + k;
      for (int outer = 0; outer < cfg.n_outer; ++outer) {
        for (int q = 0; q < k; ++q) {
          const double* cs = sp + kSlot * q;
          V3 cur_p = ld3(cs);
          V3 tx, ty;
          tangent_basis(ld3(cs + 3), tx, ty);  // slot normal = -element normal
          double best_obj = obj;
          int best_id = -1, best_anchor = -1;
          for (int mb = 0; mb < cfg.n_inner; mb += 32) {
            const int m = mb + lane;
            double v = kInf;
            int cand = -1, an = -1;
            if (m < cfg.n_inner) {
              const uint64_t* d2 = M + 2 * ((long long)(outer * k + q) * cfg.n_inner + m);
              // (sigma z1, sigma z2), precomputed by k_copt_normals
              const double u = __longlong_as_double((long long)d2[0]);
              const double vv = __longlong_as_double((long long)d2[1]);
              V3 cp = axpy(axpy(cur_p, u, tx), vv, ty);
              // project_to_domain (contact_opt.cpp:11-25): nearest element,
              // first index among equal distances.  Every lane scans the same
              // elements (broadcast loads, no divergence); pruned searches
              // (x-sorted, object-frame grid) evaluate far fewer distances but
              // diverge and measured slower.
              const double* P = el_p + 3 * off[q];
              const int ne = (int)cnt[q];
              double bd;
              int bi;
              // Every lane scans the same elements (broadcast loads, no
              // divergence): faster than the pruned search for domains of
              // a few thousand elements.
              bd = sqnorm(sub(v3(P[0], P[1], P[2]), cp));
              bi = 0;
              int e = 1;
              // peel to an even global element (16-byte aligned pairs)
              if (e < ne && ((off[q] + e) & 1)) {
                double d2v = sqnorm(sub(v3(P[3 * e], P[3 * e + 1], P[3 * e + 2]), cp));
                if (d2v < bd) {
                  bd = d2v;
                  bi = e;
                }
                ++e;
              }
              // eight independent distances in flight (twelve 16-byte
              // loads: the domain streams from L2), compared in index order
              for (; e + 8 <= ne; e += 8) {
                const double2* Q = reinterpret_cast<const double2*>(P + 3 * e);
                double2 a0 = Q[0], a1 = Q[1], a2 = Q[2], a3 = Q[3], a4 = Q[4], a5 = Q[5];
                double2 b0 = Q[6], b1 = Q[7], b2 = Q[8], b3 = Q[9], b4 = Q[10], b5 = Q[11];
                double d0 = sqnorm(sub(v3(a0.x, a0.y, a1.x), cp));
                double d1 = sqnorm(sub(v3(a1.y, a2.x, a2.y), cp));
                double d2 = sqnorm(sub(v3(a3.x, a3.y, a4.x), cp));
                double d3 = sqnorm(sub(v3(a4.y, a5.x, a5.y), cp));
                double d4 = sqnorm(sub(v3(b0.x, b0.y, b1.x), cp));
                double d5 = sqnorm(sub(v3(b1.y, b2.x, b2.y), cp));
                double d6 = sqnorm(sub(v3(b3.x, b3.y, b4.x), cp));
                double d7 = sqnorm(sub(v3(b4.y, b5.x, b5.y), cp));
                if (d0 < bd) { bd = d0; bi = e; }
                if (d1 < bd) { bd = d1; bi = e + 1; }
                if (d2 < bd) { bd = d2; bi = e + 2; }
                if (d3 < bd) { bd = d3; bi = e + 3; }
                if (d4 < bd) { bd = d4; bi = e + 4; }
                if (d5 < bd) { bd = d5; bi = e + 5; }
                if (d6 < bd) { bd = d6; bi = e + 6; }
                if (d7 < bd) { bd = d7; bi = e + 7; }
              }
              for (; e + 4 <= ne; e += 4) {
                const double2* Q = reinterpret_cast<const double2*>(P + 3 * e);
                double2 a0 = Q[0], a1 = Q[1], a2 = Q[2], a3 = Q[3], a4 = Q[4], a5 = Q[5];
                double d0 = sqnorm(sub(v3(a0.x, a0.y, a1.x), cp));
                double d1 = sqnorm(sub(v3(a1.y, a2.x, a2.y), cp));
                double d2 = sqnorm(sub(v3(a3.x, a3.y, a4.x), cp));
                double d3 = sqnorm(sub(v3(a4.y, a5.x, a5.y), cp));
                if (d0 < bd) { bd = d0; bi = e; }
                if (d1 < bd) { bd = d1; bi = e + 1; }
                if (d2 < bd) { bd = d2; bi = e + 2; }
                if (d3 < bd) { bd = d3; bi = e + 3; }
              }
              for (; e < ne; ++e) {
                double d2v = sqnorm(sub(v3(P[3 * e], P[3 * e + 1], P[3 * e + 2]), cp));
                if (d2v < bd) {
                  bd = d2v;
                  bi = e;
                }
              }
              ctr.proj += (unsigned long long)ne;
              cand = bi;
              const long long eg = off[q] + bi;
              slot_make(tslot, v3_load(el_p + 3 * eg), neg(v3_load(el_n + 3 * eg)));
              PV tw = w;
              tw.tq = q;
              // warm solve over all anchors in this lane (run_solver)
              double bobj = kInf;
              for (int anc = 0; anc < n; ++anc) {
                double va = pv_anchor<NC>(tw, anc, cfg.o, anchor >= 0 ? inc : nullptr, wst, tst, ctr);
                if (va < bobj) {
                  bobj = va;
                  an = anc;
                  for (int c = 0; c < 3 * NC; ++c) bst[c] = wst[c];
                }
              }
              v = bobj;
            }
            double bv = (v < best_obj) ? v : kInf;
            int bm = (v < best_obj) ? m : 0x7fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              double ov = __shfl_xor_sync(kFull, bv, o);
              int om = __shfl_xor_sync(kFull, bm, o);
              if (ov < bv || (ov == bv && om < bm)) {
                bv = ov;
                bm = om;
              }
            }
            if (bm != 0x7fffffff) {
              int src = bm - mb;
              best_obj = bv;
              best_id = __shfl_sync(kFull, cand, src);
              best_anchor = __shfl_sync(kFull, an, src);
              __syncwarp();
              // keep the winner's state before the next chunk reuses it; the
              // warm start (inc) stays the step's incumbent until the end
              if (lane < 3 * NC) win[lane] = lane_base[src * copt_lane<NC>() + kSlot + 3 * NC + lane];
              __syncwarp();
            }
          }
          if (best_id >= 0) {
            ids[q] = best_id;
            if (lane == 0) {
              long long e = off[q] + best_id;
              slot_make(sp + kSlot * q, v3_load(el_p + 3 * e), neg(v3_load(el_n + 3 * e)));
            }
            if (lane < 3 * NC) inc[lane] = win[lane];
            __syncwarp();
            obj = best_obj;
            anchor = best_anchor;
          }
        }
      }
      if (lane == 0) {
        double* R = res + warp * rstride;
        R[0] = obj;
        R[1] = (double)anchor;
        #pragma unroll 1
        for (int q = 0; q < k; ++q) R[2 + q] = (double)ids[q];
        for (int c = 0; c < 3 * NC; ++c) R[2 + k + c] = anchor >= 0 ? inc[c] : 0.0;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double* best = res + nw * rstride;
      for (int w2 = 0; w2 < nw && rbase + w2 < cfg.restarts; ++w2) {
        double* R = res + w2 * rstride;
        bool first = (rbase + w2) == 0;
        if (first || R[0] < best[0])
          for (int t = 0; t < rstride; ++t) best[t] = R[t];
        if (first && !(R[0] < kInf)) best[0] = kInf;
      }
    }
    __syncthreads();
  }
  ctr_flush(ctr);
  if (threadIdx.x == 0) {
    double* best = res + nw * rstride;
    out_obj[a] = best[0];
    int an = (int)best[1];
    if (!(best[0] < kInf)) an = -1;
    out_anchor[a] = an;
    #pragma unroll 1
    for (int q = 0; q < k; ++q) out_ids[a * kMaxK + q] = (int)best[2 + q];
    for (int c = 0; c < 3 * kMaxC; ++c) {
      int comp = c / kMaxC, ci = c % kMaxC;  // output keeps the [3][kMaxC] layout
      out_sol[a * 3 * kMaxC + c] = ci < NC ? best[2 + k + comp * NC + ci] : 0.0;
    }
    balanced[a] = (an >= 0 && best[0] < eps_stable) ? 1 : 0;
  }
}

template <int NC>
__host__ __forceinline__ size_t copt2_smem(int k, int nw) {
  return ((size_t)nw * copt_per_warp<NC>() + (size_t)(nw + 1) * (2 + k + 3 * NC)) * sizeof(double);
}

}  // namespace lgd
