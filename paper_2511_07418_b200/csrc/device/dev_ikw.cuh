// dev_ikw.cuh — warp-cooperative realize_grasp / solve_contact_ik: one warp
// per problem (reference ik.cpp:31-139, pipeline.cpp:185-253).
//
// Lane roles (all summations keep the oracle's exact order, so results are
// bit-identical to the serial restatement):
//   - FK: lane l computes link l's local transform, then frames are composed
//     level by level in shared memory, frames[l] = frames[parent] * local_l,
//     the same operations as the topological-order FK (hand.cpp:275-295).
//   - Jacobian: lane j owns joint column j; rows are streamed per target point.
//   - J^T J: lanes own entries (a <= b), each a row-ordered sum; mirrored.
//   - LDLT (Eigen, diagonal pivoting): lane i owns row i of the trailing
//     update; pivot = warp argmax (first index on ties).
//   - triangular solves: lane i keeps a running sum that accumulates terms in
//     the order the unknowns become final (ascending forward, descending
//     backward: the canonical orders of oracle/orc_core.cpp ldlt_solve).
#pragma once

#include "dev_ik.cuh"

namespace lgd {

constexpr unsigned kFull = 0xffffffffu;
// Shared-memory stride of one link frame (R row-major, t): 13 doubles, odd,
// so lanes reading different links' frames hit distinct banks.
constexpr int kFS = 13;

__device__ __forceinline__ Xf ld_xf(const double* p) {
  Xf x;
  x.R = m3_load(p);
  x.t = v3_load(p + 9);
  return x;
}
__device__ __forceinline__ void st_xf(double* p, const Xf& x) {
  m3_store(p, x.R);
  v3_store(p + 9, x.t);
}

// Pre-motion origin composed with the joint motion qv (hand.cpp:281-290).
__device__ __forceinline__ Xf link_local_v(int l, double qv) {
  Xf local;
  local.R = m3_load(g_hand.R[l]);
  local.t = v3_load(g_hand.t[l]);
  int jt = g_hand.jtype[l];
  if (jt == 1) {
    Xf m;
    m.R = angle_axis(qv, v3_load(g_hand.axis[l]));
    m.t = v3(0.0, 0.0, 0.0);
    local = xf_compose(local, m);
  } else if (jt == 2) {
    local.t = add(local.t, mul(local.R, scale(qv, v3_load(g_hand.axis[l]))));
  }
  return local;
}
__device__ __forceinline__ Xf link_local(int l, const double* q) {
  int j = g_hand.jidx[l];
  return link_local_v(l, j >= 0 ? q[j] : 0.0);
}

// forward_kinematics into shared memory F[n_links][12], q in shared memory.
__device__ __forceinline__ void wfk_s(const double* q, double* F, int lane) {
  const int nl = c_hand.n_links;
  Xf loc = xf_identity();
  int lvl = -1, p = -1;
  if (lane < nl) {
    loc = link_local(lane, q);
    lvl = g_hand.level[lane];
    p = g_hand.parent[lane];
  }
  for (int d = 0; d < c_hand.n_levels; ++d) {
    if (lvl == d) st_xf(F + kFS * lane, p < 0 ? loc : xf_compose(ld_xf(F + kFS * p), loc));
    __syncwarp();
  }
}

// Target layout in shared memory: [k][12] = op(3) on(3) hp(3) hn(3); links [k].
struct WTargets {
  double* t;
  int* link;
};

// The links the contact IK can see: the union of the root -> target-link
// chains.  The residual reads target-link frames and every nonzero Jacobian
// column belongs to a joint on a target chain, so solve_contact_ik never
// needs any other frame; FK is evaluated on these m links only, in G = 32/m
// lane groups (up to 4), one backtracking trial per group.
struct WChain {
  int m, G, maxlvl;
  int *link, *pslot, *lvl, *sol, *tslot, *hdr;
};
constexpr int kChainInts = 4 * kMaxLinks + kMaxK + 2;

__device__ __forceinline__ void wchain_build(WChain& C, const int* tlink, int k, int lane) {
  if (lane == 0) {
    const int nl = c_hand.n_links;
    int m = 0, maxl = 0;
    for (int l = 0; l < nl; ++l) {
      bool need = false;
      for (int i = 0; i < k; ++i) {
        int t = tlink[i];
        #pragma unroll 1
        for (int d = 0; d < g_hand.chain_len[t]; ++d) need |= g_hand.chain[t][d] == l;
      }
      // links with no joint on their chain (the palm) have constant frames:
      // computed once (wchain_static), not per trial
      const bool moving = need && g_hand.jmask[l] != 0u;
      C.sol[l] = moving ? m : (need ? -2 - l : -1);
      if (moving) {
        C.link[m] = l;
        C.lvl[m] = g_hand.level[l];
        maxl = C.lvl[m] > maxl ? C.lvl[m] : maxl;
        ++m;
      }
    }
    for (int j = 0; j < m; ++j) {  // slot, -1 (no parent) or -2 - static parent link
      int p = g_hand.parent[C.link[j]];
      C.pslot[j] = p >= 0 ? C.sol[p] : -1;
    }
    for (int i = 0; i < k; ++i) C.tslot[i] = C.sol[tlink[i]];
    C.hdr[0] = m;
    C.hdr[1] = maxl;
  }
  __syncwarp();
  C.m = C.hdr[0];
  C.maxlvl = C.hdr[1];
  int g = C.m > 0 ? 32 / C.m : 1;
  C.G = g > 4 ? 4 : g;
}

// Constant frames of the static chain links (no joint from the root) into
// the link-indexed buffer F, in level order, by one lane.
__device__ __forceinline__ void wchain_static(const int* tlink, int k, double* F, int lane) {
  if (lane == 0) {
    const int nl = c_hand.n_links;
    for (int d = 0; d < c_hand.n_levels; ++d)
      for (int l = 0; l < nl; ++l) {
        if (g_hand.level[l] != d || g_hand.jmask[l] != 0u) continue;
        bool need = false;
        for (int i = 0; i < k; ++i) {
          int t = tlink[i];
          #pragma unroll 1
          for (int e = 0; e < g_hand.chain_len[t]; ++e) need |= g_hand.chain[t][e] == l;
        }
        if (!need) continue;
        Xf loc = link_local_v(l, 0.0);
        int p = g_hand.parent[l];
        st_xf(F + kFS * l, p < 0 ? loc : xf_compose(ld_xf(F + kFS * p), loc));
      }
  }
  __syncwarp();
}

// Joint value of backtracking trial b: q + clamp(dq / 2^b) clamped to the
// limits, dq halved b times as the sequential line search does.
__device__ __forceinline__ double trial_joint(const double* q, const double* dq, int j, int b,
                                              double step_clamp) {
  double d = dq[j];
  #pragma unroll 1
  for (int h = 0; h < b; ++h) d *= 0.5;
  return dclamp(q[j] + dmin(dmax(d, -step_clamp), step_clamp), g_hand.jlo[j], g_hand.jhi[j]);
}

// FK of the chain links for ng groups into FG[g][m][kFS]; group g uses trial
// b0 + g, or q itself when b0 < 0 (one group).
__device__ __forceinline__ void wchain_fk(const WChain& C, double* FG, const double* F, int ng,
                                         const double* q, const double* dq, int b0,
                                         double step_clamp, int lane) {
  const bool on = lane < ng * C.m;
  const int g = on ? lane / C.m : 0, j = on ? lane - g * C.m : 0;
  Xf loc = xf_identity();
  int lv = -1, ps = -1;
  if (on) {
    int l = C.link[j];
    int jl = g_hand.jidx[l];
    double qv = 0.0;
    if (jl >= 0) qv = b0 < 0 ? q[jl] : trial_joint(q, dq, jl, b0 + g, step_clamp);
    loc = link_local_v(l, qv);
    lv = C.lvl[j];
    ps = C.pslot[j];
  }
  double* Fg = FG + (size_t)g * C.m * kFS;
  #pragma unroll 1
  for (int d = 0; d <= C.maxlvl; ++d) {
    if (lv == d)
      st_xf(Fg + kFS * j, ps == -1 ? loc
                                   : xf_compose(ld_xf(ps >= 0 ? Fg + kFS * ps : F + kFS * (-2 - ps)), loc));
    __syncwarp();
  }
}

// Chain frames of group g -> link-indexed frames F.
__device__ __forceinline__ void wchain_commit(const WChain& C, const double* FG, int g, double* F,
                                             int lane) {
  if (lane < C.m) {
    const double* src = FG + ((size_t)g * C.m + lane) * kFS;
    double* dst = F + kFS * C.link[lane];
    for (int a = 0; a < 12; ++a) dst[a] = src[a];
  }
  __syncwarp();
}

// Warp max of v.  Finite doubles with a clear sign bit (so not -0.0) order
// like their bit patterns, so the common case is two 32-bit warp
// reductions; anything else takes the comparison butterfly.
__device__ __forceinline__ double warp_max_d(double v) {
  if (__all_sync(kFull, __double_as_longlong(v) >= 0 && v <= 1.7976931348623157e308)) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    unsigned hi = __reduce_max_sync(kFull, (unsigned)(b >> 32));
    unsigned lo = __reduce_max_sync(kFull, (unsigned)(b >> 32) == hi ? (unsigned)b : 0u);
    return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// stacked_residual (ik.cpp:13-27): lanes < k fill r[6i..6i+5]; returns the
// row-ordered sum of squares (computed by lane 0, broadcast).
__device__ __forceinline__ double wresidual(const double* F, const WTargets& T, int k, double beta,
                                            double* r, int lane) {
  if (lane < k) {
    Xf Fl = ld_xf(F + kFS * T.link[lane]);
    const double* t = T.t + 12 * lane;
    V3 op = v3_load(t), on = v3_load(t + 3);
    V3 hp = xf_apply(Fl, v3_load(t + 6));
    V3 hn = xf_rotate(Fl, v3_load(t + 9));
    V3 a = sub(op, hp);
    V3 b = sub(axpy(op, beta, on), axpy(hp, beta, hn));
    double* o = r + 6 * lane;
    o[0] = a.x;
    o[1] = a.y;
    o[2] = a.z;
    o[3] = b.x;
    o[4] = b.y;
    o[5] = b.z;
  }
  __syncwarp();
  double s = 0.0;
  if (lane == 0)
    #pragma unroll 4
    for (int i = 0; i < 6 * k; ++i) s = s + r[i] * r[i];
  return __shfl_sync(kFull, s, 0);
}

struct WarpWs {
  double *J, *A, *r, *rt, *x, *qt, *pts;
  int* tr;
};

__host__ __device__ __forceinline__ size_t warp_ws_bytes(int k, int dof) {
  size_t d = (size_t)6 * k * dof + (size_t)dof * (dof | 1) + 12 * k + 2 * dof + 6 * k;
  return (d * sizeof(double) + (size_t)dof * sizeof(int) + 15) & ~(size_t)15;
}

__device__ __forceinline__ WarpWs warp_ws(char* base, int k, int dof) {
  WarpWs w;
  double* p = (double*)base;
  w.J = p;
  p += 6 * k * dof;
  w.A = p;
  p += dof * (dof | 1);
  w.r = p;
  p += 6 * k;
  w.rt = p;
  p += 6 * k;
  w.x = p;
  p += dof;
  w.qt = p;
  p += dof;
  w.pts = p;
  p += 6 * k;
  w.tr = (int*)p;
  return w;
}

// Final position of each diagonal entry under Eigen's diagonal pivoting
// (ldlt_inplace: step k swaps position k with the first position holding the
// largest |A(i,i)|, i >= k).  Only the diagonal decides, and at step k its
// entries i >= k are still the original ones (the left-looking update writes
// column k only; the swaps move diagonal entries as a whole), so the pivot
// order is fixed before the factorization.  Lane a < n holds v = A(a,a), not
// NaN; returns a's final position.  Non-negative doubles order like their
// bit patterns: the maximum is two 32-bit warp reductions and the first
// position among its holders a third.
__device__ __forceinline__ int pivot_positions(double v, int n, int lane) {
  const unsigned long long bits =
      lane < n ? (unsigned long long)__double_as_longlong(dabs(v)) : 0ull;
  int pos = lane;
  #pragma unroll 1
  for (int k = 0; k + 1 < n; ++k) {
    const bool act = lane < n && pos >= k;
    const unsigned hi = __reduce_max_sync(kFull, act ? (unsigned)(bits >> 32) : 0u);
    const bool t1 = act && (unsigned)(bits >> 32) == hi;
    const unsigned lo = __reduce_max_sync(kFull, t1 ? (unsigned)bits : 0u);
    const bool t2 = t1 && (unsigned)bits == lo;
    const int big = (int)__reduce_min_sync(kFull, t2 ? (unsigned)pos : 0xffffffffu);
    if (act && pos == k) pos = big;        // the entry at k moves to big
    else if (t2 && pos == big) pos = k;    // the pivot moves to k
  }
  return pos;
}

// Eigen LDLT factor + solve, warp-parallel; A (n x n, smem, lower triangle
// read and written) destroyed, x (smem) rhs in / solution out.  piv: pivot
// during the factorization (A and x in their original order); otherwise A
// and x are already symmetrically permuted to the pivot order (lane a's
// entry at position pos) and the solution is scattered back through pos.
__device__ __forceinline__ void wldlt_solve(int n, int ld, double* A, double* x, bool piv, int pos,
                                            double* tmp, int lane) {
  // pidx: the transpositions applied so far to the index vector (lane i
  // holds entry i), so P^T b is a gather and P y a scatter at the end
  int pidx = lane;
  #pragma unroll 1
  for (int k = 0; k < n; ++k) {
    if (piv) {
      // pivot = first index of max |A(i,i)|, i >= k.  Non-negative doubles
      // order like their bit patterns, so the max is two 32-bit warp
      // reductions (high word, then low word among the ties) and the first
      // lane holding it; a NaN diagonal takes the comparison-based reduction.
      const bool act = lane >= k && lane < n;
      double v = act ? dabs(A[lane * ld + lane]) : -1.0;
      int big;
      if (!__any_sync(kFull, act && v != v)) {
        unsigned long long bits = (unsigned long long)__double_as_longlong(v);
        unsigned hi = __reduce_max_sync(kFull, act ? (unsigned)(bits >> 32) : 0u);
        bool tie = act && (unsigned)(bits >> 32) == hi;
        unsigned lo = __reduce_max_sync(kFull, tie ? (unsigned)bits : 0u);
        big = __ffs(__ballot_sync(kFull, tie && (unsigned)bits == lo)) - 1;
      } else {
        int idx = act ? lane : 0x7fff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          double ov = __shfl_xor_sync(kFull, v, o);
          int oi = __shfl_xor_sync(kFull, idx, o);
          if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
          }
        }
        big = idx;
      }
      if (k != big) {
        const int pk = __shfl_sync(kFull, pidx, k), pb = __shfl_sync(kFull, pidx, big);
        if (lane == k) pidx = pb;
        else if (lane == big) pidx = pk;
        if (lane < k) {
          double t = A[k * ld + lane];
          A[k * ld + lane] = A[big * ld + lane];
          A[big * ld + lane] = t;
        }
        if (lane > big && lane < n) {
          double t = A[lane * ld + k];
          A[lane * ld + k] = A[lane * ld + big];
          A[lane * ld + big] = t;
        }
        if (lane == 0) {
          double t = A[k * ld + k];
          A[k * ld + k] = A[big * ld + big];
          A[big * ld + big] = t;
        }
        if (lane > k && lane < big) {
          double u = A[lane * ld + k];
          A[lane * ld + k] = A[big * ld + lane];
          A[big * ld + lane] = u;
        }
        __syncwarp();
      }
    }
    if (k > 0) {
      // temp_j = D_j * A(k, j), j < k, broadcast through shared memory
      if (lane < k) tmp[lane] = A[lane * ld + lane] * A[k * ld + lane];
      __syncwarp();
      if (lane >= k && lane < n) {
        double acc = 0.0;
        const double* row = A + lane * ld;
        #pragma unroll 4
        for (int j = 0; j < k; ++j) acc = acc + row[j] * tmp[j];
        A[lane * ld + k] -= acc;  // lane k: A(k,k); lanes > k: A21
      }
      __syncwarp();
    }
    double akk = A[k * ld + k];
    if (dabs(akk) > 0.0 && lane > k && lane < n) A[lane * ld + k] /= akk;
    __syncwarp();
  }
  double xi = lane < n ? x[pidx] : 0.0;  // P^T b (the forward transpositions; identity if !piv)
  __syncwarp();
  double s = 0.0;
  #pragma unroll 1
  for (int j = 0; j < n; ++j) {  // forward: L unit lower
    double xj = __shfl_sync(kFull, xi - s, j);
    if (lane == j) xi = xj;
    if (lane > j && lane < n) s = s + A[lane * ld + j] * xj;
  }
  if (lane < n) {
    double d = A[lane * ld + lane];
    if (dabs(d) > 2.2250738585072014e-308) xi /= d;
    else xi = 0.0;
  }
  s = 0.0;
  #pragma unroll 1
  for (int j = n - 1; j >= 0; --j) {  // backward: L^T
    double xj = __shfl_sync(kFull, xi - s, j);
    if (lane == j) xi = xj;
    if (lane < j) s = s + A[j * ld + lane] * xj;
  }
  if (piv) {
    if (lane < n) x[pidx] = xi;  // P y (the transpositions in reverse order)
  } else {
    const double y = __shfl_sync(kFull, xi, pos & 31);
    if (lane < n) x[lane] = y;
  }
  __syncwarp();
}

// solve_contact_ik (ik.cpp:31-139).  q (smem) in/out; F (smem) receives the
// frames at the final q; Ft is trial scratch.  Returns finite; used = OR of
// joints with a nonzero column.
__device__ __forceinline__ bool wik(double* q, const WTargets& T, int k, const IkCfg& P, int iterations,
                    unsigned long long& used, WarpWs& ws, double* F, const WChain& C, double* FG,
                    double* rtG, bool have_frames, const unsigned short* ab, Ctr& ctr, int lane,
                    int* it_out = nullptr, double* obj_out = nullptr) {
  const int dof = c_hand.dof;
  const int ld = dof | 1;  // odd row stride: column accesses hit distinct banks
  const int rows = 6 * k;
  if (lane < dof) q[lane] = dclamp(q[lane], g_hand.jlo[lane], g_hand.jhi[lane]);
  __syncwarp();
  used = 0ull;
  // A finetune round starts at the accepted q whose chain frames F already
  // holds (same FK, same inputs), and q is within its limits, so the clamp
  // above is the identity; only the first solve needs the FK.
  if (!have_frames) {
    wchain_fk(C, FG, F, 1, q, nullptr, -1, 0.0, lane);
    wchain_commit(C, FG, 0, F, lane);
  }
  ++ctr.fk;
  if (it_out) {  // IkResult.iterations / objective of the k == 0 early return
    *it_out = 0;
    *obj_out = 0.0;
  }
  if (k == 0) return true;
  bool finite = true;
  double* r = ws.r;
  double objective = wresidual(F, T, k, P.beta, r, lane);
  int iters = 0;
  for (int it = 0; it < iterations; ++it) {
    ++ctr.ik_it;
    iters = it + 1;
    // Jacobian points: lane p < 2k -> target p/2, half p%2
    if (lane < 2 * k) {
      int i = lane >> 1;
      Xf Fl = ld_xf(F + kFS * T.link[i]);
      const double* t = T.t + 12 * i;
      V3 lp = (lane & 1) ? axpy(v3_load(t + 6), P.beta, v3_load(t + 9)) : v3_load(t + 6);
      v3_store(ws.pts + 3 * lane, xf_apply(Fl, lp));
    }
    __syncwarp();
    // joint columns
    if (lane < dof) {
      int lj = g_hand.jlink[lane];
      Xf Fj = ld_xf(F + kFS * lj);
      V3 axis = mul(Fj.R, v3_load(g_hand.axis[lj]));
      bool rev = g_hand.jtype[lj] == 1;
      double cm = 0.0;
      #pragma unroll 1
      for (int p = 0; p < 2 * k; ++p) {
        bool on = (c_hand.jmask[T.link[p >> 1]] >> lane) & 1u;
        V3 col = v3(0.0, 0.0, 0.0);
        if (on) col = rev ? cross(axis, sub(v3_load(ws.pts + 3 * p), Fj.t)) : axis;
        int row = 3 * p;  // 6i + 3h
        ws.J[(row + 0) * dof + lane] = col.x;
        ws.J[(row + 1) * dof + lane] = col.y;
        ws.J[(row + 2) * dof + lane] = col.z;
        cm = dmax(cm, dabs(col.x));
        cm = dmax(cm, dabs(col.y));
        cm = dmax(cm, dabs(col.z));
      }
      if (cm > 1e-12) used |= 1ull << lane;
    }
    used = __reduce_or_sync(kFull, (unsigned)used);  // dof <= 32: one word
    __syncwarp();
    // J^T J entries (a <= b) e < ne and J^T r entries ne <= e < ne + dof
    // share one branch-free loop (same row-ordered dot product: column a of
    // J against column b of J, or against r).  Off-diagonal entries are
    // staged in the upper triangle, the diagonal in qt.
    const int ne = dof * (dof + 1) / 2;
    for (int e = lane; e < ne + dof; e += 32) {
      const bool jj = e < ne;
      const int a = jj ? (ab[e] & 0xff) : e - ne, b = jj ? (ab[e] >> 8) : 0;
      const double* o2 = jj ? ws.J + b : r;
      const int st2 = jj ? dof : 1;
      double s = 0.0;
      #pragma unroll 4
      for (int rr = 0; rr < rows; ++rr) s = s + ws.J[rr * dof + a] * o2[rr * st2];
      if (!jj) ws.x[a] = s;
      else if (a == b) ws.qt[a] = s;
      else ws.A[a * ld + b] = s;
    }
    __syncwarp();
    double tr = 0.0;
    if (lane == 0)
      #pragma unroll 4
      for (int a = 0; a < dof; ++a) tr = tr + ws.qt[a];
    tr = __shfl_sync(kFull, tr, 0);
    double lambda = dmax(P.damping_min, P.damping_scale * tr / (double)(dof > 1 ? dof : 1));
    // damped diagonal; the pivot order it implies is applied to A and J^T r
    // as they move to the lower triangle (a NaN diagonal keeps the original
    // order and pivots during the factorization)
    const double dv = lane < dof ? ws.qt[lane] + lambda : 0.0;
    const bool piv = __any_sync(kFull, lane < dof && dv != dv);
    const int pos = piv ? lane : pivot_positions(dv, dof, lane);
    const double bv = lane < dof ? ws.x[lane] : 0.0;
    if (lane < dof) ws.tr[lane] = pos;
    __syncwarp();
    if (lane < dof) {
      ws.A[pos * ld + pos] = dv;
      ws.x[pos] = bv;
    }
    for (int e = lane; e < ne; e += 32) {
      const int a = ab[e] & 0xff, b = ab[e] >> 8;
      if (a == b) continue;
      const int pa = ws.tr[a], pb = ws.tr[b];
      ws.A[(pa > pb ? pa : pb) * ld + (pa > pb ? pb : pa)] = ws.A[a * ld + b];
    }
    __syncwarp();
    wldlt_solve(dof, ld, ws.A, ws.x, piv, pos, ws.qt, lane);
    bool bad = lane < dof && !is_finite(ws.x[lane]);
    if (__any_sync(kFull, bad)) {
      finite = false;
      break;
    }
    // backtracking line search, G trials at a time; the first trial (in
    // order) with obj <= objective is the one the sequential search keeps
    bool moved = false;
    const int rk = 6 * k;
    for (int b0 = 0; b0 <= P.max_backtracks && !moved; b0 += C.G) {
      const int ng = (P.max_backtracks + 1 - b0) < C.G ? (P.max_backtracks + 1 - b0) : C.G;
      wchain_fk(C, FG, F, ng, q, ws.x, b0, P.step_clamp, lane);
      ctr.fk += ng;
      if (lane < ng * k) {  // stacked_residual (ik.cpp:13-27) per group
        int g = lane / k, i = lane - g * k;
        const int ts = C.tslot[i];  // a static target link's frame is constant
        Xf Fl = ld_xf(ts >= 0 ? FG + ((size_t)g * C.m + ts) * kFS : F + kFS * (-2 - ts));
        const double* tt = T.t + 12 * i;
        V3 op = v3_load(tt), on = v3_load(tt + 3);
        V3 hp = xf_apply(Fl, v3_load(tt + 6));
        V3 hn = xf_rotate(Fl, v3_load(tt + 9));
        V3 a = sub(op, hp);
        V3 bb = sub(axpy(op, P.beta, on), axpy(hp, P.beta, hn));
        double* o = rtG + g * rk + 6 * i;
        o[0] = a.x;
        o[1] = a.y;
        o[2] = a.z;
        o[3] = bb.x;
        o[4] = bb.y;
        o[5] = bb.z;
      }
      __syncwarp();
      double obj_try = 0.0;
      if (lane < ng)
        #pragma unroll 4
        for (int i = 0; i < rk; ++i) obj_try = obj_try + rtG[lane * rk + i] * rtG[lane * rk + i];
      unsigned accm = __ballot_sync(kFull, lane < ng && obj_try <= objective);
      if (accm) {
        const int g = __ffs(accm) - 1;
        objective = __shfl_sync(kFull, obj_try, g);
        if (lane < dof) q[lane] = trial_joint(q, ws.x, lane, b0 + g, P.step_clamp);
        if (lane < rk) r[lane] = rtG[g * rk + lane];
        wchain_commit(C, FG, g, F, lane);
        moved = true;
      }
    }
    if (!moved) break;
    double mp = 0.0;
    if (lane < k) mp = norm(v3(r[6 * lane], r[6 * lane + 1], r[6 * lane + 2]));
    mp = warp_max_d(mp);
    if (mp < P.residual_tol) break;
  }
  bool nonfin = lane < dof && !is_finite(q[lane]);
  if (__any_sync(kFull, nonfin)) finite = false;
  if (it_out) {
    *it_out = iters;
    *obj_out = objective;
  }
  return finite;
}

// realize_grasp's project (pipeline.cpp:196-220) at frames F: worst
// distance (all lanes), optionally refreshing hand points into R.
__device__ __noinline__ double wproject(const double* F, const WTargets& T, int k, WTargets* R,
                                           int lane) {
  double d = 0.0;
  if (lane < k) {
    Xf inv = xf_inverse(ld_xf(F + kFS * T.link[lane]));
    V3 sp = v3(0, 0, 0), sn = v3(0, 0, 0);
    d = closest_on_parts(T.link[lane], xf_apply(inv, v3_load(T.t + 12 * lane)), &sp, &sn);
    if (R) {
      v3_store(R->t + 12 * lane + 6, sp);
      v3_store(R->t + 12 * lane + 9, sn);
    }
  }
  __syncwarp();
  // worst = std::max(worst, d) from worst = 0.0: the max of +0.0 and the
  // non-NaN distances, so clamping each lane first gives the same value
  // (negative, -0.0 and NaN distances all leave +0.0) and keeps the
  // reduction on its two-word fast path when contacts penetrate
  return warp_max_d(0.0 < d ? d : 0.0);
}

// realize_grasp (pipeline.cpp:185-253) for one warp; q (smem) starts at q0.
// One solve site serves the initial IK (round -1) and every finetune round,
// and the residual after the last accepted round is the projection already
// computed for it (same frames, same arithmetic).  One link-indexed frame
// buffer suffices: a finetune solve starts from frames(q) (held in Fa since
// the last accepted solve) and leaves frames(qs) there; a rejected round ends
// the loop.  Only the target chains' frames are ever valid (see WChain).
__device__ bool wrealize(double* q, double* qs, const WTargets& T, WTargets& Ref, int k,
                         const IkCfg& P, int rounds, int fine_iters, double* max_res,
                         unsigned long long* used_out, WarpWs& ws, double* Fa, const WChain& C,
                         double* FG, double* rtG, const unsigned short* ab, Ctr& ctr, int lane) {
  const int dof = c_hand.dof;
  double q0 = lane < dof ? q[lane] : 0.0;
  unsigned long long used = 0ull;
  double worst = 0.0;
  // Ref = T with refreshed hand points.  The refresh at the start of a round
  // projects at frames(q) exactly as the previous round's (or the initial)
  // evaluation does, so that evaluation writes the refreshed points and the
  // round starts from them (a rejected evaluation ends the loop).
  #pragma unroll 1
  for (int a = lane; a < 12 * k; a += 32) Ref.t[a] = T.t[a];
  if (lane < k) Ref.link[lane] = T.link[lane];
  __syncwarp();
  for (int round = -1; round < rounds; ++round) {
    const bool init = round < 0;
    if (!init) {
      if (lane < dof) qs[lane] = q[lane];
      __syncwarp();
    }
    unsigned long long su = 0ull;
    double* qq = init ? q : qs;
    bool ok = wik(qq, init ? T : Ref, k, P, init ? P.iterations : fine_iters, su, ws, Fa, C, FG, rtG,
                  !init, ab, ctr, lane);
    if (!ok) {
      if (!init) break;
      if (lane < dof) q[lane] = q0;
      __syncwarp();
      *max_res = kInf;
      *used_out = 0ull;
      return false;
    }
    double w = wproject(Fa, T, k, &Ref, lane);
    if (init) {
      worst = w;
      used = su;
      continue;
    }
    if (w > worst + 1e-6) break;
    if (lane < dof) q[lane] = qs[lane];
    __syncwarp();
    worst = w;
    used |= su;
  }
  *max_res = worst;
  *used_out = used;
  bool nonfin = lane < dof && !is_finite(q[lane]);
  return !__any_sync(kFull, nonfin);
}

// Per-warp shared bytes: workspace + targets, refreshed targets, q, qs,
// link frames, chain trial frames [32][kFS], trial residuals [4][6k], links,
// chain tables (16-byte aligned).
__host__ __device__ __forceinline__ size_t realize_warp_bytes(int dof, int kmax, int nl) {
  size_t b = warp_ws_bytes(kmax, dof) +
             (size_t)(24 * kmax + 2 * dof + kFS * nl + 32 * kFS + 24 * kmax) * sizeof(double) +
             (2 * kmax + kChainInts) * sizeof(int);
  return (b + 15) & ~(size_t)15;
}

// One warp per problem; targets [t][kMaxK][12] + links [t][kMaxK]; q_out
// [t][kMaxDof] holds q0 on entry (mid_config when q_init == nullptr).
// IKO: solve_contact_ik alone (ik.cpp:30-139) instead of realize_grasp, with
// IkResult's iterations, objective, per-target position residuals and the
// clamped cosines of the normal angles in ik_out.
struct IkOut {
  int* iterations;
  double* objective;
  double* position;  // [t][kMaxK]
  double* cosine;    // [t][kMaxK]
};

template <int MINB, bool IKO = false>
__global__ void __launch_bounds__(128, MINB)
k_realize_warp(int nAct, int k, const int* kk, int kmax, IkCfg P, int rounds, int fine_iters,
               const double* tgt, int tgt_stride, const int* tl, int tl_stride,
               const double* q_init, double* q_out, double* max_res, int* finite,
               unsigned long long* used, int* next, IkOut ik_out = IkOut{}) {
  // Persistent warps: each takes the next problem when it finishes one
  // (problem cost varies by an order of magnitude, and a CTA's shared memory
  // is held until its slowest warp is done).
  extern __shared__ __align__(16) char s_ik[];
  __shared__ unsigned short s_ab[kMaxDof * (kMaxDof + 1) / 2];  // (a, b) of J^T J entry e
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int dof = c_hand.dof;
  const int nl = c_hand.n_links;
  if (threadIdx.x == 0)
    for (int a = 0, e = 0; a < dof; ++a)
      for (int b = a; b < dof; ++b) s_ab[e++] = (unsigned short)(a | (b << 8));
  __syncthreads();
  char* base = s_ik + (size_t)warp * realize_warp_bytes(dof, kmax, nl);
  double* extra = (double*)(base + warp_ws_bytes(kmax, dof));
  WTargets T, Ref;
  T.t = extra;
  Ref.t = extra + 12 * kmax;
  double* q = extra + 24 * kmax;
  double* qs = q + dof;
  double* F = qs + dof;
  double* FG = F + kFS * nl;
  double* rtG = FG + 32 * kFS;
  T.link = (int*)(rtG + 24 * kmax);
  Ref.link = T.link + kmax;
  WChain C;
  C.link = Ref.link + kmax;
  C.pslot = C.link + kMaxLinks;
  C.lvl = C.pslot + kMaxLinks;
  C.sol = C.lvl + kMaxLinks;
  C.tslot = C.sol + kMaxLinks;
  C.hdr = C.tslot + kMaxK;
  Ctr ctr = {0, 0, 0, 0, 0};
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(next, 1);
    t = __shfl_sync(kFull, t, 0);
    if (t >= nAct) break;  // warp-uniform
    const int kt = kk ? kk[t] : k;
    WarpWs ws = warp_ws(base, kt, dof);
    const double* src = tgt + (size_t)t * tgt_stride;
    #pragma unroll 1
    for (int a = lane; a < 12 * kt; a += 32) T.t[a] = src[a];
    if (lane < kt) T.link[lane] = tl[(size_t)t * tl_stride + lane];
    if (lane < dof) q[lane] = q_init ? q_init[(size_t)t * kMaxDof + lane] : g_hand.mid[lane];
    __syncwarp();
    wchain_build(C, T.link, kt, lane);
    wchain_static(T.link, kt, F, lane);
    double mr = 0.0;
    unsigned long long u;
    bool fin;
    if constexpr (IKO) {
      int its;
      double obj;
      fin = wik(q, T, kt, P, P.iterations, u, ws, F, C, FG, rtG, false, s_ab, ctr, lane, &its, &obj);
      if (lane < kt) {  // result.residuals (ik.cpp:130-137)
        const double* tt = T.t + 12 * lane;
        const V3 hn = xf_rotate(ld_xf(F + kFS * T.link[lane]), v3_load(tt + 9));
        double c = dot(hn, v3_load(tt + 3));
        c = c < -1.0 ? -1.0 : (1.0 < c ? 1.0 : c);  // std::clamp
        ik_out.position[(size_t)t * kMaxK + lane] =
            norm(v3(ws.r[6 * lane], ws.r[6 * lane + 1], ws.r[6 * lane + 2]));
        ik_out.cosine[(size_t)t * kMaxK + lane] = c;
      }
      if (lane == 0) {
        ik_out.iterations[t] = its;
        ik_out.objective[t] = obj;
      }
    } else {
      fin = wrealize(q, qs, T, Ref, kt, P, rounds, fine_iters, &mr, &u, ws, F, C, FG, rtG, s_ab, ctr,
                     lane);
    }
    if (lane < dof) q_out[(size_t)t * kMaxDof + lane] = q[lane];
    if (lane == 0) {
      max_res[t] = mr;
      finite[t] = fin ? 1 : 0;
      used[t] = u;
    }
    __syncwarp();
  }
  if (lane == 0) ctr_flush(ctr);
}

__host__ __forceinline__ size_t realize_warp_smem(int dof, int kmax, int nl, int warps) {
  return realize_warp_bytes(dof, kmax, nl) * warps;
}

}  // namespace lgd
