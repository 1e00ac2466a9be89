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

// One anchor of run_solver (wrench.cpp:179-228): cold (warm == nullptr) or
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

// ----------------------------------------------- spatial chunk index
// project_to_domain (contact_opt.cpp:11-25) returns the element with the
// smallest (squared distance, index) pair: the reference scans every element.
// The device keeps a Morton-ordered structure-of-arrays copy of each domain,
// split into chunks of 32 elements (one per lane) grouped into super-chunks
// of 32 chunks, each with its bounding box.  A warp answers its 32 mutation
// queries one after another, cooperatively: lanes test box lower bounds in
// parallel, ballot the boxes that can still hold the minimum, and evaluate a
// needed chunk with one element per lane (coalesced loads).  A box is dropped
// only when its lower bound exceeds the best distance found so far by a
// relative guard of 2^-40, which covers the roundings of the bound and of the
// distances: a dropped box can hold neither a closer element nor a tie.  All
// candidates compare lexicographically on (d2, element index), so the result
// is the reference's first minimum whatever the visit order.
constexpr int kChunk = 32;
// Domains below this size keep the plain broadcast scan (every lane reads the
// same element: one load serves the warp), which is faster when the whole
// domain sits in L1; the cooperative search pays off on large domains.
constexpr int kCoopMin = 4096;

struct DomIdx {
  const double* sx;         // sorted element positions, SoA [nel]
  const double* sy;
  const double* sz;
  const int* si;            // sorted -> element index within its domain
  const double* cb;         // chunk boxes [6][cstride] (min xyz, max xyz)
  long long cstride;
  const double* sb;         // super-chunk boxes [6][sstride]
  long long sstride;
  const int* cs;            // chunk starts (element offset in its domain), [cstride]
  const long long* choff;   // first chunk of each (candidate, slot) domain
  const long long* suoff;   // first super-chunk of each domain
};

__device__ __forceinline__ uint32_t morton_spread10(uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// Morton keys of the domain elements, quantised inside the candidate's posed
// object box (k_obj_aabb); value = element index within the domain.
__global__ void k_dom_keys(int nA, int k, const int* alive_idx, const double* aabb,
                           const long long* el_off, ElemSrc el, uint32_t* keys, int* vals) {
  const int seg = blockIdx.x;
  if (seg >= nA * k) return;
  const int i = alive_idx[seg / k];
  const long long b = el_off[seg], e = el_off[seg + 1];
  double lo[3], sc[3];
  for (int c = 0; c < 3; ++c) {
    lo[c] = aabb[6 * i + c];
    const double ext = aabb[6 * i + 3 + c] - lo[c];
    sc[c] = ext > 0.0 ? 1023.0 / ext : 0.0;
  }
  for (long long t = b + threadIdx.x; t < e; t += blockDim.x) {
    uint32_t q[3];
    const V3 pt = el.pos(t, seg / k, el.big(e - b));
    const double pc[3] = {pt.x, pt.y, pt.z};
    for (int c = 0; c < 3; ++c) {
      double v = (pc[c] - lo[c]) * sc[c];
      v = v < 0.0 ? 0.0 : (v > 1023.0 ? 1023.0 : v);
      q[c] = (uint32_t)v;
    }
    keys[t] = morton_spread10(q[0]) | (morton_spread10(q[1]) << 1) | (morton_spread10(q[2]) << 2);
    vals[t] = (int)(t - b);
  }
}

// Chunks: runs of the Morton order cut where the key changes above bit
// kSplitBit (a jump of the curve to another 2^(kSplitBit/3)-cell block: a
// chunk spanning one is long and thin, and its box is hit by many queries),
// and every 32 elements inside a run.  head(t) = run head, or (t - run
// start) % 32 == 0; the run start is a block max-scan of the head positions.
constexpr int kSplitBit = 17;

template <typename F>
__device__ void dom_chunk_heads(const uint32_t* key, int ne, F&& emit) {
  typedef cub::BlockScan<int, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_carry_run, s_carry_cnt;
  if (threadIdx.x == 0) {
    s_carry_run = 0;
    s_carry_cnt = 0;
  }
  __syncthreads();
  for (int base = 0; base < ne; base += 256) {
    const int t = base + threadIdx.x;
    const bool in = t < ne;
    const bool jump = in && (t == 0 || ((key[t] ^ key[t - 1]) >> kSplitBit) != 0);
    int run = jump ? t : -1, run_incl;
    Scan(tmp).InclusiveScan(run, run_incl, cub::Max());
    __syncthreads();
    if (run_incl < s_carry_run) run_incl = s_carry_run;
    const bool head = in && ((t - run_incl) % 32 == 0);
    int pos, total;
    Scan(tmp).ExclusiveSum(head ? 1 : 0, pos, total);
    if (head) emit(s_carry_cnt + pos, t);
    __syncthreads();
    if (threadIdx.x == 255) s_carry_run = run_incl;
    if (threadIdx.x == 0) s_carry_cnt += total;
    __syncthreads();
  }
}

// Number of chunks of each domain (block per domain; keys sorted).
__global__ void k_dom_chunk_count(int nseg, const long long* el_off, const uint32_t* keys_sorted,
                                  int* nch) {
  const int seg = blockIdx.x;
  if (seg >= nseg) return;
  const long long b = el_off[seg];
  const int ne = (int)(el_off[seg + 1] - b);
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  dom_chunk_heads(keys_sorted + b, ne, [&](int c, int) { atomicMax(&s_n, c + 1); });
  __syncthreads();
  if (threadIdx.x == 0) nch[seg] = s_n;
}

// Sorted SoA copy of each domain, its chunk starts, chunk boxes and
// super-chunk boxes (block per domain).
__global__ void k_dom_chunks(int nseg, const long long* el_off, const long long* ch_off,
                             const long long* su_off, const uint32_t* keys_sorted,
                             const int* vals_sorted, ElemSrc el, int k, DomIdx d) {
  const int seg = blockIdx.x;
  if (seg >= nseg) return;
  double* sx = const_cast<double*>(d.sx);
  double* sy = const_cast<double*>(d.sy);
  double* sz = const_cast<double*>(d.sz);
  int* si = const_cast<int*>(d.si);
  int* cs = const_cast<int*>(d.cs);
  double* cb = const_cast<double*>(d.cb);
  double* sb = const_cast<double*>(d.sb);
  const long long b = el_off[seg], e = el_off[seg + 1];
  const int ne = (int)(e - b);
  const long long c0 = ch_off[seg];
  const int nch = (int)(ch_off[seg + 1] - c0);
  dom_chunk_heads(keys_sorted + b, ne, [&](int c, int t) { cs[c0 + c] = t; });
  for (long long t = b + threadIdx.x; t < e; t += blockDim.x) {
    const int o = vals_sorted[t];
    const V3 pt = el.pos(b + o, seg / k, el.big(e - b));
    sx[t] = pt.x;
    sy[t] = pt.y;
    sz[t] = pt.z;
    si[t] = o;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    const long long j0 = b + cs[c0 + c];
    const long long j1 = b + (c + 1 < nch ? cs[c0 + c + 1] : ne);
    double mn[3] = {kInf, kInf, kInf}, mx[3] = {-kInf, -kInf, -kInf};
    for (long long j = j0; j < j1; ++j) {
      const double v[3] = {sx[j], sy[j], sz[j]};
      for (int a = 0; a < 3; ++a) {
        mn[a] = dmin(mn[a], v[a]);
        mx[a] = dmax(mx[a], v[a]);
      }
    }
    for (int a = 0; a < 3; ++a) {
      cb[a * d.cstride + c0 + c] = mn[a];
      cb[(3 + a) * d.cstride + c0 + c] = mx[a];
    }
  }
  __syncthreads();
  const long long s0 = su_off[seg];
  const int nsu = (int)(su_off[seg + 1] - s0);
  for (int t = threadIdx.x; t < nsu; t += blockDim.x) {
    const int c1 = (t + 1) * 32 < nch ? (t + 1) * 32 : nch;
    double mn[3] = {kInf, kInf, kInf}, mx[3] = {-kInf, -kInf, -kInf};
    for (int c = t * 32; c < c1; ++c)
      for (int a = 0; a < 3; ++a) {
        mn[a] = dmin(mn[a], cb[a * d.cstride + c0 + c]);
        mx[a] = dmax(mx[a], cb[(3 + a) * d.cstride + c0 + c]);
      }
    for (int a = 0; a < 3; ++a) {
      sb[a * d.sstride + s0 + t] = mn[a];
      sb[(3 + a) * d.sstride + s0 + t] = mx[a];
    }
  }
}

__device__ __forceinline__ double box_lb(const double* B, long long stride, long long i, V3 p) {
  const double ex = dmax(dmax(B[i] - p.x, p.x - B[3 * stride + i]), 0.0);
  const double ey = dmax(dmax(B[stride + i] - p.y, p.y - B[4 * stride + i]), 0.0);
  const double ez = dmax(dmax(B[2 * stride + i] - p.z, p.z - B[5 * stride + i]), 0.0);
  return ex * ex + ey * ey + ez * ez;
}

// (d, idx) lexicographic minimum over the warp.
__device__ __forceinline__ void warp_lexmin(double& d, int& o) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const double od = __shfl_xor_sync(kFull, d, s);
    const int oo = __shfl_xor_sync(kFull, o, s);
    if (od < d || (od == d && oo < o)) {
      d = od;
      o = oo;
    }
  }
}

// The 32 lanes' projections (each lane's own query point cp / act), answered
// cooperatively one query at a time.  seg = (candidate, slot) domain, cur =
// the incumbent element (index, position), a member of the domain.
__device__ int project_coop(const DomIdx& D, long long seg, long long base, int ne, V3 cp_own,
                            bool act_own, int cur_id, V3 cur_p, int lane,
                            unsigned long long& evals) {
  const long long c0 = D.choff[seg], s0 = D.suoff[seg];
  const int nch = (int)(D.choff[seg + 1] - c0);
  const int nsu = (int)(D.suoff[seg + 1] - s0);
  const int* CS = D.cs + c0;
  auto chunk_end = [&](int c) { return c + 1 < nch ? CS[c + 1] : ne; };
  const double* SX = D.sx + base;
  const double* SY = D.sy + base;
  const double* SZ = D.sz + base;
  const int* SI = D.si + base;
  int res = cur_id;
  const unsigned actm = __ballot_sync(kFull, act_own);
  for (int m = 0; m < 32; ++m) {
    if (!((actm >> m) & 1u)) continue;
    const V3 cp = v3(__shfl_sync(kFull, cp_own.x, m), __shfl_sync(kFull, cp_own.y, m),
                     __shfl_sync(kFull, cp_own.z, m));
    // pass 1: the chunk with the smallest lower bound, evaluated first
    int sbest = 0;
    if (nsu > 1) {
      double l = kInf;
      int s = 0x7fffffff;
      for (int t = lane; t < nsu; t += 32) {
        const double v = box_lb(D.sb, D.sstride, s0 + t, cp);
        if (v < l) {
          l = v;
          s = t;
        }
      }
      warp_lexmin(l, s);
      sbest = s;
    }
    double lc = kInf;
    int cbest = 0x7fffffff;
    {
      const int c = sbest * 32 + lane;
      if (c < nch) {
        lc = box_lb(D.cb, D.cstride, c0 + c, cp);
        cbest = c;
      }
      warp_lexmin(lc, cbest);
    }
    double bd = sqnorm(sub(cur_p, cp));
    int bi = cur_id;
    {
      const int j = CS[cbest] + lane;
      if (j < chunk_end(cbest)) {
        const double d = sqnorm(sub(v3(SX[j], SY[j], SZ[j]), cp));
        const int o = SI[j];
        if (d < bd || (d == bd && o < bi)) {
          bd = d;
          bi = o;
        }
      }
      warp_lexmin(bd, bi);
    }
    unsigned long long ev = (unsigned long long)(chunk_end(cbest) - CS[cbest]);
    // pass 2: every other box whose lower bound does not exceed the best
    double thr = bd * (1.0 + 0x1p-40);
    double dl = bd;
    int ol = bi;
    // the needed chunks of super-chunk ss, up to four at a time: their loads
    // are independent (the large domains stream from L2/HBM), the
    // comparisons follow
    auto eval_super = [&](int ss) {
      const int c2 = ss * 32 + lane;
      const bool nc = c2 < nch && c2 != cbest && !(box_lb(D.cb, D.cstride, c0 + c2, cp) > thr);
      unsigned mc = __ballot_sync(kFull, nc);
      {  // elements evaluated: the needed chunks' sizes
        int sz = nc ? chunk_end(c2) - CS[c2] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sz += __shfl_xor_sync(kFull, sz, o);
        ev += (unsigned long long)sz;
      }
      while (mc) {
        int jj[4], je[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          jj[u] = -1;
          je[u] = 0;
          if (mc) {
            const int cc = ss * 32 + __ffs(mc) - 1;
            jj[u] = CS[cc] + lane;
            je[u] = chunk_end(cc);
            mc &= mc - 1;
          }
        }
        double px[4], py[4], pz[4];
        int po[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = jj[u] >= 0 && jj[u] < je[u];
          const int j = ok ? jj[u] : 0;
          px[u] = ok ? SX[j] : 0.0;
          py[u] = ok ? SY[j] : 0.0;
          pz[u] = ok ? SZ[j] : 0.0;
          po[u] = ok ? SI[j] : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (po[u] < 0) continue;
          const double d = sqnorm(sub(v3(px[u], py[u], pz[u]), cp));
          if (d < dl || (d == dl && po[u] < ol)) {
            dl = d;
            ol = po[u];
          }
        }
      }
    };
    if (nsu <= 128) {
      // best first: super-chunks in ascending lower-bound order, the
      // threshold tightened to the best distance after each one, until the
      // smallest remaining bound exceeds it
      double sl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = lane + 32 * u;
        sl[u] = t < nsu ? (nsu == 1 ? 0.0 : box_lb(D.sb, D.sstride, s0 + t, cp)) : kInf;
      }
      for (;;) {
        double v = sl[0];
        int tt = lane;
#pragma unroll
        for (int u = 1; u < 4; ++u)
          if (sl[u] < v) {
            v = sl[u];
            tt = lane + 32 * u;
          }
        warp_lexmin(v, tt);
        if (!(v <= thr)) break;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (lane + 32 * u == tt) sl[u] = kInf;
        eval_super(tt);
        double bd2 = dl;
        int bi2 = ol;
        warp_lexmin(bd2, bi2);
        thr = bd2 * (1.0 + 0x1p-40);
      }
    } else {
      for (int tb = 0; tb < nsu; tb += 32) {
        const int t = tb + lane;
        const bool ns = t < nsu && !(box_lb(D.sb, D.sstride, s0 + t, cp) > thr);
        unsigned ms = __ballot_sync(kFull, ns);
        while (ms) {
          const int ss = tb + __ffs(ms) - 1;
          ms &= ms - 1;
          eval_super(ss);
        }
      }
    }
    warp_lexmin(dl, ol);
    if (lane == m) {
      res = ol;
      evals += ev;
    }
  }
  return res;
}

// Block per candidate, warp per restart, lanes over the n_inner mutations.
// NC = compile-time bound on k + statics (sizes the shared-memory layout).
// LARGE: the launch has domains of at least kCoopMin elements (cooperative
// search, elements recomputed from sample ids); the plain instance keeps the
// materialised-only code, whose smaller body stays in the instruction cache.
template <int NC, int MINB, bool LARGE>
__global__ void __launch_bounds__(128, MINB)
k_contact_opt2(int nA, const int* alive_idx, CoptCfg cfg, const int* n_static, const double* st_p,
               const double* st_n, const long long* el_off, ElemSrc el,
               DomIdx dom, const uint64_t* draws, int* out_ids, double* out_obj, int* out_anchor,
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
        const bool bg = LARGE && el.big(cnt[lane]);
        slot_make(sp + kSlot * lane, el.pos(e, a, bg), neg(el.nrm(e, a, bg)));
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
            const bool act = m < cfg.n_inner;
            double v = kInf;
            int cand = -1, an = -1;
            V3 cp = cur_p;
            if (act) {
              const uint64_t* d2 = M + 2 * ((long long)(outer * k + q) * cfg.n_inner + m);
              // (sigma z1, sigma z2), precomputed by k_copt_normals
              const double u = __longlong_as_double((long long)d2[0]);
              const double vv = __longlong_as_double((long long)d2[1]);
              cp = axpy(axpy(cur_p, u, tx), vv, ty);
            }
            const int ne = (int)cnt[q];
            double bd;
            int bi;
            if (LARGE && ne >= kCoopMin) {
              unsigned long long evals = 0;
              bi = project_coop(dom, (long long)a * k + q, off[q], ne, cp, act, ids[q], cur_p, lane,
                                evals);
              if (act) ctr.proj += evals;
            } else if (act) {
                const double* P = el.p + 3 * off[q];
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
            }
            if (act) {
              cand = bi;
              const long long eg = off[q] + bi;
              const bool bg = LARGE && el.big(cnt[q]);
              slot_make(tslot, el.pos(eg, a, bg), neg(el.nrm(eg, a, bg)));
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
              const bool bg = LARGE && el.big(cnt[q]);
              slot_make(sp + kSlot * q, el.pos(e, a, bg), neg(el.nrm(e, a, bg)));
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
