// dev_geom.cuh — per-thread device restatements of the reference's kinematics,
// convex-part queries, GJK, wrench solver and RNG streams.  FP64 throughout,
// compiled with --fmad=false; every expression follows the canonical order of
// lg_math.h so that results are bit-identical to the CPU oracle.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../lg_math.h"
#include "lg.h"

namespace lgd {

using namespace lgm;

constexpr int kMaxLinks = 32;   // device link cap (Shadow-class hands have ~25)
constexpr int kMaxDof = 24;     // device dof cap (Shadow 22 DoF)
constexpr int kMaxDepth = 10;   // device kinematic-chain depth cap
constexpr int kMaxK = LG_MAX_K;
constexpr int kMaxC = LG_MAX_CONTACTS;
constexpr double kPi = 3.14159265358979323846;
constexpr double kInf = __builtin_huge_val();

// Hand model in constant memory: every FK loop walks links uniformly across
// a warp, so constant-cache broadcast serves the whole warp per access.
struct DHand {
  int n_links, dof, root, n_parts;
  int parent[kMaxLinks], jtype[kMaxLinks], jidx[kMaxLinks], topo[kMaxLinks];
  int part_begin[kMaxLinks], part_end[kMaxLinks];
  double R[kMaxLinks][9], t[kMaxLinks][3], axis[kMaxLinks][3], lo[kMaxLinks], hi[kMaxLinks];
  double jlo[kMaxDof], jhi[kMaxDof];  // limits by joint index
  double mid[kMaxDof];                // mid_config (hand.cpp:24-32)
  // warp-parallel FK: root -> link chain per link, joints on that chain
  int chain_len[kMaxLinks];
  int chain[kMaxLinks][kMaxDepth];
  unsigned jmask[kMaxLinks];  // bit j: joint j drives link l
  int jlink[kMaxDof];         // link carrying joint j
  int level[kMaxLinks];       // depth in the kinematic tree (root = 0)
  int n_levels;
  // convex parts (global memory)
  const int* vert_off;
  const double* verts;
  const int* tri_off;
  const int* tris;
  const int* plane_off;
  const double* planes;
  const double* bounds;
};

__constant__ DHand c_hand;
// Global mirror for lane-indexed reads: the constant cache serialises a warp's
// distinct addresses, L1 serves them in one wavefront.
__device__ DHand g_hand;

// Algorithmic work counters (per thread in registers, folded into g_cnt with
// one atomic per thread at kernel exit); feed the roofline's FLOP counts.
struct Ctr {
  unsigned long long ik_it, fk, weval, wgrad, proj;
};
enum { kCntIk = 0, kCntFk, kCntWeval, kCntWgrad, kCntProj, kCntN };
__device__ unsigned long long g_cnt[kCntN];
__device__ __forceinline__ void ctr_flush(const Ctr& c) {
  if (c.ik_it) atomicAdd(&g_cnt[kCntIk], c.ik_it);
  if (c.fk) atomicAdd(&g_cnt[kCntFk], c.fk);
  if (c.weval) atomicAdd(&g_cnt[kCntWeval], c.weval);
  if (c.wgrad) atomicAdd(&g_cnt[kCntWgrad], c.wgrad);
  if (c.proj) atomicAdd(&g_cnt[kCntProj], c.proj);
}

// ------------------------------------------------------------ kinematics
// forward_kinematics (hand.cpp:275-295)
__device__ __forceinline__ void fk(const double* q, Xf* frames) {
  const int nl = c_hand.n_links;
  for (int ii = 0; ii < nl; ++ii) {
    int l = c_hand.topo[ii];
    Xf local;
    local.R = m3_load(c_hand.R[l]);
    local.t = v3_load(c_hand.t[l]);
    int jt = c_hand.jtype[l];
    if (jt == 1) {
      Xf m;
      m.R = angle_axis(q[c_hand.jidx[l]], v3_load(c_hand.axis[l]));
      m.t = v3(0.0, 0.0, 0.0);
      local = xf_compose(local, m);
    } else if (jt == 2) {
      local.t = add(local.t, mul(local.R, scale(q[c_hand.jidx[l]], v3_load(c_hand.axis[l]))));
    }
    int p = c_hand.parent[l];
    frames[l] = p < 0 ? local : xf_compose(frames[p], local);
  }
}

__device__ __forceinline__ void clamp_to_limits(double* q) {  // hand.cpp:34-43
  for (int j = 0; j < c_hand.dof; ++j) q[j] = dclamp(q[j], c_hand.jlo[j], c_hand.jhi[j]);
}

// ------------------------------------------------------------ geometry.hpp
// tangent_basis (geometry.hpp:105-126); returns false where the reference
// throws (zero or non-unit normal).
__device__ __forceinline__ bool tangent_basis(V3 n, V3& x, V3& y) {
  double len = norm(n);
  if (len < 1e-9 || dabs(len - 1.0) > 1e-6) {
    x = v3(0, 0, 0);
    y = v3(0, 0, 0);
    return false;
  }
  int axis = 0;
  double best = dabs(n.x);
  if (dabs(n.y) < best) {
    axis = 1;
    best = dabs(n.y);
  }
  if (dabs(n.z) < best) axis = 2;
  V3 e = v3(axis == 0 ? 1.0 : 0.0, axis == 1 ? 1.0 : 0.0, axis == 2 ? 1.0 : 0.0);
  x = normalized(cross(e, n));
  y = cross(n, x);
  return true;
}

__device__ __forceinline__ M3 rotation_between(V3 from, V3 to) {  // geometry.hpp:129-143
  double c = dot(from, to);
  V3 axis = cross(from, to);
  double s = norm(axis);
  if (s < 1e-12) {
    if (c > 0.0) return m3_identity();
    V3 x, y;
    tangent_basis(normalized(from), x, y);
    return angle_axis(kPi, x);
  }
  axis = divs(axis, s);
  return angle_axis(lgm::xatan2(s, c), axis);
}

// ------------------------------------------------------------------ Rng
// rng.hpp:30-90 over the lazily twisted mt19937_64 (state in local memory).
struct DRng {
  Mt64 g;
  double spare;
  bool has;
  __device__ __forceinline__ void seed(uint64_t s) {
    mt_seed(g, s);
    has = false;
    spare = 0.0;
  }
  __device__ __forceinline__ uint64_t u64() { return mt_next(g); }
  __device__ __forceinline__ double uniform() { return u01(mt_next(g)); }
  __device__ __forceinline__ double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  __device__ __forceinline__ uint64_t index(uint64_t n) { return mt_next(g) % n; }
  __device__ __forceinline__ void quaternion(double* w, double* x, double* y, double* z) {
    double u1 = uniform();
    double u2 = uniform();
    double u3 = uniform();
    double s1 = sqrt(1.0 - u1);
    double s2 = sqrt(u1);
    double t1 = 2.0 * kPi * u2;
    double t2 = 2.0 * kPi * u3;
    *w = s2 * lgm::xcos(t2);
    *x = s1 * lgm::xsin(t1);
    *y = s1 * lgm::xcos(t1);
    *z = s2 * lgm::xsin(t2);
  }
};

// Box-Muller pair from two raw draws (rng.hpp:47-61): returns r cos a and
// the cached spare r sin a.
__device__ __forceinline__ void box_muller(uint64_t d1, uint64_t d2, double* z1, double* z2) {
  double u1 = u01(d1);
  double u2 = u01(d2);
  if (u1 < 1e-300) u1 = 1e-300;
  double r = sqrt(-2.0 * lgm::xlog(u1));
  double a = 2.0 * kPi * u2;
  *z2 = r * lgm::xsin(a);
  *z1 = r * lgm::xcos(a);
}

// ------------------------------------------------------------ convex parts
__device__ __forceinline__ V3 part_vert(int p, int i) {
  return v3_load(c_hand.verts + 3 * (c_hand.vert_off[p] + i));
}
__device__ __forceinline__ int part_nverts(int p) { return c_hand.vert_off[p + 1] - c_hand.vert_off[p]; }

__device__ __forceinline__ bool part_contains(int p, V3 x) {  // convex.cpp:12-17
  for (int i = c_hand.plane_off[p]; i < c_hand.plane_off[p + 1]; ++i) {
    const double* pl = c_hand.planes + 4 * i;
    if (dot(v3(pl[0], pl[1], pl[2]), x) > pl[3] + 0.0) return false;
  }
  return true;
}

__device__ __forceinline__ double part_interior_depth(int p, V3 x) {  // convex.cpp:19-25
  double depth = kInf;
  for (int i = c_hand.plane_off[p]; i < c_hand.plane_off[p + 1]; ++i) {
    const double* pl = c_hand.planes + 4 * i;
    depth = dmin(depth, pl[3] - dot(v3(pl[0], pl[1], pl[2]), x));
  }
  return depth;
}

__device__ __forceinline__ V3 closest_point_on_triangle(V3 p, V3 a, V3 b, V3 c) {  // convex.cpp:27-63
  V3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
  double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return a;
  V3 bp = sub(p, b);
  double d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return b;
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = d1 / (d1 - d3);
    return axpy(a, v, ab);
  }
  V3 cp = sub(p, c);
  double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return c;
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = d2 / (d2 - d6);
    return axpy(a, w, ac);
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return axpy(b, w, sub(c, b));
  }
  double denom = 1.0 / (va + vb + vc);
  double v = vb * denom;
  double w = vc * denom;
  return add(add(a, v3(ab.x * v, ab.y * v, ab.z * v)), v3(ac.x * w, ac.y * w, ac.z * w));
}

__device__ V3 part_closest_surface_point(int p, V3 x, V3* normal) {  // convex.cpp:65-106
  if (part_contains(p, x)) {
    double best = kInf;
    int plane = -1;
    for (int i = c_hand.plane_off[p]; i < c_hand.plane_off[p + 1]; ++i) {
      const double* pl = c_hand.planes + 4 * i;
      double slack = pl[3] - dot(v3(pl[0], pl[1], pl[2]), x);
      if (slack < best) {
        best = slack;
        plane = i;
      }
    }
    const double* pl = c_hand.planes + 4 * plane;
    V3 n = v3(pl[0], pl[1], pl[2]);
    *normal = n;
    return axpy(x, best, n);
  }
  double best = kInf;
  V3 cp = v3(0.0, 0.0, 0.0);
  int face = 0;
  const int t0 = c_hand.tri_off[p], t1 = c_hand.tri_off[p + 1];
  for (int t = t0; t < t1; ++t) {
    const int* tri = c_hand.tris + 3 * t;
    V3 q = closest_point_on_triangle(x, part_vert(p, tri[0]), part_vert(p, tri[1]), part_vert(p, tri[2]));
    double d2 = sqnorm(sub(x, q));
    if (d2 < best) {
      best = d2;
      cp = q;
      face = t;
    }
  }
  double d = sqrt(best);
  if (d > 1e-12) {
    *normal = divs(sub(x, cp), d);
  } else {
    const int* tri = c_hand.tris + 3 * face;
    V3 e1 = sub(part_vert(p, tri[1]), part_vert(p, tri[0]));
    V3 e2 = sub(part_vert(p, tri[2]), part_vert(p, tri[0]));
    *normal = normalized(cross(e1, e2));
  }
  return cp;
}

// closest_on_parts (pipeline.cpp:55-69)
__device__ double closest_on_parts(int link, V3 x, V3* sp, V3* sn) {
  double best = kInf;
  for (int p = c_hand.part_begin[link]; p < c_hand.part_end[link]; ++p) {
    V3 n;
    V3 cp = part_closest_surface_point(p, x, &n);
    double d = norm(sub(x, cp));
    if (d < best) {
      best = d;
      *sp = cp;
      *sn = n;
    }
  }
  return best;
}

__device__ __forceinline__ V3 part_support(int p, V3 dir) {  // convex.cpp:108-119
  double best = -kInf;
  V3 out = v3(0.0, 0.0, 0.0);
  const int nv = part_nverts(p);
  for (int i = 0; i < nv; ++i) {
    V3 v = part_vert(p, i);
    double d = dot(dir, v);
    if (d > best) {
      best = d;
      out = v;
    }
  }
  return out;
}

// world_bounds (collision.cpp:10-20)
__device__ __forceinline__ void world_bounds(int p, const Xf& pose, V3* bmin, V3* bmax) {
  const double* b = c_hand.bounds + 6 * p;
  V3 mn = v3(kInf, kInf, kInf), mx = v3(-kInf, -kInf, -kInf);
  for (int i = 0; i < 8; ++i) {
    V3 corner = v3((i & 1) ? b[3] : b[0], (i & 2) ? b[4] : b[1], (i & 4) ? b[5] : b[2]);
    V3 w = xf_apply(pose, corner);
    mn = vmin(mn, w);
    mx = vmax(mx, w);
  }
  *bmin = mn;
  *bmax = mx;
}

// ------------------------------------------------------------------- GJK
// simplex_closest (collision.cpp:52-169); the degenerate-triangle recursion
// is at most one level deep (n == 2 after keep({0,1})).
// Up to a triangle (no recursion: keeps the stack size static).
__device__ __forceinline__ bool simplex_closest_le3(V3* s, int& n, V3& closest) {
  if (n == 1) {
    closest = s[0];
    return false;
  }
  if (n == 3) {
    V3 a = s[0], b = s[1], c = s[2];
    V3 ab = sub(b, a), ac = sub(c, a);
    double d1 = -dot(ab, a), d2 = -dot(ac, a);
    if (d1 <= 0.0 && d2 <= 0.0) {
      n = 1;
      closest = a;
      return false;
    }
    double d3 = -dot(ab, b), d4 = -dot(ac, b);
    if (d3 >= 0.0 && d4 <= d3) {
      s[0] = b;
      n = 1;
      closest = b;
      return false;
    }
    double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
      double v = d1 / (d1 - d3);
      n = 2;
      closest = axpy(a, v, ab);
      return false;
    }
    double d5 = -dot(ab, c), d6 = -dot(ac, c);
    if (d6 >= 0.0 && d5 <= d6) {
      s[0] = c;
      n = 1;
      closest = c;
      return false;
    }
    double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
      double w = d2 / (d2 - d6);
      s[1] = c;
      n = 2;
      closest = axpy(a, w, ac);
      return false;
    }
    double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
      double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
      s[0] = b;
      s[1] = c;
      n = 2;
      closest = axpy(b, w, sub(c, b));
      return false;
    }
    double denom = va + vb + vc;
    if (dabs(denom) < 1e-30) {
      n = 2;  // keep({0, 1}) then fall through to the segment case
    } else {
      double v = vb / denom, w = vc / denom;
      closest = axpy(axpy(a, v, ab), w, ac);
      return false;
    }
  }
  if (n == 2) {
    V3 ab = sub(s[1], s[0]);
    double t = -dot(s[0], ab);
    double len2 = sqnorm(ab);
    if (t <= 0.0 || len2 < 1e-30) {
      n = 1;
      closest = s[0];
    } else if (t >= len2) {
      s[0] = s[1];
      n = 1;
      closest = s[1];
    } else {
      closest = axpy(s[0], t / len2, ab);
    }
    return false;
  }
  return false;
}

__device__ bool simplex_closest(V3* s, int& n, V3& closest) {
  if (n <= 3) return simplex_closest_le3(s, n, closest);
  // tetrahedron
  const int faces[4][3] = {{0, 1, 2}, {0, 3, 1}, {0, 2, 3}, {1, 3, 2}};
  const int opposite[4] = {3, 2, 1, 0};
  bool inside = true;
  double best = kInf;
  V3 best_closest = v3(0.0, 0.0, 0.0);
  int best_n = 0;
  V3 best_s[3];
  for (int f = 0; f < 4; ++f) {
    V3 a = s[faces[f][0]], b = s[faces[f][1]], c = s[faces[f][2]];
    V3 nrm = cross(sub(b, a), sub(c, a));
    double side = dot(nrm, sub(s[opposite[f]], a));
    if (side > 0.0) nrm = neg(nrm);
    if (dot(nrm, neg(a)) <= 0.0) continue;
    inside = false;
    V3 sb[4] = {a, b, c, a};
    int sn = 3;
    V3 cp;
    simplex_closest_le3(sb, sn, cp);
    double d2 = sqnorm(cp);
    if (d2 < best) {
      best = d2;
      best_closest = cp;
      best_n = sn;
      for (int i = 0; i < sn; ++i) best_s[i] = sb[i];
    }
  }
  if (inside) return true;
  n = best_n;
  for (int i = 0; i < best_n; ++i) s[i] = best_s[i];
  closest = best_closest;
  return false;
}

// gjk_distance (collision.cpp:173-207)
__device__ double gjk_distance(int pa, const Xf& A, int pb, const Xf& B) {
  M3 rat = transpose(A.R);
  M3 rbt = transpose(B.R);
  auto support = [&](V3 d) {
    V3 sa = xf_apply(A, part_support(pa, mul(rat, d)));
    V3 sb = xf_apply(B, part_support(pb, mul(rbt, neg(d))));
    return sub(sa, sb);
  };
  V3 d0 = sub(A.t, B.t);
  if (sqnorm(d0) < 1e-30) d0 = v3(1.0, 0.0, 0.0);
  V3 simplex[4];
  int n = 1;
  simplex[0] = support(d0);
  for (int iter = 0; iter < 128; ++iter) {
    V3 v;
    if (simplex_closest(simplex, n, v)) return 0.0;
    double v2 = sqnorm(v);
    if (v2 < 1e-24) return 0.0;
    V3 w = support(neg(v));
    double progress = v2 - dot(v, w);
    if (progress <= 1e-12 + 1e-10 * v2) return sqrt(v2);
    if (n < 4) simplex[n++] = w;
    else return sqrt(v2);
  }
  return 0.0;
}

// ---------------------------------------------------------------- wrench
// wrench.cpp:50-226.  A problem holds n <= 6 contacts with torque arms
// precomputed; a state holds (alpha, beta_x, beta_y).
struct WProb {
  int n;
  double lambda, mu;
  V3 p[kMaxC], nn[kMaxC], tx[kMaxC], ty[kMaxC], cn[kMaxC], cx[kMaxC], cy[kMaxC];
};
struct WState {
  double a[kMaxC], bx[kMaxC], by[kMaxC];
};

__device__ __forceinline__ void wprob_set(WProb& w, int i, V3 p, V3 n) {
  w.p[i] = p;
  w.nn[i] = n;
  tangent_basis(n, w.tx[i], w.ty[i]);
  w.cn[i] = cross(p, n);
  w.cx[i] = cross(p, w.tx[i]);
  w.cy[i] = cross(p, w.ty[i]);
}

__device__ __forceinline__ void net_wrench(const WProb& w, const WState& s, V3& f, V3& t) {
  f = v3(0.0, 0.0, 0.0);
  t = v3(0.0, 0.0, 0.0);
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    if (i < w.n) {
      f = add(f, add(add(scale(s.a[i], w.nn[i]), scale(s.bx[i], w.tx[i])), scale(s.by[i], w.ty[i])));
      t = add(t, add(add(scale(s.a[i], w.cn[i]), scale(s.bx[i], w.cx[i])), scale(s.by[i], w.cy[i])));
    }
  }
}

__device__ __forceinline__ double weval(const WProb& w, const WState& s) {  // wrench.cpp:70-80
  V3 f, t;
  net_wrench(w, s, f, t);
  return sqnorm(f) + w.lambda * sqnorm(t);
}

__device__ __forceinline__ void wproject(const WProb& w, int anchor, bool fr, WState& s) {  // :82-108
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    if (i < w.n) {
      if (i == anchor) s.a[i] = 1.0;
      else if (s.a[i] < 0.0) s.a[i] = 0.0;
      if (!fr) {
        s.bx[i] = 0.0;
        s.by[i] = 0.0;
      } else {
        double cap = w.mu * s.a[i];
        double r;
        if (lgl::hypot_exceeds(s.bx[i], s.by[i], cap, &r)) {
          if (cap <= 0.0 || r <= 0.0) {
            s.bx[i] = 0.0;
            s.by[i] = 0.0;
          } else {
            double k = cap / r;
            s.bx[i] *= k;
            s.by[i] *= k;
          }
        }
      }
    }
  }
}

// descend (wrench.cpp:124-177)
__device__ double wdescend(const WProb& w, int anchor, bool fr, int iterations, double step0,
                           int max_bt, WState& s, Ctr& ctr) {
  wproject(w, anchor, fr, s);
  double current = weval(w, s);
  ++ctr.weval;
  double ga[kMaxC], gx[kMaxC], gy[kMaxC];
  WState trial = s;
  for (int it = 0; it < iterations; ++it) {
    V3 force, torque;
    net_wrench(w, s, force, torque);
    ++ctr.wgrad;
    torque = v3(torque.x * w.lambda, torque.y * w.lambda, torque.z * w.lambda);
#pragma unroll
    for (int i = 0; i < kMaxC; ++i) {
      if (i < w.n) {
        ga[i] = 2.0 * (dot(force, w.nn[i]) + dot(torque, w.cn[i]));
        if (fr) {
          gx[i] = 2.0 * (dot(force, w.tx[i]) + dot(torque, w.cx[i]));
          gy[i] = 2.0 * (dot(force, w.ty[i]) + dot(torque, w.cy[i]));
        }
      }
    }
    double step = step0;
    bool moved = false;
    for (int bt = 0; bt <= max_bt; ++bt) {
#pragma unroll
      for (int i = 0; i < kMaxC; ++i) {
        if (i < w.n) {
          trial.a[i] = s.a[i] - step * ga[i];
          if (fr) {
            trial.bx[i] = s.bx[i] - step * gx[i];
            trial.by[i] = s.by[i] - step * gy[i];
          } else {
            trial.bx[i] = 0.0;
            trial.by[i] = 0.0;
          }
        }
      }
      wproject(w, anchor, fr, trial);
      double next = weval(w, trial);
      ++ctr.weval;
      if (next <= current) {
        s = trial;
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

struct WOpts {
  int iterations, warm_iterations, max_bt;
  double step;
};

// One anchor of run_solver (wrench.cpp:179-228): cold (warm == nullptr) or
// warm-started; returns the anchor's final objective, state in s.
__device__ __forceinline__ double wsolve_anchor(const WProb& w, int anchor, bool fr,
                                                const WOpts& o, const WState* warm, WState& s,
                                                Ctr& ctr) {
  int iters = warm ? o.warm_iterations : o.iterations;
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    if (warm) {
      s.a[i] = warm->a[i];
      s.bx[i] = warm->bx[i];
      s.by[i] = warm->by[i];
    } else {
      s.a[i] = 1.0;
      s.bx[i] = 0.0;
      s.by[i] = 0.0;
    }
  }
  if (fr) {
    wdescend(w, anchor, false, iters, o.step, o.max_bt, s, ctr);
    return wdescend(w, anchor, true, iters, o.step, o.max_bt, s, ctr);
  }
  return wdescend(w, anchor, false, iters, o.step, o.max_bt, s, ctr);
}

// run_solver (wrench.cpp:179-228) sequentially over anchors in one thread;
// fr = (mu > 0) is solve() of contact_opt.cpp:37-41 / solve_gswo.
__device__ double wsolve(const WProb& w, const WOpts& o, const WState* warm, int* anchor_out,
                         WState& best, Ctr& ctr) {
  const bool fr = w.mu > 0.0;
  double best_obj = kInf;
  int best_anchor = -1;
  for (int anchor = 0; anchor < w.n; ++anchor) {
    WState s;
    double value = wsolve_anchor(w, anchor, fr, o, warm, s, ctr);
    if (value < best_obj) {
      best_obj = value;
      best_anchor = anchor;
      best = s;
    }
  }
  *anchor_out = best_anchor;
  return best_obj;
}

}  // namespace lgd
