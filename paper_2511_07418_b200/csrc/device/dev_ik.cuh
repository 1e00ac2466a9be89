// dev_ik.cuh — damped-least-squares contact IK (reference ik.cpp:31-139) and
// realize_grasp (pipeline.cpp:185-253) on the device.
//
// J (6k x dof) is never materialised: each 3-row point-Jacobian block is
// streamed into J^T J and J^T r as soon as it is formed.  Every entry of J^T J
// is still the row-ordered sum s = s + J(r,a) J(r,b), r = 0..6k-1, so the
// result is bit-identical to the oracle's dense product.  The factorisation
// is Eigen's LDLT with diagonal pivoting, unblocked, canonical order.
#pragma once

#include "dev_geom.cuh"

namespace lgd {

struct Target {
  V3 op, on;  // object point, inward normal (base frame)
  int link;
  V3 hp, hn;  // hand point / outward normal (link frame)
};

struct IkCfg {
  double beta, step_clamp, residual_tol, damping_scale, damping_min;
  int iterations, max_backtracks;
};

// stacked_residual (ik.cpp:13-27)
__device__ __forceinline__ void ik_residual(const Xf* fr, const Target* T, int k, double beta,
                                            double* r) {
  for (int i = 0; i < k; ++i) {
    const Xf& f = fr[T[i].link];
    V3 hp = xf_apply(f, T[i].hp);
    V3 hn = xf_rotate(f, T[i].hn);
    V3 a = sub(T[i].op, hp);
    V3 b = sub(axpy(T[i].op, beta, T[i].on), axpy(hp, beta, hn));
    r[6 * i + 0] = a.x;
    r[6 * i + 1] = a.y;
    r[6 * i + 2] = a.z;
    r[6 * i + 3] = b.x;
    r[6 * i + 4] = b.y;
    r[6 * i + 5] = b.z;
  }
}

__device__ __forceinline__ double sum_squares(const double* r, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = s + r[i] * r[i];
  return s;
}

// Eigen LDLT (lower, diagonal pivoting), A row-major n x n, x in/out.
__device__ void ldlt_solve(int n, double* A, double* x) {
  int tr[kMaxDof];
  double temp[kMaxDof];
  for (int k = 0; k < n; ++k) {
    int big = k;
    double best = dabs(A[k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      double v = dabs(A[i * n + i]);
      if (v > best) {
        best = v;
        big = i;
      }
    }
    tr[k] = big;
    if (k != big) {
      for (int j = 0; j < k; ++j) {
        double t = A[k * n + j];
        A[k * n + j] = A[big * n + j];
        A[big * n + j] = t;
      }
      for (int i = big + 1; i < n; ++i) {
        double t = A[i * n + k];
        A[i * n + k] = A[i * n + big];
        A[i * n + big] = t;
      }
      double t = A[k * n + k];
      A[k * n + k] = A[big * n + big];
      A[big * n + big] = t;
      for (int i = k + 1; i < big; ++i) {
        double u = A[i * n + k];
        A[i * n + k] = A[big * n + i];
        A[big * n + i] = u;
      }
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = A[j * n + j] * A[k * n + j];
      double s = 0.0;
      for (int j = 0; j < k; ++j) s = s + A[k * n + j] * temp[j];
      A[k * n + k] -= s;
      for (int i = k + 1; i < n; ++i) {
        double t = 0.0;
        for (int j = 0; j < k; ++j) t = t + A[i * n + j] * temp[j];
        A[i * n + k] -= t;
      }
    }
    double akk = A[k * n + k];
    if (dabs(akk) > 0.0)
      for (int i = k + 1; i < n; ++i) A[i * n + k] /= akk;
  }
  for (int k = 0; k < n; ++k) {
    double t = x[k];
    x[k] = x[tr[k]];
    x[tr[k]] = t;
  }
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < i; ++j) s = s + A[i * n + j] * x[j];
    x[i] -= s;
  }
  for (int i = 0; i < n; ++i) {
    double d = A[i * n + i];
    if (dabs(d) > 2.2250738585072014e-308) x[i] /= d;
    else x[i] = 0.0;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = n - 1; j > i; --j) s = s + A[j * n + i] * x[j];
    x[i] -= s;
  }
  for (int k = n - 1; k >= 0; --k) {
    double t = x[k];
    x[k] = x[tr[k]];
    x[tr[k]] = t;
  }
}

// point_jacobian (hand.cpp:343-358) as 3 x dof row-major.
__device__ __forceinline__ void point_jacobian(const Xf* fr, int link, V3 lp, double* J) {
  const int dof = c_hand.dof;
  for (int i = 0; i < 3 * dof; ++i) J[i] = 0.0;
  V3 point = xf_apply(fr[link], lp);
  for (int l = link; l >= 0; l = c_hand.parent[l]) {
    int j = c_hand.jidx[l];
    if (j < 0) continue;
    V3 axis = mul(fr[l].R, v3_load(c_hand.axis[l]));
    V3 col = c_hand.jtype[l] == 1 ? cross(axis, sub(point, fr[l].t)) : axis;
    J[j] = col.x;
    J[dof + j] = col.y;
    J[2 * dof + j] = col.z;
  }
}

__device__ __forceinline__ bool all_finite(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!is_finite(v[i])) return false;
  return true;
}

// solve_contact_ik (ik.cpp:31-139).  q in/out; returns finite.
__device__ bool ik_solve(double* q, const Target* T, int k, const IkCfg& P, int iterations,
                         unsigned long long* used, Ctr& ctr) {
  const int dof = c_hand.dof;
  const int rows = 6 * k;
  clamp_to_limits(q);
  *used = 0ull;
  bool finite = true;
  if (k == 0) return true;
  Xf fr[kMaxLinks], frt[kMaxLinks];
  double r[6 * kMaxK], rt[6 * kMaxK];
  double JtJ[kMaxDof * kMaxDof], dq[kMaxDof], qt[kMaxDof], Jp[3 * kMaxDof], cmax[kMaxDof];
  fk(q, fr);
  ++ctr.fk;
  ik_residual(fr, T, k, P.beta, r);
  double objective = sum_squares(r, rows);
  for (int it = 0; it < iterations; ++it) {
    ++ctr.ik_it;
    for (int a = 0; a < dof * dof; ++a) JtJ[a] = 0.0;
    for (int a = 0; a < dof; ++a) {
      dq[a] = 0.0;
      cmax[a] = 0.0;
    }
    for (int i = 0; i < k; ++i) {
      for (int half = 0; half < 2; ++half) {
        V3 lp = half == 0 ? T[i].hp : axpy(T[i].hp, P.beta, T[i].hn);
        point_jacobian(fr, T[i].link, lp, Jp);
        for (int rr = 0; rr < 3; ++rr) {
          const double* row = Jp + rr * dof;
          double rv = r[6 * i + 3 * half + rr];
          for (int a = 0; a < dof; ++a) {
            double ja = row[a];
            cmax[a] = dmax(cmax[a], dabs(ja));
            for (int b = 0; b < dof; ++b) JtJ[a * dof + b] = JtJ[a * dof + b] + ja * row[b];
            dq[a] = dq[a] + ja * rv;
          }
        }
      }
    }
    for (int c = 0; c < dof; ++c)
      if (cmax[c] > 1e-12) *used |= 1ull << c;
    double tr = 0.0;
    for (int a = 0; a < dof; ++a) tr = tr + JtJ[a * dof + a];
    double lambda = dmax(P.damping_min, P.damping_scale * tr / (double)(dof > 1 ? dof : 1));
    for (int a = 0; a < dof; ++a) JtJ[a * dof + a] += lambda;
    ldlt_solve(dof, JtJ, dq);
    if (!all_finite(dq, dof)) {
      finite = false;
      break;
    }
    bool moved = false;
    for (int bt = 0; bt <= P.max_backtracks; ++bt) {
      for (int c = 0; c < dof; ++c) qt[c] = q[c] + dmin(dmax(dq[c], -P.step_clamp), P.step_clamp);
      clamp_to_limits(qt);
      fk(qt, frt);
      ++ctr.fk;
      ik_residual(frt, T, k, P.beta, rt);
      double obj_try = sum_squares(rt, rows);
      if (obj_try <= objective) {
        for (int c = 0; c < dof; ++c) q[c] = qt[c];
        for (int l = 0; l < c_hand.n_links; ++l) fr[l] = frt[l];
        for (int i = 0; i < rows; ++i) r[i] = rt[i];
        objective = obj_try;
        moved = true;
        break;
      }
      for (int c = 0; c < dof; ++c) dq[c] *= 0.5;
    }
    if (!moved) break;
    double max_pos = 0.0;
    for (int i = 0; i < k; ++i) max_pos = dmax(max_pos, norm(v3(r[6 * i], r[6 * i + 1], r[6 * i + 2])));
    if (max_pos < P.residual_tol) break;
  }
  if (!all_finite(q, dof)) finite = false;
  return finite;
}

// realize_grasp's project lambda (pipeline.cpp:196-220): worst distance of
// the object points to the assigned links' parts at q; optionally refreshes
// the hand points/normals.
__device__ double realize_project(const double* q, const Target* T, int k, Target* refreshed,
                                  double* residuals, Ctr& ctr) {
  Xf fr[kMaxLinks];
  fk(q, fr);
  ++ctr.fk;
  double worst = 0.0;
  for (int i = 0; i < k; ++i) {
    Xf inv = xf_inverse(fr[T[i].link]);
    V3 sp = v3(0, 0, 0), sn = v3(0, 0, 0);
    double d = closest_on_parts(T[i].link, xf_apply(inv, T[i].op), &sp, &sn);
    worst = dmax(worst, d);
    if (refreshed) {
      refreshed[i].hp = sp;
      refreshed[i].hn = sn;
    }
    if (residuals) residuals[i] = d;
  }
  return worst;
}

// realize_grasp (pipeline.cpp:185-253) from q0 = q; q out.
__device__ bool realize_grasp(double* q, const Target* T, int k, const IkCfg& P, int rounds,
                              int fine_iters, double* max_res, unsigned long long* used_out,
                              Ctr& ctr) {
  const int dof = c_hand.dof;
  double q0[kMaxDof], qs[kMaxDof];
  for (int j = 0; j < dof; ++j) q0[j] = q[j];
  unsigned long long used = 0ull;
  *used_out = 0ull;
  if (!ik_solve(q, T, k, P, P.iterations, &used, ctr)) {
    for (int j = 0; j < dof; ++j) q[j] = q0[j];
    *max_res = kInf;
    return false;
  }
  double worst = realize_project(q, T, k, nullptr, nullptr, ctr);
  Target ref[kMaxK];
  for (int round = 0; round < rounds; ++round) {
    for (int i = 0; i < k; ++i) ref[i] = T[i];
    realize_project(q, T, k, ref, nullptr, ctr);
    for (int j = 0; j < dof; ++j) qs[j] = q[j];
    unsigned long long su = 0ull;
    if (!ik_solve(qs, ref, k, P, fine_iters, &su, ctr)) break;
    double w2 = realize_project(qs, T, k, nullptr, nullptr, ctr);
    if (w2 > worst + 1e-6) break;
    for (int j = 0; j < dof; ++j) q[j] = qs[j];
    worst = w2;
    used |= su;
  }
  *max_res = realize_project(q, T, k, nullptr, nullptr, ctr);
  *used_out = used;
  return all_finite(q, dof);
}

}  // namespace lgd
