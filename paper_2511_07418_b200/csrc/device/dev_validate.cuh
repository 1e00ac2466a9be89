// dev_validate.cuh — validate_dataset (reference validate.cpp:56-175) as one
// block per grasp.  The reference's brute-force loops — every object triangle
// per contact (distance_to_mesh, :19-28), every link triangle per contact
// (:30-42) and every object sample against every link part (:133-143) — are
// spread over the block's threads; the results are minima / maxima, which
// are order independent, so every recorded value equals the serial one.
#pragma once

#include "dev_post.cuh"

namespace lgd {

struct ValCfg {
  int dof;
  double contact_tol, penetration_margin, lambda, mu, eps_stable;
  WOpts o;
  const double* obj_v;  // [nv][3]
  const int* obj_t;     // [nt][3]
  int nt;
};

// plane_depth (validate.cpp:44-52): 0 outside any face.
__device__ __forceinline__ double plane_depth(int p, V3 x) {
  double depth = kInf;
  const int i0 = c_hand.plane_off[p], i1 = c_hand.plane_off[p + 1];
  for (int i = i0; i < i1; ++i) {
    const double* pl = c_hand.planes + 4 * i;
    double slack = pl[3] - dot(v3(pl[0], pl[1], pl[2]), x);
    if (slack < 0.0) return 0.0;
    depth = dmin(depth, slack);
  }
  return i1 > i0 ? depth : 0.0;
}

__device__ __forceinline__ double block_min(double v, double* scratch) {
  return -block_max(-v, scratch);
}

__global__ void __launch_bounds__(256)
k_validate(long long n, const lg_grasp* grasps, ValCfg C, DSamples samples, lg_grasp_check* out) {
  __shared__ double s_q[kMaxDof];
  __shared__ double s_fr[kMaxLinks * kFS];
  __shared__ double s_inv[kMaxLinks * kFS];
  __shared__ double scratch[32];
  __shared__ int s_status;
  const long long gi = blockIdx.x;
  if (gi >= n) return;
  const lg_grasp& g = grasps[gi];
  lg_grasp_check& r = out[gi];
  const int tid = threadIdx.x, lane = tid & 31;
  const int nl = c_hand.n_links;
  if (tid == 0) {
    r.status = 0;
    r.rigid_error = 0.0;
    r.n_limit = 0;
    r.n_contacts = g.n_contacts;
    r.worst_depth = 0.0;
    r.wrench_error = 0;
    r.wrench_objective = 0.0;
    for (int j = 0; j < LG_MAX_DOF; ++j) {
      r.limit_link[j] = 0;
      r.limit_value[j] = 0.0;
    }
    for (int c = 0; c < LG_MAX_CONTACTS; ++c) {
      r.contact_state[c] = 0;
      r.hand_dist[c] = 0.0;
      r.object_dist[c] = 0.0;
    }
    int st = 0;
    if (g.dof != C.dof) st = 1;
    if (!st) {
      M3 R;
      for (int a = 0; a < 9; ++a) R.m[a] = g.pose_R[a];
      r.rigid_error = orthonormal_error(R);
      if (r.rigid_error > 1e-6) st = 2;
    }
    if (!st) {
      for (int l = 0; l < nl; ++l) {  // links in order, as the reference loops
        int j = c_hand.jidx[l];
        if (j < 0) continue;
        double v = g.q[j];
        if (v < c_hand.lo[l] - 1e-9 || v > c_hand.hi[l] + 1e-9) {
          r.limit_link[r.n_limit] = l;
          r.limit_value[r.n_limit] = v;
          ++r.n_limit;
        }
      }
      if (r.n_limit) st = 3;
    }
    if (!st && g.n_contacts <= 0) st = 4;
    r.status = st;
    s_status = st;
  }
  if (tid < C.dof) s_q[tid] = g.q[tid];
  __syncthreads();
  if (s_status) return;
  if (tid < 32) wfk_s(s_q, s_fr, lane);
  __syncthreads();
  if (tid < nl) st_xf(s_inv + kFS * tid, xf_inverse(ld_xf(s_fr + kFS * tid)));
  __syncthreads();
  const Xf pose = [&] {
    Xf x;
    for (int a = 0; a < 9; ++a) x.R.m[a] = g.pose_R[a];
    x.t = v3(g.pose_t[0], g.pose_t[1], g.pose_t[2]);
    return x;
  }();
  const Xf obj_inv = xf_inverse(pose);
  // contacts (validate.cpp:99-123)
  for (int ci = 0; ci < g.n_contacts; ++ci) {
    const int link = g.contact_link[ci];
    const V3 pos = v3(g.contact_p[ci][0], g.contact_p[ci][1], g.contact_p[ci][2]);
    const V3 nrm = v3(g.contact_n[ci][0], g.contact_n[ci][1], g.contact_n[ci][2]);
    int state = 0;
    if (link < 0 || link >= nl) state = 1;
    else if (dabs(norm(nrm) - 1.0) > 1e-6) state = 2;
    if (tid == 0) r.contact_state[ci] = state;
    if (state) continue;  // block-uniform
    // distance_to_link_surface: every triangle of every part of the link
    const V3 local = xf_apply(ld_xf(s_inv + kFS * link), pos);
    double best = kInf;
    for (int p = c_hand.part_begin[link]; p < c_hand.part_end[link]; ++p) {
      const int v0 = c_hand.vert_off[p];
      for (int t = c_hand.tri_off[p] + tid; t < c_hand.tri_off[p + 1]; t += blockDim.x) {
        const int* tr = c_hand.tris + 3 * t;
        V3 cp = closest_point_on_triangle(local, v3_load(c_hand.verts + 3 * (v0 + tr[0])),
                                          v3_load(c_hand.verts + 3 * (v0 + tr[1])),
                                          v3_load(c_hand.verts + 3 * (v0 + tr[2])));
        best = dmin(best, norm(sub(local, cp)));
      }
    }
    best = block_min(best, scratch);
    if (tid == 0) r.hand_dist[ci] = best;
    // distance_to_mesh: every object triangle
    const V3 op = xf_apply(obj_inv, pos);
    double bo = kInf;
    for (int t = tid; t < C.nt; t += blockDim.x) {
      const int* tr = C.obj_t + 3 * t;
      V3 cp = closest_point_on_triangle(op, v3_load(C.obj_v + 3 * tr[0]), v3_load(C.obj_v + 3 * tr[1]),
                                        v3_load(C.obj_v + 3 * tr[2]));
      bo = dmin(bo, norm(sub(op, cp)));
    }
    bo = block_min(bo, scratch);
    if (tid == 0) r.object_dist[ci] = bo;
  }
  // object samples against every link part (validate.cpp:125-143)
  double worst = 0.0;
  for (int j = tid; j < samples.n; j += blockDim.x) {
    const V3 world = xf_apply(pose, samples.p(j));
    for (int l = 0; l < nl; ++l) {
      const int p0 = c_hand.part_begin[l], p1 = c_hand.part_end[l];
      if (p1 <= p0) continue;
      const V3 local = xf_apply(ld_xf(s_inv + kFS * l), world);
      for (int p = p0; p < p1; ++p) {
        const double* b = c_hand.bounds + 6 * p;
        if (!(local.x >= b[0] - 1e-9 && local.y >= b[1] - 1e-9 && local.z >= b[2] - 1e-9 &&
              local.x <= b[3] + 1e-9 && local.y <= b[4] + 1e-9 && local.z <= b[5] + 1e-9))
          continue;
        worst = dmax(worst, plane_depth(p, local));
      }
    }
  }
  worst = block_max(worst, scratch);
  if (tid == 0) r.worst_depth = worst;
}

// Wrench recheck (validate.cpp:145-172), thread per fully checked grasp:
// tangent_basis throws on the first contact whose normal is zero or not
// unit, otherwise solve_gswo's objective.
__global__ void k_validate_wrench(long long n, const lg_grasp* grasps, ValCfg C,
                                  lg_grasp_check* out) {
  long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gi >= n || out[gi].status) return;
  const lg_grasp& g = grasps[gi];
  int err = 0;
  for (int ci = 0; ci < g.n_contacts && !err; ++ci) {
    double len = norm(v3(g.contact_n[ci][0], g.contact_n[ci][1], g.contact_n[ci][2]));
    if (len < 1e-9) err = 1;
    else if (dabs(len - 1.0) > 1e-6) err = 2;
  }
  out[gi].wrench_error = err;
  if (err) return;
  WProb w;
  w.n = g.n_contacts;
  w.lambda = C.lambda;
  w.mu = C.mu;
  for (int ci = 0; ci < w.n; ++ci)
    wprob_set(w, ci, v3(g.contact_p[ci][0], g.contact_p[ci][1], g.contact_p[ci][2]),
              v3(g.contact_n[ci][0], g.contact_n[ci][1], g.contact_n[ci][2]));
  WState s;
  int an = -1;
  Ctr ctr = {0, 0, 0, 0, 0};
  out[gi].wrench_objective = wsolve(w, C.o, nullptr, &an, s, ctr);
}

}  // namespace lgd
