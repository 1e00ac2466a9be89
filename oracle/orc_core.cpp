// oracle/orc_core.cpp — geometry, RNG, hand kinematics, convex queries,
// collision, wrench solver, contact search and IK of the reference,
// restated for the CPU parity oracle (test infrastructure only).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <exception>
#include <mutex>
#include <thread>

#include "orc.hpp"

namespace orc {

using namespace lgm;

// ------------------------------------------------------- geometry.hpp:105-143
void tangent_basis(V3 n, V3& x, V3& y) {
  double len = norm(n);
  if (len < 1e-9) throw std::invalid_argument("tangent_basis: zero normal");
  if (std::abs(len - 1.0) > 1e-6)
    throw std::invalid_argument("tangent_basis: normal is not unit length");
  int axis = 0;
  double best = std::abs(n.x);
  if (std::abs(n.y) < best) {
    axis = 1;
    best = std::abs(n.y);
  }
  if (std::abs(n.z) < best) axis = 2;
  V3 e = v3(axis == 0 ? 1.0 : 0.0, axis == 1 ? 1.0 : 0.0, axis == 2 ? 1.0 : 0.0);
  x = normalized(cross(e, n));
  y = cross(n, x);
}

M3 rotation_between(V3 from, V3 to) {
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
  double angle = lgm::xatan2(s, c);
  return angle_axis(angle, axis);
}

// -------------------------------------------------------------- rng.hpp:30-90
Rng::Rng(uint64_t seed) { mt_seed(eng_, seed); }
uint64_t Rng::next_u64() { return mt_next(eng_); }

double Rng::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1 = uniform();
  double u2 = uniform();
  if (u1 < 1e-300) u1 = 1e-300;
  double r = std::sqrt(-2.0 * lgm::xlog(u1));
  double a = 2.0 * kPi * u2;
  spare_ = r * lgm::xsin(a);
  has_spare_ = true;
  return r * lgm::xcos(a);
}

void Rng::uniform_quaternion(double* w, double* x, double* y, double* z) {
  double u1 = uniform();
  double u2 = uniform();
  double u3 = uniform();
  double s1 = std::sqrt(1.0 - u1);
  double s2 = std::sqrt(u1);
  double t1 = 2.0 * kPi * u2;
  double t2 = 2.0 * kPi * u3;
  *w = s2 * lgm::xcos(t2);
  *x = s1 * lgm::xsin(t1);
  *y = s1 * lgm::xcos(t1);
  *z = s2 * lgm::xsin(t2);
}

V3 Rng::uniform_unit_vector() {
  double z = uniform(-1.0, 1.0);
  double a = 2.0 * kPi * uniform();
  double r = std::sqrt(dmax(0.0, 1.0 - z * z));
  return v3(r * lgm::xcos(a), r * lgm::xsin(a), z);
}

// ------------------------------------------------------------ parallel.hpp
void parallel_for(size_t begin, size_t end, int workers,
                  const std::function<void(size_t)>& fn) {
  if (begin >= end) return;
  if (workers <= 0) {
    unsigned hw = std::thread::hardware_concurrency();
    workers = hw == 0 ? 1 : (int)hw;
  }
  size_t count = end - begin;
  if (workers <= 1 || count == 1) {
    for (size_t i = begin; i < end; ++i) fn(i);
    return;
  }
  std::atomic<size_t> next{begin};
  std::atomic<bool> failed{false};
  std::exception_ptr error;
  std::mutex mu;
  auto worker = [&] {
    for (;;) {
      size_t i = next.fetch_add(1);
      if (i >= end || failed.load()) return;
      try {
        fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!failed.exchange(true)) error = std::current_exception();
        return;
      }
    }
  };
  std::vector<std::thread> threads;
  int n = (int)std::min<size_t>((size_t)workers, count);
  for (int t = 0; t < n; ++t) threads.emplace_back(worker);
  for (auto& t : threads) t.join();
  if (failed.load() && error) std::rethrow_exception(error);
}

// ------------------------------------------------------------ convex.cpp
bool Part::contains(V3 p, double tol) const {  // convex.cpp:12-17
  for (size_t i = 0; i < plane_n.size(); ++i)
    if (dot(plane_n[i], p) > plane_d[i] + tol) return false;
  return true;
}

double Part::interior_depth(V3 p) const {  // convex.cpp:19-25
  double depth = kInf;
  for (size_t i = 0; i < plane_n.size(); ++i)
    depth = dmin(depth, plane_d[i] - dot(plane_n[i], p));
  return depth;
}

V3 closest_point_on_triangle(V3 p, V3 a, V3 b, V3 c) {  // convex.cpp:27-63
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
  // a + ab * v + ac * w
  return add(add(a, v3(ab.x * v, ab.y * v, ab.z * v)), v3(ac.x * w, ac.y * w, ac.z * w));
}

V3 Part::closest_surface_point(V3 p, V3* normal) const {  // convex.cpp:65-106
  if (contains(p)) {
    double best = kInf;
    int plane = -1;
    for (size_t i = 0; i < plane_n.size(); ++i) {
      double slack = plane_d[i] - dot(plane_n[i], p);
      if (slack < best) {
        best = slack;
        plane = (int)i;
      }
    }
    if (normal) *normal = plane_n[plane];
    return axpy(p, best, plane_n[plane]);
  }
  double best = kInf;
  V3 cp = v3(0.0, 0.0, 0.0);
  int face = 0;
  for (size_t t = 0; t < tris.size(); ++t) {
    V3 q = closest_point_on_triangle(p, verts[tris[t][0]], verts[tris[t][1]], verts[tris[t][2]]);
    double d2 = sqnorm(sub(p, q));
    if (d2 < best) {
      best = d2;
      cp = q;
      face = (int)t;
    }
  }
  if (normal) {
    double d = std::sqrt(best);
    if (d > 1e-12) {
      *normal = divs(sub(p, cp), d);
    } else {
      V3 e1 = sub(verts[tris[face][1]], verts[tris[face][0]]);
      V3 e2 = sub(verts[tris[face][2]], verts[tris[face][0]]);
      *normal = normalized(cross(e1, e2));
    }
  }
  return cp;
}

V3 Part::support(V3 dir) const {  // convex.cpp:108-119
  double best = -kInf;
  V3 out = v3(0.0, 0.0, 0.0);
  for (const V3& v : verts) {
    double d = dot(dir, v);
    if (d > best) {
      best = d;
      out = v;
    }
  }
  return out;
}

// -------------------------------------------------------------- hand.cpp
Hand Hand::from_desc(const lg_hand_desc& d) {
  Hand h;
  h.root = d.root;
  h.dof = d.dof;
  h.links.resize(d.n_links);
  for (int l = 0; l < d.n_links; ++l) {
    Link& k = h.links[l];
    k.parent = d.parent[l];
    k.jtype = d.joint_type[l];
    k.jidx = d.joint_index[l];
    k.origin.R = m3_load(d.origin_R + 9 * l);
    k.origin.t = v3_load(d.origin_t + 3 * l);
    k.axis = v3_load(d.axis + 3 * l);
    k.lo = d.limit_lo[l];
    k.hi = d.limit_hi[l];
  }
  h.topo.assign(d.topo_order, d.topo_order + d.n_links);
  h.parts.resize(d.n_parts);
  for (int p = 0; p < d.n_parts; ++p) {
    Part& part = h.parts[p];
    for (int v = d.part_vert_off[p]; v < d.part_vert_off[p + 1]; ++v)
      part.verts.push_back(v3_load(d.part_verts + 3 * v));
    for (int t = d.part_tri_off[p]; t < d.part_tri_off[p + 1]; ++t)
      part.tris.push_back({d.part_tris[3 * t], d.part_tris[3 * t + 1], d.part_tris[3 * t + 2]});
    for (int i = d.part_plane_off[p]; i < d.part_plane_off[p + 1]; ++i) {
      part.plane_n.push_back(v3_load(d.part_planes + 4 * i));
      part.plane_d.push_back(d.part_planes[4 * i + 3]);
    }
    part.bounds.min = v3_load(d.part_bounds + 6 * p);
    part.bounds.max = v3_load(d.part_bounds + 6 * p + 3);
    h.links[d.part_link[p]].parts.push_back(p);
  }
  return h;
}

std::vector<double> Hand::mid_config() const {
  std::vector<double> q(dof, 0.0);
  for (const Link& l : links)
    if (l.jidx >= 0) q[l.jidx] = 0.5 * (l.lo + l.hi);
  return q;
}

void Hand::clamp_to_limits(std::vector<double>& q) const {
  for (const Link& l : links)
    if (l.jidx >= 0) q[l.jidx] = dclamp(q[l.jidx], l.lo, l.hi);
}

std::vector<Xf> forward_kinematics(const Hand& h, const double* q) {
  std::vector<Xf> frames(h.links.size());
  for (int l : h.topo) {
    const Link& link = h.links[l];
    Xf local = link.origin;
    if (link.jtype == 1) {
      Xf m;
      m.R = angle_axis(q[link.jidx], link.axis);
      m.t = v3(0.0, 0.0, 0.0);
      local = xf_compose(local, m);
    } else if (link.jtype == 2) {
      local.t = add(local.t, mul(local.R, scale(q[link.jidx], link.axis)));
    }
    frames[l] = link.parent < 0 ? local : xf_compose(frames[link.parent], local);
  }
  return frames;
}

void point_jacobian(const Hand& h, const std::vector<Xf>& frames, int link, V3 lp,
                    double* J) {
  for (int i = 0; i < 3 * h.dof; ++i) J[i] = 0.0;
  V3 point = xf_apply(frames[link], lp);
  for (int l = link; l >= 0; l = h.links[l].parent) {
    const Link& lk = h.links[l];
    if (lk.jidx < 0) continue;
    V3 axis = mul(frames[l].R, lk.axis);
    V3 o = frames[l].t;
    V3 col = lk.jtype == 1 ? cross(axis, sub(point, o)) : axis;
    J[0 * h.dof + lk.jidx] = col.x;
    J[1 * h.dof + lk.jidx] = col.y;
    J[2 * h.dof + lk.jidx] = col.z;
  }
}

int Groups::group_of(int link) const {  // hand.cpp:365-372
  for (size_t g = 0; g < groups.size(); ++g)
    if (std::binary_search(groups[g].begin(), groups[g].end(), link)) return (int)g;
  return -1;
}

Groups dependency_groups(const Hand& h) {  // hand.cpp:374-411
  int n = (int)h.links.size();
  std::vector<bool> is_static(n, false);
  for (int l : h.topo) {
    const Link& link = h.links[l];
    if (link.parent < 0) is_static[l] = true;
    else if (is_static[link.parent] && link.jtype == 0) is_static[l] = true;
  }
  Groups out;
  std::vector<int> group_of(n, -1);
  std::map<int, std::vector<int>> by_seed;
  for (int l : h.topo) {
    if (is_static[l]) {
      out.static_links.push_back(l);
      continue;
    }
    int parent = h.links[l].parent;
    if (parent >= 0 && !is_static[parent]) group_of[l] = group_of[parent];
    else group_of[l] = l;
    by_seed[group_of[l]].push_back(l);
  }
  for (auto& kv : by_seed) {
    std::sort(kv.second.begin(), kv.second.end());
    out.groups.push_back(kv.second);
  }
  std::sort(out.groups.begin(), out.groups.end(),
            [](const std::vector<int>& a, const std::vector<int>& b) { return a[0] < b[0]; });
  std::sort(out.static_links.begin(), out.static_links.end());
  return out;
}

// ------------------------------------------------------------ collision.cpp
Aabb world_bounds(const Part& part, const Xf& pose) {  // collision.cpp:10-20
  Aabb out;
  const Aabb& b = part.bounds;
  for (int i = 0; i < 8; ++i) {
    V3 corner = v3((i & 1) ? b.max.x : b.min.x, (i & 2) ? b.max.y : b.min.y,
                   (i & 4) ? b.max.z : b.min.z);
    out.expand(xf_apply(pose, corner));
  }
  return out;
}

namespace {

// simplex_closest (collision.cpp:52-169)
bool simplex_closest(V3* s, int& n, V3& closest) {
  auto keep = [&](std::initializer_list<int> ids) {
    V3 tmp[4];
    int m = 0;
    for (int id : ids) tmp[m++] = s[id];
    for (int i = 0; i < m; ++i) s[i] = tmp[i];
    n = m;
  };
  if (n == 1) {
    closest = s[0];
    return false;
  }
  if (n == 2) {
    V3 ab = sub(s[1], s[0]);
    double t = -dot(s[0], ab);
    double len2 = sqnorm(ab);
    if (t <= 0.0 || len2 < 1e-30) {
      keep({0});
      closest = s[0];
    } else if (t >= len2) {
      keep({1});
      closest = s[1];
    } else {
      closest = axpy(s[0], t / len2, ab);
    }
    return false;
  }
  if (n == 3) {
    V3 a = s[0], b = s[1], c = s[2];
    V3 ab = sub(b, a), ac = sub(c, a);
    double d1 = -dot(ab, a), d2 = -dot(ac, a);
    if (d1 <= 0.0 && d2 <= 0.0) {
      keep({0});
      closest = a;
      return false;
    }
    double d3 = -dot(ab, b), d4 = -dot(ac, b);
    if (d3 >= 0.0 && d4 <= d3) {
      keep({1});
      closest = b;
      return false;
    }
    double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
      double v = d1 / (d1 - d3);
      keep({0, 1});
      closest = axpy(a, v, ab);
      return false;
    }
    double d5 = -dot(ab, c), d6 = -dot(ac, c);
    if (d6 >= 0.0 && d5 <= d6) {
      keep({2});
      closest = c;
      return false;
    }
    double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
      double w = d2 / (d2 - d6);
      keep({0, 2});
      closest = axpy(a, w, ac);
      return false;
    }
    double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
      double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
      keep({1, 2});
      closest = axpy(b, w, sub(c, b));
      return false;
    }
    double denom = va + vb + vc;
    if (std::abs(denom) < 1e-30) {
      keep({0, 1});
      return simplex_closest(s, n, closest);
    }
    double v = vb / denom, w = vc / denom;
    closest = axpy(axpy(a, v, ab), w, ac);
    return false;
  }
  static const int faces[4][3] = {{0, 1, 2}, {0, 3, 1}, {0, 2, 3}, {1, 3, 2}};
  static const int opposite[4] = {3, 2, 1, 0};
  bool inside = true;
  double best = kInf;
  V3 best_closest = v3(0.0, 0.0, 0.0);
  int best_n = 0;
  V3 best_simplex[4];
  for (int f = 0; f < 4; ++f) {
    V3 a = s[faces[f][0]], b = s[faces[f][1]], c = s[faces[f][2]];
    V3 nrm = cross(sub(b, a), sub(c, a));
    double side = dot(nrm, sub(s[opposite[f]], a));
    if (side > 0.0) nrm = neg(nrm);
    if (dot(nrm, neg(a)) <= 0.0) continue;
    inside = false;
    V3 sb[4] = {a, b, c, a};
    int sub_n = 3;
    V3 cp;
    simplex_closest(sb, sub_n, cp);
    double d2 = sqnorm(cp);
    if (d2 < best) {
      best = d2;
      best_closest = cp;
      best_n = sub_n;
      for (int i = 0; i < sub_n; ++i) best_simplex[i] = sb[i];
    }
  }
  if (inside) return true;
  n = best_n;
  for (int i = 0; i < best_n; ++i) s[i] = best_simplex[i];
  closest = best_closest;
  return false;
}

}  // namespace

double gjk_distance(const Part& a, const Xf& pa, const Part& b, const Xf& pb) {
  M3 rat = transpose(pa.R);
  M3 rbt = transpose(pb.R);
  auto support = [&](V3 d) {
    V3 sa = xf_apply(pa, a.support(mul(rat, d)));
    V3 sb = xf_apply(pb, b.support(mul(rbt, neg(d))));
    return sub(sa, sb);
  };
  V3 d0 = sub(pa.t, pb.t);
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
    if (progress <= 1e-12 + 1e-10 * v2) return std::sqrt(v2);
    if (n < 4) simplex[n++] = w;
    else return std::sqrt(v2);
  }
  return 0.0;
}

PenetrationResult object_penetration(const std::vector<Sample>& samples, const Part& part,
                                     const Xf& pose, double margin) {
  if (part.plane_n.empty())
    throw std::invalid_argument("object_penetration: part has no face planes");
  Xf inv = xf_inverse(pose);
  PenetrationResult r;
  Aabb bb = part.bounds.inflated(1e-9);
  for (size_t i = 0; i < samples.size(); ++i) {
    V3 local = xf_apply(inv, samples[i].p);
    if (!bb.contains(local)) continue;
    double depth = part.interior_depth(local);
    if (depth > margin) {
      r.offending.push_back((int)i);
      r.max_depth = dmax(r.max_depth, depth);
    }
  }
  return r;
}

CollisionReport validate_grasp_collisions(const Hand& h, const double* q,
                                          const std::vector<Sample>& samples,
                                          const Xf& pose, double margin) {
  auto frames = forward_kinematics(h, q);
  struct Posed {
    int part;
    int link;
  };
  std::vector<Posed> parts;
  for (size_t l = 0; l < h.links.size(); ++l)
    for (int p : h.links[l].parts) parts.push_back({p, (int)l});
  auto world = transform_samples(samples, pose);
  bool have_obj = !world.empty();
  Aabb obj;
  for (const Sample& s : world) obj.expand(s.p);

  // broad_phase (collision.cpp:22-45)
  if (margin < 0.0) throw std::invalid_argument("broad_phase: negative margin");
  std::vector<Aabb> boxes;
  for (const Posed& p : parts)
    boxes.push_back(world_bounds(h.parts[p.part], frames[p.link]).inflated(margin));
  std::vector<std::pair<int, int>> cand;
  Aabb obj_inf = obj.inflated(margin);
  for (size_t i = 0; i < parts.size(); ++i) {
    for (size_t j = i + 1; j < parts.size(); ++j)
      if (boxes[i].overlaps(boxes[j])) cand.push_back({(int)i, (int)j});
    if (have_obj && boxes[i].overlaps(obj_inf)) cand.push_back({(int)i, -1});
  }

  CollisionReport rep;
  rep.broad_pairs = (long)cand.size();
  struct Viol {
    int a, b;
    double depth;
  };
  std::vector<Viol> viol;
  auto record = [&](int la, int lb, double depth) {
    for (auto& v : viol) {
      if (v.a == la && v.b == lb) {
        v.depth = dmax(v.depth, depth);
        return;
      }
    }
    viol.push_back({la, lb, depth});
  };
  auto adjacent = [&](int la, int lb) {
    return h.links[la].parent == lb || h.links[lb].parent == la;
  };
  for (const auto& pr : cand) {
    const Posed& pa = parts[pr.first];
    if (pr.second >= 0) {
      const Posed& pb = parts[pr.second];
      if (pa.link == pb.link || adjacent(pa.link, pb.link)) continue;
      ++rep.narrow_gjk;
      if (gjk_distance(h.parts[pa.part], frames[pa.link], h.parts[pb.part], frames[pb.link]) ==
          0.0)
        record(std::min(pa.link, pb.link), std::max(pa.link, pb.link), 0.0);
    } else {
      ++rep.narrow_halfplane;
      auto pen = object_penetration(world, h.parts[pa.part], frames[pa.link], margin);
      if (!pen.offending.empty()) {
        record(pa.link, -1, pen.max_depth);
        rep.max_penetration = dmax(rep.max_penetration, pen.max_depth);
      }
    }
  }
  rep.n_violations = (int)viol.size();
  return rep;
}

// --------------------------------------------------------------- wrench.cpp
WrenchProblem make_wrench_problem(const std::vector<V3>& p, const std::vector<V3>& n,
                                  double lambda, double mu) {  // wrench.cpp:31-45
  WrenchProblem w;
  w.p = p;
  w.n = n;
  w.lambda = lambda;
  w.mu = mu;
  w.tx.resize(p.size());
  w.ty.resize(p.size());
  for (size_t i = 0; i < p.size(); ++i) tangent_basis(w.n[i], w.tx[i], w.ty[i]);
  return w;
}

namespace {

struct Precomp {  // wrench.cpp:50-64
  std::vector<V3> cn, cx, cy;
  explicit Precomp(const WrenchProblem& p) {
    size_t n = p.size();
    cn.resize(n);
    cx.resize(n);
    cy.resize(n);
    for (size_t i = 0; i < n; ++i) {
      cn[i] = cross(p.p[i], p.n[i]);
      cx[i] = cross(p.p[i], p.tx[i]);
      cy[i] = cross(p.p[i], p.ty[i]);
    }
  }
};

struct State {
  std::vector<double> a, bx, by;
};

// force/torque accumulation shared by eval and the gradient
void net_wrench(const WrenchProblem& p, const Precomp& pre, const State& s, V3& force,
                V3& torque) {
  force = v3(0.0, 0.0, 0.0);
  torque = v3(0.0, 0.0, 0.0);
  for (size_t i = 0; i < p.size(); ++i) {
    V3 f = add(add(scale(s.a[i], p.n[i]), scale(s.bx[i], p.tx[i])), scale(s.by[i], p.ty[i]));
    force = add(force, f);
    V3 t = add(add(scale(s.a[i], pre.cn[i]), scale(s.bx[i], pre.cx[i])),
               scale(s.by[i], pre.cy[i]));
    torque = add(torque, t);
  }
}

double eval(const WrenchProblem& p, const Precomp& pre, const State& s) {  // :70-80
  V3 f, t;
  net_wrench(p, pre, s, f, t);
  return sqnorm(f) + p.lambda * sqnorm(t);
}

void project(const WrenchProblem& p, int anchor, bool fr, State& s) {  // :82-108
  for (size_t i = 0; i < s.a.size(); ++i) {
    if ((int)i == anchor) s.a[i] = 1.0;
    else if (s.a[i] < 0.0) s.a[i] = 0.0;
    if (!fr) {
      s.bx[i] = 0.0;
      s.by[i] = 0.0;
      continue;
    }
    double cap = p.mu * s.a[i];
    double r = lgm::xhypot(s.bx[i], s.by[i]);
    if (r > cap) {
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

double descend(const WrenchProblem& p, const Precomp& pre, int anchor, bool fr, int iterations,
               const WrenchOpts& o, State& s) {  // :124-177
  project(p, anchor, fr, s);
  double current = eval(p, pre, s);
  size_t n = p.size();
  std::vector<double> ga(n), gx(n), gy(n);
  State trial = s;
  for (int it = 0; it < iterations; ++it) {
    V3 force, torque;
    net_wrench(p, pre, s, force, torque);
    torque = v3(torque.x * p.lambda, torque.y * p.lambda, torque.z * p.lambda);
    for (size_t i = 0; i < n; ++i) {
      ga[i] = 2.0 * (dot(force, p.n[i]) + dot(torque, pre.cn[i]));
      if (fr) {
        gx[i] = 2.0 * (dot(force, p.tx[i]) + dot(torque, pre.cx[i]));
        gy[i] = 2.0 * (dot(force, p.ty[i]) + dot(torque, pre.cy[i]));
      }
    }
    double step = o.step;
    bool moved = false;
    for (int bt = 0; bt <= o.max_backtracks; ++bt) {
      for (size_t i = 0; i < n; ++i) {
        trial.a[i] = s.a[i] - step * ga[i];
        if (fr) {
          trial.bx[i] = s.bx[i] - step * gx[i];
          trial.by[i] = s.by[i] - step * gy[i];
        } else {
          trial.bx[i] = 0.0;
          trial.by[i] = 0.0;
        }
      }
      project(p, anchor, fr, trial);
      double next = eval(p, pre, trial);
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

WrenchSolution run_solver(const WrenchProblem& prob, bool fr, const WrenchOpts& o,
                          const WrenchSolution* warm) {  // :179-226
  if (prob.size() == 0) throw std::invalid_argument("wrench solve: no contacts");
  size_t n = prob.size();
  Precomp pre(prob);
  bool use_warm = warm && warm->valid() && warm->alpha.size() == n;
  int iterations = use_warm ? o.warm_iterations : o.iterations;
  WrenchSolution best;
  for (int anchor = 0; anchor < (int)n; ++anchor) {
    State s;
    if (use_warm) {
      s.a = warm->alpha;
      s.bx = warm->bx.size() == n ? warm->bx : std::vector<double>(n, 0.0);
      s.by = warm->by.size() == n ? warm->by : std::vector<double>(n, 0.0);
    } else {
      s.a.assign(n, 1.0);
      s.bx.assign(n, 0.0);
      s.by.assign(n, 0.0);
    }
    double value;
    if (fr) {
      descend(prob, pre, anchor, false, iterations, o, s);
      value = descend(prob, pre, anchor, true, iterations, o, s);
    } else {
      value = descend(prob, pre, anchor, false, iterations, o, s);
    }
    if (value < best.objective) {
      best.objective = value;
      best.anchor = anchor;
      best.alpha = s.a;
      best.bx = s.bx;
      best.by = s.by;
    }
  }
  return best;
}

}  // namespace

double wrench_objective(const WrenchProblem& p, const WrenchSolution& sol) {  // :229-245
  if (sol.alpha.size() != p.size())
    throw std::invalid_argument("wrench_objective: size mismatch");
  Precomp pre(p);
  State s;
  s.a = sol.alpha;
  s.bx = sol.bx.size() == p.size() ? sol.bx : std::vector<double>(p.size(), 0.0);
  s.by = sol.by.size() == p.size() ? sol.by : std::vector<double>(p.size(), 0.0);
  return eval(p, pre, s);
}

WrenchSolution solve_fswo(const WrenchProblem& p, const WrenchOpts& o,
                          const WrenchSolution* warm) {
  return run_solver(p, false, o, warm);
}

WrenchSolution solve_gswo(const WrenchProblem& p, const WrenchOpts& o,
                          const WrenchSolution* warm) {
  if (p.mu == 0.0) return solve_fswo(p, o, warm);
  return run_solver(p, true, o, warm);
}

bool is_stable(const WrenchProblem& p, double eps, WrenchSolution* sol, const WrenchOpts& o) {
  if (eps <= 0.0) throw std::invalid_argument("is_stable: eps must be > 0");
  WrenchSolution s = solve_gswo(p, o, nullptr);
  bool stable = s.objective < eps;
  if (sol) *sol = s;
  return stable;
}

// ---------------------------------------------------------- contact_opt.cpp
int project_to_domain(V3 c, const Domain& d) {  // contact_opt.cpp:11-25
  if (d.elements.empty()) throw std::invalid_argument("project_to_domain: empty domain");
  int best = 0;
  double best_d2 = sqnorm(sub(d.elements[0].position, c));
  for (int i = 1; i < (int)d.elements.size(); ++i) {
    double d2 = sqnorm(sub(d.elements[i].position, c));
    if (d2 < best_d2) {
      best_d2 = d2;
      best = i;
    }
  }
  return best;
}

namespace {

void write_slot(WrenchProblem& prob, int i, const DomainElement& el) {  // :31-35
  prob.p[i] = el.position;
  prob.n[i] = neg(el.normal);
  tangent_basis(prob.n[i], prob.tx[i], prob.ty[i]);
}

WrenchSolution solve(const WrenchProblem& p, const WrenchOpts& o, const WrenchSolution* warm) {
  return p.mu > 0.0 ? solve_gswo(p, o, warm) : solve_fswo(p, o, warm);
}

}  // namespace

ContactOptResult optimize_contacts(const std::vector<const Domain*>& domains,
                                   const ContactOptParams& params,
                                   const std::vector<StaticContact>& statics,
                                   uint64_t seed) {  // contact_opt.cpp:45-142
  const int k = (int)domains.size();
  if (k < 1) throw std::invalid_argument("optimize_contacts: no domains");
  for (const Domain* d : domains)
    if (!d || d->elements.empty()) throw std::invalid_argument("optimize_contacts: empty domain");
  if (params.sigma <= 0.0 || params.n_inner < 1 || params.n_outer < 0 || params.restarts < 1)
    throw std::invalid_argument("optimize_contacts: bad parameters");
  Rng rng(seed);
  const int s = (int)statics.size();
  WrenchProblem prob;
  prob.lambda = params.lambda;
  prob.mu = params.mu;
  prob.p.resize(k + s);
  prob.n.resize(k + s);
  prob.tx.resize(k + s);
  prob.ty.resize(k + s);
  for (int j = 0; j < s; ++j) {
    prob.p[k + j] = statics[j].position;
    prob.n[k + j] = statics[j].normal;
    tangent_basis(prob.n[k + j], prob.tx[k + j], prob.ty[k + j]);
  }
  ContactOptResult result;
  int evaluations = 0;
  for (int restart = 0; restart < params.restarts; ++restart) {
    ContactOptResult run;
    run.element_ids.resize(k);
    for (int i = 0; i < k; ++i) {
      run.element_ids[i] = (int)rng.uniform_index(domains[i]->elements.size());
      write_slot(prob, i, domains[i]->elements[run.element_ids[i]]);
    }
    run.solution = solve(prob, params.solve, nullptr);
    run.objective = run.solution.objective;
    ++evaluations;
    WrenchProblem trial = prob;
    for (int outer = 0; outer < params.n_outer; ++outer) {
      for (int i = 0; i < k; ++i) {
        const Domain& domain = *domains[i];
        const DomainElement& cur = domain.elements[run.element_ids[i]];
        V3 tx, ty;
        tangent_basis(neg(cur.normal), tx, ty);
        int best_id = -1;
        double best_obj = run.objective;
        WrenchSolution best_sol;
        for (int m = 0; m < params.n_inner; ++m) {
          double u = params.sigma * rng.normal();
          double v = params.sigma * rng.normal();
          V3 cp = axpy(axpy(cur.position, u, tx), v, ty);
          int cand = project_to_domain(cp, domain);
          write_slot(trial, i, domain.elements[cand]);
          WrenchSolution sol = solve(trial, params.solve, &run.solution);
          ++evaluations;
          if (sol.objective < best_obj) {
            best_obj = sol.objective;
            best_id = cand;
            best_sol = sol;
          }
        }
        if (best_id >= 0) {
          run.element_ids[i] = best_id;
          write_slot(prob, i, domain.elements[best_id]);
          run.solution = best_sol;
          run.objective = best_obj;
        }
        trial.p[i] = prob.p[i];
        trial.n[i] = prob.n[i];
        trial.tx[i] = prob.tx[i];
        trial.ty[i] = prob.ty[i];
      }
    }
    if (run.objective < result.objective) result = run;
  }
  result.evaluations = evaluations;
  result.elements.clear();
  for (int i = 0; i < k; ++i) result.elements.push_back(domains[i]->elements[result.element_ids[i]]);
  return result;
}

// ------------------------------------------------------------------- ik.cpp
namespace {

// stacked_residual (ik.cpp:13-27)
void stacked_residual(const std::vector<Xf>& frames, const std::vector<ContactTarget>& t,
                      double beta, std::vector<double>& r) {
  r.resize(6 * t.size());
  for (size_t i = 0; i < t.size(); ++i) {
    const Xf& f = frames[t[i].link];
    V3 hp = xf_apply(f, t[i].hand_point);
    V3 hn = xf_rotate(f, t[i].hand_normal);
    V3 a = sub(t[i].object_point, hp);
    V3 b = sub(axpy(t[i].object_point, beta, t[i].object_normal), axpy(hp, beta, hn));
    r[6 * i + 0] = a.x;
    r[6 * i + 1] = a.y;
    r[6 * i + 2] = a.z;
    r[6 * i + 3] = b.x;
    r[6 * i + 4] = b.y;
    r[6 * i + 5] = b.z;
  }
}

double sum_squares(const std::vector<double>& r) {
  double s = 0.0;
  for (double v : r) s = s + v * v;
  return s;
}

// Eigen LDLT<MatrixXd> (lower, diagonal pivoting) factor + solve, unblocked,
// canonical summation order.  A is n x n row-major, destroyed.
void ldlt_solve(int n, double* A, double* x) {
  int tr[LG_MAX_DOF];
  double temp[LG_MAX_DOF];
  for (int k = 0; k < n; ++k) {
    int big = k;
    double best = std::abs(A[k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      double v = std::abs(A[i * n + i]);
      if (v > best) {
        best = v;
        big = i;
      }
    }
    tr[k] = big;
    if (k != big) {
      for (int j = 0; j < k; ++j) std::swap(A[k * n + j], A[big * n + j]);
      for (int i = big + 1; i < n; ++i) std::swap(A[i * n + k], A[i * n + big]);
      std::swap(A[k * n + k], A[big * n + big]);
      for (int i = k + 1; i < big; ++i) {
        double t = A[i * n + k];
        A[i * n + k] = A[big * n + i];
        A[big * n + i] = t;
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
    if (std::abs(akk) > 0.0)
      for (int i = k + 1; i < n; ++i) A[i * n + k] /= akk;
  }
  for (int k = 0; k < n; ++k) std::swap(x[k], x[tr[k]]);
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < i; ++j) s = s + A[i * n + j] * x[j];
    x[i] -= s;
  }
  for (int i = 0; i < n; ++i) {
    double d = A[i * n + i];
    if (std::abs(d) > 2.2250738585072014e-308) x[i] /= d;
    else x[i] = 0.0;
  }
  // L^T back substitution; canonical order: the sum for x[i] accumulates
  // j = n-1 down to i+1 (the order in which the x[j] become final).
  for (int i = n - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = n - 1; j > i; --j) s = s + A[j * n + i] * x[j];
    x[i] -= s;
  }
  for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[tr[k]]);
}

bool all_finite(const std::vector<double>& v) {
  for (double d : v)
    if (!std::isfinite(d)) return false;
  return true;
}

}  // namespace

IkResult solve_contact_ik(const Hand& h, const std::vector<double>& q0,
                          const std::vector<ContactTarget>& targets, const IkParams& p) {
  if ((int)q0.size() != h.dof)
    throw std::invalid_argument("solve_contact_ik: config dimension mismatch");
  if (p.beta <= 0.0) throw std::invalid_argument("solve_contact_ik: beta must be > 0");
  for (const auto& t : targets)
    if (t.link < 0 || t.link >= (int)h.links.size())
      throw std::invalid_argument("solve_contact_ik: invalid target link");
  const int dof = h.dof;
  const size_t k = targets.size();
  IkResult res;
  res.q = q0;
  h.clamp_to_limits(res.q);
  res.used.assign(dof, false);
  res.res_pos.assign(k, 0.0);
  res.res_angle.assign(k, 0.0);
  if (k == 0) return res;
  auto frames = forward_kinematics(h, res.q.data());
  std::vector<double> r, r_try;
  stacked_residual(frames, targets, p.beta, r);
  double objective = sum_squares(r);
  const int rows = (int)(6 * k);
  std::vector<double> J(rows * dof), Jp(3 * dof), JtJ(dof * dof), dq(dof);
  for (int it = 0; it < p.iterations; ++it) {
    res.iterations = it + 1;
    for (size_t i = 0; i < k; ++i) {
      const ContactTarget& t = targets[i];
      point_jacobian(h, frames, t.link, t.hand_point, Jp.data());
      for (int rr = 0; rr < 3; ++rr)
        for (int c = 0; c < dof; ++c) J[(6 * i + rr) * dof + c] = Jp[rr * dof + c];
      point_jacobian(h, frames, t.link, axpy(t.hand_point, p.beta, t.hand_normal), Jp.data());
      for (int rr = 0; rr < 3; ++rr)
        for (int c = 0; c < dof; ++c) J[(6 * i + 3 + rr) * dof + c] = Jp[rr * dof + c];
    }
    for (int c = 0; c < dof; ++c) {
      if (res.used[c]) continue;
      double mx = 0.0;
      for (int rr = 0; rr < rows; ++rr) mx = dmax(mx, std::abs(J[rr * dof + c]));
      if (mx > 1e-12) res.used[c] = true;
    }
    for (int a = 0; a < dof; ++a)
      for (int b = 0; b < dof; ++b) {
        double s = 0.0;
        for (int rr = 0; rr < rows; ++rr) s = s + J[rr * dof + a] * J[rr * dof + b];
        JtJ[a * dof + b] = s;
      }
    double tr = 0.0;
    for (int a = 0; a < dof; ++a) tr = tr + JtJ[a * dof + a];
    double lambda = dmax(p.damping_min, p.damping_scale * tr / (double)std::max(1, dof));
    for (int a = 0; a < dof; ++a) JtJ[a * dof + a] += lambda;
    for (int a = 0; a < dof; ++a) {
      double s = 0.0;
      for (int rr = 0; rr < rows; ++rr) s = s + J[rr * dof + a] * r[rr];
      dq[a] = s;
    }
    ldlt_solve(dof, JtJ.data(), dq.data());
    if (!all_finite(dq)) {
      res.finite = false;
      break;
    }
    bool moved = false;
    std::vector<double> q_try(dof);
    for (int bt = 0; bt <= p.max_backtracks; ++bt) {
      for (int c = 0; c < dof; ++c) {
        double st = dmin(dmax(dq[c], -p.step_clamp), p.step_clamp);
        q_try[c] = res.q[c] + st;
      }
      h.clamp_to_limits(q_try);
      auto frames_try = forward_kinematics(h, q_try.data());
      stacked_residual(frames_try, targets, p.beta, r_try);
      double obj_try = sum_squares(r_try);
      if (obj_try <= objective) {
        res.q = q_try;
        frames = frames_try;
        r = r_try;
        objective = obj_try;
        moved = true;
        break;
      }
      for (int c = 0; c < dof; ++c) dq[c] *= 0.5;
    }
    if (!moved) break;
    double max_pos = 0.0;
    for (size_t i = 0; i < k; ++i)
      max_pos = dmax(max_pos, norm(v3(r[6 * i], r[6 * i + 1], r[6 * i + 2])));
    if (max_pos < p.residual_tol) break;
  }
  if (!all_finite(res.q)) res.finite = false;
  res.objective = objective;
  for (size_t i = 0; i < k; ++i) {
    const Xf& f = frames[targets[i].link];
    res.res_pos[i] = norm(v3(r[6 * i], r[6 * i + 1], r[6 * i + 2]));
    V3 hn = xf_rotate(f, targets[i].hand_normal);
    double c = dclamp(dot(hn, targets[i].object_normal), -1.0, 1.0);
    res.res_angle[i] = std::acos(c);
  }
  return res;
}

}  // namespace orc
