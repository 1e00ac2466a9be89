// hull.cpp — incremental 3D quickhull producing the convex collision parts
// of hand links (reference convex.cpp:139-359).  Load time only; the device
// receives the resulting vertices, triangles and distinct face planes, and
// their ORDER matters (support() and closest_surface_point() break ties by
// lowest index), so the construction order follows the reference exactly.
#include <cmath>
#include <map>
#include <unordered_map>

#include "host.hpp"

namespace lgh {

using namespace lgm;

namespace {
struct Face {
  int a, b, c;
  V3 n;
  double off;
  bool alive = true;
  std::vector<int> outside;
  int far_point = -1;
  double far_dist = 0.0;
};
}  // namespace

Part convex_hull(const std::vector<V3>& P) {
  if (P.size() < 4) fail_invalid("convex_hull: need at least 4 points");
  V3 bmin = v3(INFINITY, INFINITY, INFINITY), bmax = v3(-INFINITY, -INFINITY, -INFINITY);
  for (const V3& p : P) {
    if (!std::isfinite(p.x) || !std::isfinite(p.y) || !std::isfinite(p.z))
      fail_invalid("convex_hull: non-finite input point");
    bmin = vmin(bmin, p);
    bmax = vmax(bmax, p);
  }
  V3 ext = sub(bmax, bmin);
  double scl = dmax(dmax(dmax(ext.x, ext.y), ext.z), 1e-9);
  const double eps = 1e-10 * scl;
  const int n = (int)P.size();

  int i0 = 0, i1 = 0;
  {
    double best = -1.0;
    for (int axis = 0; axis < 3; ++axis) {
      int lo = 0, hi = 0;
      for (int i = 1; i < n; ++i) {
        if (comp(P[i], axis) < comp(P[lo], axis)) lo = i;
        if (comp(P[i], axis) > comp(P[hi], axis)) hi = i;
      }
      double d = comp(P[hi], axis) - comp(P[lo], axis);
      if (d > best) {
        best = d;
        i0 = lo;
        i1 = hi;
      }
    }
    if (best <= eps) fail_invalid("convex_hull: degenerate point set");
  }
  V3 dir = normalized(sub(P[i1], P[i0]));
  int i2 = -1;
  {
    double best = eps;
    for (int i = 0; i < n; ++i) {
      V3 d = sub(P[i], P[i0]);
      double dist = norm(sub(d, scale(dot(d, dir), dir)));
      if (dist > best) {
        best = dist;
        i2 = i;
      }
    }
    if (i2 < 0) fail_invalid("convex_hull: collinear point set");
  }
  V3 pn = normalized(cross(sub(P[i1], P[i0]), sub(P[i2], P[i0])));
  double pd = dot(pn, P[i0]);
  int i3 = -1;
  {
    double best = eps;
    for (int i = 0; i < n; ++i) {
      double dist = std::abs(dot(pn, P[i]) - pd);
      if (dist > best) {
        best = dist;
        i3 = i;
      }
    }
    if (i3 < 0) fail_invalid("convex_hull: coplanar point set");
  }
  if (dot(pn, P[i3]) - pd > 0.0) std::swap(i1, i2);

  std::vector<Face> faces;
  auto add_face = [&](int a, int b, int c) {
    Face f;
    f.a = a;
    f.b = b;
    f.c = c;
    V3 nrm = cross(sub(P[b], P[a]), sub(P[c], P[a]));
    double len = norm(nrm);
    f.n = len > 0.0 ? divs(nrm, len) : v3(0, 0, 1);
    f.off = dot(f.n, P[a]);
    faces.push_back(std::move(f));
    return (int)faces.size() - 1;
  };
  auto sdist = [&](const Face& f, V3 p) { return dot(f.n, p) - f.off; };
  add_face(i0, i1, i2);
  add_face(i0, i2, i3);
  add_face(i0, i3, i1);
  add_face(i1, i3, i2);
  for (int i = 0; i < n; ++i) {
    if (i == i0 || i == i1 || i == i2 || i == i3) continue;
    for (auto& f : faces) {
      double d = sdist(f, P[i]);
      if (d > eps) {
        f.outside.push_back(i);
        if (d > f.far_dist) {
          f.far_dist = d;
          f.far_point = i;
        }
        break;
      }
    }
  }
  for (;;) {
    int grow = -1;
    for (int fi = 0; fi < (int)faces.size(); ++fi)
      if (faces[fi].alive && !faces[fi].outside.empty()) {
        grow = fi;
        break;
      }
    if (grow < 0) break;
    int apex = faces[grow].far_point;
    V3 p = P[apex];
    std::vector<int> visible;
    for (int fi = 0; fi < (int)faces.size(); ++fi)
      if (faces[fi].alive && sdist(faces[fi], p) > eps) visible.push_back(fi);
    std::map<std::pair<int, int>, int> edges;
    for (int fi = 0; fi < (int)faces.size(); ++fi) {
      if (!faces[fi].alive) continue;
      const Face& f = faces[fi];
      edges[{f.a, f.b}] = fi;
      edges[{f.b, f.c}] = fi;
      edges[{f.c, f.a}] = fi;
    }
    std::vector<bool> is_vis(faces.size(), false);
    for (int fi : visible) is_vis[fi] = true;
    std::vector<std::pair<int, int>> horizon;
    for (int fi : visible) {
      const Face& f = faces[fi];
      const std::pair<int, int> es[3] = {{f.a, f.b}, {f.b, f.c}, {f.c, f.a}};
      for (const auto& e : es) {
        auto twin = edges.find({e.second, e.first});
        if (twin == edges.end() || !is_vis[twin->second]) horizon.push_back(e);
      }
    }
    std::vector<int> orphaned;
    for (int fi : visible) {
      faces[fi].alive = false;
      for (int i : faces[fi].outside)
        if (i != apex) orphaned.push_back(i);
      faces[fi].outside.clear();
    }
    std::vector<int> created;
    for (const auto& e : horizon) created.push_back(add_face(e.first, e.second, apex));
    for (int i : orphaned) {
      for (int fi : created) {
        double d = sdist(faces[fi], P[i]);
        if (d > eps) {
          faces[fi].outside.push_back(i);
          if (d > faces[fi].far_dist) {
            faces[fi].far_dist = d;
            faces[fi].far_point = i;
          }
          break;
        }
      }
    }
  }
  Part part;
  std::unordered_map<int, int> remap;
  for (const Face& f : faces) {
    if (!f.alive) continue;
    int idx[3] = {f.a, f.b, f.c};
    std::array<int, 3> tri;
    for (int k = 0; k < 3; ++k) {
      auto it = remap.find(idx[k]);
      if (it == remap.end()) {
        int id = (int)part.verts.size();
        part.verts.push_back(P[idx[k]]);
        remap.emplace(idx[k], id);
        tri[k] = id;
      } else {
        tri[k] = it->second;
      }
    }
    part.tris.push_back(tri);
    bool merged = false;
    for (size_t i = 0; i < part.plane_n.size(); ++i) {
      if (dot(part.plane_n[i], f.n) > 1.0 - 1e-9 &&
          std::abs(part.plane_d[i] - f.off) < 1e-7 * scl + 1e-12) {
        merged = true;
        break;
      }
    }
    if (!merged) {
      part.plane_n.push_back(f.n);
      part.plane_d.push_back(f.off);
    }
  }
  part.bmin = v3(INFINITY, INFINITY, INFINITY);
  part.bmax = v3(-INFINITY, -INFINITY, -INFINITY);
  for (const V3& v : part.verts) {
    part.bmin = vmin(part.bmin, v);
    part.bmax = vmax(part.bmax, v);
  }
  return part;
}

Part scale_part(const Part& p, double s) {  // convex.cpp:665-676
  Part out;
  for (const V3& v : p.verts) out.verts.push_back(scale(s, v));
  out.tris = p.tris;
  out.plane_n = p.plane_n;
  for (double d : p.plane_d) out.plane_d.push_back(s * d);
  out.bmin = v3(INFINITY, INFINITY, INFINITY);
  out.bmax = v3(-INFINITY, -INFINITY, -INFINITY);
  for (const V3& v : out.verts) {
    out.bmin = vmin(out.bmin, v);
    out.bmax = vmax(out.bmax, v);
  }
  return out;
}

}  // namespace lgh
