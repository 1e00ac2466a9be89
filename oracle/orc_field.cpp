// oracle/orc_field.cpp — surface sampling, patch decomposition, contact-field
// index build (std::map accumulation + median-split BVHs) and the BVH query /
// reverse lookup of the reference, restated for the CPU parity oracle.
#include <algorithm>
#include <cmath>

#include "orc.hpp"

namespace orc {

using namespace lgm;

namespace {
constexpr uint64_t kTagPatch = 0x70617463;   // contact_field.cpp:16
constexpr uint64_t kTagSubset = 0x73756273;  // contact_field.cpp:17
constexpr uint64_t kTagConfig = 0x636f6e66;  // contact_field.cpp:18
constexpr double kBoundsEps = 1e-9;          // contact_field.cpp:22

V3 face_normal(const std::vector<V3>& v, const std::array<int, 3>& t) {  // mesh.cpp:16-24
  V3 n = cross(sub(v[t[1]], v[t[0]]), sub(v[t[2]], v[t[0]]));
  double len = norm(n);
  if (len < 1e-300) return v3(0.0, 0.0, 1.0);
  return divs(n, len);
}
double face_area(const std::vector<V3>& v, const std::array<int, 3>& t) {  // mesh.cpp:26-31
  return 0.5 * norm(cross(sub(v[t[1]], v[t[0]]), sub(v[t[2]], v[t[0]])));
}
}  // namespace

std::vector<Sample> sample_surface(const std::vector<V3>& verts,
                                   const std::vector<std::array<int, 3>>& tris,
                                   double spc, uint64_t seed) {  // mesh.cpp:297-339
  if (tris.empty()) return {};
  double area = 0.0;
  for (const auto& t : tris) area += face_area(verts, t);
  size_t count = (size_t)std::llround(area * 1e4 * spc);
  if (count == 0) count = 1;
  std::vector<double> cum(tris.size());
  double acc = 0.0;
  for (size_t t = 0; t < tris.size(); ++t) {
    acc += face_area(verts, tris[t]);
    cum[t] = acc;
  }
  Rng rng(seed);
  std::vector<Sample> out;
  out.reserve(count);
  for (size_t i = 0; i < count; ++i) {
    double pick = rng.uniform() * acc;
    size_t t = std::lower_bound(cum.begin(), cum.end(), pick) - cum.begin();
    t = std::min(t, tris.size() - 1);
    double u = rng.uniform();
    double v = rng.uniform();
    if (u + v > 1.0) {
      u = 1.0 - u;
      v = 1.0 - v;
    }
    V3 a = verts[tris[t][0]], b = verts[tris[t][1]], c = verts[tris[t][2]];
    Sample s;
    s.p = axpy(axpy(a, u, sub(b, a)), v, sub(c, a));
    s.n = face_normal(verts, tris[t]);
    out.push_back(s);
  }
  return out;
}

std::vector<Sample> transform_samples(const std::vector<Sample>& s, const Xf& t) {
  std::vector<Sample> out;
  out.reserve(s.size());
  for (const Sample& x : s) out.push_back({xf_apply(t, x.p), xf_rotate(t, x.n)});
  return out;
}

std::vector<Patch> patches_from_desc(const lg_patches_desc& d) {
  std::vector<Patch> out(d.n_patches);
  for (int p = 0; p < d.n_patches; ++p) {
    Patch& P = out[p];
    P.id = p;
    P.link = d.link[p];
    for (int i = d.point_off[p]; i < d.point_off[p + 1]; ++i) {
      P.points.push_back(v3_load(d.points + 3 * i));
      P.normals.push_back(v3_load(d.normals + 3 * i));
    }
    for (int i = d.fp_off[p]; i < d.fp_off[p + 1]; ++i) P.field_points.push_back(d.field_points[i]);
  }
  return out;
}

std::vector<Patch> decompose_patches(const Hand& h,
                                     const std::vector<std::vector<Sample>>& per_link,
                                     double patch_radius, uint64_t seed,
                                     int cap) {  // contact_field.cpp:26-99
  if (per_link.size() != h.links.size())
    throw std::invalid_argument("decompose_patches: per-link sample mismatch");
  if (patch_radius <= 0.0 || cap < 1)
    throw std::invalid_argument("decompose_patches: bad radius or cap");
  size_t total = 0;
  for (const auto& s : per_link) total += s.size();
  if (total == 0) throw std::invalid_argument("decompose_patches: no surface samples");
  const double gather = 0.5 * patch_radius;
  std::vector<Patch> patches;
  for (size_t link = 0; link < per_link.size(); ++link) {
    const auto& S = per_link[link];
    if (S.empty()) continue;
    Rng rng(mix_seed(seed, kTagPatch, link));
    std::vector<int> uncovered(S.size());
    for (size_t i = 0; i < S.size(); ++i) uncovered[i] = (int)i;
    while (!uncovered.empty()) {
      size_t pick = rng.uniform_index(uncovered.size());
      int sid = uncovered[pick];
      V3 center = S[sid].p;
      Patch P;
      P.id = (int)patches.size();
      P.link = (int)link;
      std::vector<int> rest;
      P.points.push_back(center);
      P.normals.push_back(S[sid].n);
      for (int id : uncovered) {
        if (id == sid) continue;
        if (norm(sub(S[id].p, center)) <= gather) {
          P.points.push_back(S[id].p);
          P.normals.push_back(S[id].n);
        } else {
          rest.push_back(id);
        }
      }
      uncovered.swap(rest);
      int m = (int)P.points.size();
      if (m <= cap) {
        for (int i = 0; i < m; ++i) P.field_points.push_back(i);
      } else {
        Rng sr(mix_seed(seed, kTagSubset, (uint64_t)P.id));
        std::vector<int> pool(m - 1);
        for (int i = 1; i < m; ++i) pool[i - 1] = i;
        P.field_points.push_back(0);
        for (int i = 0; i < cap - 1; ++i) {
          size_t j = i + sr.uniform_index(pool.size() - i);
          std::swap(pool[i], pool[j]);
          P.field_points.push_back(pool[i]);
        }
        std::sort(P.field_points.begin(), P.field_points.end());
      }
      patches.push_back(std::move(P));
    }
  }
  return patches;
}

std::vector<double> field_config(const Hand& h, uint64_t seed, int c) {  // :101-114
  Rng rng(mix_seed(seed, kTagConfig, (uint64_t)c));
  std::vector<double> q(h.dof, 0.0);
  std::vector<std::pair<int, int>> act;
  for (size_t l = 0; l < h.links.size(); ++l)
    if (h.links[l].jidx >= 0) act.push_back({h.links[l].jidx, (int)l});
  std::sort(act.begin(), act.end());
  for (const auto& a : act) q[a.first] = rng.uniform(h.links[a.second].lo, h.links[a.second].hi);
  return q;
}

std::vector<V3> make_codebook(int size) {  // :144-158 (glibc cos/sin, host side)
  if (size < 1 || size > 65536) throw std::invalid_argument("make_codebook: size out of range");
  std::vector<V3> dirs(size);
  const double golden = kPi * (3.0 - std::sqrt(5.0));
  for (int i = 0; i < size; ++i) {
    double z = 1.0 - 2.0 * (i + 0.5) / size;
    double r = std::sqrt(dmax(0.0, 1.0 - z * z));
    double a = golden * i;
    dirs[i] = v3(r * std::cos(a), r * std::sin(a), z);
  }
  return dirs;
}

uint16_t quantize_normal(const std::vector<V3>& cb, V3 n) {  // :160-172
  int best = 0;
  double best_dot = -2.0;
  for (int i = 0; i < (int)cb.size(); ++i) {
    double d = dot(cb[i], n);
    if (d > best_dot) {
      best_dot = d;
      best = i;
    }
  }
  return (uint16_t)best;
}

std::array<int64_t, 3> cell_of(V3 p, double w) {  // :176-180
  return {(int64_t)std::floor(p.x / w), (int64_t)std::floor(p.y / w),
          (int64_t)std::floor(p.z / w)};
}

namespace {

Aabb cell_bounds(const std::array<int64_t, 3>& c, double w) {  // :182-187
  Aabb b;
  b.min = v3(c[0] * w, c[1] * w, c[2] * w);
  b.max = v3((c[0] + 1) * w, (c[1] + 1) * w, (c[2] + 1) * w);
  return b;
}

int32_t build_bvh(std::vector<BvhNode>& nodes, std::vector<std::pair<Aabb, int32_t>>& items,
                  int lo, int hi) {  // :190-224
  if (hi - lo == 1) {
    BvhNode leaf;
    leaf.bounds = items[lo].first;
    leaf.leaf = items[lo].second;
    nodes.push_back(leaf);
    return (int32_t)nodes.size() - 1;
  }
  Aabb cb;
  for (int i = lo; i < hi; ++i) cb.expand(items[i].first.center());
  V3 ext = cb.extents();
  int axis = 0;
  if (ext.y > ext.x) axis = 1;
  if (ext.z > comp(ext, axis)) axis = 2;
  std::sort(items.begin() + lo, items.begin() + hi,
            [axis](const std::pair<Aabb, int32_t>& a, const std::pair<Aabb, int32_t>& b) {
              double ca = comp(a.first.center(), axis);
              double cbv = comp(b.first.center(), axis);
              return ca != cbv ? ca < cbv : a.second < b.second;
            });
  int mid = lo + (hi - lo) / 2;
  int32_t left = build_bvh(nodes, items, lo, mid);
  int32_t right = build_bvh(nodes, items, mid, hi);
  BvhNode node;
  node.bounds = nodes[left].bounds;
  node.bounds.expand(nodes[right].bounds);
  node.left = left;
  node.right = right;
  nodes.push_back(node);
  return (int32_t)nodes.size() - 1;
}

struct PatchAcc {
  int link = -1;
  std::map<std::array<int64_t, 3>, std::map<uint16_t, IndexRep>> boxes;
};

}  // namespace

FieldIndex build_field_index(const Hand& h, const std::vector<Patch>& patches, int N, double w,
                             uint64_t seed, int C) {  // :306-334 + finalize_index :234-277
  if (patches.empty()) throw std::invalid_argument("index build: no patches");
  if (w <= 0.0 || N < 1) throw std::invalid_argument("index build: bad box width or N");
  FieldIndex idx;
  idx.codebook = make_codebook(C);
  idx.box_width = w;
  std::map<int, PatchAcc> acc;
  for (int c = 0; c < N; ++c) {
    auto q = field_config(h, seed, c);
    auto frames = forward_kinematics(h, q.data());
    for (const Patch& P : patches) {
      const Xf& f = frames[P.link];
      for (int fp : P.field_points) {
        V3 pos = xf_apply(f, P.points[fp]);
        V3 nrm = xf_rotate(f, P.normals[fp]);
        PatchAcc& pa = acc[P.id];  // insert_vector :279-288
        if (pa.link < 0) pa.link = P.link;
        uint16_t code = quantize_normal(idx.codebook, nrm);
        IndexRep rep;
        rep.link = P.link;
        rep.point = P.points[fp];
        rep.normal = P.normals[fp];
        pa.boxes[cell_of(pos, w)].emplace(code, rep);
        ++idx.n_vectors;
      }
    }
  }
  for (auto& kv : acc) {
    PatchIndex pi;
    pi.patch_id = kv.first;
    pi.link = kv.second.link;
    for (auto& bx : kv.second.boxes) {
      IndexBox box;
      box.cell = bx.first;
      for (auto& cr : bx.second) {
        box.codes.push_back(cr.first);
        box.reps.push_back(cr.second);
      }
      pi.boxes.push_back(std::move(box));
    }
    std::vector<std::pair<Aabb, int32_t>> items;
    for (size_t b = 0; b < pi.boxes.size(); ++b)
      items.push_back({cell_bounds(pi.boxes[b].cell, w).inflated(kBoundsEps), (int32_t)b});
    pi.root = build_bvh(pi.nodes, items, 0, (int)items.size());
    idx.patches.push_back(std::move(pi));
  }
  if (!idx.patches.empty()) {
    std::vector<std::pair<Aabb, int32_t>> tops;
    for (size_t p = 0; p < idx.patches.size(); ++p)
      tops.push_back({idx.patches[p].nodes[idx.patches[p].root].bounds, (int32_t)p});
    idx.top_root = build_bvh(idx.top_nodes, tops, 0, (int)tops.size());
  }
  return idx;
}

namespace {
template <typename Visit>
void traverse(const std::vector<BvhNode>& nodes, int32_t root, V3 p, Visit&& visit) {
  if (root < 0) return;
  int32_t stack[64];
  int top = 0;
  stack[top++] = root;
  while (top > 0) {
    const BvhNode& node = nodes[stack[--top]];
    if (!node.bounds.contains(p)) continue;
    if (node.leaf >= 0) {
      visit(node.leaf);
    } else {
      stack[top++] = node.left;
      stack[top++] = node.right;
    }
  }
}
}  // namespace

std::vector<Domain> query_domains(const FieldIndex& idx, const std::vector<Sample>& samples,
                                  const Xf& pose, double theta, const Hand& h,
                                  const Groups& g) {  // :380-448
  std::vector<Domain> domains(g.groups.size());
  for (size_t i = 0; i < domains.size(); ++i) domains[i].group = (int)i;
  if (idx.patches.empty()) return domains;
  std::vector<int> patch_group(idx.patches.size(), -1);
  for (size_t p = 0; p < idx.patches.size(); ++p) {
    int link = idx.patches[p].link;
    if (link < 0 || link >= (int)h.links.size())
      throw std::invalid_argument("query_domains: index link out of range");
    patch_group[p] = g.group_of(link);
  }
  struct Hit {
    int patch, box;
    double score;
  };
  std::vector<Hit> hits;
  for (size_t si = 0; si < samples.size(); ++si) {
    V3 p = xf_apply(pose, samples[si].p);
    V3 n = xf_rotate(pose, samples[si].n);
    auto cell = cell_of(p, idx.box_width);
    hits.clear();
    traverse(idx.top_nodes, idx.top_root, p, [&](int32_t pi) {
      const PatchIndex& patch = idx.patches[pi];
      traverse(patch.nodes, patch.root, p, [&](int32_t bi) {
        const IndexBox& box = patch.boxes[bi];
        if (box.cell != cell) return;
        double best = -2.0;
        for (uint16_t code : box.codes) best = dmax(best, -dot(idx.codebook[code], n));
        if (best >= theta) hits.push_back({(int)pi, (int)bi, best});
      });
    });
    if (hits.empty()) continue;
    std::sort(hits.begin(), hits.end(), [](const Hit& a, const Hit& b) {
      return a.patch != b.patch ? a.patch < b.patch : a.box < b.box;
    });
    for (size_t gi = 0; gi < domains.size(); ++gi) {
      DomainElement el;
      for (const Hit& ht : hits) {
        if (patch_group[ht.patch] != (int)gi) continue;
        el.hit_patches.push_back(idx.patches[ht.patch].patch_id);
        el.hit_boxes.push_back(ht.box);
        el.score = dmax(el.score, ht.score);
      }
      if (el.hit_patches.empty()) continue;
      el.position = p;
      el.normal = n;
      el.sample = (int)si;
      domains[gi].elements.push_back(std::move(el));
    }
  }
  return domains;
}

IndexRep reverse_lookup(const FieldIndex& idx, const DomainElement& el,
                        uint64_t seed) {  // :450-484
  if (el.hit_patches.empty() || el.hit_patches.size() != el.hit_boxes.size())
    throw std::out_of_range("reverse_lookup: element has no hits");
  Rng rng(seed);
  size_t pick = rng.uniform_index(el.hit_patches.size());
  int patch_id = el.hit_patches[pick];
  int box_id = el.hit_boxes[pick];
  const PatchIndex* patch = nullptr;
  for (const auto& p : idx.patches)
    if (p.patch_id == patch_id) {
      patch = &p;
      break;
    }
  if (!patch || box_id < 0 || box_id >= (int)patch->boxes.size())
    throw std::out_of_range("reverse_lookup: stale element");
  const IndexBox& box = patch->boxes[box_id];
  int best = -1;
  double best_dot = -2.0;
  for (size_t i = 0; i < box.codes.size(); ++i) {
    double d = -dot(idx.codebook[box.codes[i]], el.normal);
    if (d > best_dot) {
      best_dot = d;
      best = (int)i;
    }
  }
  return box.reps[best];
}

}  // namespace orc
