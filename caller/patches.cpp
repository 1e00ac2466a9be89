// patches.cpp — build_field's caller-side hand steps (pipeline.cpp:277-285):
// per-link surface samples with stream 'hnds' (mesh.cpp:297-339) and the
// random greedy patch cover decompose_patches (contact_field.cpp:26-99), from
// the flat hand description and its visual meshes.  The same steps run on the
// GPU behind lg_hand_patches_device; tests/test_caller.py checks this host
// version against the reference's output.
#include <algorithm>
#include <random>

#include "caller.hpp"

namespace lgh {

lg_patches_desc Patches::desc() const {
  lg_patches_desc d;
  d.n_patches = (int)link.size();
  d.link = link.data();
  d.point_off = point_off.data();
  d.points = pts.data();
  d.normals = nrm.data();
  d.fp_off = fp_off.data();
  d.field_points = fps.data();
  return d;
}

Patches make_patches(const lg_hand_desc& h, const lg_visual_desc& vis, double spc, double radius,
                     uint64_t seed, int cap) {
  const uint64_t kTagHandSamples = 0x686e6473;  // pipeline.cpp:20
  const uint64_t kTagPatch = 0x70617463;        // contact_field.cpp:16
  const uint64_t kTagSubset = 0x73756273;       // contact_field.cpp:17
  if (vis.n_links != h.n_links) fail_invalid("decompose_patches: per-link sample mismatch");
  std::vector<std::vector<Sample>> per((size_t)h.n_links);
  size_t total = 0;
  for (int l = 0; l < h.n_links; ++l) {
    Mesh m;
    for (int v = vis.vert_off[l]; v < vis.vert_off[l + 1]; ++v)
      m.verts.push_back(lgm::v3_load(vis.verts + 3 * v));
    for (int t = vis.tri_off[l]; t < vis.tri_off[l + 1]; ++t)
      m.tris.push_back({vis.tris[3 * t], vis.tris[3 * t + 1], vis.tris[3 * t + 2]});
    if (m.verts.empty()) continue;
    per[l] = sample_surface(m, spc, lgm::mix_seed(seed, kTagHandSamples, (uint64_t)l));
    total += per[l].size();
  }
  if (radius <= 0.0 || cap < 1) fail_invalid("decompose_patches: bad radius or cap");
  if (total == 0) fail_invalid("decompose_patches: no surface samples");
  const double gather = 0.5 * radius;
  Patches P;
  P.point_off.push_back(0);
  P.fp_off.push_back(0);
  int next_id = 0;
  for (size_t link = 0; link < per.size(); ++link) {
    const auto& S = per[link];
    if (S.empty()) continue;
    std::mt19937_64 rng(lgm::mix_seed(seed, kTagPatch, link));
    std::vector<int> uncovered(S.size());
    for (size_t i = 0; i < S.size(); ++i) uncovered[i] = (int)i;
    while (!uncovered.empty()) {
      size_t pick = rng() % uncovered.size();
      int sid = uncovered[pick];
      V3 center = S[sid].p;
      std::vector<V3> pts = {center}, nrm = {S[sid].n};
      std::vector<int> rest;
      for (int id : uncovered) {
        if (id == sid) continue;
        if (lgm::norm(lgm::sub(S[id].p, center)) <= gather) {
          pts.push_back(S[id].p);
          nrm.push_back(S[id].n);
        } else {
          rest.push_back(id);
        }
      }
      uncovered.swap(rest);
      int id = next_id++;
      int m = (int)pts.size();
      std::vector<int> fp;
      if (m <= cap) {
        for (int i = 0; i < m; ++i) fp.push_back(i);
      } else {
        std::mt19937_64 sr(lgm::mix_seed(seed, kTagSubset, (uint64_t)id));
        std::vector<int> pool(m - 1);
        for (int i = 1; i < m; ++i) pool[i - 1] = i;
        fp.push_back(0);
        for (int i = 0; i < cap - 1; ++i) {
          size_t j = i + sr() % (pool.size() - i);
          std::swap(pool[i], pool[j]);
          fp.push_back(pool[i]);
        }
        std::sort(fp.begin(), fp.end());
      }
      P.link.push_back((int)link);
      for (int i = 0; i < m; ++i) {
        P.pts.insert(P.pts.end(), {pts[i].x, pts[i].y, pts[i].z});
        P.nrm.insert(P.nrm.end(), {nrm[i].x, nrm[i].y, nrm[i].z});
      }
      P.point_off.push_back((int)(P.pts.size() / 3));
      P.fps.insert(P.fps.end(), fp.begin(), fp.end());
      P.fp_off.push_back((int)P.fps.size());
    }
  }
  return P;
}

}  // namespace lgh
