// oracle/orc_api.cpp — flat C entry points over the CPU oracle, loaded with
// ctypes by tests/ and bench.py (checker / cpu_baseline only).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "orc.hpp"

using namespace orc;
using namespace lgm;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return LG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return LG_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return LG_ERR_OUT_OF_RANGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LG_ERR_RUNTIME;
  }
}

std::vector<Sample> samples_from(const double* s, int n) {
  std::vector<Sample> out(n);
  for (int i = 0; i < n; ++i) {
    out[i].p = v3_load(s + 6 * i);
    out[i].n = v3_load(s + 6 * i + 3);
  }
  return out;
}

Xf pose_from(const double* p) {
  Xf x;
  x.R = m3_load(p);
  x.t = v3_load(p + 9);
  return x;
}

struct OrcField {
  FieldIndex idx;
  // flattened export
  std::vector<double> codebook, rep_point, rep_normal;
  std::vector<int> patch_link, patch_box_off, rep_link;
  std::vector<long long> box_cell, box_code_off;
  std::vector<uint16_t> codes;
};

struct OrcPatches {
  std::vector<Patch> patches;
  std::vector<int> link, point_off, fp_off, fps;
  std::vector<double> pts, nrm;
};

}  // namespace

struct orc_result {
  RunOutput out;
};

extern "C" {

int orc_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    std::strncpy(buf, g_err.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return (int)g_err.size();
}

uint64_t orc_mix_seed(uint64_t s, uint64_t a, uint64_t b) { return mix_seed(s, a, b); }

void orc_rng_u64(uint64_t seed, int n, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}
void orc_rng_normal(uint64_t seed, int n, double* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.normal();
}
void orc_rng_unit_vectors(uint64_t seed, int n, double* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) v3_store(out + 3 * i, r.uniform_unit_vector());
}
void orc_rng_quaternions(uint64_t seed, int n, double* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) r.uniform_quaternion(out + 4 * i, out + 4 * i + 1, out + 4 * i + 2, out + 4 * i + 3);
}
void orc_libm(int which, int n, const double* x, const double* y, double* out) {
  for (int i = 0; i < n; ++i) {
    switch (which) {
      case 0: out[i] = lgm::xsin(x[i]); break;
      case 1: out[i] = lgm::xcos(x[i]); break;
      case 2: out[i] = lgm::xlog(x[i]); break;
      case 3: out[i] = lgm::xatan2(x[i], y[i]); break;
      default: out[i] = lgm::xhypot(x[i], y[i]); break;
    }
  }
}

// The host glibc itself (std::sin / cos / log / atan2 / hypot, what the
// reference calls) for the same argument arrays, to check lgm:: (and the
// device) against it bit for bit.
void orc_glibc(int which, long long n, const double* x, const double* y, double* out) {
  for (long long i = 0; i < n; ++i) {
    switch (which) {
      case 0: out[i] = std::sin(x[i]); break;
      case 1: out[i] = std::cos(x[i]); break;
      case 2: out[i] = std::log(x[i]); break;
      case 3: out[i] = std::atan2(x[i], y[i]); break;
      default: out[i] = std::hypot(x[i], y[i]); break;
    }
  }
}

// lgl::hypot_exceeds (the friction-disc test of wrench.cpp:96-104 without
// evaluating hypot when a bound settles it): out[i] = hypot(x, y) > cap.
void orc_hypot_exceeds(long long n, const double* x, const double* y, const double* cap,
                       unsigned char* out) {
  for (long long i = 0; i < n; ++i) {
    double r = 0.0;
    out[i] = lgl::hypot_exceeds(x[i], y[i], cap[i], &r) ? 1 : 0;
  }
}

// random_problem of test_wrench.cpp:13-25 (fixture generator): points on a
// 5 cm sphere, roughly inward unit normals.
void orc_random_wrench_problem(uint64_t seed, int n, double* pts, double* nrm) {
  Rng rng(seed);
  for (int i = 0; i < n; ++i) {
    V3 p = scale(0.05, rng.uniform_unit_vector());
    // Vec3(normal(), normal(), normal()): argument evaluation order is
    // unspecified in C++; g++ on x86-64 evaluates right to left.
    double c = rng.normal(), b = rng.normal(), a = rng.normal();
    V3 nin = normalized(add(neg(p), scale(0.3, v3(a, b, c))));
    v3_store(pts + 3 * i, p);
    v3_store(nrm + 3 * i, nin);
  }
}

int orc_tangent_basis(const double* n, double* x, double* y) {
  return guard([&] {
    V3 a, b;
    tangent_basis(v3_load(n), a, b);
    v3_store(x, a);
    v3_store(y, b);
  });
}
int orc_rotation_between(const double* from, const double* to, double* R) {
  return guard([&] { m3_store(R, rotation_between(v3_load(from), v3_load(to))); });
}

int orc_fk(const lg_hand_desc* hd, const double* q, double* frames) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    auto f = forward_kinematics(h, q);
    for (size_t l = 0; l < f.size(); ++l) {
      m3_store(frames + 12 * l, f[l].R);
      v3_store(frames + 12 * l + 9, f[l].t);
    }
  });
}
int orc_point_jacobian(const lg_hand_desc* hd, const double* q, int link, const double* lp,
                       double* J) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    if (link < 0 || link >= (int)h.links.size())
      throw std::invalid_argument("point_jacobian: invalid link");
    auto f = forward_kinematics(h, q);
    point_jacobian(h, f, link, v3_load(lp), J);
  });
}
int orc_groups(const lg_hand_desc* hd, int* group_of_link, int* n_groups) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    Groups g = dependency_groups(h);
    for (size_t l = 0; l < h.links.size(); ++l) group_of_link[l] = g.group_of((int)l);
    *n_groups = (int)g.groups.size();
  });
}

int orc_sample_surface(const double* verts, int nv, const int* tris, int nt, double spc,
                       uint64_t seed, double* out, size_t cap, size_t* n) {
  return guard([&] {
    std::vector<V3> v(nv);
    for (int i = 0; i < nv; ++i) v[i] = v3_load(verts + 3 * i);
    std::vector<std::array<int, 3>> t(nt);
    for (int i = 0; i < nt; ++i) t[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    auto s = sample_surface(v, t, spc, seed);
    *n = s.size();
    if (!out) return;
    for (size_t i = 0; i < s.size() && i < cap; ++i) {
      v3_store(out + 6 * i, s[i].p);
      v3_store(out + 6 * i + 3, s[i].n);
    }
  });
}

// decompose_patches over per-link samples given as one concatenated [n][6]
// array with link offsets [n_links+1].
int orc_decompose_patches(const lg_hand_desc* hd, const double* samples, const int* link_off,
                          double patch_radius, uint64_t seed, int cap, void** out) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    std::vector<std::vector<Sample>> per(h.links.size());
    for (size_t l = 0; l < h.links.size(); ++l)
      per[l] = samples_from(samples + 6 * link_off[l], link_off[l + 1] - link_off[l]);
    auto* P = new OrcPatches;
    P->patches = decompose_patches(h, per, patch_radius, seed, cap);
    P->point_off.push_back(0);
    P->fp_off.push_back(0);
    for (const Patch& p : P->patches) {
      P->link.push_back(p.link);
      for (size_t i = 0; i < p.points.size(); ++i) {
        P->pts.insert(P->pts.end(), {p.points[i].x, p.points[i].y, p.points[i].z});
        P->nrm.insert(P->nrm.end(), {p.normals[i].x, p.normals[i].y, p.normals[i].z});
      }
      P->point_off.push_back((int)(P->pts.size() / 3));
      P->fps.insert(P->fps.end(), p.field_points.begin(), p.field_points.end());
      P->fp_off.push_back((int)P->fps.size());
    }
    *out = P;
  });
}
int orc_patches_export(void* p, lg_patches_desc* d) {
  auto* P = (OrcPatches*)p;
  d->n_patches = (int)P->patches.size();
  d->link = P->link.data();
  d->point_off = P->point_off.data();
  d->points = P->pts.data();
  d->normals = P->nrm.data();
  d->fp_off = P->fp_off.data();
  d->field_points = P->fps.data();
  return LG_OK;
}
void orc_patches_destroy(void* p) { delete (OrcPatches*)p; }

int orc_field_build(const lg_hand_desc* hd, const lg_patches_desc* pd, int N, double w,
                    uint64_t seed, int C, void** out) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    auto patches = patches_from_desc(*pd);
    auto* f = new OrcField;
    f->idx = build_field_index(h, patches, N, w, seed, C);
    for (const V3& c : f->idx.codebook) f->codebook.insert(f->codebook.end(), {c.x, c.y, c.z});
    f->patch_box_off.push_back(0);
    f->box_code_off.push_back(0);
    for (const auto& p : f->idx.patches) {
      f->patch_link.push_back(p.link);
      for (const auto& b : p.boxes) {
        f->box_cell.insert(f->box_cell.end(), {b.cell[0], b.cell[1], b.cell[2]});
        for (size_t i = 0; i < b.codes.size(); ++i) {
          f->codes.push_back(b.codes[i]);
          f->rep_link.push_back(b.reps[i].link);
          f->rep_point.insert(f->rep_point.end(), {b.reps[i].point.x, b.reps[i].point.y, b.reps[i].point.z});
          f->rep_normal.insert(f->rep_normal.end(), {b.reps[i].normal.x, b.reps[i].normal.y, b.reps[i].normal.z});
        }
        f->box_code_off.push_back((long long)f->codes.size());
      }
      f->patch_box_off.push_back((int)(f->box_cell.size() / 3));
    }
    *out = f;
  });
}
int orc_field_export(void* fp, lg_field_csr* o) {
  auto* f = (OrcField*)fp;
  o->box_width = f->idx.box_width;
  o->codebook_size = (int)f->idx.codebook.size();
  o->codebook = f->codebook.data();
  o->n_patches = (int)f->idx.patches.size();
  o->patch_link = f->patch_link.data();
  o->patch_box_off = f->patch_box_off.data();
  o->n_boxes = (long long)(f->box_cell.size() / 3);
  o->box_cell = f->box_cell.data();
  o->box_code_off = f->box_code_off.data();
  o->n_codes = (long long)f->codes.size();
  o->codes = f->codes.data();
  o->rep_link = f->rep_link.data();
  o->rep_point = f->rep_point.data();
  o->rep_normal = f->rep_normal.data();
  o->n_vectors = f->idx.n_vectors;
  return LG_OK;
}
// BVH sizes (for the memory accounting of contact_field.cpp:336-353)
long long orc_field_nodes(void* fp) {
  auto* f = (OrcField*)fp;
  long long n = (long long)f->idx.top_nodes.size();
  for (const auto& p : f->idx.patches) n += (long long)p.nodes.size();
  return n;
}
void orc_field_destroy(void* f) { delete (OrcField*)f; }

// validate_dataset (validate.cpp:56-175) restated per grasp, recording every
// quantity the reference's checks read (the issue texts are formatted from
// these by the library's lg_validation_issues).
int orc_validate(const lg_hand_desc* hd, const lg_grasp* grasps, long long n,
                 const double* verts, int nv, const int* tris, int nt, const double* samples,
                 int ns, const lg_run_params* p, lg_grasp_check* out) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    const int nl = (int)h.links.size();
    (void)nv;
    for (long long gi = 0; gi < n; ++gi) {
      const lg_grasp& g = grasps[gi];
      lg_grasp_check r;
      std::memset(&r, 0, sizeof(r));
      r.n_contacts = g.n_contacts;
      out[gi] = r;
      lg_grasp_check& c = out[gi];
      if (g.dof != h.dof) {
        c.status = 1;
        continue;
      }
      lgm::M3 R;
      for (int a = 0; a < 9; ++a) R.m[a] = g.pose_R[a];
      c.rigid_error = lgm::orthonormal_error(R);
      if (c.rigid_error > 1e-6) {
        c.status = 2;
        continue;
      }
      for (int l = 0; l < nl; ++l) {
        const Link& L = h.links[l];
        if (L.jidx < 0) continue;
        double v = g.q[L.jidx];
        if (v < L.lo - 1e-9 || v > L.hi + 1e-9) {
          c.limit_link[c.n_limit] = l;
          c.limit_value[c.n_limit] = v;
          ++c.n_limit;
        }
      }
      if (c.n_limit) {
        c.status = 3;
        continue;
      }
      if (g.n_contacts <= 0) {
        c.status = 4;
        continue;
      }
      auto frames = forward_kinematics(h, g.q);
      Xf pose;
      for (int a = 0; a < 9; ++a) pose.R.m[a] = g.pose_R[a];
      pose.t = lgm::v3(g.pose_t[0], g.pose_t[1], g.pose_t[2]);
      Xf obj_inv = lgm::xf_inverse(pose);
      for (int ci = 0; ci < g.n_contacts; ++ci) {
        int link = g.contact_link[ci];
        V3 pos = lgm::v3(g.contact_p[ci][0], g.contact_p[ci][1], g.contact_p[ci][2]);
        V3 nrm = lgm::v3(g.contact_n[ci][0], g.contact_n[ci][1], g.contact_n[ci][2]);
        if (link < 0 || link >= nl) {
          c.contact_state[ci] = 1;
          continue;
        }
        if (std::abs(lgm::norm(nrm) - 1.0) > 1e-6) {
          c.contact_state[ci] = 2;
          continue;
        }
        V3 local = lgm::xf_apply(lgm::xf_inverse(frames[link]), pos);
        double dh = kInf;  // distance_to_link_surface (:30-42)
        for (int pi : h.links[link].parts) {
          const Part& P = h.parts[pi];
          for (const auto& t : P.tris) {
            V3 cp = closest_point_on_triangle(local, P.verts[t[0]], P.verts[t[1]], P.verts[t[2]]);
            dh = std::min(dh, lgm::norm(lgm::sub(local, cp)));
          }
        }
        c.hand_dist[ci] = dh;
        V3 op = lgm::xf_apply(obj_inv, pos);
        double dobj = kInf;  // distance_to_mesh (:19-28)
        for (int t = 0; t < nt; ++t) {
          const int* tr = tris + 3 * t;
          V3 cp = closest_point_on_triangle(op, lgm::v3_load(verts + 3 * tr[0]),
                                            lgm::v3_load(verts + 3 * tr[1]),
                                            lgm::v3_load(verts + 3 * tr[2]));
          dobj = std::min(dobj, lgm::norm(lgm::sub(op, cp)));
        }
        c.object_dist[ci] = dobj;
      }
      double worst = 0.0;  // object samples vs every link part (:125-143)
      std::vector<Xf> inv(nl);
      for (int l = 0; l < nl; ++l) inv[l] = lgm::xf_inverse(frames[l]);
      for (int j = 0; j < ns; ++j) {
        V3 world = lgm::xf_apply(pose, lgm::v3_load(samples + 6 * j));
        for (int l = 0; l < nl; ++l) {
          if (h.links[l].parts.empty()) continue;
          V3 local = lgm::xf_apply(inv[l], world);
          for (int pi : h.links[l].parts) {
            const Part& P = h.parts[pi];
            const Aabb& b = P.bounds;
            if (!(local.x >= b.min.x - 1e-9 && local.y >= b.min.y - 1e-9 && local.z >= b.min.z - 1e-9 &&
                  local.x <= b.max.x + 1e-9 && local.y <= b.max.y + 1e-9 && local.z <= b.max.z + 1e-9))
              continue;
            double depth = kInf;  // plane_depth (:44-52)
            bool outside = false;
            for (size_t k = 0; k < P.plane_n.size(); ++k) {
              double slack = P.plane_d[k] - lgm::dot(P.plane_n[k], local);
              if (slack < 0.0) {
                outside = true;
                break;
              }
              depth = std::min(depth, slack);
            }
            double d = (outside || P.plane_n.empty()) ? 0.0 : depth;
            worst = std::max(worst, d);
          }
        }
      }
      c.worst_depth = worst;
      std::vector<V3> pts, nrms;
      for (int ci = 0; ci < g.n_contacts; ++ci) {
        pts.push_back(lgm::v3(g.contact_p[ci][0], g.contact_p[ci][1], g.contact_p[ci][2]));
        nrms.push_back(lgm::v3(g.contact_n[ci][0], g.contact_n[ci][1], g.contact_n[ci][2]));
      }
      try {
        WrenchProblem wp = make_wrench_problem(pts, nrms, p->lambda_torque, p->mu);
        WrenchOpts o;
        o.iterations = p->pgd_iterations;
        o.warm_iterations = p->pgd_warm_iterations;
        o.step = p->pgd_step;
        c.wrench_objective = solve_gswo(wp, o, nullptr).objective;
      } catch (const std::invalid_argument& e) {
        c.wrench_error = std::string(e.what()).find("zero") != std::string::npos ? 1 : 2;
      }
    }
  });
}


// ContactFieldIndex::save (contact_field.cpp:570-600): the GGCF v1 stream,
// field by field, from the oracle's map-built index and its BVHs.
extern "C++" {
namespace {
template <typename T>
void fput(FILE* f, const T& v) { std::fwrite(&v, sizeof(T), 1, f); }
void fput_v3(FILE* f, const V3& v) { fput(f, v.x); fput(f, v.y); fput(f, v.z); }
void fput_nodes(FILE* f, const std::vector<BvhNode>& nodes, int32_t root) {
  fput(f, (uint64_t)nodes.size());
  for (const BvhNode& n : nodes) {
    fput_v3(f, n.bounds.min);
    fput_v3(f, n.bounds.max);
    fput(f, n.left);
    fput(f, n.right);
    fput(f, n.leaf);
  }
  fput(f, root);
}
}  // namespace
}  // extern "C++"
int orc_field_save(void* fp, const char* path, uint64_t key) {
  return guard([&] {
    const FieldIndex& idx = ((OrcField*)fp)->idx;
    FILE* f = std::fopen(path, "wb");
    if (!f) throw std::runtime_error(std::string("cannot write index file: ") + path);
    fput(f, (uint32_t)0x47474346u);
    fput(f, (uint32_t)1u);
    fput(f, key);
    fput(f, idx.box_width);
    fput(f, (uint32_t)idx.codebook.size());
    for (const V3& d : idx.codebook) fput_v3(f, d);
    fput(f, (uint64_t)idx.patches.size());
    for (const PatchIndex& p : idx.patches) {
      fput(f, (int32_t)p.patch_id);
      fput(f, (int32_t)p.link);
      fput(f, (uint64_t)p.boxes.size());
      for (const IndexBox& b : p.boxes) {
        fput(f, b.cell[0]);
        fput(f, b.cell[1]);
        fput(f, b.cell[2]);
        fput(f, (uint32_t)b.codes.size());
        for (size_t i = 0; i < b.codes.size(); ++i) {
          fput(f, b.codes[i]);
          fput(f, (int32_t)b.reps[i].link);
          fput_v3(f, b.reps[i].point);
          fput_v3(f, b.reps[i].normal);
        }
      }
      fput_nodes(f, p.nodes, p.root);
    }
    fput_nodes(f, idx.top_nodes, idx.top_root);
    bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad) throw std::runtime_error(std::string("short write on index file: ") + path);
  });
}


// query_domains for one pose: masks[n] bitmask of groups whose domain holds
// an element for sample i, scores[n] element score (0 when no element).
int orc_query(void* fp, const lg_hand_desc* hd, const double* samples, int n,
              const double* pose, double theta, uint32_t* masks, double* scores,
              int* domain_sizes) {
  return guard([&] {
    auto* f = (OrcField*)fp;
    Hand h = Hand::from_desc(*hd);
    Groups g = dependency_groups(h);
    auto s = samples_from(samples, n);
    auto d = query_domains(f->idx, s, pose_from(pose), theta, h, g);
    for (int i = 0; i < n; ++i) {
      masks[i] = 0;
      if (scores) scores[i] = 0.0;
    }
    for (size_t gi = 0; gi < d.size(); ++gi) {
      if (domain_sizes) domain_sizes[gi] = (int)d[gi].elements.size();
      for (const auto& el : d[gi].elements) {
        masks[el.sample] |= 1u << gi;
        if (scores) scores[el.sample] = dmax(scores[el.sample], el.score);
      }
    }
  });
}

// reverse_lookup of the element (sample, group) under a pose.
int orc_reverse_lookup(void* fp, const lg_hand_desc* hd, const double* samples, int n,
                       const double* pose, double theta, int sample, int group, uint64_t seed,
                       int* link, double* point, double* normal) {
  return guard([&] {
    auto* f = (OrcField*)fp;
    Hand h = Hand::from_desc(*hd);
    Groups g = dependency_groups(h);
    auto s = samples_from(samples, n);
    auto d = query_domains(f->idx, s, pose_from(pose), theta, h, g);
    for (const auto& el : d.at(group).elements) {
      if (el.sample != sample) continue;
      IndexRep r = reverse_lookup(f->idx, el, seed);
      *link = r.link;
      v3_store(point, r.point);
      v3_store(normal, r.normal);
      return;
    }
    throw std::out_of_range("reverse_lookup: element has no hits");
  });
}

int orc_preprocess(const double* samples, int n, double hw, double dt, uint8_t* keep) {
  return guard([&] {
    auto s = samples_from(samples, n);
    if (hw <= 0.0 || dt < 0.0)
      throw std::invalid_argument("preprocess_object: bad probe dimensions");
    auto kept = preprocess_object(s, hw, dt);
    // map back by identity order (preprocess is order preserving)
    size_t j = 0;
    for (int i = 0; i < n; ++i) {
      bool k = j < kept.size() && std::memcmp(&kept[j], &s[i], sizeof(Sample)) == 0;
      keep[i] = k ? 1 : 0;
      if (k) ++j;
    }
  });
}

int orc_wrench_solve(int n, const double* pts, const double* nrm, double lambda, double mu,
                     int mode, int iters, int warm_iters, double step, int max_bt,
                     const double* warm_alpha, const double* warm_bx, const double* warm_by,
                     double* objective, int* anchor, double* alpha, double* bx, double* by) {
  return guard([&] {
    std::vector<V3> p(n), nn(n);
    for (int i = 0; i < n; ++i) {
      p[i] = v3_load(pts + 3 * i);
      nn[i] = v3_load(nrm + 3 * i);
    }
    WrenchProblem wp = make_wrench_problem(p, nn, lambda, mu);
    WrenchOpts o;
    o.iterations = iters;
    o.warm_iterations = warm_iters;
    o.step = step;
    o.max_backtracks = max_bt;
    WrenchSolution warm;
    const WrenchSolution* wptr = nullptr;
    if (warm_alpha) {
      warm.anchor = 0;
      warm.alpha.assign(warm_alpha, warm_alpha + n);
      warm.bx.assign(warm_bx, warm_bx + n);
      warm.by.assign(warm_by, warm_by + n);
      wptr = &warm;
    }
    WrenchSolution s = mode ? solve_gswo(wp, o, wptr) : solve_fswo(wp, o, wptr);
    *objective = s.objective;
    *anchor = s.anchor;
    for (int i = 0; i < n && s.valid(); ++i) {
      alpha[i] = s.alpha[i];
      bx[i] = s.bx[i];
      by[i] = s.by[i];
    }
  });
}

int orc_wrench_objective(int n, const double* pts, const double* nrm, double lambda, double mu,
                         const double* alpha, const double* bx, const double* by, double* out) {
  return guard([&] {
    std::vector<V3> p(n), nn(n);
    for (int i = 0; i < n; ++i) {
      p[i] = v3_load(pts + 3 * i);
      nn[i] = v3_load(nrm + 3 * i);
    }
    WrenchProblem wp = make_wrench_problem(p, nn, lambda, mu);
    WrenchSolution s;
    s.anchor = 0;
    s.alpha.assign(alpha, alpha + n);
    s.bx.assign(bx, bx + n);
    s.by.assign(by, by + n);
    *out = wrench_objective(wp, s);
  });
}

// optimize_contacts over k synthetic domains: domain i has counts[i]
// elements with positions/normals [*][3] concatenated.
int orc_optimize_contacts(int k, const int* counts, const double* pos, const double* nrm,
                          int n_static, const double* spos, const double* snrm, int n_outer,
                          int n_inner, int restarts, double sigma, double lambda, double mu,
                          uint64_t seed, int* ids, double* objective, int* evaluations) {
  return guard([&] {
    std::vector<Domain> doms(k);
    size_t off = 0;
    for (int i = 0; i < k; ++i) {
      for (int e = 0; e < counts[i]; ++e, ++off) {
        DomainElement el;
        el.position = v3_load(pos + 3 * off);
        el.normal = v3_load(nrm + 3 * off);
        el.sample = e;
        doms[i].elements.push_back(el);
      }
    }
    std::vector<const Domain*> dp;
    for (auto& d : doms) dp.push_back(&d);
    std::vector<StaticContact> st(n_static);
    for (int i = 0; i < n_static; ++i) {
      st[i].position = v3_load(spos + 3 * i);
      st[i].normal = v3_load(snrm + 3 * i);
    }
    ContactOptParams p;
    p.n_outer = n_outer;
    p.n_inner = n_inner;
    p.restarts = restarts;
    p.sigma = sigma;
    p.lambda = lambda;
    p.mu = mu;
    auto r = optimize_contacts(dp, p, st, seed);
    for (int i = 0; i < k; ++i) ids[i] = r.element_ids[i];
    *objective = r.objective;
    *evaluations = r.evaluations;
  });
}

int orc_collision(const lg_hand_desc* hd, const double* q, const double* pose,
                  const double* samples, int n, double margin, int* clean, double* max_pen,
                  int* n_viol) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    auto s = samples_from(samples, n);
    auto r = validate_grasp_collisions(h, q, s, pose_from(pose), margin);
    *clean = r.clean();
    *max_pen = r.max_penetration;
    *n_viol = r.n_violations;
  });
}

// GJK between two parts of a hand description (part ids) at given poses.
int orc_gjk(const lg_hand_desc* hd, int pa, const double* pose_a, int pb, const double* pose_b,
            double* dist) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    *dist = gjk_distance(h.parts.at(pa), pose_from(pose_a), h.parts.at(pb), pose_from(pose_b));
  });
}

int orc_closest_on_parts(const lg_hand_desc* hd, int link, const double* p, double* sp,
                         double* sn, double* d) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    V3 a = v3(0, 0, 0), b = v3(0, 0, 0);
    *d = closest_on_parts(h, link, v3_load(p), &a, &b);
    v3_store(sp, a);
    v3_store(sn, b);
  });
}

static std::vector<ContactTarget> targets_from(int k, const double* op, const double* on,
                                               const int* links, const double* hp,
                                               const double* hn) {
  std::vector<ContactTarget> t(k);
  for (int i = 0; i < k; ++i) {
    t[i].object_point = v3_load(op + 3 * i);
    t[i].object_normal = v3_load(on + 3 * i);
    t[i].link = links[i];
    t[i].hand_point = v3_load(hp + 3 * i);
    t[i].hand_normal = v3_load(hn + 3 * i);
  }
  return t;
}

int orc_ik(const lg_hand_desc* hd, const double* q0, int k, const double* op, const double* on,
           const int* links, const double* hp, const double* hn, double beta, int iterations,
           double step_clamp, double residual_tol, double damping_scale, double* q,
           int* iters_out, double* objective, int* finite, unsigned long long* used,
           double* res_pos, double* res_angle) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    IkParams p;
    p.beta = beta;
    p.iterations = iterations;
    p.step_clamp = step_clamp;
    p.residual_tol = residual_tol;
    p.damping_scale = damping_scale;
    std::vector<double> q0v(q0, q0 + h.dof);
    auto r = solve_contact_ik(h, q0v, targets_from(k, op, on, links, hp, hn), p);
    for (int j = 0; j < h.dof; ++j) q[j] = r.q[j];
    *iters_out = r.iterations;
    *objective = r.objective;
    *finite = r.finite;
    unsigned long long m = 0;
    for (int j = 0; j < h.dof && j < 64; ++j)
      if (r.used[j]) m |= 1ull << j;
    *used = m;
    for (int i = 0; i < k; ++i) {
      if (res_pos) res_pos[i] = r.res_pos[i];
      if (res_angle) res_angle[i] = r.res_angle[i];
    }
  });
}

int orc_realize(const lg_hand_desc* hd, const double* q0, int k, const double* op,
                const double* on, const int* links, const double* hp, const double* hn,
                double beta, int iterations, double step_clamp, double residual_tol,
                double damping_scale, int rounds, int fine_iters, double* q, double* max_res,
                int* finite, unsigned long long* used) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    IkParams p;
    p.beta = beta;
    p.iterations = iterations;
    p.step_clamp = step_clamp;
    p.residual_tol = residual_tol;
    p.damping_scale = damping_scale;
    std::vector<double> q0v(q0, q0 + h.dof);
    auto r = realize_grasp(h, q0v, targets_from(k, op, on, links, hp, hn), p, rounds, fine_iters);
    for (int j = 0; j < h.dof; ++j) q[j] = r.q[j];
    *max_res = r.max_residual;
    *finite = r.finite;
    unsigned long long m = 0;
    for (int j = 0; j < h.dof && j < 64; ++j)
      if (r.used[j]) m |= 1ull << j;
    *used = m;
  });
}

int orc_run_batch(const lg_hand_desc* hd, const lg_patches_desc* pd, const double* raw,
                  int n_raw, const lg_run_params* cfg, int workers, orc_result** out) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    auto patches = patches_from_desc(*pd);
    auto s = samples_from(raw, n_raw);
    auto* r = new orc_result;
    try {
      r->out = run_batch(h, patches, s, *cfg, workers);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}
// run_batch over a prebuilt index (the reference's cache=true mode).
int orc_run_batch_field(void* fp, const lg_hand_desc* hd, const lg_patches_desc* pd,
                        const double* raw, int n_raw, const lg_run_params* cfg, int workers,
                        orc_result** out) {
  return guard([&] {
    Hand h = Hand::from_desc(*hd);
    auto patches = patches_from_desc(*pd);
    auto s = samples_from(raw, n_raw);
    auto* r = new orc_result;
    try {
      r->out = run_batch(h, patches, s, *cfg, workers, &((OrcField*)fp)->idx);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

int orc_result_profile(const orc_result* r, lg_profile* p) {
  *p = r->out.profile;
  return LG_OK;
}
long long orc_result_num_grasps(const orc_result* r) { return (long long)r->out.grasps.size(); }
const lg_grasp* orc_result_grasps(const orc_result* r) { return r->out.grasps.data(); }
long long orc_result_num_traces(const orc_result* r) { return (long long)r->out.traces.size(); }
const lg_trace* orc_result_traces(const orc_result* r) { return r->out.traces.data(); }
void orc_result_destroy(orc_result* r) { delete r; }

}  // extern "C"
