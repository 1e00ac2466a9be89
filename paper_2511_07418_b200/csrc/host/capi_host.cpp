// capi_host.cpp — C-ABI for the caller-side (host) steps: loaders, sampling,
// patches, config and result writers.
#include <cstring>
#include <string>

#include "../capi_common.hpp"
#include <cstdio>
#include <algorithm>
#include "capi_types.hpp"

namespace lgc {
thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }
}  // namespace lgc

using lgc::guard;

namespace {
void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}
}  // namespace

extern "C" {

int lg_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    std::strncpy(buf, lgc::g_error.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return (int)lgc::g_error.size();
}

void lg_run_params_default(lg_run_params* p) { lgh::params_default(p); }

int lg_config_parse(const char* path, const char* hand, const char* object, const char* out,
                    const long long* seed, const int* batch, const int* workers,
                    lg_run_params* p) {
  return guard([&] {
    require(p != nullptr, "lg_config_parse: null params");
    lgh::params_default(p);
    lgh::parse_config(path, p);
    if (hand) std::strncpy(p->hand, hand, 511);
    if (object) std::strncpy(p->object, object, 511);
    if (out) std::strncpy(p->out, out, 511);
    if (seed) p->seed = (uint64_t)*seed;
    if (batch) {
      if (*batch < 1) throw std::runtime_error("config: batch must be >= 1");
      p->batch = *batch;
    }
    if (workers) {
      if (*workers < 0) throw std::runtime_error("config: workers must be >= 0");
      p->workers = *workers;
    }
    auto exists = [](const char* f) {
      FILE* fp = std::fopen(f, "rb");
      if (fp) std::fclose(fp);
      return fp != nullptr;
    };
    if (p->hand[0] && !exists(p->hand))
      throw std::runtime_error(std::string("config: hand file not found: ") + p->hand);
    if (p->object[0] && !exists(p->object))
      throw std::runtime_error(std::string("config: object file not found: ") + p->object);
  });
}

int lg_index_cache_key(const lg_run_params* p, uint64_t* key) {
  return guard([&] { *key = lgh::cache_key(p); });
}

uint64_t lg_mix_seed(uint64_t seed, uint64_t a, uint64_t b) { return lgm::mix_seed(seed, a, b); }

// ------------------------------------------------------------------ hand
int lg_hand_load(const char* path, double scale, lg_hand** out) {
  return guard([&] {
    require(path && out, "lg_hand_load: null argument");
    auto* h = new lg_hand;
    try {
      h->h = lgh::load_hand(path, scale);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int lg_hand_export(const lg_hand* h, lg_hand_desc* out) {
  return guard([&] {
    require(h && out, "lg_hand_export: null argument");
    *out = h->h.desc();
  });
}

int lg_hand_link_name(const lg_hand* h, int link, char* buf, size_t cap) {
  return guard([&] {
    require(h && link >= 0 && link < (int)h->h.links.size(), "lg_hand_link_name: bad link");
    std::strncpy(buf, h->h.links[link].name.c_str(), cap - 1);
    buf[cap - 1] = 0;
  });
}

int lg_hand_groups(const lg_hand* h, int* group_of_link, int* n_groups) {
  return guard([&] {
    require(h != nullptr, "lg_hand_groups: null hand");
    auto g = lgh::dependency_group_of(h->h, n_groups);
    for (size_t i = 0; i < g.size(); ++i) group_of_link[i] = g[i];
  });
}

int lg_hand_link_visual(const lg_hand* h, int link, lg_mesh** out) {
  return guard([&] {
    require(h && link >= 0 && link < (int)h->h.links.size(), "lg_hand_link_visual: bad link");
    auto* m = new lg_mesh;
    m->m = h->h.links[link].visual;
    *out = m;
  });
}

void lg_hand_destroy(lg_hand* h) { delete h; }

// ------------------------------------------------------------------ mesh
int lg_mesh_load(const char* path, lg_load_report* report, lg_mesh** out) {
  return guard([&] {
    require(path && out, "lg_mesh_load: null argument");
    lgh::LoadReport r;
    auto* m = new lg_mesh;
    try {
      m->m = lgh::load_mesh(path, &r);
    } catch (...) {
      delete m;
      throw;
    }
    if (report) {
      report->triangles_read = r.read;
      report->triangles_kept = r.kept;
      report->degenerate_dropped = r.dropped;
    }
    *out = m;
  });
}

int lg_mesh_box(double sx, double sy, double sz, lg_mesh** out) {
  return guard([&] {
    auto* m = new lg_mesh;
    m->m = lgh::make_box(lgm::v3(sx, sy, sz), lgm::v3(0, 0, 0));
    *out = m;
  });
}
int lg_mesh_icosphere(double r, int sub, lg_mesh** out) {
  return guard([&] {
    require(sub >= 0 && sub <= 8, "lg_mesh_icosphere: subdivisions out of range");
    auto* m = new lg_mesh;
    m->m = lgh::make_icosphere(r, sub, lgm::v3(0, 0, 0));
    *out = m;
  });
}
int lg_mesh_cylinder(double r, double len, int segments, lg_mesh** out) {
  return guard([&] {
    require(segments >= 3, "lg_mesh_cylinder: need >= 3 segments");
    auto* m = new lg_mesh;
    m->m = lgh::make_cylinder(r, len, segments);
    *out = m;
  });
}
int lg_mesh_from_arrays(const double* verts, int nv, const int* tris, int nt, lg_mesh** out) {
  return guard([&] {
    auto* m = new lg_mesh;
    for (int i = 0; i < nv; ++i) m->m.verts.push_back(lgm::v3_load(verts + 3 * i));
    for (int i = 0; i < nt; ++i) {
      for (int k = 0; k < 3; ++k)
        if (tris[3 * i + k] < 0 || tris[3 * i + k] >= nv) {
          delete m;
          throw std::invalid_argument("lg_mesh_from_arrays: index out of range");
        }
      m->m.tris.push_back({tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]});
    }
    *out = m;
  });
}
int lg_mesh_scale(lg_mesh* m, double s) {
  return guard([&] {
    for (auto& v : m->m.verts) v = lgm::scale(s, v);
  });
}
int lg_mesh_info(const lg_mesh* m, int* nv, int* nt, double* area) {
  return guard([&] {
    if (nv) *nv = (int)m->m.verts.size();
    if (nt) *nt = (int)m->m.tris.size();
    if (area) *area = m->m.surface_area();
  });
}
int lg_mesh_arrays(const lg_mesh* mc, const double** verts, const int** tris) {
  return guard([&] {
    auto* m = const_cast<lg_mesh*>(mc);
    m->fv.clear();
    m->ft.clear();
    for (const auto& v : m->m.verts) m->fv.insert(m->fv.end(), {v.x, v.y, v.z});
    for (const auto& t : m->m.tris) m->ft.insert(m->ft.end(), {t[0], t[1], t[2]});
    *verts = m->fv.data();
    *tris = m->ft.data();
  });
}
int lg_mesh_save_obj(const lg_mesh* m, const char* path) {
  return guard([&] { lgh::save_obj(m->m, path); });
}
void lg_mesh_destroy(lg_mesh* m) { delete m; }

int lg_sample_surface(const lg_mesh* m, double spc, uint64_t seed, double* out, size_t cap,
                      size_t* n) {
  return guard([&] {
    require(m && n, "lg_sample_surface: null argument");
    auto s = lgh::sample_surface(m->m, spc, seed);
    *n = s.size();
    if (!out) return;
    for (size_t i = 0; i < s.size() && i < cap; ++i) {
      lgm::v3_store(out + 6 * i, s[i].p);
      lgm::v3_store(out + 6 * i + 3, s[i].n);
    }
  });
}

// ---------------------------------------------------------------- patches
int lg_hand_patches(const lg_hand* h, double spc, double radius, uint64_t seed, int cap,
                    lg_patches** out) {
  return guard([&] {
    require(h && out, "lg_hand_patches: null argument");
    auto* p = new lg_patches;
    try {
      p->p = lgh::make_patches(h->h, spc, radius, seed, cap);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}
int lg_patches_export(const lg_patches* p, lg_patches_desc* out) {
  return guard([&] { *out = p->p.desc(); });
}
void lg_patches_destroy(lg_patches* p) { delete p; }

// ---------------------------------------------------------------- results
int lg_write_dataset(const char* path, const lg_grasp* g, long long n) {
  return guard([&] { lgh::write_dataset(path, g, n); });
}
int lg_write_profile(const char* path, const lg_profile* p) {
  return guard([&] { lgh::write_profile(path, *p); });
}

// ValidationReport issue texts (validate.cpp:56-175); numbers as an ostream
// with default formatting prints them (%g, 6 significant digits).
int lg_validation_issues(const lg_hand* hand, const lg_grasp_check* checks, long long n,
                         const lg_run_params* p, char* buf, size_t cap, size_t* needed,
                         long long* n_issues) {
  return guard([&] {
    if (!hand || (!checks && n) || !p) throw std::invalid_argument("lg_validation_issues: null argument");
    std::string out;
    long long count = 0;
    auto num = [](double v) {
      char t[64];
      std::snprintf(t, sizeof(t), "%g", v);
      return std::string(t);
    };
    auto add = [&](long long gi, const std::string& what) {
      out += std::to_string(gi) + "\t" + what + "\n";
      ++count;
    };
    const auto& links = hand->h.links;
    for (long long gi = 0; gi < n; ++gi) {
      const lg_grasp_check& c = checks[gi];
      if (c.status == 1) {
        add(gi, "joint vector size mismatch");
        continue;
      }
      if (c.status == 2) {
        add(gi, "pose not rigid: transform rotation is not orthonormal");
        continue;
      }
      if (c.status == 3) {
        for (int k = 0; k < c.n_limit; ++k) {
          int l = c.limit_link[k];
          std::string name = (l >= 0 && l < (int)links.size()) ? links[l].joint_name : std::string("?");
          add(gi, "joint " + name + " out of limits: " + num(c.limit_value[k]));
        }
        continue;
      }
      if (c.status == 4) {
        add(gi, "no contacts");
        continue;
      }
      for (int ci = 0; ci < c.n_contacts; ++ci) {
        if (c.contact_state[ci] == 1) {
          add(gi, "contact with invalid link id");
          continue;
        }
        if (c.contact_state[ci] == 2) {
          add(gi, "contact normal not unit length");
          continue;
        }
        if (c.hand_dist[ci] > p->contact_tol)
          add(gi, "contact " + std::to_string(ci) + " is " + num(c.hand_dist[ci]) +
                      " m off the hand surface (limit " + num(p->contact_tol) + ")");
        if (c.object_dist[ci] > p->contact_tol)
          add(gi, "contact " + std::to_string(ci) + " is " + num(c.object_dist[ci]) +
                      " m off the object surface (limit " + num(p->contact_tol) + ")");
      }
      if (c.worst_depth > p->penetration_margin)
        add(gi, "object penetrates the hand by " + num(c.worst_depth) + " m (limit " +
                    num(p->penetration_margin) + ")");
      if (c.wrench_error == 1) {
        add(gi, "wrench recheck failed: tangent_basis: zero normal");
      } else if (c.wrench_error == 2) {
        add(gi, "wrench recheck failed: tangent_basis: normal is not unit length");
      } else if (!(c.wrench_objective < p->eps_stable)) {
        add(gi, "wrench objective " + num(c.wrench_objective) + " not under stability threshold " +
                    num(p->eps_stable));
      }
    }
    if (needed) *needed = out.size() + 1;
    if (n_issues) *n_issues = count;
    if (buf && cap) {
      size_t m = std::min(cap - 1, out.size());
      std::memcpy(buf, out.data(), m);
      buf[m] = '\0';
    }
  });
}

}  // extern "C"
