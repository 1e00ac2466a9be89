// capi_caller.cpp — C-ABI of the caller-side helpers (caller/lg_caller.h):
// config parsing, meshes and surface sampling, the hand's host patches and
// the JSONL writer.  Not part of the product library.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "caller.hpp"
#include "lg_caller.h"

struct lgc_mesh {
  lgh::Mesh m;
  std::vector<double> fv;
  std::vector<int> ft;
};
struct lgc_patches {
  lgh::Patches p;
};

namespace {
thread_local std::string g_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return LG_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return LG_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return LG_ERR_OUT_OF_RANGE;
  } catch (const std::bad_alloc&) {
    g_error = "out of memory";
    return LG_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return LG_ERR_RUNTIME;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}
}  // namespace

extern "C" {

int lgc_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    std::strncpy(buf, g_error.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return (int)g_error.size();
}

void lgc_run_params_default(lg_run_params* p) { lgh::params_default(p); }

int lgc_config_parse(const char* path, const char* hand, const char* object, const char* out,
                     const long long* seed, const int* batch, const int* workers,
                     lg_run_params* p) {
  return guard([&] {
    require(p != nullptr, "lgc_config_parse: null params");
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

int lgc_index_cache_key(const lg_run_params* p, uint64_t* key) {
  return guard([&] { *key = lgh::cache_key(p); });
}

// ------------------------------------------------------------------ mesh
int lgc_mesh_load(const char* path, lgc_load_report* report, lgc_mesh** out) {
  return guard([&] {
    require(path && out, "lgc_mesh_load: null argument");
    lgh::LoadReport r;
    auto* m = new lgc_mesh;
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

int lgc_mesh_box(double sx, double sy, double sz, lgc_mesh** out) {
  return guard([&] {
    auto* m = new lgc_mesh;
    m->m = lgh::make_box(lgm::v3(sx, sy, sz), lgm::v3(0, 0, 0));
    *out = m;
  });
}
int lgc_mesh_icosphere(double r, int sub, lgc_mesh** out) {
  return guard([&] {
    require(sub >= 0 && sub <= 8, "lgc_mesh_icosphere: subdivisions out of range");
    auto* m = new lgc_mesh;
    m->m = lgh::make_icosphere(r, sub, lgm::v3(0, 0, 0));
    *out = m;
  });
}
int lgc_mesh_cylinder(double r, double len, int segments, lgc_mesh** out) {
  return guard([&] {
    require(segments >= 3, "lgc_mesh_cylinder: need >= 3 segments");
    auto* m = new lgc_mesh;
    m->m = lgh::make_cylinder(r, len, segments);
    *out = m;
  });
}
int lgc_mesh_from_arrays(const double* verts, int nv, const int* tris, int nt, lgc_mesh** out) {
  return guard([&] {
    auto* m = new lgc_mesh;
    for (int i = 0; i < nv; ++i) m->m.verts.push_back(lgm::v3_load(verts + 3 * i));
    for (int i = 0; i < nt; ++i) {
      for (int k = 0; k < 3; ++k)
        if (tris[3 * i + k] < 0 || tris[3 * i + k] >= nv) {
          delete m;
          throw std::invalid_argument("lgc_mesh_from_arrays: index out of range");
        }
      m->m.tris.push_back({tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]});
    }
    *out = m;
  });
}
int lgc_mesh_scale(lgc_mesh* m, double s) {
  return guard([&] {
    for (auto& v : m->m.verts) v = lgm::scale(s, v);
  });
}
int lgc_mesh_info(const lgc_mesh* m, int* nv, int* nt, double* area) {
  return guard([&] {
    if (nv) *nv = (int)m->m.verts.size();
    if (nt) *nt = (int)m->m.tris.size();
    if (area) *area = m->m.surface_area();
  });
}
int lgc_mesh_arrays(const lgc_mesh* mc, const double** verts, const int** tris) {
  return guard([&] {
    auto* m = const_cast<lgc_mesh*>(mc);
    m->fv.clear();
    m->ft.clear();
    for (const auto& v : m->m.verts) m->fv.insert(m->fv.end(), {v.x, v.y, v.z});
    for (const auto& t : m->m.tris) m->ft.insert(m->ft.end(), {t[0], t[1], t[2]});
    *verts = m->fv.data();
    *tris = m->ft.data();
  });
}
int lgc_mesh_save_obj(const lgc_mesh* m, const char* path) {
  return guard([&] { lgh::save_obj(m->m, path); });
}
void lgc_mesh_destroy(lgc_mesh* m) { delete m; }

int lgc_sample_surface(const lgc_mesh* m, double spc, uint64_t seed, double* out, size_t cap,
                      size_t* n) {
  return guard([&] {
    require(m && n, "lgc_sample_surface: null argument");
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
int lgc_hand_patches(const lg_hand_desc* h, const lg_visual_desc* vis, double spc, double radius,
                     uint64_t seed, int cap, lgc_patches** out) {
  return guard([&] {
    require(h && vis && out, "lgc_hand_patches: null argument");
    auto* p = new lgc_patches;
    try {
      p->p = lgh::make_patches(*h, *vis, spc, radius, seed, cap);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}
int lgc_patches_export(const lgc_patches* p, lg_patches_desc* out) {
  return guard([&] { *out = p->p.desc(); });
}
void lgc_patches_destroy(lgc_patches* p) { delete p; }

// ---------------------------------------------------------------- results
int lgc_write_dataset(const char* path, const lg_grasp* g, long long n) {
  return guard([&] { lgh::write_dataset(path, g, n); });
}
int lgc_write_profile(const char* path, const lg_profile* p) {
  return guard([&] { lgh::write_profile(path, *p); });
}

}  // extern "C"
