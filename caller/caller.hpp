// caller.hpp — the CALLER side of the drop-in boundary (not the product).
//
// The reference keeps these steps on the host and the north star leaves them
// there (SURVEY.md §8(b) "What stays"): OBJ/STL meshes and primitives
// (mesh.cpp), area-weighted surface sampling (mesh.cpp:297-339), the hand's
// surface samples + decompose_patches (pipeline.cpp:277-285,
// contact_field.cpp:26-99), run configuration (config.cpp) and the JSONL
// result format (dataset.cpp).  A production caller (the reference's own
// graspgen CLI) uses the reference's code for them; this
// library is the stand-in caller the bench and the tests drive, and it never
// runs on the GPU.  The hand model itself comes from the reference's own
// load_hand via the fixtures in assets/prepared/ (tools/prepare_hands.py);
// there is no URDF parser or convex-hull code here.
//
// Everything it produces is a flat lg_*_desc view (include/lg.h) — the only
// thing libgraspgen_b200.so accepts.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "lg.h"
#include "lg_math.h"

namespace lgh {

using lgm::M3;
using lgm::V3;
using lgm::Xf;

struct Mesh {  // TriMesh, mesh.hpp:13-21
  std::vector<V3> verts;
  std::vector<std::array<int, 3>> tris;
  double face_area(int t) const;
  V3 face_normal(int t) const;
  double surface_area() const;
};

struct Sample {
  V3 p, n;
};

struct Patches {
  std::vector<int> link, point_off, fp_off, fps;
  std::vector<double> pts, nrm;
  lg_patches_desc desc() const;
};

struct LoadReport {
  long long read = 0, kept = 0, dropped = 0;
};

// mesh.cpp
Mesh load_mesh(const std::string& path, LoadReport* rep = nullptr, double area_eps = 1e-12);
Mesh make_box(V3 size, V3 center);
Mesh make_icosphere(double r, int subdivisions, V3 center);
Mesh make_cylinder(double r, double len, int segments);
void save_obj(const Mesh& m, const std::string& path);
std::vector<Sample> sample_surface(const Mesh& m, double spc, uint64_t seed);

// patches.cpp: per-link hand samples + decompose_patches from the flat hand
// description and its visual meshes.
Patches make_patches(const lg_hand_desc& h, const lg_visual_desc& vis, double spc, double radius,
                     uint64_t seed, int cap);

// config.cpp
void params_default(lg_run_params* p);
void parse_config(const char* path, lg_run_params* p);
uint64_t cache_key(const lg_run_params* p);
uint64_t fnv1a(const void* data, size_t n, uint64_t h);

// dataset.cpp
std::string json_double(double v);
void write_dataset(const std::string& path, const lg_grasp* g, long long n);
void write_profile(const std::string& path, const lg_profile& p);

[[noreturn]] void fail_runtime(const std::string& msg);
[[noreturn]] void fail_invalid(const std::string& msg);

}  // namespace lgh
