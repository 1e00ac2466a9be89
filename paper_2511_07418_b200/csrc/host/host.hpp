// host.hpp — caller-side model types and loaders of the drop-in boundary.
//
// These are the steps the reference keeps on the host and the north star
// leaves in place: URDF-subset hand loading with convex collision parts
// (hand.cpp:265-414, convex.cpp:139-359), OBJ/STL meshes and primitives
// (mesh.cpp), area-weighted surface sampling (mesh.cpp:297-339), patch
// decomposition (contact_field.cpp:26-99), dependency groups (hand.cpp:
// 515-552), run configuration (config.cpp) and the JSONL result format
// (dataset.cpp).  They produce the flat lg_*_desc views that the device
// library consumes.
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

struct Part {  // ConvexPart, convex.hpp:20-38
  std::vector<V3> verts;
  std::vector<std::array<int, 3>> tris;
  std::vector<V3> plane_n;
  std::vector<double> plane_d;
  V3 bmin, bmax;
};

struct Link {
  std::string name;
  int parent = -1;
  Xf origin = lgm::xf_identity();
  int jtype = 0;
  std::string joint_name;
  V3 axis = lgm::v3(1, 0, 0);
  double lo = 0.0, hi = 0.0;
  int jidx = -1;
  Mesh visual;
  std::vector<Part> parts;
};

struct Hand {
  std::vector<Link> links;
  int root = -1;
  int dof = 0;
  std::vector<int> topo;
  std::string source_dir;
  // flat view storage
  std::vector<int> f_parent, f_jtype, f_jidx, f_part_link, f_vert_off, f_tri_off, f_plane_off,
      f_tris;
  std::vector<double> f_R, f_t, f_axis, f_lo, f_hi, f_verts, f_planes, f_bounds;
  void flatten();
  lg_hand_desc desc() const;
  int link_index(const std::string& n) const;
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

// convex.cpp
Part convex_hull(const std::vector<V3>& pts);
Part scale_part(const Part& p, double s);

// hand.cpp
Hand load_hand(const std::string& path, double scale);
std::vector<int> dependency_group_of(const Hand& h, int* n_groups);  // per link, -1 static
Patches make_patches(const Hand& h, double spc, double radius, uint64_t seed, int cap);

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
