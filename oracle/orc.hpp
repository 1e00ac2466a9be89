// oracle/orc.hpp — CPU restatement of the Lightning Grasp reference forward
// pass (/root/reference/proj/src), used ONLY as the parity checker by tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
// Nothing in the product path links or calls this code.
//
// Parity status: the reference itself cannot be compiled here (it needs
// Eigen, Boost.PropertyTree and Catch2, none of which exist in the image;
// see DESIGN.md "Oracle").  This restatement follows the reference file by
// file (each function cites file:line) and is pinned against every
// known-answer and property test the reference's own Catch2 suite holds for
// the hot path (tests/test_oracle_pins.py).  Arithmetic uses the canonical
// Eigen-equivalent order and deterministic libm from lg_math.h, shared with
// the device so that device-vs-oracle comparisons can be bit-exact.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "lg.h"
#include "lg_math.h"

namespace orc {

using lgm::M3;
using lgm::V3;
using lgm::Xf;

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double kPi = 3.14159265358979323846;

// ------------------------------------------------------------- geometry.hpp
struct Aabb {  // geometry.hpp:65-101
  V3 min = lgm::v3(kInf, kInf, kInf);
  V3 max = lgm::v3(-kInf, -kInf, -kInf);
  bool empty() const { return min.x > max.x || min.y > max.y || min.z > max.z; }
  void expand(V3 p) {
    min = lgm::vmin(min, p);
    max = lgm::vmax(max, p);
  }
  void expand(const Aabb& b) {
    min = lgm::vmin(min, b.min);
    max = lgm::vmax(max, b.max);
  }
  Aabb inflated(double m) const {
    Aabb r;
    r.min = lgm::v3(min.x - m, min.y - m, min.z - m);
    r.max = lgm::v3(max.x + m, max.y + m, max.z + m);
    return r;
  }
  bool contains(V3 p) const {
    return p.x >= min.x && p.y >= min.y && p.z >= min.z && p.x <= max.x &&
           p.y <= max.y && p.z <= max.z;
  }
  bool overlaps(const Aabb& b) const {
    return min.x <= b.max.x && min.y <= b.max.y && min.z <= b.max.z &&
           max.x >= b.min.x && max.y >= b.min.y && max.z >= b.min.z;
  }
  V3 center() const {
    return lgm::v3(0.5 * (min.x + max.x), 0.5 * (min.y + max.y), 0.5 * (min.z + max.z));
  }
  V3 extents() const { return lgm::sub(max, min); }
};

void tangent_basis(V3 n, V3& x, V3& y);    // geometry.hpp:105-126
M3 rotation_between(V3 from, V3 to);       // geometry.hpp:129-143

// ------------------------------------------------------------------ rng.hpp
class Rng {  // rng.hpp:30-90 (std::mt19937_64 engine)
 public:
  explicit Rng(uint64_t seed);
  uint64_t next_u64();
  double uniform() { return lgm::u01(next_u64()); }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint64_t uniform_index(uint64_t n) { return next_u64() % n; }
  double normal();
  void uniform_quaternion(double* w, double* x, double* y, double* z);
  V3 uniform_unit_vector();

 private:
  lgm::Mt64 eng_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

// -------------------------------------------------------- convex / hand
struct Part {  // convex.hpp:20-38
  std::vector<V3> verts;
  std::vector<std::array<int, 3>> tris;
  std::vector<V3> plane_n;
  std::vector<double> plane_d;
  Aabb bounds;
  bool contains(V3 p, double tol = 0.0) const;
  double interior_depth(V3 p) const;
  V3 closest_surface_point(V3 p, V3* normal) const;
  V3 support(V3 dir) const;
};
V3 closest_point_on_triangle(V3 p, V3 a, V3 b, V3 c);  // convex.cpp:27-63

struct Link {  // hand.hpp:19-35
  int parent = -1;
  Xf origin;
  int jtype = 0;  // 0 fixed 1 revolute 2 prismatic
  V3 axis;
  double lo = 0, hi = 0;
  int jidx = -1;
  std::vector<int> parts;  // indices into Hand::parts
};

struct Hand {  // hand.hpp:37-46
  std::vector<Link> links;
  std::vector<Part> parts;
  int root = -1;
  int dof = 0;
  std::vector<int> topo;
  static Hand from_desc(const lg_hand_desc& d);
  std::vector<double> mid_config() const;                       // hand.cpp:24-32
  void clamp_to_limits(std::vector<double>& q) const;           // hand.cpp:34-43
};

std::vector<Xf> forward_kinematics(const Hand& h, const double* q);  // hand.cpp:275-295
// point_jacobian (hand.cpp:343-358): J is 3 x dof, row-major [r*dof + c]
void point_jacobian(const Hand& h, const std::vector<Xf>& frames, int link,
                    V3 local_point, double* J);

struct Groups {  // hand.hpp:66-73
  std::vector<std::vector<int>> groups;
  std::vector<int> static_links;
  int group_of(int link) const;
};
Groups dependency_groups(const Hand& h);  // hand.cpp:374-411

// ------------------------------------------------------------ mesh sampling
struct Sample {
  V3 p, n;
};
// sample_surface (mesh.cpp:297-339) over a flat triangle mesh.
std::vector<Sample> sample_surface(const std::vector<V3>& verts,
                                   const std::vector<std::array<int, 3>>& tris,
                                   double samples_per_cm2, uint64_t seed);
std::vector<Sample> transform_samples(const std::vector<Sample>& s, const Xf& t);

// ------------------------------------------------------------ contact field
struct Patch {  // contact_field.hpp:20-30
  int id = -1, link = -1;
  std::vector<V3> points, normals;
  std::vector<int> field_points;
};
std::vector<Patch> patches_from_desc(const lg_patches_desc& d);
std::vector<Patch> decompose_patches(const Hand& h,
                                     const std::vector<std::vector<Sample>>& per_link,
                                     double patch_radius, uint64_t seed, int cap);

struct IndexRep {
  int link = -1;
  V3 point, normal;
};
struct IndexBox {
  std::array<int64_t, 3> cell;
  std::vector<uint16_t> codes;
  std::vector<IndexRep> reps;
};
struct BvhNode {
  Aabb bounds;
  int32_t left = -1, right = -1, leaf = -1;
};
struct PatchIndex {
  int patch_id = -1, link = -1;
  std::vector<IndexBox> boxes;
  std::vector<BvhNode> nodes;
  int32_t root = -1;
};
struct FieldIndex {  // contact_field.hpp:112-137
  double box_width = 0;
  std::vector<V3> codebook;
  std::vector<PatchIndex> patches;
  std::vector<BvhNode> top_nodes;
  int32_t top_root = -1;
  long long n_vectors = 0;
};
std::vector<V3> make_codebook(int size);                      // :144-158
uint16_t quantize_normal(const std::vector<V3>& cb, V3 n);    // :160-172
std::array<int64_t, 3> cell_of(V3 p, double w);               // :176-180
std::vector<double> field_config(const Hand& h, uint64_t seed, int c);  // :101-114
FieldIndex build_field_index(const Hand& h, const std::vector<Patch>& patches, int N,
                             double w, uint64_t seed, int C);  // :306-334

struct DomainElement {  // contact_field.hpp:95-102
  V3 position, normal;
  std::vector<int> hit_patches, hit_boxes;
  double score = 0.0;
  int sample = -1;  // index of the field sample behind the element
};
struct Domain {
  int group = -1;
  std::vector<DomainElement> elements;
};
std::vector<Domain> query_domains(const FieldIndex& idx, const std::vector<Sample>& samples,
                                  const Xf& pose, double theta, const Hand& h,
                                  const Groups& g);            // :380-448
IndexRep reverse_lookup(const FieldIndex& idx, const DomainElement& el,
                        uint64_t seed);                        // :450-484

// ------------------------------------------------------------------ wrench
struct WrenchProblem {  // wrench.hpp:13-29
  std::vector<V3> p, n, tx, ty;
  double lambda = 10.0, mu = 0.0;
  size_t size() const { return p.size(); }
};
struct WrenchSolution {  // wrench.hpp:36-44
  double objective = kInf;
  int anchor = -1;
  std::vector<double> alpha, bx, by;
  bool valid() const { return anchor >= 0; }
};
struct WrenchOpts {
  int iterations = 64, warm_iterations = 8;
  double step = 0.1;
  int max_backtracks = 20;
};
WrenchProblem make_wrench_problem(const std::vector<V3>& p, const std::vector<V3>& n,
                                  double lambda, double mu);
double wrench_objective(const WrenchProblem& p, const WrenchSolution& s);
WrenchSolution solve_fswo(const WrenchProblem& p, const WrenchOpts& o,
                          const WrenchSolution* warm);
WrenchSolution solve_gswo(const WrenchProblem& p, const WrenchOpts& o,
                          const WrenchSolution* warm);
bool is_stable(const WrenchProblem& p, double eps, WrenchSolution* sol, const WrenchOpts& o);

// -------------------------------------------------------------- contact opt
struct StaticContact {
  V3 position, normal;
};
struct ContactOptParams {  // contact_opt.hpp:14-22
  int n_outer = 8, n_inner = 32, restarts = 4;
  double sigma = 0.01, lambda = 10.0, mu = 0.3;
  WrenchOpts solve;
};
struct ContactOptResult {  // contact_opt.hpp:33-39
  std::vector<int> element_ids;
  std::vector<DomainElement> elements;
  double objective = kInf;
  WrenchSolution solution;
  int evaluations = 0;
};
int project_to_domain(V3 c, const Domain& d);  // contact_opt.cpp:11-25
ContactOptResult optimize_contacts(const std::vector<const Domain*>& domains,
                                   const ContactOptParams& params,
                                   const std::vector<StaticContact>& statics,
                                   uint64_t seed);  // contact_opt.cpp:45-142

// ---------------------------------------------------------------------- IK
struct ContactTarget {  // ik.hpp:13-19
  V3 object_point, object_normal;
  int link = -1;
  V3 hand_point, hand_normal;
};
struct IkParams {  // ik.hpp:21-29
  double beta = 0.01;
  int iterations = 30;
  double step_clamp = 0.2, residual_tol = 1e-4, damping_scale = 1e-4,
         damping_min = 1e-6;
  int max_backtracks = 10;
};
struct IkResult {
  std::vector<double> q;
  std::vector<double> res_pos, res_angle;
  std::vector<bool> used;
  bool finite = true;
  int iterations = 0;
  double objective = 0.0;
};
IkResult solve_contact_ik(const Hand& h, const std::vector<double>& q0,
                          const std::vector<ContactTarget>& t, const IkParams& p);

// --------------------------------------------------------------- collision
struct CollisionReport {
  int n_violations = 0;
  double max_penetration = 0.0;
  long broad_pairs = 0, narrow_gjk = 0, narrow_halfplane = 0;
  bool clean() const { return n_violations == 0; }
};
double gjk_distance(const Part& a, const Xf& pa, const Part& b, const Xf& pb);
struct PenetrationResult {
  double max_depth = 0.0;
  std::vector<int> offending;
};
PenetrationResult object_penetration(const std::vector<Sample>& s, const Part& part,
                                     const Xf& pose, double margin);
CollisionReport validate_grasp_collisions(const Hand& h, const double* q,
                                          const std::vector<Sample>& samples,
                                          const Xf& pose, double margin);
Aabb world_bounds(const Part& part, const Xf& pose);

// ---------------------------------------------------------------- pipeline
double closest_on_parts(const Hand& h, int link, V3 p, V3* sp, V3* sn);
std::vector<Sample> preprocess_object(const std::vector<Sample>& s, double h, double d);

struct RealizeResult {  // pipeline.hpp:108-115
  std::vector<double> q;
  std::vector<bool> used;
  std::vector<V3> real_p, real_n;
  std::vector<int> real_link;
  std::vector<double> residuals;
  double max_residual = 0.0;
  bool finite = true;
};
RealizeResult realize_grasp(const Hand& h, const std::vector<double>& q0,
                            const std::vector<ContactTarget>& targets, const IkParams& p,
                            int finetune_rounds, int finetune_iterations);

struct RunOutput {
  lg_profile profile;
  std::vector<lg_grasp> grasps;
  std::vector<lg_trace> traces;
};
// run_batch (pipeline.cpp:308-625) minus the loaders: the caller passes the
// loaded hand, its decomposed patches and the raw object samples.
RunOutput run_batch(const Hand& h, const std::vector<Patch>& patches,
                    const std::vector<Sample>& raw, const lg_run_params& cfg,
                    int workers, const FieldIndex* cached = nullptr);

// parallel_for (parallel.hpp:24-56)
void parallel_for(size_t begin, size_t end, int workers,
                  const std::function<void(size_t)>& fn);

}  // namespace orc
