// integration/graspgen_b200.cpp — the adapter a maintainer adds to the
// reference (/root/reference/proj) to swap its hot path for the B200 path.
//
// It is compiled against the reference's own headers and defines, with the
// reference's exact C++ signatures, the entry points the device takes over:
//
//   run_batch                 (pipeline.hpp:150, pipeline.cpp:308-625)
//   optimize_contacts         (contact_opt.hpp:49-52, contact_opt.cpp:45-142)
//   validate_grasp_collisions (collision.hpp:71-74, collision.cpp:230-288)
//   solve_contact_ik          (ik.hpp:49-51, ik.cpp:30-139)
//   ContactFieldIndex::build  (contact_field.hpp:125-128, contact_field.cpp:306-334)
//   query_domains             (contact_field.hpp:147-150, contact_field.cpp:380-448)
//   reverse_lookup            (contact_field.hpp:154-156, contact_field.cpp:450-484)
//   solve_fswo / solve_gswo / is_stable (wrench.hpp:56-77, wrench.cpp:179-267)
//   validate_dataset          (validate.hpp:26-29, validate.cpp:56-175)
//
// Everything the reference keeps on the host stays the reference's code:
// parse_config, load_hand (URDF + quickhull parts), load_mesh,
// sample_surface, decompose_patches, dependency_groups, write_dataset.  The
// adapter flattens those results into the lg.h descriptors, calls
// libgraspgen_b200.so and maps the results and status codes back (an lg.h
// LG_ERR_INVALID_ARGUMENT becomes std::invalid_argument, LG_ERR_OUT_OF_RANGE
// std::out_of_range, everything else std::runtime_error, with the library's
// message — so REQUIRE_THROWS in the reference's tests keeps working).
//
// oracle/Makefile links it in place of the reference's definitions
// (objcopy --weaken-symbol on the reference objects, no source edits) into
//   oracle/_ref/graspgen_b200          the reference CLI on the device
//   oracle/_ref/test_contact_opt_b200  the reference's Catch2 tests
//   oracle/_ref/test_collision_b200    against the device entry points
//   oracle/_ref/test_ik_b200
//   oracle/_ref/test_contact_field_b200
//   oracle/_ref/test_wrench_b200
// and tests/test_integration.py runs them on the GPU.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <unistd.h>
#include <vector>

#include "graspgen/collision.hpp"
#include "graspgen/contact_field.hpp"
#include "graspgen/contact_opt.hpp"
#include "graspgen/hand.hpp"
#include "graspgen/ik.hpp"
#include "graspgen/mesh.hpp"
#include "graspgen/pipeline.hpp"
#include "graspgen/rng.hpp"
#include "graspgen/validate.hpp"
#include "graspgen/wrench.hpp"
#include "lg.h"

namespace graspgen {
namespace {

void check(int rc) {
  if (rc == LG_OK) return;
  char msg[2048];
  lg_last_error(msg, sizeof msg);
  if (rc == LG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == LG_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// One context (GPU 0, one stream) per process; the library serialises calls
// on it (one in-flight call per lg_ctx).
lg_ctx* context() {
  static std::once_flag once;
  static lg_ctx* ctx = nullptr;
  std::call_once(once, [] { check(lg_ctx_create(0, &ctx)); });
  return ctx;
}

void put3(double* d, const Vec3& v) {
  d[0] = v.x();
  d[1] = v.y();
  d[2] = v.z();
}
Vec3 get3(const double* d) { return Vec3(d[0], d[1], d[2]); }

struct FlatHand {  // owns the arrays behind an lg_hand_desc
  std::vector<int> parent, type, jidx, topo, part_link, voff{0}, toff{0}, poff{0}, tris;
  std::vector<double> R, t, axis, lo, hi, verts, planes, bounds;
  lg_hand_desc d{};
  explicit FlatHand(const HandModel& m) {
    for (const Link& l : m.links) {
      parent.push_back(l.parent);
      type.push_back(l.joint == JointType::kFixed ? 0 : l.joint == JointType::kRevolute ? 1 : 2);
      jidx.push_back(l.joint_index);
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) R.push_back(l.origin.rotation(r, c));
      for (int a = 0; a < 3; ++a) {
        t.push_back(l.origin.translation[a]);
        axis.push_back(l.axis[a]);
      }
      lo.push_back(l.limit_lo);
      hi.push_back(l.limit_hi);
    }
    for (std::size_t l = 0; l < m.links.size(); ++l)
      for (const ConvexPart& p : m.links[l].parts) {
        part_link.push_back(static_cast<int>(l));
        for (const Vec3& v : p.vertices) verts.insert(verts.end(), {v.x(), v.y(), v.z()});
        for (const auto& tr : p.triangles) tris.insert(tris.end(), {tr[0], tr[1], tr[2]});
        for (const FacePlane& f : p.planes)
          planes.insert(planes.end(), {f.normal.x(), f.normal.y(), f.normal.z(), f.offset});
        bounds.insert(bounds.end(), {p.bounds.min.x(), p.bounds.min.y(), p.bounds.min.z(),
                                     p.bounds.max.x(), p.bounds.max.y(), p.bounds.max.z()});
        voff.push_back(static_cast<int>(verts.size() / 3));
        toff.push_back(static_cast<int>(tris.size() / 3));
        poff.push_back(static_cast<int>(planes.size() / 4));
      }
    topo = m.topo_order;
    d = {static_cast<int>(m.links.size()), m.actuated_count, m.root, parent.data(), type.data(),
         jidx.data(), topo.data(), R.data(), t.data(), axis.data(), lo.data(), hi.data(),
         static_cast<int>(part_link.size()), part_link.data(), voff.data(), verts.data(),
         toff.data(), tris.data(), poff.data(), planes.data(), bounds.data()};
  }
};

struct FlatPatches {
  std::vector<int> link, point_off{0}, fp_off{0}, fps;
  std::vector<double> pts, nrm;
  lg_patches_desc d{};
  explicit FlatPatches(const std::vector<ContactPatch>& ps) {
    for (const ContactPatch& p : ps) {
      link.push_back(p.link);
      for (std::size_t i = 0; i < p.points.size(); ++i) {
        pts.insert(pts.end(), {p.points[i].x(), p.points[i].y(), p.points[i].z()});
        nrm.insert(nrm.end(), {p.normals[i].x(), p.normals[i].y(), p.normals[i].z()});
      }
      point_off.push_back(static_cast<int>(pts.size() / 3));
      fps.insert(fps.end(), p.field_points.begin(), p.field_points.end());
      fp_off.push_back(static_cast<int>(fps.size()));
    }
    d = {static_cast<int>(ps.size()), link.data(), point_off.data(), pts.data(), nrm.data(),
         fp_off.data(), fps.data()};
  }
};

std::vector<double> flat_samples(const std::vector<SurfaceSample>& s) {
  std::vector<double> out;
  out.reserve(6 * s.size());
  for (const SurfaceSample& x : s)
    out.insert(out.end(), {x.position.x(), x.position.y(), x.position.z(), x.normal.x(),
                           x.normal.y(), x.normal.z()});
  return out;
}

lg_run_params params_of(const RunConfig& c) {
  lg_run_params p;
  std::memset(&p, 0, sizeof p);
  std::snprintf(p.hand, sizeof p.hand, "%s", c.hand.c_str());
  std::snprintf(p.object, sizeof p.object, "%s", c.object.c_str());
  std::snprintf(p.out, sizeof p.out, "%s", c.out.c_str());
  p.seed = c.seed;
  p.batch = c.batch;
  p.workers = c.workers;
  p.passes = c.passes;
  p.cache = c.cache;
  p.export_obj = c.export_obj;
  p.k_contacts = c.k_contacts;
  p.samples_per_cm2 = c.samples_per_cm2;
  p.object_scale = c.object_scale;
  p.probe_half_width = c.probe_half_width;
  p.probe_depth_threshold = c.probe_depth_threshold;
  p.hand_scale = c.hand_scale;
  p.field_configs = c.field_configs;
  p.box_width = c.box_width;
  p.patch_radius = c.patch_radius;
  p.field_points_per_patch = c.field_points_per_patch;
  p.codebook_size = c.codebook_size;
  p.theta_hit = c.theta_hit;
  p.placement_mode = c.placement_mode == PlacementMode::kExhaustive ? 0 : 1;
  p.static_contact_prob = c.static_contact_prob;
  put3(p.canonical_center, c.canonical_center);
  put3(p.canonical_half_extents, c.canonical_half_extents);
  p.penetration_margin = c.penetration_margin;
  p.lambda_torque = c.lambda_torque;
  p.mu = c.mu;
  p.eps_stable = c.eps_stable;
  p.pgd_iterations = c.pgd_iterations;
  p.pgd_warm_iterations = c.pgd_warm_iterations;
  p.pgd_step = c.pgd_step;
  p.n_outer = c.n_outer;
  p.n_inner = c.n_inner;
  p.restarts = c.restarts;
  p.sigma = c.sigma;
  p.beta = c.beta;
  p.ik_iterations = c.ik_iterations;
  p.step_clamp = c.step_clamp;
  p.residual_tol = c.residual_tol;
  p.damping_scale = c.damping_scale;
  p.finetune_rounds = c.finetune_rounds;
  p.finetune_iterations = c.finetune_iterations;
  p.lookup_attempts = c.lookup_attempts;
  p.unused_attempts = c.unused_attempts;
  p.contact_tol = c.contact_tol;
  p.shard_rank = 0;
  p.shard_count = 1;
  return p;
}

constexpr std::uint64_t kTagObjectSamples = 0x6f626a73;  // pipeline.cpp:19
constexpr std::uint64_t kTagHandSamples = 0x686e6473;    // pipeline.cpp:20

}  // namespace

// run_batch (pipeline.cpp:308-625): the reference's loaders on the host, the
// forward pass (field build included) on the GPU.
RunResult run_batch(const RunConfig& cfg) {
  auto wall0 = std::chrono::steady_clock::now();
  RunResult out;
  HandModel model = load_hand(cfg.hand, cfg.hand_scale);
  std::vector<std::vector<SurfaceSample>> link_samples(model.links.size());
  for (std::size_t l = 0; l < model.links.size(); ++l) {
    if (model.links[l].visual.vertices.empty()) continue;
    link_samples[l] = sample_surface(model.links[l].visual, cfg.samples_per_cm2,
                                     mix_seed(cfg.seed, kTagHandSamples, l));
  }
  std::vector<ContactPatch> patches =
      decompose_patches(model, link_samples, cfg.patch_radius, cfg.seed, cfg.field_points_per_patch);
  LoadReport object_report;
  TriMesh object = load_mesh(cfg.object, &object_report);
  if (cfg.object_scale != 1.0) object = scale_mesh(object, cfg.object_scale);
  out.loads.object = object_report;
  out.loads.hand_links = static_cast<long>(model.links.size());
  out.loads.hand_joints = model.actuated_count;
  for (const auto& link : model.links) out.loads.hand_parts += static_cast<long>(link.parts.size());
  auto raw = flat_samples(
      sample_surface(object, cfg.samples_per_cm2, mix_seed(cfg.seed, kTagObjectSamples)));

  FlatHand hand(model);
  FlatPatches flat(patches);
  lg_run_params p = params_of(cfg);
  lg_result* res = nullptr;
  check(lg_run_batch(context(), &hand.d, &flat.d, raw.data(), static_cast<int>(raw.size() / 6), &p,
                     &res));
  std::unique_ptr<lg_result, void (*)(lg_result*)> own(res, lg_result_destroy);
  lg_profile prof;
  check(lg_result_profile(res, &prof));
  const long long n = lg_result_num_grasps(res);
  const lg_grasp* g = lg_result_grasps(res);
  for (long long i = 0; i < n; ++i) {
    Grasp gr;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) gr.object_pose.rotation(r, c) = g[i].pose_R[3 * r + c];
    gr.object_pose.translation = get3(g[i].pose_t);
    gr.q = Eigen::VectorXd(g[i].dof);
    for (int j = 0; j < g[i].dof; ++j) gr.q[j] = g[i].q[j];
    for (int c = 0; c < g[i].n_contacts; ++c)
      gr.contacts.push_back({get3(g[i].contact_p[c]), get3(g[i].contact_n[c]), g[i].contact_link[c]});
    gr.objective = g[i].objective;
    gr.flags.penetration_free = g[i].penetration_free != 0;
    gr.flags.stable = g[i].stable != 0;
    gr.flags.ik_converged = g[i].ik_converged != 0;
    out.dataset.grasps.push_back(std::move(gr));
  }
  StageProfile& sp = out.profile;
  sp.placement_domains = prof.placement_domains;
  sp.contact_optimization = prof.contact_optimization;
  sp.kinematics_optimization = prof.kinematics_optimization;
  sp.postprocessing = prof.postprocessing;
  sp.candidates = prof.candidates;
  sp.placements_accepted = prof.placements_accepted;
  sp.contact_sets_balanced = prof.contact_sets_balanced;
  sp.ik_finite = prof.ik_finite;
  sp.penetration_free = prof.penetration_free;
  sp.ik_converged = prof.ik_converged;
  sp.stable = prof.stable;
  sp.valid = prof.valid;
  out.index.patches = static_cast<std::size_t>(prof.patches);
  out.index.boxes = static_cast<std::size_t>(prof.boxes);
  out.index.from_cache = prof.index_from_cache != 0;
  // ContactFieldIndex::total_memory_bytes (contact_field.cpp:336-353) of the
  // same index: every patch in the index holds >= 1 box, and each BVH is a
  // binary tree with one leaf per item (2 b - 1 nodes per patch, 2 P - 1 on
  // top), so the count follows from P, B and the code count
  if (prof.patches > 0) {
    const std::size_t P = static_cast<std::size_t>(prof.patches);
    const std::size_t B = static_cast<std::size_t>(prof.boxes);
    const std::size_t R = static_cast<std::size_t>(prof.index_codes);
    out.index.memory_bytes = sizeof(ContactFieldIndex) +
                             static_cast<std::size_t>(cfg.codebook_size) * sizeof(Vec3) +
                             (2 * P - 1) * sizeof(BvhNode) + P * sizeof(PatchIndex) +
                             B * sizeof(IndexBox) + R * (sizeof(std::uint16_t) + sizeof(IndexRep)) +
                             (2 * B - P) * sizeof(BvhNode);
  }
  sp.total = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  sp.grasps_per_second = sp.total > 0.0 ? sp.valid / sp.total : 0.0;
  return out;
}

// optimize_contacts (contact_opt.cpp:45-142) on the device.
ContactOptResult optimize_contacts(const std::vector<const ContactDomain*>& domains,
                                   const ContactOptParams& params,
                                   const std::vector<StaticContact>& static_contacts,
                                   std::uint64_t seed) {
  const int k = static_cast<int>(domains.size());
  if (k < 1) throw std::invalid_argument("optimize_contacts: no domains");
  for (const auto* d : domains)
    if (!d || d->elements.empty()) throw std::invalid_argument("optimize_contacts: empty domain");
  std::vector<long long> off{0};
  std::vector<double> pos, nrm;
  for (const auto* d : domains) {
    for (const DomainElement& e : d->elements) {
      pos.insert(pos.end(), {e.position.x(), e.position.y(), e.position.z()});
      nrm.insert(nrm.end(), {e.normal.x(), e.normal.y(), e.normal.z()});
    }
    off.push_back(static_cast<long long>(pos.size() / 3));
  }
  int ns = static_cast<int>(static_contacts.size());
  double sp[3] = {0, 0, 0}, sn[3] = {0, 0, 0};
  if (ns > 0) {
    put3(sp, static_contacts[0].position);
    put3(sn, static_contacts[0].normal);
  }
  lg_run_params p;
  std::memset(&p, 0, sizeof p);
  p.n_outer = params.n_outer;
  p.n_inner = params.n_inner;
  p.restarts = params.restarts;
  p.sigma = params.sigma;
  p.lambda_torque = params.lambda_torque;
  p.mu = params.mu;
  p.pgd_iterations = params.solve.iterations;
  p.pgd_warm_iterations = params.solve.warm_iterations;
  p.pgd_step = params.solve.step;
  std::vector<int> ids(k);
  double obj = 0.0;
  int anchor = -1;
  double al[6], bx[6], by[6];
  long long evals = 0;
  check(lg_optimize_contacts_batch(context(), 1, k, off.data(), pos.data(), nrm.data(), &ns, sp, sn,
                                   &p, &seed, ids.data(), &obj, &anchor, al, bx, by, &evals));
  ContactOptResult r;
  r.element_ids = ids;
  for (int q = 0; q < k; ++q) r.elements.push_back(domains[q]->elements[ids[q]]);
  r.objective = obj;
  r.solution.objective = obj;
  r.solution.anchor = anchor;
  if (anchor >= 0) {  // run_solver keeps n-sized alpha / beta (zero beta without friction)
    r.solution.alpha.assign(al, al + k + ns);
    r.solution.beta_x.assign(bx, bx + k + ns);
    r.solution.beta_y.assign(by, by + k + ns);
  }
  r.evaluations = static_cast<int>(evals);
  return r;
}

// validate_grasp_collisions (collision.cpp:230-288) on the device.
CollisionReport validate_grasp_collisions(const HandModel& model, const Eigen::VectorXd& q,
                                          const std::vector<SurfaceSample>& object_samples,
                                          const RigidTransform& object_pose, double margin) {
  if (q.size() != model.actuated_count)
    throw std::invalid_argument("forward_kinematics: config dimension mismatch");
  FlatHand hand(model);
  std::vector<double> qq(q.data(), q.data() + q.size());
  double pose[12];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) pose[3 * r + c] = object_pose.rotation(r, c);
  put3(pose + 9, object_pose.translation);
  auto s = flat_samples(object_samples);
  const int cap = 256;
  int nv = 0, la[cap], lb[cap], pairs[3];
  double depth[cap], maxpen = 0.0;
  check(lg_collision_report_batch(context(), &hand.d, 1, qq.data(), pose, s.data(),
                                  static_cast<int>(object_samples.size()), margin, cap, &nv, la, lb,
                                  depth, &maxpen, pairs));
  CollisionReport rep;
  for (int i = 0; i < nv && i < cap; ++i) rep.violations.push_back({la[i], lb[i], depth[i]});
  rep.max_penetration = maxpen;
  rep.broad_pairs = static_cast<std::size_t>(pairs[0]);
  rep.narrow_gjk = static_cast<std::size_t>(pairs[1]);
  rep.narrow_halfplane = static_cast<std::size_t>(pairs[2]);
  return rep;
}

namespace {

// The contact-field index crosses between host and device as its GGCF v1
// file: the library writes and reads the reference's format byte for byte,
// so a device-built index loads into the reference's ContactFieldIndex and a
// host index (built, loaded or edited by the caller) loads onto the device.
std::string ggcf_scratch() {
  static std::atomic<long> n{0};
  const char* dir = std::getenv("TMPDIR");
  return std::string(dir ? dir : "/tmp") + "/graspgen_b200_" + std::to_string(getpid()) + "_" +
         std::to_string(n++) + ".ggcf";
}

struct DeviceIndex {
  lg_field* f = nullptr;
  DeviceIndex(const ContactFieldIndex& index, const HandModel& model) {
    const std::string path = ggcf_scratch();
    index.save(path);
    FlatHand hand(model);
    const int rc = lg_field_load(context(), &hand.d, path.c_str(), index.cache_key, &f);
    std::remove(path.c_str());
    check(rc);
    if (!f) throw std::runtime_error("graspgen_b200: the index did not load on the device");
  }
  ~DeviceIndex() { lg_field_destroy(f); }
  DeviceIndex(const DeviceIndex&) = delete;
  DeviceIndex& operator=(const DeviceIndex&) = delete;
};

}  // namespace

// ContactFieldIndex::build (contact_field.cpp:306-334) on the device.
ContactFieldIndex ContactFieldIndex::build(const HandModel& model,
                                           const std::vector<ContactPatch>& patches, int N,
                                           double box_width, std::uint64_t seed,
                                           int codebook_size) {
  FlatHand hand(model);
  FlatPatches flat(patches);
  lg_field* f = nullptr;
  check(lg_field_build(context(), &hand.d, &flat.d, N, box_width, seed, codebook_size, &f));
  std::unique_ptr<lg_field, void (*)(lg_field*)> own(f, lg_field_destroy);
  const std::string path = ggcf_scratch();
  check(lg_field_save(f, path.c_str(), 0));
  std::optional<ContactFieldIndex> index = ContactFieldIndex::load(path, 0);
  std::remove(path.c_str());
  if (!index) throw std::runtime_error("graspgen_b200: the device index did not load");
  return std::move(*index);
}

// query_domains (contact_field.cpp:380-448) on the device.
std::vector<ContactDomain> query_domains(const ContactFieldIndex& index,
                                         const std::vector<SurfaceSample>& samples,
                                         const RigidTransform& object_pose, double theta_hit,
                                         const HandModel& model, const DependencyGroups& groups) {
  const int G = static_cast<int>(groups.groups.size());
  std::vector<ContactDomain> domains(G);
  for (int g = 0; g < G; ++g) domains[g].group = g;
  if (index.patches.empty()) return domains;
  int max_id = 0;
  for (const PatchIndex& p : index.patches) max_id = std::max(max_id, p.patch_id);
  std::vector<int> group_of_patch(static_cast<std::size_t>(max_id) + 1, -1);
  for (const PatchIndex& p : index.patches) {
    if (p.link < 0 || p.link >= static_cast<int>(model.links.size()))
      throw std::invalid_argument("query_domains: index link out of range");
    group_of_patch[p.patch_id] = groups.group_of(p.link);
  }
  if (samples.empty()) return domains;
  DeviceIndex dev(index, model);
  auto s = flat_samples(samples);
  double pose[12];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) pose[3 * r + c] = object_pose.rotation(r, c);
  put3(pose + 9, object_pose.translation);
  lg_domains* d = nullptr;
  check(lg_query_domains_elements(context(), dev.f, group_of_patch.data(), G, s.data(),
                                  static_cast<int>(samples.size()), pose, theta_hit, &d));
  std::unique_ptr<lg_domains, void (*)(lg_domains*)> own(d, lg_domains_destroy);
  long long ne = 0;
  const int *sample = nullptr, *hp = nullptr, *hb = nullptr;
  const double *pos = nullptr, *nrm = nullptr, *score = nullptr;
  const long long* hoff = nullptr;
  check(lg_domains_elements(d, &ne, &sample, &pos, &nrm, &score, &hoff, &hp, &hb));
  for (int g = 0; g < G; ++g) {
    long long first = 0, count = 0;
    check(lg_domains_group(d, g, &first, &count));
    for (long long e = first; e < first + count; ++e) {
      DomainElement el;
      el.position = get3(pos + 3 * e);
      el.normal = get3(nrm + 3 * e);
      el.score = score[e];
      el.hit_patches.assign(hp + hoff[e], hp + hoff[e + 1]);
      el.hit_boxes.assign(hb + hoff[e], hb + hoff[e + 1]);
      domains[g].elements.push_back(std::move(el));
    }
  }
  return domains;
}

// reverse_lookup (contact_field.cpp:450-484) on the device.
IndexRep reverse_lookup(const ContactFieldIndex& index, const DomainElement& element,
                        std::uint64_t choice_seed) {
  if (element.hit_patches.empty() || element.hit_patches.size() != element.hit_boxes.size())
    throw std::out_of_range("reverse_lookup: element has no hits");
  // the device needs only the links of the index's patches: a stand-in
  // model with one link per patch link id
  HandModel model;
  int max_link = 0;
  for (const PatchIndex& p : index.patches) max_link = std::max(max_link, p.link);
  model.links.resize(static_cast<std::size_t>(max_link) + 1);
  for (std::size_t l = 0; l < model.links.size(); ++l) {
    model.links[l].parent = l == 0 ? -1 : 0;
    model.topo_order.push_back(static_cast<int>(l));
  }
  DeviceIndex dev(index, model);
  const long long hoff[2] = {0, static_cast<long long>(element.hit_patches.size())};
  double n[3];
  put3(n, element.normal);
  int link = -1;
  double pt[3], nr[3];
  check(lg_reverse_lookup_batch(context(), dev.f, 1, hoff, element.hit_patches.data(),
                                element.hit_boxes.data(), n, &choice_seed, &link, pt, nr));
  IndexRep rep;
  rep.link = link;
  rep.point = get3(pt);
  rep.normal = get3(nr);
  return rep;
}

namespace {

// run_solver (wrench.cpp:179-228) for one problem on the device.
WrenchSolution wrench_device(const WrenchProblem& p, bool gswo, const WrenchSolveOptions& opts,
                             const WrenchSolution* warm) {
  const std::size_t n = p.size();
  if (n == 0) throw std::invalid_argument("wrench solve: no contacts");
  double pts[18] = {}, nrm[18] = {}, tx[18] = {}, ty[18] = {};
  for (std::size_t i = 0; i < n && i < 6; ++i) {
    put3(pts + 3 * i, p.points[i]);
    put3(nrm + 3 * i, p.normals[i]);
    put3(tx + 3 * i, p.tangent_x[i]);
    put3(ty + 3 * i, p.tangent_y[i]);
  }
  const int nn = static_cast<int>(n);
  const bool use_warm = warm && warm->valid() && warm->alpha.size() == n;
  const int uw = use_warm ? 1 : 0;
  double wa[6] = {}, wx[6] = {}, wy[6] = {};
  if (use_warm)
    for (std::size_t i = 0; i < n && i < 6; ++i) {
      wa[i] = warm->alpha[i];
      wx[i] = warm->beta_x.size() == n ? warm->beta_x[i] : 0.0;
      wy[i] = warm->beta_y.size() == n ? warm->beta_y[i] : 0.0;
    }
  double obj = 0.0, a[6], bx[6], by[6];
  int anchor = -1;
  check(lg_wrench_problem_batch(context(), 1, &nn, pts, nrm, tx, ty, &p.lambda_torque, &p.mu,
                                gswo ? 1 : 0, opts.iterations, opts.warm_iterations, opts.step,
                                opts.max_backtracks, &uw, wa, wx, wy, &obj, &anchor, a, bx, by));
  WrenchSolution best;
  if (anchor < 0) return best;  // no anchor improved on +inf
  best.objective = obj;
  best.anchor = anchor;
  best.alpha.assign(a, a + n);
  best.beta_x.assign(bx, bx + n);
  best.beta_y.assign(by, by + n);
  return best;
}

}  // namespace

// solve_fswo / solve_gswo / is_stable (wrench.cpp:247-267) on the device.
WrenchSolution solve_fswo(const WrenchProblem& problem, const WrenchSolveOptions& opts,
                          const WrenchSolution* warm) {
  return wrench_device(problem, false, opts, warm);
}

WrenchSolution solve_gswo(const WrenchProblem& problem, const WrenchSolveOptions& opts,
                          const WrenchSolution* warm) {
  return wrench_device(problem, problem.mu != 0.0, opts, warm);
}

bool is_stable(const WrenchProblem& problem, double eps, WrenchSolution* solution,
               const WrenchSolveOptions& opts) {
  if (eps <= 0.0) throw std::invalid_argument("is_stable: eps must be > 0");
  WrenchSolution s = solve_gswo(problem, opts);
  const bool stable = s.objective < eps;
  if (solution) *solution = std::move(s);
  return stable;
}

// validate_dataset (validate.cpp:56-175): the object samples are the
// reference's sample_surface (stream 'objs', as validate.cpp:63-65 re-draws
// them); every check runs on the device and the issue texts come from
// lg_validation_issues.
ValidationReport validate_dataset(const GraspDataset& dataset, const HandModel& model,
                                  const TriMesh& object, const RunConfig& config) {
  ValidationReport report;
  report.checked = static_cast<long>(dataset.grasps.size());
  if (dataset.grasps.empty()) return report;
  FlatHand hand(model);
  std::vector<lg_grasp> gs(dataset.grasps.size());
  for (std::size_t i = 0; i < gs.size(); ++i) {
    const Grasp& g = dataset.grasps[i];
    lg_grasp& o = gs[i];
    std::memset(&o, 0, sizeof o);
    o.g = static_cast<long long>(i);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) o.pose_R[3 * r + c] = g.object_pose.rotation(r, c);
    put3(o.pose_t, g.object_pose.translation);
    o.dof = static_cast<int>(g.q.size());
    for (int j = 0; j < o.dof && j < LG_MAX_DOF; ++j) o.q[j] = g.q[j];
    if (g.contacts.size() > LG_MAX_CONTACTS)
      throw std::invalid_argument("validate_dataset: the device checks at most 6 contacts per grasp");
    o.n_contacts = static_cast<int>(g.contacts.size());
    for (int c = 0; c < o.n_contacts; ++c) {
      put3(o.contact_p[c], g.contacts[c].position);
      put3(o.contact_n[c], g.contacts[c].normal);
      o.contact_link[c] = g.contacts[c].link;
    }
    o.objective = g.objective;
  }
  std::vector<double> verts;
  std::vector<int> tris;
  for (const Vec3& v : object.vertices) verts.insert(verts.end(), {v.x(), v.y(), v.z()});
  for (const auto& t : object.triangles) tris.insert(tris.end(), {t[0], t[1], t[2]});
  auto samples = flat_samples(sample_surface(object, config.samples_per_cm2,
                                             mix_seed(config.seed, kTagObjectSamples)));
  const lg_run_params p = params_of(config);
  std::vector<lg_grasp_check> checks(gs.size());
  check(lg_validate_batch(context(), &hand.d, gs.data(), static_cast<long long>(gs.size()),
                          verts.data(), static_cast<int>(object.vertices.size()), tris.data(),
                          static_cast<int>(object.triangles.size()), samples.data(),
                          static_cast<int>(samples.size() / 6), &p, checks.data()));
  std::vector<const char*> names;
  for (const Link& l : model.links) names.push_back(l.joint_name.c_str());
  std::size_t need = 0;
  long long n_issues = 0;
  check(lg_validation_issues(names.data(), static_cast<int>(names.size()), checks.data(),
                             static_cast<long long>(checks.size()), &p, nullptr, 0, &need,
                             &n_issues));
  std::vector<char> buf(need + 1, '\0');
  check(lg_validation_issues(names.data(), static_cast<int>(names.size()), checks.data(),
                             static_cast<long long>(checks.size()), &p, buf.data(), buf.size(),
                             &need, &n_issues));
  const std::string text(buf.data());
  std::size_t pos = 0;
  while (pos < text.size()) {
    const std::size_t eol = text.find('\n', pos), tab = text.find('\t', pos);
    if (eol == std::string::npos || tab == std::string::npos || tab > eol) break;
    report.issues.push_back({std::stol(text.substr(pos, tab - pos)), text.substr(tab + 1, eol - tab - 1)});
    pos = eol + 1;
  }
  return report;
}

// solve_contact_ik (ik.cpp:30-139) on the device.  The device returns each
// target's clamped normal cosine; normal_angle is its std::acos, as in
// ik.cpp:136-137.
IkResult solve_contact_ik(const HandModel& model, const Eigen::VectorXd& q0,
                          const std::vector<ContactTarget>& targets, const IkParams& params) {
  if (q0.size() != model.actuated_count)
    throw std::invalid_argument("solve_contact_ik: config dimension mismatch");
  FlatHand hand(model);
  const int k = static_cast<int>(targets.size());
  std::vector<double> op, on, hp, hn;
  std::vector<int> links;
  for (const ContactTarget& t : targets) {
    op.insert(op.end(), {t.object_point.x(), t.object_point.y(), t.object_point.z()});
    on.insert(on.end(), {t.object_normal.x(), t.object_normal.y(), t.object_normal.z()});
    hp.insert(hp.end(), {t.hand_point_local.x(), t.hand_point_local.y(), t.hand_point_local.z()});
    hn.insert(hn.end(), {t.hand_normal_local.x(), t.hand_normal_local.y(), t.hand_normal_local.z()});
    links.push_back(t.link);
  }
  const int dof = model.actuated_count;
  std::vector<double> qi(q0.data(), q0.data() + dof), q(std::max(dof, 1));
  std::vector<double> pos(std::max(k, 1)), cosv(std::max(k, 1));
  int finite = 0, iters = 0;
  unsigned long long used = 0;
  double objective = 0.0;
  check(lg_contact_ik_batch(context(), &hand.d, 1, &k, qi.data(), op.data(), on.data(), links.data(),
                            hp.data(), hn.data(), params.beta, params.iterations, params.step_clamp,
                            params.residual_tol, params.damping_scale, params.damping_min,
                            params.max_backtracks, q.data(), &finite, &used, &iters, &objective,
                            pos.data(), cosv.data()));
  IkResult res;
  res.q = Eigen::VectorXd(dof);
  for (int j = 0; j < dof; ++j) res.q[j] = q[j];
  res.used_joints.assign(dof, false);
  for (int j = 0; j < dof; ++j) res.used_joints[j] = ((used >> j) & 1ull) != 0;
  res.finite = finite != 0;
  res.iterations = iters;
  res.objective = objective;
  res.residuals.resize(k);
  for (int i = 0; i < k; ++i) {
    res.residuals[i].position = pos[i];
    res.residuals[i].normal_angle = std::acos(cosv[i]);
  }
  return res;
}

}  // namespace graspgen
