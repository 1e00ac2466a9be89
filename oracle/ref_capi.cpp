// oracle/ref_capi.cpp — C entry points over the REFERENCE ITSELF, compiled
// from /root/reference/proj/src/*.cpp (unmodified) against the shims in
// oracle/shim into oracle/_ref/libgraspgen_ref.so.
//
// TEST INFRASTRUCTURE ONLY.  tests/, __graft_entry__.smoke() and bench.py's
// reference arm load it through oracle/ref_py.py to (a) obtain the reference's
// own inputs (load_hand, sample_surface, decompose_patches, parse_config) in
// the flat lg.h descriptor layout the device consumes, and (b) run the
// reference's public functions on them (run_batch, ContactFieldIndex::build,
// query_domains, optimize_contacts, reverse_lookup, place_object,
// realize_grasp, validate_grasp_collisions, solve_fswo / solve_gswo,
// preprocess_object) so every device result is compared with the reference's
// own output on identical inputs.  Nothing in the product links this file.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "graspgen/collision.hpp"
#include "graspgen/config.hpp"
#include "graspgen/contact_field.hpp"
#include "graspgen/contact_opt.hpp"
#include "graspgen/hand.hpp"
#include "graspgen/ik.hpp"
#include "graspgen/mesh.hpp"
#include "graspgen/pipeline.hpp"
#include "graspgen/rng.hpp"
#include "graspgen/wrench.hpp"
#include "lg.h"

using namespace graspgen;

namespace {

thread_local std::string g_err;

constexpr std::uint64_t kTagObjectSamples = 0x6f626a73;  // pipeline.cpp:19
constexpr std::uint64_t kTagHandSamples = 0x686e6473;    // pipeline.cpp:20

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

void put3(double* d, const Vec3& v) {
  d[0] = v.x();
  d[1] = v.y();
  d[2] = v.z();
}
Vec3 get3(const double* d) { return Vec3(d[0], d[1], d[2]); }

void put_rigid(double* R, double* t, const RigidTransform& x) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = x.rotation(i, j);
  put3(t, x.translation);
}
RigidTransform get_pose12(const double* p) {
  RigidTransform x;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) x.rotation(i, j) = p[3 * i + j];
  x.translation = get3(p + 9);
  return x;
}

// Flat HandModel (lg_hand_desc layout, lg.h) built from the reference's own
// loaded model.
struct FlatHand {
  std::vector<int> parent, jtype, jidx, topo, part_link, vert_off{0}, tri_off{0}, plane_off{0}, tris;
  std::vector<double> R, t, axis, lo, hi, verts, planes, bounds;
  lg_hand_desc d{};

  void build(const HandModel& m) {
    const int n = static_cast<int>(m.links.size());
    for (int l = 0; l < n; ++l) {
      const Link& k = m.links[l];
      parent.push_back(k.parent);
      jtype.push_back(k.joint == JointType::kFixed ? 0 : k.joint == JointType::kRevolute ? 1 : 2);
      jidx.push_back(k.joint_index);
      R.resize(R.size() + 9);
      t.resize(t.size() + 3);
      put_rigid(&R[9 * l], &t[3 * l], k.origin);
      axis.resize(axis.size() + 3);
      put3(&axis[3 * l], k.axis);
      lo.push_back(k.limit_lo);
      hi.push_back(k.limit_hi);
      for (const ConvexPart& p : k.parts) {
        part_link.push_back(l);
        for (const Vec3& v : p.vertices) verts.insert(verts.end(), {v.x(), v.y(), v.z()});
        for (const auto& tr : p.triangles) tris.insert(tris.end(), {tr[0], tr[1], tr[2]});
        for (const FacePlane& pl : p.planes)
          planes.insert(planes.end(), {pl.normal.x(), pl.normal.y(), pl.normal.z(), pl.offset});
        bounds.insert(bounds.end(), {p.bounds.min.x(), p.bounds.min.y(), p.bounds.min.z(),
                                     p.bounds.max.x(), p.bounds.max.y(), p.bounds.max.z()});
        vert_off.push_back(static_cast<int>(verts.size() / 3));
        tri_off.push_back(static_cast<int>(tris.size() / 3));
        plane_off.push_back(static_cast<int>(planes.size() / 4));
      }
    }
    topo = m.topo_order;
    d.n_links = n;
    d.dof = m.actuated_count;
    d.root = m.root;
    d.parent = parent.data();
    d.joint_type = jtype.data();
    d.joint_index = jidx.data();
    d.topo_order = topo.data();
    d.origin_R = R.data();
    d.origin_t = t.data();
    d.axis = axis.data();
    d.limit_lo = lo.data();
    d.limit_hi = hi.data();
    d.n_parts = static_cast<int>(part_link.size());
    d.part_link = part_link.data();
    d.part_vert_off = vert_off.data();
    d.part_verts = verts.data();
    d.part_tri_off = tri_off.data();
    d.part_tris = tris.data();
    d.part_plane_off = plane_off.data();
    d.part_planes = planes.data();
    d.part_bounds = bounds.data();
  }
};

struct FlatPatches {
  std::vector<int> link, point_off{0}, fp_off{0}, fps;
  std::vector<double> pts, nrm;
  lg_patches_desc d{};
  void build(const std::vector<ContactPatch>& ps) {
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
    d.n_patches = static_cast<int>(ps.size());
    d.link = link.data();
    d.point_off = point_off.data();
    d.points = pts.data();
    d.normals = nrm.data();
    d.fp_off = fp_off.data();
    d.field_points = fps.data();
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
std::vector<SurfaceSample> unflat_samples(const double* s, int n) {
  std::vector<SurfaceSample> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    out[i].position = get3(s + 6 * i);
    out[i].normal = get3(s + 6 * i + 3);
  }
  return out;
}

void export_params(const RunConfig& c, lg_run_params* p) {
  std::memset(p, 0, sizeof(*p));
  std::snprintf(p->hand, sizeof(p->hand), "%s", c.hand.c_str());
  std::snprintf(p->object, sizeof(p->object), "%s", c.object.c_str());
  std::snprintf(p->out, sizeof(p->out), "%s", c.out.c_str());
  p->seed = c.seed;
  p->batch = c.batch;
  p->workers = c.workers;
  p->passes = c.passes;
  p->cache = c.cache ? 1 : 0;
  p->export_obj = c.export_obj ? 1 : 0;
  p->k_contacts = c.k_contacts;
  p->samples_per_cm2 = c.samples_per_cm2;
  p->object_scale = c.object_scale;
  p->probe_half_width = c.probe_half_width;
  p->probe_depth_threshold = c.probe_depth_threshold;
  p->hand_scale = c.hand_scale;
  p->field_configs = c.field_configs;
  p->box_width = c.box_width;
  p->patch_radius = c.patch_radius;
  p->field_points_per_patch = c.field_points_per_patch;
  p->codebook_size = c.codebook_size;
  p->theta_hit = c.theta_hit;
  p->placement_mode = c.placement_mode == PlacementMode::kExhaustive ? 0 : 1;
  p->static_contact_prob = c.static_contact_prob;
  put3(p->canonical_center, c.canonical_center);
  put3(p->canonical_half_extents, c.canonical_half_extents);
  p->penetration_margin = c.penetration_margin;
  p->lambda_torque = c.lambda_torque;
  p->mu = c.mu;
  p->eps_stable = c.eps_stable;
  p->pgd_iterations = c.pgd_iterations;
  p->pgd_warm_iterations = c.pgd_warm_iterations;
  p->pgd_step = c.pgd_step;
  p->n_outer = c.n_outer;
  p->n_inner = c.n_inner;
  p->restarts = c.restarts;
  p->sigma = c.sigma;
  p->beta = c.beta;
  p->ik_iterations = c.ik_iterations;
  p->step_clamp = c.step_clamp;
  p->residual_tol = c.residual_tol;
  p->damping_scale = c.damping_scale;
  p->finetune_rounds = c.finetune_rounds;
  p->finetune_iterations = c.finetune_iterations;
  p->lookup_attempts = c.lookup_attempts;
  p->unused_attempts = c.unused_attempts;
  p->contact_tol = c.contact_tol;
  p->shard_rank = 0;
  p->shard_count = 1;
}

void export_grasp(const Grasp& g, long long id, lg_grasp* o) {
  std::memset(o, 0, sizeof(*o));
  o->g = id;
  put_rigid(o->pose_R, o->pose_t, g.object_pose);
  o->dof = static_cast<int>(g.q.size());
  for (int j = 0; j < o->dof && j < LG_MAX_DOF; ++j) o->q[j] = g.q[j];
  o->n_contacts = static_cast<int>(g.contacts.size());
  for (int i = 0; i < o->n_contacts && i < LG_MAX_CONTACTS; ++i) {
    put3(o->contact_p[i], g.contacts[i].position);
    put3(o->contact_n[i], g.contacts[i].normal);
    o->contact_link[i] = g.contacts[i].link;
  }
  o->objective = g.objective;
  o->penetration_free = g.flags.penetration_free;
  o->stable = g.flags.stable;
  o->ik_converged = g.flags.ik_converged;
}

}  // namespace

// ----------------------------------------------------------------- handles
struct ref_inputs {
  RunConfig cfg;
  HandModel model;
  DependencyGroups groups;
  std::vector<ContactPatch> patches;
  std::vector<SurfaceSample> raw;
  std::vector<double> raw_flat;
  std::vector<int> group_of_link, group_of_patch;
  FlatHand hand;
  FlatPatches pflat;
  LoadReport object_report;
  std::unique_ptr<ContactFieldIndex> index;
};

struct ref_result {
  RunResult r;
  std::vector<lg_grasp> grasps;
};

struct ref_hand {
  HandModel model;
  DependencyGroups groups;
  FlatHand flat;
  std::vector<int> vis_vert_off{0}, vis_tri_off{0}, vis_tris, group_of_link;
  std::vector<double> vis_verts;
};

struct ref_field {
  ContactFieldIndex idx;
  std::vector<int> patch_link, box_off{0};
  std::vector<long long> cells, code_off{0};
  std::vector<uint16_t> codes;
  std::vector<int> rep_link;
  std::vector<double> codebook, rep_point, rep_normal;
};

extern "C" {

int ref_last_error(char* buf, size_t cap) {
  if (buf && cap) std::snprintf(buf, cap, "%s", g_err.c_str());
  return static_cast<int>(g_err.size());
}

// parse_config(cfg_path + extra "key = value" lines, overrides) followed by
// build_field's and run_batch's host input steps (pipeline.cpp:273-331):
// load_hand, per-link sample_surface ('hnds'), decompose_patches, object
// load_mesh / scale / sample_surface ('objs').
int ref_prepare(const char* cfg_path, const char* extra, const char* hand, const char* object,
                const char* out_dir, long long seed, int batch, int workers, ref_inputs** out) {
  return guard([&] {
    std::string text;
    if (cfg_path && *cfg_path) {
      std::ifstream in(cfg_path);
      if (!in) throw std::runtime_error(std::string("config: cannot open ") + cfg_path);
      std::stringstream ss;
      ss << in.rdbuf();
      text = ss.str();
    }
    if (extra) text += std::string("\n") + extra + "\n";
    auto tmp = std::filesystem::temp_directory_path() /
               ("ref_cfg_" + std::to_string(reinterpret_cast<uintptr_t>(&text)) + ".cfg");
    {
      std::ofstream o(tmp);
      o << text;
    }
    ConfigOverrides ov;
    if (hand) ov.hand = std::string(hand);
    if (object) ov.object = std::string(object);
    if (out_dir) ov.out = std::string(out_dir);
    if (seed >= 0) ov.seed = static_cast<std::uint64_t>(seed);
    if (batch > 0) ov.batch = batch;
    if (workers >= 0) ov.workers = workers;
    auto in = std::make_unique<ref_inputs>();
    try {
      in->cfg = parse_config(tmp.string(), ov);
    } catch (...) {
      std::filesystem::remove(tmp);
      throw;
    }
    std::filesystem::remove(tmp);
    const RunConfig& cfg = in->cfg;
    in->model = load_hand(cfg.hand, cfg.hand_scale);
    std::vector<std::vector<SurfaceSample>> link_samples(in->model.links.size());
    for (std::size_t l = 0; l < in->model.links.size(); ++l) {
      if (in->model.links[l].visual.vertices.empty()) continue;
      link_samples[l] = sample_surface(in->model.links[l].visual, cfg.samples_per_cm2,
                                       mix_seed(cfg.seed, kTagHandSamples, l));
    }
    in->patches = decompose_patches(in->model, link_samples, cfg.patch_radius, cfg.seed,
                                    cfg.field_points_per_patch);
    TriMesh obj = load_mesh(cfg.object, &in->object_report);
    if (cfg.object_scale != 1.0) obj = scale_mesh(obj, cfg.object_scale);
    in->raw = sample_surface(obj, cfg.samples_per_cm2, mix_seed(cfg.seed, kTagObjectSamples));
    in->raw_flat = flat_samples(in->raw);
    in->groups = dependency_groups(in->model);
    in->group_of_link.assign(in->model.links.size(), -1);
    for (std::size_t l = 0; l < in->model.links.size(); ++l)
      in->group_of_link[l] = in->groups.group_of(static_cast<int>(l));
    for (const ContactPatch& p : in->patches) in->group_of_patch.push_back(in->group_of_link[p.link]);
    in->hand.build(in->model);
    in->pflat.build(in->patches);
    *out = in.release();
  });
}

void ref_inputs_destroy(ref_inputs* in) { delete in; }

int ref_params(const ref_inputs* in, lg_run_params* p) {
  return guard([&] { export_params(in->cfg, p); });
}
int ref_hand_desc(const ref_inputs* in, lg_hand_desc* d) {
  return guard([&] { *d = in->hand.d; });
}
int ref_patches_desc(const ref_inputs* in, lg_patches_desc* d) {
  return guard([&] { *d = in->pflat.d; });
}
int ref_raw_samples(const ref_inputs* in, const double** s, int* n) {
  return guard([&] {
    *s = in->raw_flat.data();
    *n = static_cast<int>(in->raw.size());
  });
}
// group id per link and per patch (-1 static), number of groups.
int ref_groups(const ref_inputs* in, int* group_of_link, int* group_of_patch, int* n_groups) {
  return guard([&] {
    if (group_of_link)
      std::copy(in->group_of_link.begin(), in->group_of_link.end(), group_of_link);
    if (group_of_patch)
      std::copy(in->group_of_patch.begin(), in->group_of_patch.end(), group_of_patch);
    if (n_groups) *n_groups = static_cast<int>(in->groups.groups.size());
  });
}
int ref_link_name(const ref_inputs* in, int link, char* buf, size_t cap) {
  return guard([&] { std::snprintf(buf, cap, "%s", in->model.links.at(link).name.c_str()); });
}
// Visual mesh of a link (link-local): counts, then arrays when non-NULL.
int ref_link_visual(const ref_inputs* in, int link, int* nv, int* nt, double* verts, int* tris) {
  return guard([&] {
    const TriMesh& m = in->model.links.at(link).visual;
    *nv = static_cast<int>(m.vertices.size());
    *nt = static_cast<int>(m.triangles.size());
    if (verts)
      for (int i = 0; i < *nv; ++i) put3(verts + 3 * i, m.vertices[i]);
    if (tris)
      for (int i = 0; i < *nt; ++i)
        for (int k = 0; k < 3; ++k) tris[3 * i + k] = m.triangles[i][k];
  });
}
int ref_index_cache_key(const ref_inputs* in, uint64_t* key) {
  return guard([&] { *key = index_cache_key(in->cfg); });
}

// ---- load_hand (hand.cpp:124-273) alone: the reference's HandModel (with
// its quickhull collision parts) flattened, its visual meshes and its
// dependency groups (hand.cpp:374-411).  Used to write the caller-side hand
// fixtures (tools/prepare_hands.py).
int ref_hand_load(const char* urdf, double scale, ref_hand** out) {
  return guard([&] {
    auto h = std::make_unique<ref_hand>();
    h->model = load_hand(urdf, scale);
    h->groups = dependency_groups(h->model);
    h->flat.build(h->model);
    for (std::size_t l = 0; l < h->model.links.size(); ++l) {
      const TriMesh& m = h->model.links[l].visual;
      for (const Vec3& v : m.vertices) h->vis_verts.insert(h->vis_verts.end(), {v.x(), v.y(), v.z()});
      for (const auto& t : m.triangles) h->vis_tris.insert(h->vis_tris.end(), {t[0], t[1], t[2]});
      h->vis_vert_off.push_back(static_cast<int>(h->vis_verts.size() / 3));
      h->vis_tri_off.push_back(static_cast<int>(h->vis_tris.size() / 3));
      h->group_of_link.push_back(h->groups.group_of(static_cast<int>(l)));
    }
    *out = h.release();
  });
}
int ref_hand_desc_of(const ref_hand* h, lg_hand_desc* d) {
  return guard([&] { *d = h->flat.d; });
}
// visual meshes as CSR over links; group id per link; counts first.
int ref_hand_visual(const ref_hand* h, const int** vert_off, const double** verts, const int** tri_off,
                    const int** tris, const int** group_of_link, int* n_groups) {
  return guard([&] {
    *vert_off = h->vis_vert_off.data();
    *verts = h->vis_verts.data();
    *tri_off = h->vis_tri_off.data();
    *tris = h->vis_tris.data();
    *group_of_link = h->group_of_link.data();
    *n_groups = static_cast<int>(h->groups.groups.size());
  });
}
int ref_hand_link_name(const ref_hand* h, int link, char* buf, size_t cap) {
  return guard([&] { std::snprintf(buf, cap, "%s", h->model.links.at(link).name.c_str()); });
}
int ref_hand_joint_name(const ref_hand* h, int link, char* buf, size_t cap) {
  return guard([&] { std::snprintf(buf, cap, "%s", h->model.links.at(link).joint_name.c_str()); });
}
void ref_hand_destroy(ref_hand* h) { delete h; }

// ---- the whole forward pass: the reference's own run_batch(cfg)
int ref_run_batch(const ref_inputs* in, ref_result** out) {
  return guard([&] {
    auto r = std::make_unique<ref_result>();
    r->r = run_batch(in->cfg);
    r->grasps.resize(r->r.dataset.grasps.size());
    for (std::size_t i = 0; i < r->grasps.size(); ++i)
      export_grasp(r->r.dataset.grasps[i], -1, &r->grasps[i]);
    *out = r.release();
  });
}
long long ref_result_num_grasps(const ref_result* r) { return static_cast<long long>(r->grasps.size()); }
const lg_grasp* ref_result_grasps(const ref_result* r) { return r->grasps.data(); }
int ref_result_profile(const ref_result* r, lg_profile* p) {
  return guard([&] {
    std::memset(p, 0, sizeof(*p));
    const StageProfile& s = r->r.profile;
    p->placement_domains = s.placement_domains;
    p->contact_optimization = s.contact_optimization;
    p->kinematics_optimization = s.kinematics_optimization;
    p->postprocessing = s.postprocessing;
    p->total = s.total;
    p->candidates = s.candidates;
    p->placements_accepted = s.placements_accepted;
    p->contact_sets_balanced = s.contact_sets_balanced;
    p->ik_finite = s.ik_finite;
    p->penetration_free = s.penetration_free;
    p->ik_converged = s.ik_converged;
    p->stable = s.stable;
    p->valid = s.valid;
    p->grasps_per_second = s.grasps_per_second;
    p->patches = static_cast<long long>(r->r.index.patches);
    p->boxes = static_cast<long long>(r->r.index.boxes);
    p->index_from_cache = r->r.index.from_cache ? 1 : 0;
  });
}
// RunResult.index.memory_bytes and LoadSummary (pipeline.cpp:322-340).
int ref_result_extras(const ref_result* r, long long* index_memory_bytes, long long* hand_links,
                      long long* hand_joints, long long* hand_parts, long long* tri_read,
                      long long* tri_kept, long long* tri_dropped) {
  return guard([&] {
    *index_memory_bytes = static_cast<long long>(r->r.index.memory_bytes);
    *hand_links = r->r.loads.hand_links;
    *hand_joints = r->r.loads.hand_joints;
    *hand_parts = r->r.loads.hand_parts;
    *tri_read = static_cast<long long>(r->r.loads.object.triangles_read);
    *tri_kept = static_cast<long long>(r->r.loads.object.triangles_kept);
    *tri_dropped = static_cast<long long>(r->r.loads.object.degenerate_dropped);
  });
}
void ref_result_destroy(ref_result* r) { delete r; }

// ---- ContactFieldIndex::build on the reference inputs, exported as lg.h CSR
int ref_field_build(const ref_inputs* in, int N, ref_field** out) {
  return guard([&] {
    const RunConfig& c = in->cfg;
    auto f = std::make_unique<ref_field>();
    f->idx = ContactFieldIndex::build(in->model, in->patches, N > 0 ? N : c.field_configs,
                                      c.box_width, c.seed, c.codebook_size);
    for (const Vec3& v : f->idx.codebook) f->codebook.insert(f->codebook.end(), {v.x(), v.y(), v.z()});
    for (const PatchIndex& p : f->idx.patches) {
      f->patch_link.push_back(p.link);
      for (const IndexBox& b : p.boxes) {
        f->cells.insert(f->cells.end(), {b.cell[0], b.cell[1], b.cell[2]});
        for (std::size_t k = 0; k < b.codes.size(); ++k) {
          f->codes.push_back(b.codes[k]);
          f->rep_link.push_back(b.reps[k].link);
          f->rep_point.insert(f->rep_point.end(), {b.reps[k].point.x(), b.reps[k].point.y(), b.reps[k].point.z()});
          f->rep_normal.insert(f->rep_normal.end(),
                               {b.reps[k].normal.x(), b.reps[k].normal.y(), b.reps[k].normal.z()});
        }
        f->code_off.push_back(static_cast<long long>(f->codes.size()));
      }
      f->box_off.push_back(static_cast<int>(f->cells.size() / 3));
    }
    *out = f.release();
  });
}
int ref_field_export(const ref_field* f, lg_field_csr* o) {
  return guard([&] {
    std::memset(o, 0, sizeof(*o));
    o->box_width = f->idx.box_width;
    o->codebook_size = static_cast<int>(f->idx.codebook.size());
    o->codebook = f->codebook.data();
    o->n_patches = static_cast<int>(f->patch_link.size());
    o->patch_link = f->patch_link.data();
    o->patch_box_off = f->box_off.data();
    o->n_boxes = static_cast<long long>(f->cells.size() / 3);
    o->box_cell = f->cells.data();
    o->box_code_off = f->code_off.data();
    o->n_codes = static_cast<long long>(f->codes.size());
    o->codes = f->codes.data();
    o->rep_link = f->rep_link.data();
    o->rep_point = f->rep_point.data();
    o->rep_normal = f->rep_normal.data();
  });
}
int ref_field_save(const ref_field* f, const char* path, uint64_t key) {
  return guard([&] {
    ContactFieldIndex idx = f->idx;
    idx.cache_key = key;
    idx.save(path);
  });
}
long long ref_field_memory_bytes(const ref_field* f) {
  return static_cast<long long>(f->idx.total_memory_bytes());
}
void ref_field_destroy(ref_field* f) { delete f; }

// ---- stage functions on explicit inputs ---------------------------------

// preprocess_object (pipeline.cpp:71-98): keep[i] = 1 when sample i survives.
int ref_preprocess(const double* samples, int n, double h, double d, uint8_t* keep) {
  return guard([&] {
    auto in = unflat_samples(samples, n);
    auto kept = preprocess_object(in, h, d);
    std::size_t j = 0;
    for (int i = 0; i < n; ++i) {
      bool k = j < kept.size() && kept[j].position == in[i].position && kept[j].normal == in[i].normal;
      keep[i] = k ? 1 : 0;
      if (k) ++j;
    }
  });
}

// query_domains (contact_field.cpp:380-448) for one pose: the domains'
// elements flattened group by group.  Two-call protocol: with cap too small
// (or NULL arrays) only the counts are written.
//   n_elem[g]              elements of group g (sample order)
//   elem_pos/nrm [*][3], elem_score [*], elem_hit_off [*+1] into
//   hit_patch/hit_box [*]
int ref_query_domains(const ref_field* f, const ref_inputs* in, const double* samples, int n,
                      const double* pose12, double theta_hit, int* n_groups, int* n_elem,
                      long long* total_elems, long long* total_hits, long long cap_elems,
                      long long cap_hits, double* elem_pos, double* elem_nrm, double* elem_score,
                      long long* elem_hit_off, int* hit_patch, int* hit_box) {
  return guard([&] {
    auto s = unflat_samples(samples, n);
    auto doms = query_domains(f->idx, s, get_pose12(pose12), theta_hit, in->model, in->groups);
    *n_groups = static_cast<int>(doms.size());
    long long te = 0, th = 0;
    for (std::size_t g = 0; g < doms.size(); ++g) {
      n_elem[g] = static_cast<int>(doms[g].elements.size());
      te += n_elem[g];
      for (const auto& e : doms[g].elements) th += static_cast<long long>(e.hit_patches.size());
    }
    *total_elems = te;
    *total_hits = th;
    if (!elem_pos || te > cap_elems || th > cap_hits) return;
    long long k = 0, h = 0;
    elem_hit_off[0] = 0;
    for (const auto& d : doms)
      for (const auto& e : d.elements) {
        put3(elem_pos + 3 * k, e.position);
        put3(elem_nrm + 3 * k, e.normal);
        elem_score[k] = e.score;
        for (std::size_t i = 0; i < e.hit_patches.size(); ++i, ++h) {
          hit_patch[h] = e.hit_patches[i];
          hit_box[h] = e.hit_boxes[i];
        }
        ++k;
        elem_hit_off[k] = h;
      }
  });
}

// reverse_lookup (contact_field.cpp:450-484) for one element given by its
// hit list.
int ref_reverse_lookup(const ref_field* f, int n_hits, const int* hit_patch, const int* hit_box,
                       const double* pos, const double* nrm, uint64_t seed, int* link,
                       double* point, double* normal) {
  return guard([&] {
    DomainElement e;
    e.position = get3(pos);
    e.normal = get3(nrm);
    e.hit_patches.assign(hit_patch, hit_patch + n_hits);
    e.hit_boxes.assign(hit_box, hit_box + n_hits);
    IndexRep r = reverse_lookup(f->idx, e, seed);
    *link = r.link;
    put3(point, r.point);
    put3(normal, r.normal);
  });
}

// place_object (pipeline.cpp:122-183) for candidate seed stream c.
int ref_place(const ref_inputs* in, const double* field_samples, int n, uint64_t seed, double* pose12,
              int* accepted, double* penetration, int* n_static, double* static_p, double* static_n,
              int* static_link) {
  return guard([&] {
    auto fs = unflat_samples(field_samples, n);
    StaticSurface st = collect_static_surface(in->model, in->patches, in->groups);
    PlacementSpec spec;
    spec.mode = in->cfg.placement_mode;
    spec.canonical_center = in->cfg.canonical_center;
    spec.canonical_half_extents = in->cfg.canonical_half_extents;
    spec.static_contact_prob = in->cfg.static_contact_prob;
    spec.penetration_margin = in->cfg.penetration_margin;
    PlacementRecord pr = place_object(spec, in->model, in->patches, fs, st, seed);
    put_rigid(pose12, pose12 + 9, pr.pose);
    *accepted = pr.accepted ? 1 : 0;
    *penetration = pr.penetration;
    *n_static = static_cast<int>(pr.static_contacts.size());
    for (std::size_t i = 0; i < pr.static_contacts.size(); ++i) {
      put3(static_p + 3 * i, pr.static_contacts[i].position);
      put3(static_n + 3 * i, pr.static_contacts[i].normal);
      static_link[i] = pr.static_links[i];
    }
  });
}

// optimize_contacts (contact_opt.cpp:45-142): k domains given as element
// arrays (positions/normals/[hits ignored]), statics, params.
int ref_optimize_contacts(int k, const int* dom_n, const double* dom_pos, const double* dom_nrm,
                          int n_static, const double* static_p, const double* static_n, int n_outer,
                          int n_inner, int restarts, double sigma, double lambda_torque, double mu,
                          int iterations, int warm_iterations, double step, uint64_t seed,
                          int* element_ids, double* objective, int* anchor, double* alpha,
                          double* beta_x, double* beta_y, int* evaluations, int* valid) {
  return guard([&] {
    std::vector<ContactDomain> doms(static_cast<std::size_t>(k));
    long long off = 0;
    for (int i = 0; i < k; ++i) {
      doms[i].group = i;
      for (int e = 0; e < dom_n[i]; ++e, ++off) {
        DomainElement el;
        el.position = get3(dom_pos + 3 * off);
        el.normal = get3(dom_nrm + 3 * off);
        doms[i].elements.push_back(el);
      }
    }
    std::vector<const ContactDomain*> ptrs;
    for (auto& d : doms) ptrs.push_back(&d);
    std::vector<StaticContact> st;
    for (int i = 0; i < n_static; ++i) st.push_back({get3(static_p + 3 * i), get3(static_n + 3 * i)});
    ContactOptParams p;
    p.n_outer = n_outer;
    p.n_inner = n_inner;
    p.restarts = restarts;
    p.sigma = sigma;
    p.lambda_torque = lambda_torque;
    p.mu = mu;
    p.solve.iterations = iterations;
    p.solve.warm_iterations = warm_iterations;
    p.solve.step = step;
    ContactOptResult r = optimize_contacts(ptrs, p, st, seed);
    for (std::size_t i = 0; i < r.element_ids.size(); ++i) element_ids[i] = r.element_ids[i];
    *objective = r.objective;
    *anchor = r.solution.anchor;
    for (std::size_t i = 0; i < r.solution.alpha.size(); ++i) {
      alpha[i] = r.solution.alpha[i];
      beta_x[i] = i < r.solution.beta_x.size() ? r.solution.beta_x[i] : 0.0;
      beta_y[i] = i < r.solution.beta_y.size() ? r.solution.beta_y[i] : 0.0;
    }
    *evaluations = r.evaluations;
    *valid = r.solution.valid() ? 1 : 0;
  });
}

// solve_fswo / solve_gswo (wrench.cpp:245-258) on make_wrench_problem.
int ref_wrench_solve(int n, const double* points, const double* normals, double lambda_torque,
                     double mu, int gswo, int iterations, int warm_iterations, double step,
                     double* objective, int* anchor, double* alpha, double* beta_x, double* beta_y) {
  return guard([&] {
    std::vector<Vec3> p, nn;
    for (int i = 0; i < n; ++i) {
      p.push_back(get3(points + 3 * i));
      nn.push_back(get3(normals + 3 * i));
    }
    WrenchProblem wp = make_wrench_problem(p, nn, lambda_torque, mu);
    WrenchSolveOptions o;
    o.iterations = iterations;
    o.warm_iterations = warm_iterations;
    o.step = step;
    WrenchSolution s = gswo ? solve_gswo(wp, o) : solve_fswo(wp, o);
    *objective = s.objective;
    *anchor = s.anchor;
    for (int i = 0; i < n; ++i) {
      alpha[i] = i < static_cast<int>(s.alpha.size()) ? s.alpha[i] : 0.0;
      beta_x[i] = i < static_cast<int>(s.beta_x.size()) ? s.beta_x[i] : 0.0;
      beta_y[i] = i < static_cast<int>(s.beta_y.size()) ? s.beta_y[i] : 0.0;
    }
  });
}

// realize_grasp (pipeline.cpp:185-253) from q0 with k targets.
int ref_realize(const ref_inputs* in, const double* q0, int k, const double* obj_p, const double* obj_n,
                const int* link, const double* hand_p, const double* hand_n, double beta,
                int iterations, double step_clamp, double residual_tol, double damping_scale,
                int finetune_rounds, int finetune_iterations, double* q, double* max_residual,
                int* finite, unsigned long long* used_joints, double* realized_p,
                double* realized_n, int* realized_link, double* residuals) {
  return guard([&] {
    const int dof = in->model.actuated_count;
    Eigen::VectorXd q0v(dof);
    for (int j = 0; j < dof; ++j) q0v[j] = q0[j];
    std::vector<ContactTarget> t(static_cast<std::size_t>(k));
    for (int i = 0; i < k; ++i) {
      t[i].object_point = get3(obj_p + 3 * i);
      t[i].object_normal = get3(obj_n + 3 * i);
      t[i].link = link[i];
      t[i].hand_point_local = get3(hand_p + 3 * i);
      t[i].hand_normal_local = get3(hand_n + 3 * i);
    }
    IkParams ikp;
    ikp.beta = beta;
    ikp.iterations = iterations;
    ikp.step_clamp = step_clamp;
    ikp.residual_tol = residual_tol;
    ikp.damping_scale = damping_scale;
    RealizeResult r = realize_grasp(in->model, q0v, t, ikp, finetune_rounds, finetune_iterations);
    for (int j = 0; j < dof; ++j) q[j] = r.q[j];
    *max_residual = r.max_position_residual;
    *finite = r.finite ? 1 : 0;
    unsigned long long m = 0;
    for (std::size_t j = 0; j < r.used_joints.size(); ++j)
      if (r.used_joints[j]) m |= 1ull << j;
    *used_joints = m;
    for (std::size_t i = 0; i < r.realized.size(); ++i) {
      if (realized_p) put3(realized_p + 3 * i, r.realized[i].position);
      if (realized_n) put3(realized_n + 3 * i, r.realized[i].normal);
      if (realized_link) realized_link[i] = r.realized[i].link;
    }
    if (residuals)
      for (std::size_t i = 0; i < r.position_residuals.size(); ++i) residuals[i] = r.position_residuals[i];
  });
}

// solve_contact_ik (ik.cpp:30-139) with every IkParams field: q, finite,
// used joints, iterations, objective, per-target residuals.
int ref_contact_ik(const ref_inputs* in, const double* q0, int k, const double* obj_p,
                   const double* obj_n, const int* link, const double* hand_p, const double* hand_n,
                   double beta, int iterations, double step_clamp, double residual_tol,
                   double damping_scale, double damping_min, int max_backtracks, double* q,
                   int* finite, unsigned long long* used_joints, int* iters, double* objective,
                   double* position, double* normal_angle) {
  return guard([&] {
    const int dof = in->model.actuated_count;
    Eigen::VectorXd q0v(dof);
    for (int j = 0; j < dof; ++j) q0v[j] = q0[j];
    std::vector<ContactTarget> t(static_cast<std::size_t>(k));
    for (int i = 0; i < k; ++i) {
      t[i].object_point = get3(obj_p + 3 * i);
      t[i].object_normal = get3(obj_n + 3 * i);
      t[i].link = link[i];
      t[i].hand_point_local = get3(hand_p + 3 * i);
      t[i].hand_normal_local = get3(hand_n + 3 * i);
    }
    IkParams ikp;
    ikp.beta = beta;
    ikp.iterations = iterations;
    ikp.step_clamp = step_clamp;
    ikp.residual_tol = residual_tol;
    ikp.damping_scale = damping_scale;
    ikp.damping_min = damping_min;
    ikp.max_backtracks = max_backtracks;
    IkResult r = solve_contact_ik(in->model, q0v, t, ikp);
    for (int j = 0; j < dof; ++j) q[j] = r.q[j];
    *finite = r.finite ? 1 : 0;
    unsigned long long m = 0;
    for (std::size_t j = 0; j < r.used_joints.size(); ++j)
      if (r.used_joints[j]) m |= 1ull << j;
    *used_joints = m;
    *iters = r.iterations;
    *objective = r.objective;
    for (int i = 0; i < k; ++i) {
      position[i] = r.residuals[i].position;
      normal_angle[i] = r.residuals[i].normal_angle;
    }
  });
}

// validate_grasp_collisions (collision.cpp:230-288): the report's clean flag,
// max penetration and the violation list (link_b = -1 for the object).
int ref_collision(const ref_inputs* in, const double* q, const double* pose12, const double* samples,
                  int n, double margin, int* clean, double* max_penetration, int* n_viol, int cap,
                  int* viol_a, int* viol_b, double* viol_depth, int* broad_pairs) {
  return guard([&] {
    const int dof = in->model.actuated_count;
    Eigen::VectorXd qv(dof);
    for (int j = 0; j < dof; ++j) qv[j] = q[j];
    auto s = unflat_samples(samples, n);
    CollisionReport r = validate_grasp_collisions(in->model, qv, s, get_pose12(pose12), margin);
    *clean = r.clean() ? 1 : 0;
    *max_penetration = r.max_penetration;
    if (broad_pairs) *broad_pairs = static_cast<int>(r.broad_pairs);
    *n_viol = static_cast<int>(r.violations.size());
    for (int i = 0; i < *n_viol && i < cap; ++i) {
      const CollisionViolation& v = r.violations[i];
      viol_a[i] = v.link_a;
      viol_b[i] = v.link_b;
      viol_depth[i] = v.depth;
    }
  });
}

}  // extern "C"
