// oracle/orc_pipeline.cpp — pipeline.cpp of the reference restated for the
// CPU parity oracle: preprocess_object, statics, place_object,
// realize_grasp and the four-stage run_batch loop with its thread pool.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "orc.hpp"

namespace orc {

using namespace lgm;

namespace {
constexpr uint64_t kTagPlacement = 0x706c6163;   // pipeline.cpp:21
constexpr uint64_t kTagGroups = 0x67727073;      // pipeline.cpp:22
constexpr uint64_t kTagContactOpt = 0x636f7074;  // pipeline.cpp:23
constexpr uint64_t kTagReverse = 0x72657673;     // pipeline.cpp:24
constexpr uint64_t kTagUnused = 0x756e7573;      // pipeline.cpp:25

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

struct Statics {  // pipeline.hpp:84-89
  std::vector<Sample> samples;
  std::vector<int> sample_links;
  std::vector<std::pair<int, int>> parts;  // (part, link)
  std::vector<Xf> part_pose;
};

struct Placement {  // pipeline.hpp:91-97
  Xf pose = xf_identity();
  std::vector<StaticContact> statics;
  std::vector<int> static_links;
  bool accepted = false;
  double penetration = 0.0;
};

Statics collect_static_surface(const Hand& h, const std::vector<Patch>& patches,
                               const Groups& g) {  // pipeline.cpp:100-120
  Statics out;
  auto mid = h.mid_config();
  auto frames = forward_kinematics(h, mid.data());
  for (int link : g.static_links)
    for (int p : h.links[link].parts) {
      out.parts.push_back({p, link});
      out.part_pose.push_back(frames[link]);
    }
  for (const Patch& P : patches) {
    if (g.group_of(P.link) != -1) continue;
    const Xf& f = frames[P.link];
    for (size_t i = 0; i < P.points.size(); ++i) {
      out.samples.push_back({xf_apply(f, P.points[i]), xf_rotate(f, P.normals[i])});
      out.sample_links.push_back(P.link);
    }
  }
  return out;
}

Placement place_object(const lg_run_params& cfg, const Hand& h, const std::vector<Patch>& patches,
                       const std::vector<Sample>& obj, const Statics& st,
                       uint64_t seed) {  // pipeline.cpp:122-183
  if (obj.empty()) throw std::invalid_argument("place_object: no object samples");
  Rng rng(seed);
  Placement rec;
  bool want_static = rng.uniform() < cfg.static_contact_prob;
  const Sample& os = obj[rng.uniform_index(obj.size())];
  if (want_static && !st.samples.empty()) {
    size_t si = rng.uniform_index(st.samples.size());
    const Sample& ss = st.samples[si];
    double roll = rng.uniform(0.0, 2.0 * kPi);
    M3 r = mul(angle_axis(roll, ss.n), rotation_between(os.n, neg(ss.n)));
    rec.pose.R = r;
    rec.pose.t = sub(ss.p, mul(r, os.p));
    rec.statics.push_back({ss.p, ss.n});
    rec.static_links.push_back(st.sample_links[si]);
  } else if (cfg.placement_mode == 0) {
    if (patches.empty()) throw std::invalid_argument("place_object: no patches");
    const Patch& P = patches[rng.uniform_index(patches.size())];
    int fp = P.field_points[rng.uniform_index(P.field_points.size())];
    std::vector<double> q(h.dof, 0.0);
    std::vector<std::pair<double, double>> lims(h.dof, {0.0, 0.0});
    for (const Link& l : h.links)
      if (l.jidx >= 0) lims[l.jidx] = {l.lo, l.hi};
    for (int j = 0; j < h.dof; ++j) q[j] = rng.uniform(lims[j].first, lims[j].second);
    auto frames = forward_kinematics(h, q.data());
    V3 x = xf_apply(frames[P.link], P.points[fp]);
    V3 m = xf_rotate(frames[P.link], P.normals[fp]);
    double roll = rng.uniform(0.0, 2.0 * kPi);
    M3 r = mul(angle_axis(roll, m), rotation_between(os.n, neg(m)));
    rec.pose.R = r;
    rec.pose.t = sub(x, mul(r, os.p));
  } else {
    double t[3] = {cfg.canonical_center[0], cfg.canonical_center[1], cfg.canonical_center[2]};
    for (int a = 0; a < 3; ++a)
      t[a] += rng.uniform(-cfg.canonical_half_extents[a], cfg.canonical_half_extents[a]);
    double w, x, y, z;
    rng.uniform_quaternion(&w, &x, &y, &z);
    rec.pose.R = quat_to_matrix(w, x, y, z);
    rec.pose.t = v3(t[0], t[1], t[2]);
  }
  auto world = transform_samples(obj, rec.pose);
  for (size_t i = 0; i < st.parts.size(); ++i) {
    auto pen = object_penetration(world, h.parts[st.parts[i].first], st.part_pose[i],
                                  cfg.penetration_margin);
    rec.penetration = dmax(rec.penetration, pen.max_depth);
  }
  rec.accepted = rec.penetration <= cfg.penetration_margin;
  return rec;
}

}  // namespace

double closest_on_parts(const Hand& h, int link, V3 p, V3* sp, V3* sn) {  // pipeline.cpp:55-69
  double best = kInf;
  for (int pi : h.links[link].parts) {
    V3 n;
    V3 cp = h.parts[pi].closest_surface_point(p, &n);
    double d = norm(sub(p, cp));
    if (d < best) {
      best = d;
      if (sp) *sp = cp;
      if (sn) *sn = n;
    }
  }
  return best;
}

std::vector<Sample> preprocess_object(const std::vector<Sample>& s, double hw,
                                      double dt) {  // pipeline.cpp:71-98
  if (hw <= 0.0 || dt < 0.0)
    throw std::invalid_argument("preprocess_object: bad probe dimensions");
  std::vector<Sample> kept;
  for (size_t i = 0; i < s.size(); ++i) {
    V3 c = axpy(s[i].p, dt, s[i].n);
    bool blocked = false;
    for (size_t j = 0; j < s.size() && !blocked; ++j) {
      if (j == i) continue;
      V3 d = sub(s[j].p, c);
      if (std::abs(d.x) > hw || std::abs(d.y) > hw || std::abs(d.z) > hw) continue;
      if (dot(s[j].n, s[i].n) < 0.0) blocked = true;
    }
    if (!blocked) kept.push_back(s[i]);
  }
  return kept;
}

RealizeResult realize_grasp(const Hand& h, const std::vector<double>& q0,
                            const std::vector<ContactTarget>& targets, const IkParams& params,
                            int rounds, int fine_iters) {  // pipeline.cpp:185-253
  RealizeResult rr;
  rr.q = q0;
  rr.used.assign(h.dof, false);
  if (targets.empty()) throw std::invalid_argument("realize_grasp: no targets");
  auto project = [&](const std::vector<double>& q, std::vector<ContactTarget>* refreshed,
                     RealizeResult* realized) {
    auto frames = forward_kinematics(h, q.data());
    double worst = 0.0;
    for (size_t i = 0; i < targets.size(); ++i) {
      const ContactTarget& t = targets[i];
      Xf inv = xf_inverse(frames[t.link]);
      V3 sp = v3(0, 0, 0), sn = v3(0, 0, 0);
      double d = closest_on_parts(h, t.link, xf_apply(inv, t.object_point), &sp, &sn);
      worst = dmax(worst, d);
      if (refreshed) {
        (*refreshed)[i].hand_point = sp;
        (*refreshed)[i].hand_normal = sn;
      }
      if (realized) {
        realized->real_p.push_back(xf_apply(frames[t.link], sp));
        realized->real_n.push_back(xf_rotate(frames[t.link], sn));
        realized->real_link.push_back(t.link);
        realized->residuals.push_back(d);
      }
    }
    return worst;
  };
  IkResult ik = solve_contact_ik(h, q0, targets, params);
  if (!ik.finite) {
    rr.finite = false;
    rr.max_residual = kInf;
    return rr;
  }
  std::vector<double> q = ik.q;
  rr.used = ik.used;
  double worst = project(q, nullptr, nullptr);
  IkParams fine = params;
  fine.iterations = fine_iters;
  for (int round = 0; round < rounds; ++round) {
    std::vector<ContactTarget> refreshed = targets;
    project(q, &refreshed, nullptr);
    IkResult step = solve_contact_ik(h, q, refreshed, fine);
    if (!step.finite) break;
    double w2 = project(step.q, nullptr, nullptr);
    if (w2 > worst + 1e-6) break;
    q = step.q;
    worst = w2;
    for (size_t j = 0; j < rr.used.size(); ++j)
      if (step.used[j]) rr.used[j] = true;
  }
  rr.q = q;
  rr.max_residual = project(q, nullptr, &rr);
  rr.finite = true;
  for (double v : q)
    if (!std::isfinite(v)) rr.finite = false;
  return rr;
}

namespace {

struct Slot {  // pipeline.cpp:257-269
  const Placement* place = nullptr;
  const std::vector<Domain>* domains = nullptr;
  std::vector<int> chosen;
  ContactOptResult opt;
  std::vector<ContactTarget> targets;
  RealizeResult real;
  lg_grasp grasp;
  bool alive = false;
  bool valid = false;
  lg_trace* tr = nullptr;
};

void v3out(double* d, V3 v) {
  d[0] = v.x;
  d[1] = v.y;
  d[2] = v.z;
}

}  // namespace

RunOutput run_batch(const Hand& h, const std::vector<Patch>& patches,
                    const std::vector<Sample>& raw, const lg_run_params& cfg, int workers,
                    const FieldIndex* cached) {  // pipeline.cpp:308-625
  auto wall0 = Clock::now();
  RunOutput out;
  std::memset(&out.profile, 0, sizeof(out.profile));
  // build_field (pipeline.cpp:273-306): build, or reuse a cached index
  FieldIndex built;
  if (!cached)
    built = build_field_index(h, patches, cfg.field_configs, cfg.box_width, cfg.seed,
                              cfg.codebook_size);
  const FieldIndex& index = cached ? *cached : built;
  out.profile.field_build = since(wall0);
  auto field = preprocess_object(raw, cfg.probe_half_width, cfg.probe_depth_threshold);
  if (field.empty())
    throw std::runtime_error("run_batch: preprocessing stripped every object sample");
  out.profile.patches = (long long)index.patches.size();
  for (const auto& p : index.patches) out.profile.boxes += (long long)p.boxes.size();
  out.profile.field_vectors = index.n_vectors;
  out.profile.object_samples = (long long)raw.size();
  out.profile.field_samples = (long long)field.size();

  Groups groups = dependency_groups(h);
  Statics statics = collect_static_surface(h, patches, groups);
  std::vector<std::pair<double, double>> lims(h.dof, {0.0, 0.0});
  for (const Link& l : h.links)
    if (l.jidx >= 0) lims[l.jidx] = {l.lo, l.hi};

  ContactOptParams copt;
  copt.n_outer = cfg.n_outer;
  copt.n_inner = cfg.n_inner;
  copt.restarts = cfg.restarts;
  copt.sigma = cfg.sigma;
  copt.lambda = cfg.lambda_torque;
  copt.mu = cfg.mu;
  copt.solve.iterations = cfg.pgd_iterations;
  copt.solve.warm_iterations = cfg.pgd_warm_iterations;
  copt.solve.step = cfg.pgd_step;
  IkParams ikp;
  ikp.beta = cfg.beta;
  ikp.iterations = cfg.ik_iterations;
  ikp.step_clamp = cfg.step_clamp;
  ikp.residual_tol = cfg.residual_tol;
  ikp.damping_scale = cfg.damping_scale;

  const std::vector<double> q_start = h.mid_config();
  const int B = cfg.batch;
  int c_lo = 0, c_hi = B;
  if (cfg.shard_count > 1) {
    c_lo = (int)((long long)cfg.shard_rank * B / cfg.shard_count);
    c_hi = (int)((long long)(cfg.shard_rank + 1) * B / cfg.shard_count);
  }
  std::vector<Placement> places(B);
  std::vector<std::vector<Domain>> doms(B);
  const int chunk = 64;
  const int G = (int)groups.groups.size();
  const int k = cfg.k_contacts;

  for (int pass = 0; pass < cfg.passes; ++pass) {
    for (int cs = c_lo; cs < c_hi; cs += chunk) {
      int nc = std::min(chunk, c_hi - cs);
      std::vector<Slot> slots(nc);
      std::vector<lg_trace> traces(cfg.want_trace ? nc : 0);
      for (int i = 0; i < nc; ++i) {
        std::memset(&slots[i].grasp, 0, sizeof(lg_grasp));
        if (cfg.want_trace) {
          std::memset(&traces[i], 0, sizeof(lg_trace));
          slots[i].tr = &traces[i];
        }
      }
      auto t = Clock::now();
      parallel_for(0, nc, workers, [&](size_t i) {  // stage 1, pipeline.cpp:391-439
        Slot& s = slots[i];
        int c = cs + (int)i;
        uint64_t g = (uint64_t)pass * B + c;
        if (pass == 0) {
          places[c] = place_object(cfg, h, patches, field, statics,
                                   mix_seed(cfg.seed, kTagPlacement, c));
          if (places[c].accepted)
            doms[c] = query_domains(index, field, places[c].pose, cfg.theta_hit, h, groups);
        }
        s.place = &places[c];
        s.domains = &doms[c];
        if (s.tr) {
          lg_trace& tr = *s.tr;
          tr.g = (long long)g;
          tr.pass = pass;
          tr.c = c;
          tr.accepted = s.place->accepted;
          tr.penetration = s.place->penetration;
          m3_store(tr.pose_R, s.place->pose.R);
          v3out(tr.pose_t, s.place->pose.t);
          tr.n_static = (int)s.place->statics.size();
          tr.static_link = s.place->static_links.empty() ? -1 : s.place->static_links[0];
          if (!s.place->statics.empty()) {
            v3out(tr.static_p, s.place->statics[0].position);
            v3out(tr.static_n, s.place->statics[0].normal);
          }
          tr.n_groups = G;
          for (int gi = 0; gi < G && gi < LG_MAX_GROUPS && gi < (int)s.domains->size(); ++gi)
            tr.domain_size[gi] = (int)(*s.domains)[gi].elements.size();
        }
        s.alive = s.place->accepted;
        if (!s.alive) return;
        std::vector<int> nonempty;
        for (size_t di = 0; di < s.domains->size(); ++di)
          if (!(*s.domains)[di].elements.empty()) nonempty.push_back((int)di);
        if ((int)nonempty.size() < k) {
          s.alive = false;
          return;
        }
        Rng gr(mix_seed(cfg.seed, kTagGroups, g));
        for (int pick = 0; pick < k; ++pick) {
          size_t j = pick + gr.uniform_index(nonempty.size() - pick);
          std::swap(nonempty[pick], nonempty[j]);
        }
        s.chosen.assign(nonempty.begin(), nonempty.begin() + k);
        if (s.tr) {
          s.tr->picked = 1;
          for (int q = 0; q < k; ++q) s.tr->chosen[q] = s.chosen[q];
        }
      });
      out.profile.placement_domains += since(t);
      for (auto& s : slots) out.profile.placements_accepted += s.alive ? 1 : 0;

      t = Clock::now();
      parallel_for(0, nc, workers, [&](size_t i) {  // stage 2, pipeline.cpp:444-458
        Slot& s = slots[i];
        if (!s.alive) return;
        uint64_t g = (uint64_t)pass * B + cs + i;
        std::vector<const Domain*> picked;
        for (int di : s.chosen) picked.push_back(&(*s.domains)[di]);
        s.opt = optimize_contacts(picked, copt, s.place->statics,
                                  mix_seed(cfg.seed, kTagContactOpt, g));
        if (!s.opt.solution.valid() || s.opt.objective >= cfg.eps_stable) s.alive = false;
        if (s.tr) {
          lg_trace& tr = *s.tr;
          for (int q = 0; q < k; ++q) {
            tr.opt_element[q] = s.opt.element_ids[q];
            tr.opt_sample[q] = s.opt.elements[q].sample;
          }
          tr.opt_objective = s.opt.objective;
          tr.opt_anchor = s.opt.solution.anchor;
          tr.opt_evaluations = s.opt.evaluations;
          for (size_t q = 0; q < s.opt.solution.alpha.size() && q < LG_MAX_CONTACTS; ++q) {
            tr.opt_alpha[q] = s.opt.solution.alpha[q];
            tr.opt_bx[q] = s.opt.solution.bx[q];
            tr.opt_by[q] = s.opt.solution.by[q];
          }
          tr.balanced = s.alive;
        }
      });
      out.profile.contact_optimization += since(t);
      for (auto& s : slots) out.profile.contact_sets_balanced += s.alive ? 1 : 0;

      t = Clock::now();
      parallel_for(0, nc, workers, [&](size_t i) {  // stage 3, pipeline.cpp:465-523
        Slot& s = slots[i];
        if (!s.alive) return;
        uint64_t g = (uint64_t)pass * B + cs + i;
        bool have = false, best_clear = false;
        int attempts_run = 0, best_attempt = -1;
        for (int attempt = 0; attempt < cfg.lookup_attempts; ++attempt) {
          ++attempts_run;
          std::vector<ContactTarget> targets;
          for (size_t slot = 0; slot < s.opt.elements.size(); ++slot) {
            const DomainElement& el = s.opt.elements[slot];
            IndexRep rep = reverse_lookup(
                index, el,
                mix_seed(cfg.seed, kTagReverse, (g << 6) + ((uint64_t)attempt << 3) + slot));
            ContactTarget tg;
            tg.object_point = el.position;
            tg.object_normal = neg(el.normal);
            tg.link = rep.link;
            tg.hand_point = rep.point;
            tg.hand_normal = rep.normal;
            targets.push_back(tg);
          }
          RealizeResult real = realize_grasp(h, q_start, targets, ikp, cfg.finetune_rounds,
                                             cfg.finetune_iterations);
          if (!real.finite) continue;
          bool conv = real.max_residual <= cfg.contact_tol;
          bool clear = false;
          if (conv)
            clear = validate_grasp_collisions(h, real.q.data(), raw, s.place->pose,
                                              cfg.penetration_margin)
                        .clean();
          bool better;
          if (!have) better = true;
          else if (clear != best_clear) better = clear;
          else better = real.max_residual < s.real.max_residual;
          if (better) {
            s.real = real;
            s.targets = targets;
            best_clear = clear;
            have = true;
            best_attempt = attempt;
          }
          if (best_clear) break;
        }
        if (!have) s.alive = false;
        if (s.tr) {
          lg_trace& tr = *s.tr;
          tr.realized = have;
          tr.attempts_run = attempts_run;
          tr.best_attempt = best_attempt;
          tr.best_clear = best_clear;
          if (have) {
            tr.max_residual = s.real.max_residual;
            for (int j = 0; j < h.dof && j < LG_MAX_DOF; ++j) tr.real_q[j] = s.real.q[j];
            unsigned long long m = 0;
            for (int j = 0; j < h.dof && j < 64; ++j)
              if (s.real.used[j]) m |= 1ull << j;
            tr.used_joints = m;
            for (size_t q = 0; q < s.targets.size() && q < LG_MAX_K; ++q) {
              tr.target_link[q] = s.targets[q].link;
              v3out(tr.target_point[q], s.targets[q].hand_point);
              v3out(tr.target_normal[q], s.targets[q].hand_normal);
            }
          }
        }
      });
      out.profile.kinematics_optimization += since(t);
      for (auto& s : slots) out.profile.ik_finite += s.alive ? 1 : 0;

      t = Clock::now();
      parallel_for(0, nc, workers, [&](size_t i) {  // stage 4, pipeline.cpp:528-604
        Slot& s = slots[i];
        if (!s.alive) return;
        uint64_t g = (uint64_t)pass * B + cs + i;
        Rng ur(mix_seed(cfg.seed, kTagUnused, g));
        std::vector<double> q;
        CollisionReport report;
        int used_attempt = -1;
        for (int attempt = 0; attempt < cfg.unused_attempts; ++attempt) {
          q = s.real.q;
          for (int j = 0; j < h.dof; ++j) {
            if (j < (int)s.real.used.size() && s.real.used[j]) continue;
            q[j] = ur.uniform(lims[j].first, lims[j].second);
          }
          report = validate_grasp_collisions(h, q.data(), raw, s.place->pose,
                                             cfg.penetration_margin);
          used_attempt = attempt;
          if (report.clean()) break;
        }
        if (s.tr) {
          s.tr->unused_attempt = used_attempt;
          for (int j = 0; j < h.dof && j < LG_MAX_DOF; ++j) s.tr->final_q[j] = q[j];
        }
        auto frames = forward_kinematics(h, q.data());
        auto world_field = transform_samples(field, s.place->pose);
        double worst = 0.0;
        lg_grasp& gr = s.grasp;
        gr.n_contacts = 0;
        for (const auto& tg : s.targets) {
          Xf inv = xf_inverse(frames[tg.link]);
          V3 sp = v3(0, 0, 0), sn = v3(0, 0, 0);
          double d = closest_on_parts(h, tg.link, xf_apply(inv, tg.object_point), &sp, &sn);
          if (!std::isfinite(d)) {
            if (s.tr) s.tr->dropped = 1;
            return;
          }
          worst = dmax(worst, d);
          V3 pw = xf_apply(frames[tg.link], sp);
          size_t nearest = 0;
          double best_d2 = kInf;
          for (size_t fi = 0; fi < world_field.size(); ++fi) {
            double d2 = sqnorm(sub(world_field[fi].p, pw));
            if (d2 < best_d2) {
              best_d2 = d2;
              nearest = fi;
            }
          }
          int ci = gr.n_contacts++;
          v3out(gr.contact_p[ci], pw);
          v3out(gr.contact_n[ci], neg(world_field[nearest].n));
          gr.contact_link[ci] = tg.link;
        }
        for (size_t si = 0; si < s.place->statics.size(); ++si) {
          int ci = gr.n_contacts++;
          v3out(gr.contact_p[ci], s.place->statics[si].position);
          v3out(gr.contact_n[ci], s.place->statics[si].normal);
          gr.contact_link[ci] = s.place->static_links[si];
        }
        gr.ik_converged = worst <= cfg.contact_tol;
        gr.penetration_free = report.clean();
        std::vector<V3> pts, nrms;
        for (int ci = 0; ci < gr.n_contacts; ++ci) {
          pts.push_back(v3_load(gr.contact_p[ci]));
          nrms.push_back(v3_load(gr.contact_n[ci]));
        }
        WrenchProblem wp = make_wrench_problem(pts, nrms, cfg.lambda_torque, cfg.mu);
        WrenchSolution sol;
        gr.stable = is_stable(wp, cfg.eps_stable, &sol, copt.solve);
        gr.g = (long long)g;
        m3_store(gr.pose_R, s.place->pose.R);
        v3out(gr.pose_t, s.place->pose.t);
        gr.dof = h.dof;
        for (int j = 0; j < h.dof && j < LG_MAX_DOF; ++j) gr.q[j] = q[j];
        gr.objective = sol.objective;
        s.valid = gr.penetration_free && gr.stable && gr.ik_converged;
      });
      out.profile.postprocessing += since(t);
      for (auto& s : slots) {
        if (s.alive) {
          out.profile.penetration_free += s.grasp.penetration_free ? 1 : 0;
          out.profile.ik_converged += s.grasp.ik_converged ? 1 : 0;
          out.profile.stable += s.grasp.stable ? 1 : 0;
        }
        if (s.tr) {
          s.tr->penetration_free = s.grasp.penetration_free;
          s.tr->ik_converged = s.grasp.ik_converged;
          s.tr->stable = s.grasp.stable;
          s.tr->valid = s.valid;
          s.tr->objective = s.grasp.objective;
        }
        if (s.valid) out.grasps.push_back(s.grasp);
      }
      for (auto& tr : traces) out.traces.push_back(tr);
    }
  }
  out.profile.candidates = (long long)cfg.passes * (c_hi - c_lo);
  out.profile.valid = (long long)out.grasps.size();
  out.profile.total = since(wall0);
  out.profile.grasps_per_second =
      out.profile.total > 0.0 ? out.profile.valid / out.profile.total : 0.0;
  return out;
}

}  // namespace orc
