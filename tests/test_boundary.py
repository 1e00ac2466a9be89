"""The stage-level C-ABI entry points against the reference's
own functions (oracle/_ref) on identical inputs, bit for bit:

  lg_query_domains_elements  <-> query_domains      (contact_field.cpp:380-448)
  lg_reverse_lookup_batch    <-> reverse_lookup     (contact_field.cpp:450-484)
  lg_place_batch             <-> place_object       (pipeline.cpp:122-183)
  lg_optimize_contacts_batch <-> optimize_contacts  (contact_opt.cpp:45-142)
  lg_realize_batch + lg_realized_contacts_batch <-> realize_grasp (pipeline.cpp:185-253)
  lg_collision_report_batch  <-> validate_grasp_collisions (collision.cpp:230-288)
"""
import os
import types

import numpy as np
import pytest

from conftest import ASSETS
from oracle import ref_py as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]

TAG_PLAC, TAG_COPT, TAG_REVS = 0x706C6163, 0x636F7074, 0x72657673


def mix_seed(seed, a, b=0):
    import caller
    return caller.mix_seed(seed, a, b)


@pytest.fixture(scope="module", params=[
    ("four_finger.cfg", "four_finger.urdf", "sphere_r030.obj"),
    ("allegro.cfg", "allegro_like.urdf", "box_050.obj"),
], ids=["four_finger", "allegro"])
def setup(request, ctx):
    import paper_2511_07418_b200 as lg
    cfg, hand, obj = request.param
    inp = R.RefInputs(config=os.path.join(ASSETS, "configs", cfg),
                      extra="field_configs = 128\n",
                      hand=os.path.join(ASSETS, "hands", hand),
                      object=os.path.join(ASSETS, "objects", obj), batch=32, workers=8)
    H = types.SimpleNamespace(desc=inp.hand_desc, dof=inp.hand_desc.dof)
    Pt = types.SimpleNamespace(desc=inp.patches_desc)
    dev_field = lg.ContactFieldIndex.build(ctx, H, Pt, inp.params.field_configs,
                                           inp.params.box_width, inp.params.seed,
                                           inp.params.codebook_size)
    ref_field = inp.field()
    keep = R.preprocess(inp.raw, inp.params.probe_half_width, inp.params.probe_depth_threshold)
    fs = inp.raw[keep.astype(bool)]
    return types.SimpleNamespace(inp=inp, H=H, Pt=Pt, dev_field=dev_field, ref_field=ref_field,
                                 fs=fs, p=inp.params)


def _placements(s, ctx, c0=0, m=24):
    import paper_2511_07418_b200 as lg
    return lg.api.place_batch(ctx, s.H, s.Pt, s.inp.raw, s.p, c0, m, field=s.dev_field)


def test_place_batch_matches_reference(setup, ctx):
    s = setup
    dev = _placements(s, ctx, 3, 24)
    for t in range(24):
        ref = R.place(s.inp, s.fs, mix_seed(s.p.seed, TAG_PLAC, 3 + t))
        assert dev["pose"][t].tobytes() == ref["pose"].tobytes(), t
        assert dev["accepted"][t] == ref["accepted"]
        assert dev["penetration"][t] == ref["penetration"]
        assert dev["n_static"][t] == len(ref["static_p"])
        if len(ref["static_p"]):
            assert dev["static_p"][t].tobytes() == ref["static_p"][0].tobytes()
            assert dev["static_n"][t].tobytes() == ref["static_n"][0].tobytes()
            assert dev["static_link"][t] == ref["static_link"][0]


def _domains(s, ctx, pose):
    import paper_2511_07418_b200 as lg
    dev = lg.api.query_domains_elements(ctx, s.dev_field, s.inp.group_of_patch, s.inp.n_groups,
                                        s.fs, pose, s.p.theta_hit)
    ref = s.ref_field.query(s.fs, pose, s.p.theta_hit)
    return dev, ref


def test_query_domains_elements_match_reference(setup, ctx):
    s = setup
    pl = _placements(s, ctx, 0, 12)
    checked = 0
    for t in np.flatnonzero(pl["accepted"])[:6]:
        dev, ref = _domains(s, ctx, pl["pose"][t])
        assert len(dev) == len(ref)
        for g in range(len(ref)):
            assert len(dev[g]) == len(ref[g]), (t, g)
            for a, b in zip(dev[g], ref[g]):
                assert a["pos"].tobytes() == b["pos"].tobytes()
                assert a["nrm"].tobytes() == b["nrm"].tobytes()
                assert a["score"] == b["score"]
                assert a["hits"] == b["hits"]
                checked += 1
    assert checked > 100


def test_reverse_lookup_matches_reference(setup, ctx):
    import paper_2511_07418_b200 as lg
    s = setup
    pl = _placements(s, ctx, 0, 8)
    t = int(np.flatnonzero(pl["accepted"])[0])
    _, ref_doms = _domains(s, ctx, pl["pose"][t])
    els = [e for d in ref_doms for e in d][:400]
    seeds = [mix_seed(s.p.seed, TAG_REVS, (i << 6) + 3) for i in range(len(els))]
    link, pt, nn = lg.api.reverse_lookup_batch(ctx, s.dev_field, els, seeds)
    for i, e in enumerate(els):
        rl, rp, rn = s.ref_field.reverse_lookup(e, seeds[i])
        assert link[i] == rl and pt[i].tobytes() == rp.tobytes() and nn[i].tobytes() == rn.tobytes()
    bad = dict(els[0])
    bad["hits"] = []
    with pytest.raises(IndexError, match="no hits"):
        lg.api.reverse_lookup_batch(ctx, s.dev_field, [bad], [1])


def test_optimize_contacts_matches_reference(setup, ctx):
    import paper_2511_07418_b200 as lg
    s = setup
    k = s.p.k_contacts
    pl = _placements(s, ctx, 0, 16)
    problems, seeds, refs = [], [], []
    for t in np.flatnonzero(pl["accepted"]):
        _, doms = _domains(s, ctx, pl["pose"][t])
        nonempty = [d for d in doms if d]
        if len(nonempty) < k:
            continue
        dd = [(np.array([e["pos"] for e in d]), np.array([e["nrm"] for e in d]))
              for d in nonempty[:k]]
        st = [(pl["static_p"][t], pl["static_n"][t])] if pl["n_static"][t] else []
        sd = mix_seed(s.p.seed, TAG_COPT, int(t))
        problems.append((dd, st))
        seeds.append(sd)
        refs.append(R.optimize_contacts(dd, st, n_outer=s.p.n_outer, n_inner=s.p.n_inner,
                                        restarts=s.p.restarts, sigma=s.p.sigma,
                                        lambda_torque=s.p.lambda_torque, mu=s.p.mu,
                                        iterations=s.p.pgd_iterations,
                                        warm_iterations=s.p.pgd_warm_iterations,
                                        step=s.p.pgd_step, seed=sd))
        if len(problems) == 6:
            break
    assert problems
    dev = lg.api.optimize_contacts_batch(ctx, problems, s.p, seeds)
    for i, ref in enumerate(refs):
        n = k + len(problems[i][1])
        assert dev["element_ids"][i].tolist() == ref["element_ids"].tolist()
        assert dev["objective"][i] == ref["objective"]
        assert dev["anchor"][i] == ref["anchor"]
        for f in ("alpha", "beta_x", "beta_y"):
            assert dev[f][i][:n].tobytes() == ref[f][:n].tobytes(), f
        assert dev["evaluations"][i] == ref["evaluations"]


def test_realize_and_realized_contacts_match_reference(setup, ctx):
    import paper_2511_07418_b200 as lg
    s = setup
    pl = _placements(s, ctx, 0, 8)
    t = int(np.flatnonzero(pl["accepted"])[0])
    _, doms = _domains(s, ctx, pl["pose"][t])
    els = [d[len(d) // 2] for d in doms if d][:2]
    targets = []
    for j, e in enumerate(els):
        l, hp, hn = s.ref_field.reverse_lookup(e, 11 + j)
        targets.append((e["pos"], -e["nrm"], l, hp, hn))
    q0 = np.zeros(s.inp.hand_desc.dof)
    d = s.inp.hand_desc
    for l in range(d.n_links):
        if d.joint_index[l] >= 0:
            q0[d.joint_index[l]] = 0.5 * (d.limit_lo[l] + d.limit_hi[l])
    kw = dict(beta=s.p.beta, iterations=s.p.ik_iterations, step_clamp=s.p.step_clamp,
              residual_tol=s.p.residual_tol, damping_scale=s.p.damping_scale,
              finetune_rounds=s.p.finetune_rounds, finetune_iterations=s.p.finetune_iterations)
    ref = R.realize(s.inp, q0, targets, **kw)
    q, mr, fin, used = lg.api.realize_batch(ctx, s.H, q0[None], [targets], **kw)
    assert q[0].tobytes() == ref["q"].tobytes() and mr[0] == ref["max_residual"]
    rp, rn, rl, rs = lg.api.realized_contacts_batch(ctx, s.H, q, [[(tg[2], tg[0]) for tg in targets]])
    assert rp.tobytes() == ref["realized_p"].tobytes()
    assert rn.tobytes() == ref["realized_n"].tobytes()
    assert rl.tolist() == ref["realized_link"].tolist()
    assert rs.tobytes() == ref["residuals"].tobytes()


def test_collision_report_matches_reference(setup, ctx):
    import paper_2511_07418_b200 as lg
    s = setup
    pl = _placements(s, ctx, 0, 16)
    d = s.inp.hand_desc
    lo = np.zeros(d.dof)
    hi = np.zeros(d.dof)
    for l in range(d.n_links):
        j = d.joint_index[l]
        if j >= 0:
            lo[j], hi[j] = d.limit_lo[l], d.limit_hi[l]
    rng = np.random.default_rng(4)
    q = rng.uniform(lo, hi, size=(16, d.dof))
    dev = lg.api.collision_report_batch(ctx, s.H, q, pl["pose"], s.inp.raw, s.p.penetration_margin)
    dirty = 0
    for i in range(16):
        ref = R.collision(s.inp, q[i], pl["pose"][i], s.inp.raw, s.p.penetration_margin)
        assert dev[i]["n_violations"] == ref["n_violations"], i
        assert dev[i]["violations"] == ref["violations"], i
        assert dev[i]["max_penetration"] == ref["max_penetration"]
        assert dev[i]["broad_pairs"] == ref["broad_pairs"]
        dirty += ref["n_violations"] > 0
    assert dirty > 0


def test_collision_batch_grid_path_matches_reference(ctx):
    """lg_collision_batch on >= 20k object samples (the object-sample grid
    path of k_collision3) == validate_grasp_collisions' clean() and
    max_penetration, on placements of the Allegro-class hand around a dense
    icosphere and random joint values (many of them penetrating)."""
    import paper_2511_07418_b200 as lg
    inp = R.RefInputs(config=os.path.join(ASSETS, "configs", "allegro.cfg"),
                      extra="samples_per_cm2 = 250\nfield_configs = 64\n",
                      hand=os.path.join(ASSETS, "hands", "allegro_like.urdf"),
                      object=os.path.join(ASSETS, "objects", "icosphere_r030_s6.obj"),
                      batch=24, workers=8)
    assert len(inp.raw) >= 20000
    H = types.SimpleNamespace(desc=inp.hand_desc, dof=inp.hand_desc.dof)
    Pt = types.SimpleNamespace(desc=inp.patches_desc)
    pl = lg.api.place_batch(ctx, H, Pt, inp.raw, inp.params, 0, 24)
    d = inp.hand_desc
    lo, hi = np.zeros(d.dof), np.zeros(d.dof)
    for l in range(d.n_links):
        j = d.joint_index[l]
        if j >= 0:
            lo[j], hi[j] = d.limit_lo[l], d.limit_hi[l]
    q = np.random.default_rng(9).uniform(lo, hi, size=(24, d.dof))
    clean, depth = lg.api.collision_batch(ctx, H, q, pl["pose"], inp.raw, inp.params.penetration_margin)
    dirty = 0
    for i in range(24):
        ref = R.collision(inp, q[i], pl["pose"][i], inp.raw, inp.params.penetration_margin)
        assert bool(clean[i]) == (ref["n_violations"] == 0), i
        assert depth[i] == ref["max_penetration"], i
        dirty += ref["n_violations"] > 0
    assert dirty > 0


def test_contact_ik_matches_reference(setup, ctx):
    """lg_contact_ik_batch == solve_contact_ik (ik.cpp:30-139): q, finite,
    used joints, iterations, objective and residuals, bit for bit, from
    mid-range and random starts, with default and tightened IkParams."""
    import math
    import paper_2511_07418_b200 as lg
    s = setup
    pl = _placements(s, ctx, 0, 8)
    t = int(np.flatnonzero(pl["accepted"])[0])
    _, doms = _domains(s, ctx, pl["pose"][t])
    d = s.inp.hand_desc
    lo, hi = np.zeros(d.dof), np.zeros(d.dof)
    for l in range(d.n_links):
        j = d.joint_index[l]
        if j >= 0:
            lo[j], hi[j] = d.limit_lo[l], d.limit_hi[l]
    rng = np.random.default_rng(5)
    problems, starts = [], []
    for r in range(12):
        els = [dm[(r * 7 + 3 * g) % len(dm)] for g, dm in enumerate(doms) if dm][: 1 + r % 3]
        targets = []
        for j, e in enumerate(els):
            lk, hp, hn = s.ref_field.reverse_lookup(e, 100 * r + j)
            targets.append((e["pos"], -e["nrm"], lk, hp, hn))
        problems.append(targets)
        starts.append(0.5 * (lo + hi) if r % 2 == 0 else rng.uniform(lo, hi))
    problems.append([])  # k == 0: clamp only
    starts.append(rng.uniform(lo - 0.5, hi + 0.5))
    for kw in (dict(), dict(beta=0.02, iterations=40, step_clamp=0.1, residual_tol=1e-6,
                            damping_scale=1e-3, damping_min=1e-5, max_backtracks=6)):
        dev = lg.api.contact_ik_batch(ctx, s.H, np.array(starts), problems, **kw)
        for i, targets in enumerate(problems):
            ref = R.contact_ik(s.inp, starts[i], targets, **kw)
            assert dev["q"][i].tobytes() == ref["q"].tobytes(), i
            assert dev["finite"][i] == ref["finite"]
            assert int(dev["used_joints"][i]) == ref["used_joints"]
            assert dev["iterations"][i] == ref["iterations"]
            assert dev["objective"][i] == ref["objective"]
            assert dev["position"][i].tobytes() == ref["position"].tobytes()
            assert [math.acos(c) for c in dev["cosine"][i]] == ref["normal_angle"].tolist()
