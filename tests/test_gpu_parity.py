"""Device-vs-oracle parity on the B200 (run with -m gpu).  Every test calls
the sm_100a path through the C-ABI and compares with the CPU oracle on the
same inputs: integer / index / decision outputs bit-exact, and - because
the device evaluates the oracle's exact FP64 operation order with the same
libm - every floating-point output bit-exact as well (the north-star
tolerance of 1e-4 rad / 1e-4 m is therefore met with zero error)."""
import types

import numpy as np
import pytest

import caller as lc
import paper_2511_07418_b200 as lg
from oracle import orc_py as orc
from oracle import ref_py as R
from conftest import asset, cfg1, mismatched_fields

pytestmark = pytest.mark.gpu


def _poses(n, seed=0, z0=0.05):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        q = rng.normal(size=4)
        w, x, y, z = q / np.linalg.norm(q)
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                      [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                      [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
        out.append(np.concatenate([R.ravel(), rng.normal(scale=0.01, size=3) + [0, 0, z0]]))
    return np.array(out)


@pytest.mark.parametrize("hand_name,N,C", [("four_finger", 256, 256), ("two_finger", 64, 64)])
def test_field_build_bit_exact(ctx, hand_name, N, C):
    p = cfg1(hand=hand_name)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    dev = lg.ContactFieldIndex.build(ctx, hand, patches, N, p.box_width, p.seed, C).export()
    ref = orc.OrcField(hand.desc, patches.desc, N, p.box_width, p.seed, C).export()
    for k in ref:
        assert np.array_equal(np.asarray(dev[k]), np.asarray(ref[k])), k


def test_query_masks_bit_exact(ctx, four_finger):
    p = cfg1()
    hand, patches, raw, _ = lc.prepare_inputs(p)
    f = lg.ContactFieldIndex.build(ctx, hand, patches, p.field_configs, p.box_width, p.seed, 256)
    fo = orc.OrcField(hand.desc, patches.desc, p.field_configs, p.box_width, p.seed, 256)
    gl, _ = hand.groups()
    gop = gl[patches.link_of_patch()]
    poses = _poses(24)
    md, sd = lg.query_domains_batch(ctx, f, gop, raw, poses, p.theta_hit, with_scores=True)
    total = 0
    for i, pose in enumerate(poses):
        mo, so, _ = fo.query(hand.desc, raw, pose, p.theta_hit)
        assert np.array_equal(md[i], mo), i
        assert np.array_equal(sd[i], so), i  # element scores (contact_field.cpp:443)
        total += int((mo != 0).sum())
    assert total > 0
    # theta_hit = 1.0 admits no hit: empty domains everywhere
    assert not lg.query_domains_batch(ctx, f, gop, raw, poses[:2], 1.0).any()


def test_preprocess_bit_exact(ctx):
    a = lc.Mesh.box((0.04, 0.04, 0.002))
    va, ta = a.arrays()
    slab = lc.Mesh.from_arrays(np.vstack([va, va + [0, 0, 0.006]]), np.vstack([ta, ta + len(va)]))
    kept = []
    for mesh in (slab, lc.load_mesh(asset("objects", "scan_test.obj"))):
        s = lc.sample_surface(mesh, 40.0, 5)
        kd = lg.preprocess_object(ctx, s, 0.01, 0.005)
        assert np.array_equal(kd, orc.preprocess(s, 0.01, 0.005))
        if R.available():
            assert np.array_equal(kd, R.preprocess(s, 0.01, 0.005))  # the reference itself
        kept.append(kd)
    # the 6 mm slab is a thin slot: its facing samples are stripped
    assert 0 < kept[0].sum() < len(kept[0])


def test_wrench_batch_bit_exact(ctx):
    probs, ref = [], []
    for seed in range(1, 120):
        n = 1 + seed % 6
        p, q = np.zeros((n, 3)), np.zeros((n, 3))
        orc.lib().orc_random_wrench_problem(seed, n, orc._p(p), orc._p(q))
        probs.append((p, q))
    for mu in (0.0, 0.3):
        obj, anchor, al, bx, by = lg.api.wrench_solve_batch(ctx, probs, mu=mu)
        for i, (p, q) in enumerate(probs):
            o, a, ra, rbx, rby = orc.wrench_solve(p, q, mu=mu)
            n = len(p)
            assert obj[i] == o and anchor[i] == a
            assert al[i, :n].tobytes() == ra.tobytes() and bx[i, :n].tobytes() == rbx.tobytes()


def test_collision_batch_bit_exact(ctx, four_finger):
    s = lc.sample_surface(lc.load_mesh(asset("objects", "sphere_r030.obj")), 30.0, 1)
    lo, hi = four_finger.limits()
    rng = np.random.default_rng(3)
    q = rng.uniform(lo, hi, size=(64, four_finger.dof))
    poses = _poses(64, seed=4, z0=0.06)
    clean, depth = lg.api.collision_batch(ctx, four_finger, q, poses, s)
    n_clean = 0
    for i in range(64):
        c, d, _ = orc.collision(four_finger.desc, q[i], poses[i], s)
        assert clean[i] == c and depth[i] == d, i
        n_clean += c
    assert 0 < n_clean < 64


def test_realize_batch_bit_exact(ctx, four_finger):
    rng = np.random.default_rng(9)
    probs = []
    for _ in range(32):
        k = int(rng.integers(1, 4))
        ts = []
        for _ in range(k):
            n = rng.normal(size=3)
            m = rng.normal(size=3)
            ts.append((np.array([rng.uniform(-.05, .05), rng.uniform(-.05, .05), rng.uniform(.03, .1)]),
                       n / np.linalg.norm(n), int(rng.integers(1, four_finger.n_links)),
                       0.005 * rng.normal(size=3), m / np.linalg.norm(m)))
        probs.append(ts)
    q0 = four_finger.mid_config()
    q, mr, fin, used = lg.api.realize_batch(ctx, four_finger, q0, probs, beta=0.05,
                                            iterations=60, finetune_rounds=3,
                                            finetune_iterations=10)
    for i, ts in enumerate(probs):
        r = orc.realize(four_finger.desc, q0, ts, beta=0.05, iterations=60, rounds=3,
                        fine_iters=10)
        assert fin[i] == r["finite"] and used[i] == r["used"]
        assert q[i].tobytes() == r["q"].tobytes() and mr[i] == r["max_residual"], i


def _run_both(p):
    hand, patches, raw, _ = lc.prepare_inputs(p)
    ctx = lg.Context(0)
    dev = lg.run_batch(ctx, hand, patches, raw, p)
    ref = orc.run_batch(hand.desc, patches.desc, raw, p, workers=0)
    ctx.close()
    return dev, ref


GRASP_FIELDS = ["g", "pose_R", "pose_t", "dof", "q", "n_contacts", "contact_p", "contact_n",
                "contact_link", "objective", "penetration_free", "stable", "ik_converged"]
FUNNEL = ["candidates", "placements_accepted", "contact_sets_balanced", "ik_finite",
          "penetration_free", "ik_converged", "stable", "valid", "patches", "boxes",
          "field_vectors", "field_samples"]


@pytest.mark.parametrize("case", [
    dict(batch=128, passes=2),                                   # cfg1 sphere, multi-pass reuse
    dict(batch=96, obj="box_040.obj"),                           # cfg1 box
    dict(batch=96, hand="two_finger"),                           # two-finger cfg
    dict(batch=64, placement_mode=0),                            # exhaustive placement
    dict(batch=48, static_contact_prob=1.0),                     # every candidate pinned
    dict(batch=32, k_contacts=3),                                # k = 3 of 4 groups
    dict(batch=32, k_contacts=4, static_contact_prob=0.5),       # k = 4 (+ statics): 5-6 contacts
])
def test_run_batch_stage_traces_bit_exact(case):
    case = dict(case)
    p = cfg1(batch=case.pop("batch"), **{k: case.pop(k) for k in ("passes", "obj", "hand")
                                         if k in case}, **case)
    dev, ref = _run_both(p)
    for k in FUNNEL:
        assert dev.profile[k] == ref.profile[k], k
    assert dev.profile["gpu_launches"] > 0
    assert mismatched_fields(dev.traces, ref.traces) == {}
    assert mismatched_fields(dev.grasps, ref.grasps, GRASP_FIELDS) == {}


def test_two_finger_k3_never_succeeds():  # pipeline.cpp:429-432 (2 groups < k)
    dev, ref = _run_both(cfg1(batch=32, hand="two_finger", k_contacts=3))
    assert dev.profile["placements_accepted"] == 0 == ref.profile["placements_accepted"]
    assert dev.profile["valid"] == 0


def test_sharded_full_size_against_oracle_shard():
    """Size-independent property at a full batch: the device runs all 2048
    candidates; the oracle re-runs one 1/32 shard and every candidate of that
    shard must agree bit for bit (per-candidate streams depend only on
    (seed, c, pass))."""
    p = cfg1(batch=2048)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    ctx = lg.Context(0)
    dev = lg.run_batch(ctx, hand, patches, raw, p)
    ctx.close()
    from paper_2511_07418_b200 import dist as ldist
    sp = ldist.shard_params(p, 13, 32)
    ref = orc.run_batch(hand.desc, patches.desc, raw, sp, workers=0)
    lo, hi = ldist.shard_range(2048, 13, 32)
    sub = dev.traces[(dev.traces["c"] >= lo) & (dev.traces["c"] < hi)]
    assert mismatched_fields(sub, ref.traces) == {}
    gsub = dev.grasps[(dev.grasps["g"] >= lo) & (dev.grasps["g"] < hi)]
    assert mismatched_fields(gsub, ref.grasps, GRASP_FIELDS) == {}


def _cfg(hand, obj, cfg, batch, **over):
    p = lc.parse_config(asset("configs", cfg), hand=asset("hands", hand),
                        object=asset("objects", obj), batch=batch)
    p.want_trace = 1
    for k, v in over.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("args", [
    # BASELINE config 3: LEAP-class hand on a tool-like union (reduced field)
    ("leap_like.urdf", "mug.obj", "leap.cfg", 48, dict(field_configs=128)),
    ("leap_like.urdf", "drill.obj", "leap.cfg", 32, dict(field_configs=128)),
    # config 4: Shadow-class 22 DoF, k = 3 of 5 groups (reduced sampling)
    ("shadow_like.urdf", "icosphere_r030_s6.obj", "shadow.cfg", 32,
     dict(field_configs=64, samples_per_cm2=20.0, patch_radius=0.012)),
    # config 2 hand, cylinder object
    ("allegro_like.urdf", "cylinder_r025_l100.obj", "allegro.cfg", 64, dict(field_configs=256)),
])
def test_run_batch_synthetic_hands_bit_exact(args):
    p = _cfg(*args[:4], **args[4])
    dev, ref = _run_both(p)
    for k in FUNNEL:
        assert dev.profile[k] == ref.profile[k], k
    assert mismatched_fields(dev.traces, ref.traces) == {}
    assert mismatched_fields(dev.grasps, ref.grasps, GRASP_FIELDS) == {}


def _patch_arrays(pt):
    d = pt.desc
    P = d.n_patches
    arr = np.ctypeslib.as_array
    po = arr(d.point_off, shape=(P + 1,)).copy()
    fo = arr(d.fp_off, shape=(P + 1,)).copy()
    return dict(link=arr(d.link, shape=(P,)).copy(), point_off=po, fp_off=fo,
                points=arr(d.points, shape=(3 * po[-1],)).copy(),
                normals=arr(d.normals, shape=(3 * po[-1],)).copy(),
                field_points=arr(d.field_points, shape=(fo[-1],)).copy())


@pytest.mark.parametrize("hand_name,spc,radius,cap", [
    ("four_finger.urdf", 30.0, 0.014, 8),
    ("allegro_like.urdf", 30.0, 0.012, 8),
    ("shadow_like.urdf", 1000.0, 0.008, 8),   # config 4: ~810k hand samples
    ("shadow_like.urdf", 200.0, 0.008, 3),
    ("shadow_like.urdf", 30.0, 0.020, 16),    # large patches: the maximum field cap
])
def test_patches_device_identical(ctx, hand_name, spc, radius, cap):
    """Hand sampling + decompose_patches on the GPU ==
    the reference's own (sample_surface per link with stream 'hnds',
    decompose_patches: contact_field.cpp:26-99, run by oracle/_ref)."""
    if not R.available():
        pytest.skip("oracle/_ref not built")
    hand = lc.load_hand(asset("hands", hand_name))
    ref = R.RefInputs(extra=f"samples_per_cm2 = {spc}\npatch_radius = {radius}\n"
                            f"field_points_per_patch = {cap}\nseed = 7\n",
                      hand=asset("hands", hand_name), object=asset("objects", "box_040.obj"),
                      batch=1)
    a = _patch_arrays(types.SimpleNamespace(desc=ref.patches_desc))
    b = _patch_arrays(lg.hand_patches_device(ctx, hand, spc, radius, 7, cap))
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_device_errors_map_to_reference_exceptions(ctx, four_finger):
    """Bad arguments raise the reference's exception class with its message
    (ValueError <- std::invalid_argument) instead of running."""
    p = cfg1(batch=8)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    p.k_contacts = 9
    with pytest.raises(ValueError, match="k_contacts"):
        lg.run_batch(ctx, hand, patches, raw, p)
    with pytest.raises(ValueError, match="box width"):
        lg.ContactFieldIndex.build(ctx, hand, patches, 16, 0.0, 0, 64)
    with pytest.raises(ValueError, match="1..6 contacts"):
        lg.api.wrench_solve_batch(ctx, [(np.zeros((7, 3)), np.tile([0.0, 0.0, 1.0], (7, 1)))])
    with pytest.raises(ValueError, match="no samples|stripped|no object samples"):
        lg.run_batch(ctx, hand, patches, np.zeros((0, 6)), cfg1(batch=8))
    # the context stays usable after an error
    ok = lg.run_batch(ctx, hand, patches, raw, cfg1(batch=8))
    assert ok.profile["candidates"] == 8


def test_empty_batch_matches_oracle(ctx, four_finger):
    """batch = 0 (or passes = 0) past the config layer: the reference's
    run_batch builds the field and returns no candidates, no grasps
    (pipeline.cpp:385 loop never runs); the device does the same."""
    p = cfg1(batch=8)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    for field, val in (("batch", 0), ("passes", 0)):
        q = cfg1(batch=8)
        setattr(q, field, val)
        q.want_trace = 1
        dev = lg.run_batch(ctx, hand, patches, raw, q)
        ref = orc.run_batch(hand.desc, patches.desc, raw, q, workers=0)
        assert len(dev.traces) == len(ref.traces) == 0
        assert len(dev.grasps) == len(ref.grasps) == 0
        for k in FUNNEL + ["patches", "boxes", "field_vectors", "object_samples", "field_samples"]:
            assert dev.profile[k] == ref.profile[k], (field, k)


def test_bench_config_against_oracle_shard():
    """The bench workload itself (Allegro-class hand, 5 cm box, 10k seeds):
    the device's full batch, compared candidate by candidate with the
    oracle's re-run of one 1/40 shard (field built by each side)."""
    import bench
    cfg, hand_path, obj = bench.workload_paths("allegro_box")
    p = lc.parse_config(cfg, hand=hand_path, object=obj)
    p.want_trace = 1
    hand, patches, raw, _ = lc.prepare_inputs(p)
    ctx = lg.Context(0)
    dev = lg.run_batch(ctx, hand, patches, raw, p)
    ctx.close()
    from paper_2511_07418_b200 import dist as ldist
    sp = ldist.shard_params(p, 7, 40)
    ref = orc.run_batch(hand.desc, patches.desc, raw, sp, workers=0)
    lo, hi = ldist.shard_range(p.batch, 7, 40)
    sub = dev.traces[(dev.traces["c"] >= lo) & (dev.traces["c"] < hi)]
    assert len(sub) == hi - lo
    assert mismatched_fields(sub, ref.traces) == {}
    gsub = dev.grasps[(dev.grasps["g"] >= lo) & (dev.grasps["g"] < hi)]
    assert mismatched_fields(gsub, ref.grasps, GRASP_FIELDS) == {}


def test_untraced_run_matches_oracle():
    """The production path (want_trace = 0: funnel counts and kept grasps
    compacted on the device) returns the same grasps and funnel."""
    p = cfg1(batch=160, passes=2)
    p.want_trace = 0
    dev, ref = _run_both(p)
    for k in FUNNEL:
        assert dev.profile[k] == ref.profile[k], k
    assert len(dev.grasps) > 0
    assert mismatched_fields(dev.grasps, ref.grasps, GRASP_FIELDS) == {}
