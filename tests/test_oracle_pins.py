"""Pins the CPU oracle to the reference's own known answers and property
tests (proj/tests/*.cpp).  The reference ships no golden vectors; these are
the analytic / known-answer / oracle-comparison checks its Catch2 suite holds
for the hot path, restated against oracle/liborc.so."""
import math
import os

import numpy as np
import pytest

import caller as lc
import paper_2511_07418_b200 as lg
from oracle import orc_py as orc
from oracle import ref_py as R
from conftest import asset, cfg1, mismatched_fields


# ------------------------------------------------------------- rng / geometry
def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th draw of a default-seeded mt19937_64
    assert int(orc.rng_u64(5489, 10000)[-1]) == 9981545732273789042


def test_uniform_deciles():  # test_geometry.cpp:95-105
    u = (orc.rng_u64(15, 20000) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    assert (u >= 0).all() and (u < 1).all()
    assert len(set((u * 10).astype(int))) == 10


def test_normal_moments():  # test_geometry.cpp:107-120
    x = orc.rng_normal(16, 200000)
    assert abs(x.mean()) < 0.01
    assert abs(x.var() - 1.0) < 0.02


def test_unit_vectors_and_quaternions():  # test_geometry.cpp:122-166
    v = orc.rng_unit_vectors(17, 80000)
    assert np.allclose(np.linalg.norm(v, axis=1), 1.0, atol=1e-12)
    oct_ = (v[:, 0] > 0) + 2 * (v[:, 1] > 0) + 4 * (v[:, 2] > 0)
    cnt = np.bincount(oct_, minlength=8)
    assert (np.abs(cnt - 10000) < 5 * math.sqrt(10000)).all()
    q = orc.rng_quaternions(18, 80000)
    assert np.allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-9)


def test_mix_seed_grid_has_no_collisions():  # test_geometry.cpp:122-133
    seen = {orc.mix_seed(s, a, b) for s in range(4) for a in range(8) for b in range(8)}
    assert len(seen) == 4 * 8 * 8
    assert orc.mix_seed(1, 2, 3) == orc.mix_seed(1, 2, 3) == lg.mix_seed(1, 2, 3)


@pytest.mark.parametrize("fn", ["sin", "cos", "log", "atan2", "hypot"])
def test_libm_within_one_ulp_of_glibc(fn):
    """The deterministic libm shared by the oracle and the device stays
    within 1 ulp of glibc (Python's math module) over the pipeline's ranges."""
    rng = np.random.default_rng(1)
    n = 20000
    if fn == "log":
        x = rng.uniform(1e-12, 1.0, n)
        y = None
        ref = np.array([math.log(a) for a in x])
    elif fn in ("sin", "cos"):
        x = rng.uniform(-8.0, 8.0, n)
        y = None
        ref = np.array([getattr(math, fn)(a) for a in x])
    else:
        x = rng.uniform(-2, 2, n)
        y = rng.uniform(-2, 2, n)
        f = math.atan2 if fn == "atan2" else math.hypot
        ref = np.array([f(a, b) for a, b in zip(x, y)])
    got = orc.libm(fn, x, y)
    ulps = np.abs(got.view(np.int64) - ref.view(np.int64))
    assert ulps.max() <= 1


def test_tangent_basis_frame():  # test_geometry.cpp:42-57
    for n in orc.rng_unit_vectors(13, 200):
        x, y = orc.tangent_basis(n)
        assert abs(np.linalg.norm(x) - 1) < 1e-12 and abs(np.linalg.norm(y) - 1) < 1e-12
        assert abs(x @ n) < 1e-12 and abs(y @ n) < 1e-12 and abs(x @ y) < 1e-12
        assert np.linalg.norm(np.cross(x, y) - n) < 1e-12
    with pytest.raises(ValueError):
        orc.tangent_basis([0.0, 0.0, 0.0])
    with pytest.raises(ValueError):
        orc.tangent_basis([2.0, 0.0, 0.0])


def test_rotation_between():  # test_geometry.cpp:59-74
    v = orc.rng_unit_vectors(14, 400)
    for a, b in zip(v[::2], v[1::2]):
        R = orc.rotation_between(a, b)
        assert np.linalg.norm(R @ a - b) < 1e-9
        assert np.linalg.norm(R @ R.T - np.eye(3)) < 1e-9
        assert abs(np.linalg.det(R) - 1) < 1e-9
    a = np.array([0.0, 0.0, 1.0])
    R = orc.rotation_between(a, -a)
    assert np.linalg.norm(R @ a + a) < 1e-12


# ------------------------------------------------------------------- wrench
def rproblem(seed, n):
    p, q = np.zeros((n, 3)), np.zeros((n, 3))
    orc.lib().orc_random_wrench_problem(seed, n, orc._p(p), orc._p(q))
    return p, q


def grid_oracle(p, n, hi=4.0, step=5e-3, lam=10.0):  # test_wrench.cpp:29-71
    f = n
    t = np.cross(p, n)
    m = int(hi / step) + 1
    a = np.arange(m) * step
    best = np.inf
    for anchor in range(len(p)):
        free = [i for i in range(len(p)) if i != anchor]
        if not free:
            best = min(best, f[anchor] @ f[anchor] + lam * t[anchor] @ t[anchor])
        elif len(free) == 1:
            F = f[anchor] + a[:, None] * f[free[0]]
            T = t[anchor] + a[:, None] * t[free[0]]
            best = min(best, ((F * F).sum(1) + lam * (T * T).sum(1)).min())
        else:
            F = f[anchor] + a[:, None, None] * f[free[0]] + a[None, :, None] * f[free[1]]
            T = t[anchor] + a[:, None, None] * t[free[0]] + a[None, :, None] * t[free[1]]
            best = min(best, ((F * F).sum(-1) + lam * (T * T).sum(-1)).min())
    return best


def test_wrench_objective_hand_computed():  # test_wrench.cpp:75-91
    pts = [[0.1, 0, 0], [-0.1, 0, 0]]
    nrm = [[-1, 0, 0], [1, 0, 0]]
    assert orc.wrench_objective(pts, nrm, [1.0, 0.5]) == pytest.approx(0.25, abs=1e-12)
    assert orc.wrench_objective(pts, nrm, [1.0, 1.0]) == pytest.approx(0.0, abs=1e-12)


def test_antipodal_and_symmetric_balance():  # test_wrench.cpp:112-137
    obj, anchor, al, bx, by = orc.wrench_solve([[0.03, 0, 0], [-0.03, 0, 0]],
                                               [[-1, 0, 0], [1, 0, 0]])
    assert anchor >= 0 and obj <= 1e-6
    pts = [[0.04 * math.cos(2 * math.pi * i / 3), 0.04 * math.sin(2 * math.pi * i / 3), 0]
           for i in range(3)]
    nrm = [-np.array(p) / np.linalg.norm(p) for p in pts]
    obj, anchor, al, _, _ = orc.wrench_solve(pts, nrm)
    assert obj <= 1e-6
    assert abs(al[0] - al[1]) < 1e-3 and abs(al[1] - al[2]) < 1e-3


def test_single_contact_never_balances():  # test_wrench.cpp:139-147
    for seed in range(1, 11):
        p, n = rproblem(seed, 1)
        obj, *_ = orc.wrench_solve(p, n)
        assert obj >= 1.0 - 1e-12


def test_fswo_matches_grid_oracle():  # test_wrench.cpp:149-160
    for seed in range(1, 9):
        n = 2 + seed % 2
        p, q = rproblem(seed * 31, n)
        obj, *_ = orc.wrench_solve(p, q)
        g = grid_oracle(p, q)
        assert obj <= g + 1e-3
        assert obj >= g - 1e-2


def test_anchor_and_cone_invariants():  # test_wrench.cpp:162-187
    for seed in range(40, 52):
        n = 2 + seed % 4
        mu = 0.4 if seed % 2 else 0.0
        p, q = rproblem(seed, n)
        obj, anchor, al, bx, by = orc.wrench_solve(p, q, mu=mu)
        assert 0 <= anchor < n
        assert al[anchor] == pytest.approx(1.0, abs=1e-12)
        assert (al >= 0).all()
        assert orc.wrench_objective(p, q, al, bx, by, mu=mu) == pytest.approx(obj, abs=1e-9)
        assert (np.hypot(bx, by) <= mu * al + 1e-9).all()


def test_friction_never_hurts():  # test_wrench.cpp:189-204
    for seed in range(100, 120):
        p, q = rproblem(seed, 2 + seed % 3)
        f0, a0, *_ = orc.wrench_solve(p, q, mu=0.0, mode=0)
        g0, ag, *_ = orc.wrench_solve(p, q, mu=0.0, mode=1)
        assert g0 == f0 and ag == a0
        g5, *_ = orc.wrench_solve(p, q, mu=0.5, mode=1)
        assert g5 <= f0 + 1e-9


def test_wrench_solver_deterministic():  # test_wrench.cpp:250-259
    p, q = rproblem(5, 4)
    a = orc.wrench_solve(p, q, mu=0.3)
    b = orc.wrench_solve(p, q, mu=0.3)
    assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])


# -------------------------------------------------------------- contact_opt
def sphere_domain(seed, r=0.03, count=200):  # test_contact_opt.cpp:16-32
    n = orc.rng_unit_vectors(seed, count)
    return r * n, n


def test_antipodal_convergence_on_sphere_domains():  # test_contact_opt.cpp:83-104
    ok = 0
    for seed in range(20):
        d0, d1 = sphere_domain(1000 + seed), sphere_domain(2000 + seed)
        ids, obj, ev = orc.optimize_contacts([d0, d1], mu=0.0, seed=seed)
        ok += obj < 0.05
        assert ev == 4 * (1 + 8 * 2 * 32)
    assert ok >= 18


def test_contact_opt_deterministic_and_restarts_never_worse():  # :131-164
    d0, d1 = sphere_domain(7), sphere_domain(8)
    a = orc.optimize_contacts([d0, d1], seed=3)
    b = orc.optimize_contacts([d0, d1], seed=3)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]
    one = orc.optimize_contacts([d0, d1], restarts=1, seed=3)
    four = orc.optimize_contacts([d0, d1], restarts=4, seed=3)
    assert four[1] <= one[1]


def test_single_cap_cannot_balance():  # test_contact_opt.cpp:190-201
    rng = np.random.default_rng(0)
    n = rng.normal(size=(400, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    cap = n[n[:, 2] > math.cos(0.3)][:50]
    ids, obj, _ = orc.optimize_contacts([(0.03 * cap, cap)], mu=0.0, seed=1)
    assert obj >= 0.5


def test_empty_domain_rejected():  # test_contact_opt.cpp:203-211
    with pytest.raises(ValueError):
        orc.optimize_contacts([(np.zeros((0, 3)), np.zeros((0, 3)))])


# -------------------------------------------------------------- kinematics
def test_fk_analytic_four_finger(four_finger):  # test_hand.cpp:107-147
    d = four_finger.desc
    q = np.zeros(d.dof)
    th = 0.4
    q[0] = th  # finger_a_base about +y
    fr = orc.fk(d, q)
    names = [four_finger.link_name(l) for l in range(d.n_links)]
    prox = fr[names.index("finger_a_proximal")]
    mid = fr[names.index("finger_a_middle")]
    assert np.allclose(prox[9:], [-0.046, 0, 0.012], atol=1e-12)
    exp = np.array([-0.046, 0, 0.012]) + 0.04 * np.array([math.sin(th), 0, math.cos(th)])
    assert np.allclose(mid[9:], exp, atol=1e-12)


def test_point_jacobian_matches_finite_differences(four_finger):  # test_ik.cpp:49-82
    d = four_finger.desc
    lo, hi = four_finger.limits()
    rng = np.random.default_rng(17)
    h = 1e-6
    worst = 0.0
    for _ in range(50):
        q = rng.uniform(lo, hi)
        link = int(rng.integers(1, d.n_links))
        lp = 0.01 * rng.normal(size=3)
        J = orc.point_jacobian(d, q, link, lp)
        for j in range(d.dof):
            qp, qm = q.copy(), q.copy()
            qp[j] += h
            qm[j] -= h
            fp, fm = orc.fk(d, qp)[link], orc.fk(d, qm)[link]
            pp = fp[:9].reshape(3, 3) @ lp + fp[9:]
            pm = fm[:9].reshape(3, 3) @ lp + fm[9:]
            worst = max(worst, np.abs((pp - pm) / (2 * h) - J[:, j]).max())
    assert worst < 1e-5


PLANAR = """<?xml version="1.0"?>
<robot name="arm">
  <link name="base"><visual><geometry><box size="0.02 0.02 0.02"/></geometry></visual></link>
  <link name="upper"><visual><geometry><box size="0.01 0.01 0.1"/></geometry></visual></link>
  <link name="lower"><visual><geometry><box size="0.01 0.01 0.08"/></geometry></visual></link>
  <joint name="shoulder" type="revolute">
    <parent link="base"/><child link="upper"/>
    <origin xyz="0 0 0" rpy="0 0 0"/><axis xyz="0 1 0"/>
    <limit lower="-3.1" upper="3.1"/>
  </joint>
  <joint name="elbow" type="revolute">
    <parent link="upper"/><child link="lower"/>
    <origin xyz="0 0 0.1" rpy="0 0 0"/><axis xyz="0 1 0"/>
    <limit lower="-3.1" upper="3.1"/>
  </joint>
</robot>
"""


def test_planar_reach_matches_analytic(tmp_path):  # test_ik.cpp:115-157
    path = tmp_path / "arm.urdf"
    path.write_text(PLANAR)
    if not R.available():
        pytest.skip("oracle/_ref not built (the reference parses the URDF)")
    arm = lc.HandModel(R.load_hand_arrays(str(path)))
    rng = np.random.default_rng(5)
    solved = 0
    l1, l2 = 0.1, 0.08
    for _ in range(100):
        reach = rng.uniform(0.6, 0.95) * (l1 + l2)
        ang = rng.uniform(-1.2, 1.2)
        tgt = np.array([reach * math.sin(ang), 0, reach * math.cos(ang)])
        r = orc.ik(arm.desc, [0.3, 0.3], [(tgt, [0, 1, 0], 2, [0, 0, l2], [0, 1, 0])],
                   iterations=1000, residual_tol=1e-6)
        assert r["finite"]
        fr = orc.fk(arm.desc, r["q"])[2]
        tip = fr[:9].reshape(3, 3) @ [0, 0, l2] + fr[9:]
        if np.linalg.norm(tip - tgt) <= 1e-4:
            solved += 1
            c = (reach ** 2 - l1 ** 2 - l2 ** 2) / (2 * l1 * l2)
            assert math.cos(r["q"][1]) == pytest.approx(c, abs=1e-3)
    assert solved >= 95


def _random_targets(rng, hand, count):
    out = []
    for _ in range(count):
        n = rng.normal(size=3)
        m = rng.normal(size=3)
        out.append((np.array([rng.uniform(-.08, .08), rng.uniform(-.04, .04), rng.uniform(.02, .12)]),
                    n / np.linalg.norm(n), int(rng.integers(1, hand.n_links)),
                    0.01 * rng.normal(size=3), m / np.linalg.norm(m)))
    return out


def test_ik_objective_monotone_and_limits(two_finger):  # test_ik.cpp:159-222
    d = two_finger.desc
    lo, hi = two_finger.limits()
    q0 = two_finger.mid_config()
    rng = np.random.default_rng(23)
    for _ in range(40):
        tg = _random_targets(rng, two_finger, int(rng.integers(1, 4)))
        r = orc.ik(d, q0, tg, iterations=40)
        assert r["finite"]
        fr = orc.fk(d, q0)
        start = 0.0
        for op, on, link, hp, hn in tg:
            R, t = fr[link][:9].reshape(3, 3), fr[link][9:]
            sp, sn = R @ hp + t, R @ hn
            start += ((op - sp) ** 2).sum() + (((op + 0.01 * on) - (sp + 0.01 * sn)) ** 2).sum()
        assert r["objective"] <= start + 1e-12
        assert (r["q"] >= lo).all() and (r["q"] <= hi).all()


def test_ik_unreachable_stays_finite(two_finger):  # test_ik.cpp:298-315
    r = orc.ik(two_finger.desc, two_finger.mid_config(),
               [([5.0, 5.0, 5.0], [0, 0, 1], 3, [0, 0, 0], [0, 0, 1])])
    assert r["finite"] and np.isfinite(r["q"]).all()


# ---------------------------------------------------------------- collision
def test_gjk_box_distances(four_finger):  # test_collision.cpp:55-97
    d = four_finger.desc
    I = np.concatenate([np.eye(3).ravel(), [0, 0, 0]])
    # parts 1 and 4 are the proximal boxes (0.018 x 0.018 x 0.04, z in [0, .04])
    for gap in (0.001, 0.01, 0.05):
        T = np.concatenate([np.eye(3).ravel(), [0.018 + gap, 0, 0]])
        assert orc.gjk(d, 1, I, 4, T) == pytest.approx(gap, abs=1e-9)
    T = np.concatenate([np.eye(3).ravel(), [0.01, 0, 0.0]])
    assert orc.gjk(d, 1, I, 4, T) == 0.0


def test_halfplane_depth_exact(four_finger):  # test_collision.cpp:201-225
    d = four_finger.desc
    q = four_finger.mid_config()
    I = np.concatenate([np.eye(3).ravel(), [0, 0, 0]])
    # palm box 0.11 x 0.11 x 0.02 centred at the origin: a sample 3 mm below
    # the top face penetrates by exactly 3 mm
    s = np.array([[0.0, 0.0, 0.007, 0, 0, 1]])
    clean, depth, nv = orc.collision(d, q, I, s)
    assert not clean and depth == pytest.approx(0.003, abs=1e-15)
    s[0, 2] = 0.0095  # 0.5 mm deep: under the 2 mm margin
    clean, depth, nv = orc.collision(d, q, I, s)
    assert depth == 0.0


# -------------------------------------------------------------------- field
def test_query_equals_linear_scan(two_finger, tmp_path):  # test_contact_field.cpp:218-273
    import paper_2511_07418_b200.api as api
    d = two_finger.desc
    patches = lc.hand_patches(two_finger, 20.0, 0.01, 42)
    N, w, theta = 24, 0.01, 0.9397
    f = orc.OrcField(d, patches.desc, N, w, 7, 64)
    ex = f.export()
    cb = ex["codebook"]
    ball = lc.Mesh.icosphere(0.03, 2)
    samples = lc.sample_surface(ball, 30.0, 11)
    pose = np.concatenate([np.eye(3).ravel(), [0.0, 0.0, 0.09]])
    masks, scores, _ = f.query(d, samples, pose, theta)
    # linear scan over the materialised vectors, scored through their codes
    gl, _ = two_finger.groups()
    P = patches.desc
    plink = np.ctypeslib.as_array(P.link, shape=(P.n_patches,))
    poff = np.ctypeslib.as_array(P.point_off, shape=(P.n_patches + 1,))
    foff = np.ctypeslib.as_array(P.fp_off, shape=(P.n_patches + 1,))
    fps = np.ctypeslib.as_array(P.field_points, shape=(foff[-1],))
    pts = np.ctypeslib.as_array(P.points, shape=(poff[-1] * 3,)).reshape(-1, 3)
    nrm = np.ctypeslib.as_array(P.normals, shape=(poff[-1] * 3,)).reshape(-1, 3)
    lo, hi = two_finger.limits()
    cells, codes, pids = [], [], []
    for c in range(N):
        rng_draws = orc.rng_u64(orc.mix_seed(7, 0x636f6e66, c), d.dof)
        q = lo + (hi - lo) * ((rng_draws >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
        fr = orc.fk(d, q)
        for p in range(P.n_patches):
            R, t = fr[plink[p]][:9].reshape(3, 3), fr[plink[p]][9:]
            for fp in fps[foff[p]:foff[p + 1]]:
                x = R @ pts[poff[p] + fp] + t
                n = R @ nrm[poff[p] + fp]
                cells.append(np.floor(x / w).astype(np.int64))
                codes.append(int(np.argmax(cb @ n)))
                pids.append(p)
    cells = np.array(cells)
    expect = np.zeros(len(samples), dtype=np.uint32)
    for i, s in enumerate(samples):
        p = s[:3] + pose[9:]
        n = s[3:]
        cell = np.floor(p / w).astype(np.int64)
        hit = np.nonzero((cells == cell).all(1))[0]
        for v in hit:
            if -(n @ cb[codes[v]]) < theta:
                continue
            g = gl[plink[pids[v]]]
            if g >= 0:
                expect[i] |= np.uint32(1 << g)
    assert np.array_equal(masks, expect)
    assert (scores[masks != 0] >= theta).all()


def test_index_boxes_sorted_codes_unique(two_finger):  # test_contact_field.cpp:192-216
    patches = lc.hand_patches(two_finger, 20.0, 0.01, 42)
    ex = orc.OrcField(two_finger.desc, patches.desc, 24, 0.01, 7, 64).export()
    pbo, cells, bco, codes = ex["patch_box_off"], ex["box_cell"], ex["box_code_off"], ex["codes"]
    for p in range(len(pbo) - 1):
        c = [tuple(x) for x in cells[pbo[p]:pbo[p + 1]]]
        assert c == sorted(c) and len(set(c)) == len(c)
    for b in range(len(bco) - 1):
        cs = codes[bco[b]:bco[b + 1]]
        assert len(cs) > 0 and (np.diff(cs.astype(int)) > 0).all()


def test_reverse_lookup_returns_hit_rep(two_finger):  # test_contact_field.cpp:297-346
    patches = lc.hand_patches(two_finger, 20.0, 0.01, 42)
    f = orc.OrcField(two_finger.desc, patches.desc, 24, 0.01, 7, 256)
    ball = lc.Mesh.icosphere(0.03, 2)
    s = lc.sample_surface(ball, 30.0, 11)
    pose = np.concatenate([np.eye(3).ravel(), [0.0, 0.0, 0.09]])
    masks, _, _ = f.query(two_finger.desc, s, pose, 0.9397)
    idx = np.nonzero(masks)[0][:20]
    assert len(idx) > 0
    ex = f.export()
    for i in idx:
        g = (int(masks[i]) & -int(masks[i])).bit_length() - 1
        a = f.reverse_lookup(two_finger.desc, s, pose, 0.9397, i, g, 99)
        b = f.reverse_lookup(two_finger.desc, s, pose, 0.9397, i, g, 99)
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
        assert abs(np.linalg.norm(a[2]) - 1) < 1e-9
        hits = (ex["rep_link"] == a[0]) & (ex["rep_point"] == a[1]).all(1)
        assert hits.any()
    with pytest.raises(IndexError):
        f.reverse_lookup(two_finger.desc, s, pose, 0.9397, int(np.nonzero(masks == 0)[0][0]), 0, 1)


# ---------------------------------------------------------------- pipeline
def test_preprocess_drops_thin_slots():  # pipeline.cpp:71-98
    a = lc.Mesh.box((0.04, 0.04, 0.002))
    va, ta = a.arrays()
    vb = va + [0, 0, 0.006]  # second plate 4 mm above the first
    slab = lc.Mesh.from_arrays(np.vstack([va, vb]), np.vstack([ta, ta + len(va)]))
    s = lc.sample_surface(slab, 30.0, 3)
    keep = orc.preprocess(s, 0.01, 0.005)
    inner = ((np.abs(s[:, 2] - 0.001) < 1e-9) & (s[:, 5] > 0)) | \
            ((np.abs(s[:, 2] - 0.005) < 1e-9) & (s[:, 5] < 0))
    assert not keep[inner].any()
    ball = lc.sample_surface(lc.Mesh.icosphere(0.03, 3), 30.0, 1)
    assert orc.preprocess(ball, 0.01, 0.005).all()
    with pytest.raises(ValueError):
        orc.preprocess(ball, 0.0, 0.005)


def test_run_batch_worker_invariant_and_deterministic():  # parallel.hpp:20-23
    p = cfg1(batch=24, field_configs=48)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    a = orc.run_batch(hand.desc, patches.desc, raw, p, workers=1)
    b = orc.run_batch(hand.desc, patches.desc, raw, p, workers=4)
    assert mismatched_fields(a.traces, b.traces) == {}
    assert a.profile["valid"] == b.profile["valid"]
    assert a.profile["placements_accepted"] > 0
