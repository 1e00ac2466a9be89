"""validate_dataset (reference validate.cpp:56-175) — the independent
acceptance check, on the GPU (§8(f) rank 2).

CPU: the oracle's restatement plus the library's issue formatter reproduce
the reference's messages on crafted grasps (limits, rigidity, contacts off
the surfaces, penetration, wrench).  GPU: lg_validate_batch's records equal
the oracle's bit for bit, on a real run's grasps and on the crafted ones, and
every grasp the pipeline marks valid passes validation."""
import numpy as np
import pytest

import caller as lc
import paper_2511_07418_b200 as lg
from oracle import orc_py as orc
from conftest import cfg1, mismatched_fields


def _inputs(batch=96):
    p = cfg1(batch=batch)
    p.want_trace = 0
    hand, patches, raw, mesh = lc.prepare_inputs(p)
    return p, hand, patches, raw, mesh


def _crafted(grasps, hand):
    """Copies of the first grasp with one defect each (reference check order)."""
    g0 = grasps[0]
    out = [g0.copy() for _ in range(8)]
    out[0]["dof"] = g0["dof"] - 1                      # joint vector size mismatch
    out[1]["pose_R"] = g0["pose_R"] * 1.01             # pose not rigid
    lo, hi = hand.limits()
    out[2]["q"][0] = hi[0] + 0.5                       # joint out of limits
    out[3]["n_contacts"] = 0                           # no contacts
    out[4]["contact_link"][0] = 999                    # invalid link id
    out[5]["contact_n"][0] = g0["contact_n"][0] * 2.0  # not unit (and wrench recheck fails)
    out[6]["contact_p"][0] = g0["contact_p"][0] + 0.05 # off hand and object surfaces
    out[7]["pose_t"] = g0["pose_t"] + np.array([0.0, 0.0, -0.02])  # object pushed into the hand
    return np.array(out, dtype=grasps.dtype)


def _oracle_run(p, hand, patches, raw):
    return orc.run_batch(hand.desc, patches.desc, raw, p, workers=0)


def test_oracle_validation_messages():
    p, hand, patches, raw, mesh = _inputs()
    ref = _oracle_run(p, hand, patches, raw)
    assert len(ref.grasps) > 0
    v, t = mesh.arrays()
    checks = orc.validate(hand.desc, ref.grasps, v, t, raw, p)
    issues = lg.validation_issues(hand.joint_names, checks, p)
    # every grasp the pipeline flags valid passes the independent check
    flagged = set(gi for gi, _ in issues)
    for gi, g in enumerate(ref.grasps):
        if g["penetration_free"] and g["stable"] and g["ik_converged"]:
            assert gi not in flagged, [w for i, w in issues if i == gi]
    bad = _crafted(ref.grasps, hand)
    msgs = lg.validation_issues(hand.joint_names, orc.validate(hand.desc, bad, v, t, raw, p), p)
    by = {}
    for gi, what in msgs:
        by.setdefault(gi, []).append(what)
    assert by[0] == ["joint vector size mismatch"]
    assert by[1] == ["pose not rigid: transform rotation is not orthonormal"]
    assert len(by[2]) == 1 and by[2][0].startswith("joint ") and " out of limits: " in by[2][0]
    assert by[3] == ["no contacts"]
    assert "contact with invalid link id" in by[4]
    assert "contact normal not unit length" in by[5]
    assert "wrench recheck failed: tangent_basis: normal is not unit length" in by[5]
    assert any("m off the hand surface (limit" in w for w in by[6])
    assert any("m off the object surface (limit" in w for w in by[6])
    assert any(w.startswith("object penetrates the hand by ") for w in by.get(7, [])), by.get(7)


@pytest.mark.gpu
def test_validate_batch_bit_exact():
    p, hand, patches, raw, mesh = _inputs()
    ctx = lg.Context(0)
    dev = lg.run_batch(ctx, hand, patches, raw, p)
    assert len(dev.grasps) > 0
    v, t = mesh.arrays()
    grasps = np.concatenate([dev.grasps, _crafted(dev.grasps, hand)])
    got = lg.validate_batch(ctx, hand, grasps, mesh, raw, p)
    ctx.close()
    want = orc.validate(hand.desc, grasps, v, t, raw, p)
    assert mismatched_fields(got, want) == {}
    assert lg.validation_issues(hand.joint_names, got, p) == lg.validation_issues(hand.joint_names, want, p)
