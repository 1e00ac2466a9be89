"""Parity against THE REFERENCE ITSELF (oracle/_ref: /root/reference/proj/src
compiled unmodified against oracle/shim, linked with the host glibc).

* The reference's own 99 Catch2 cases run green on that build.
* The CPU restatement (oracle/liborc.so, which carries per-candidate stage
  traces) reproduces the reference's run_batch bit for bit.
* The device (libgraspgen_b200.so, through the C-ABI) reproduces the
  reference's run_batch bit for bit on the reference's own inputs: every kept
  grasp (pose, q, contacts, objective, flags) and every funnel counter.

Inputs come from the reference (parse_config, load_hand, sample_surface,
decompose_patches via oracle/ref_capi.cpp) and are handed to the device in the
lg.h descriptor layout, so both sides see identical bits.
"""
import filecmp
import os
import subprocess
import types

import numpy as np
import pytest

from conftest import ASSETS, ROOT
from oracle import ref_py as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")

FUNNEL = ("placements_accepted", "contact_sets_balanced", "ik_finite", "penetration_free",
          "ik_converged", "stable", "valid")
GRASP_FIELDS = ("pose_R", "pose_t", "dof", "q", "n_contacts", "contact_p", "contact_n",
                "contact_link", "objective", "penetration_free", "stable", "ik_converged")
REF_TESTS = ("geometry", "mesh", "convex", "wrench", "hand", "ik", "collision", "contact_field",
             "contact_opt")


def asset(*p):
    return os.path.join(ASSETS, *p)


def ref_inputs(cfg, hand, obj, batch, extra="", workers=8):
    return R.RefInputs(config=asset("configs", cfg), extra=extra, hand=asset("hands", hand),
                       object=asset("objects", obj), batch=batch, workers=workers,
                       out="/tmp/lg_ref_out")


def grasp_mismatches(a, b):
    assert len(a) == len(b), (len(a), len(b))
    bad = {}
    if len(a) == 0:
        return bad
    for f in GRASP_FIELDS:
        x = np.ascontiguousarray(a[f]).view(np.uint8).reshape(len(a), -1)
        y = np.ascontiguousarray(b[f]).view(np.uint8).reshape(len(b), -1)
        rows = np.nonzero((x != y).any(axis=1))[0] if len(a) else []
        if len(rows):
            bad[f] = list(rows)
    return bad


# ----------------------------------------------------------------- CPU side
def test_bundled_assets_are_the_references():
    ref_assets = "/root/reference/proj/assets"
    if not os.path.isdir(ref_assets):
        pytest.skip("reference tree not present (GPU box)")
    for dp, _, files in os.walk(ref_assets):
        for f in files:
            src = os.path.join(dp, f)
            dst = os.path.join(ROOT, "assets", os.path.relpath(src, ref_assets))
            assert filecmp.cmp(src, dst, shallow=False), dst


@pytest.mark.parametrize("name", REF_TESTS)
def test_reference_catch2_suite(name):
    """The reference's own unit tests (tests/test_<name>.cpp) on oracle/_ref."""
    exe = os.path.join(R.REF_DIR, f"test_{name}")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "All tests passed" in out.stdout


CPU_CASES = [
    ("four_finger.cfg", "four_finger.urdf", "sphere_r030.obj", 192, "passes = 2"),
    ("four_finger.cfg", "four_finger.urdf", "box_040.obj", 128, "passes = 1"),
    ("two_finger.cfg", "two_finger.urdf", "sphere_r030.obj", 192, "passes = 2"),
    ("four_finger.cfg", "four_finger.urdf", "scan_test.obj", 64,
     "passes = 1\nplacement_mode = exhaustive"),
]


@pytest.mark.parametrize("case", CPU_CASES, ids=lambda c: f"{c[1]}-{c[2]}-{c[3]}")
def test_oracle_restatement_matches_reference_run_batch(case):
    from oracle import orc_py as orc
    cfg, hand, obj, batch, extra = case
    inp = ref_inputs(cfg, hand, obj, batch, extra)
    ref = inp.run_batch()
    got = orc.run_batch(inp.hand_desc, inp.patches_desc, inp.raw, inp.params, workers=8)
    assert [got.profile[k] for k in FUNNEL] == [ref.profile[k] for k in FUNNEL]
    assert ref.profile["valid"] > 0
    assert grasp_mismatches(got.grasps, ref.grasps) == {}


def test_reference_inputs_round_trip():
    """The flat descriptors exported from the reference's HandModel are
    self-consistent (parts grouped by link, offsets monotone)."""
    inp = ref_inputs("four_finger.cfg", "four_finger.urdf", "sphere_r030.obj", 8)
    h = inp.hand_desc
    assert h.n_links == 13 and h.dof == 12
    pl = [h.part_link[i] for i in range(h.n_parts)]
    assert pl == sorted(pl)
    assert inp.raw.shape[1] == 6 and len(inp.raw) > 3000
    assert inp.n_groups == 4 and inp.patches_desc.n_patches > 100


# ----------------------------------------------------------------- GPU side
def _device_run(ctx, inp, field=None):
    import paper_2511_07418_b200 as lg
    hand = types.SimpleNamespace(desc=inp.hand_desc)
    patches = types.SimpleNamespace(desc=inp.patches_desc)
    return lg.run_batch(ctx, hand, patches, inp.raw, inp.params, field=field)


GPU_CASES = CPU_CASES + [
    # BASELINE configs[1] (Allegro-class, 5 cm box, bench settings), a shard
    ("allegro.cfg", "allegro_like.urdf", "box_050.obj", 384, ""),
    ("allegro.cfg", "allegro_like.urdf", "cylinder_r025_l100.obj", 256, ""),
    # configs[2] (LEAP-class on tools) at leap.cfg as written
    ("leap.cfg", "leap_like.urdf", "mug.obj", 192, ""),
    ("leap.cfg", "leap_like.urdf", "drill.obj", 256, ""),
    # k = 3 and k = 4 on small domains: the NC = 4 and NC = 6 instances of
    # the plain contact search
    ("allegro.cfg", "allegro_like.urdf", "box_050.obj", 160, "k_contacts = 3"),
    ("leap.cfg", "leap_like.urdf", "mug.obj", 128, "k_contacts = 4\nstatic_contact_prob = 0.5"),
    # the largest codebook the config accepts in shared memory for the query
    # kernels (C = 2048: 48 KiB of codebook plus the kernels' static arrays)
    ("four_finger.cfg", "four_finger.urdf", "sphere_r030.obj", 96,
     "codebook_size = 2048\nfield_configs = 48"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GPU_CASES, ids=lambda c: f"{c[1]}-{c[2]}-{c[3]}")
def test_device_matches_reference_run_batch(ctx, case):
    cfg, hand, obj, batch, extra = case
    inp = ref_inputs(cfg, hand, obj, batch, extra, workers=16)
    ref = inp.run_batch()
    dev = _device_run(ctx, inp)
    assert dev.profile["gpu_launches"] > 0
    assert [dev.profile[k] for k in FUNNEL] == [ref.profile[k] for k in FUNNEL]
    assert grasp_mismatches(dev.grasps, ref.grasps) == {}
