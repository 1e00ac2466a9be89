"""The drop-in, end to end: integration/graspgen_b200.cpp (the adapter a
maintainer adds to the reference) linked into the reference's own binaries
in place of run_batch, optimize_contacts, validate_grasp_collisions,
solve_contact_ik, ContactFieldIndex::build, query_domains, reverse_lookup,
solve_fswo / solve_gswo / is_stable and validate_dataset (oracle/Makefile
`integration`):

* the reference's CLI on the device: `synthesize` writes the same
  grasps.jsonl, byte for byte, as the unmodified reference CLI; `build-index`
  writes the same index_cache.bin and report; `validate` reports the same
  issues;
* the reference's own Catch2 suites (contact_opt, collision, ik,
  contact_field, wrench) pass with those functions served by the device.
"""
import json
import os
import subprocess

import pytest

from conftest import ASSETS
from oracle import ref_py as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(os.path.join(R.REF_DIR, "graspgen_b200")),
                                 reason="oracle/_ref integration binaries not built")]


def _run(exe, *args, timeout=900):
    out = subprocess.run([os.path.join(R.REF_DIR, exe), *args], capture_output=True, text=True,
                         timeout=timeout)
    return out


@pytest.mark.parametrize("suite", ["contact_opt", "collision", "ik", "contact_field", "wrench"])
def test_reference_catch2_suite_on_the_device(suite):
    out = _run(f"test_{suite}_b200")
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "All tests passed" in out.stdout


@pytest.mark.parametrize("hand,obj,cfg,batch", [
    ("four_finger.urdf", "sphere_r030.obj", "four_finger.cfg", 256),
    ("two_finger.urdf", "box_040.obj", "two_finger.cfg", 256),
])
def test_reference_cli_on_the_device_writes_the_same_dataset(tmp_path, hand, obj, cfg, batch):
    args = ["synthesize", "--hand", os.path.join(ASSETS, "hands", hand),
            "--object", os.path.join(ASSETS, "objects", obj),
            "--config", os.path.join(ASSETS, "configs", cfg), "--seed", "0",
            "--batch", str(batch), "--workers", "0"]
    ref = _run("graspgen", *args, "--out", str(tmp_path / "ref"))
    dev = _run("graspgen_b200", *args, "--out", str(tmp_path / "dev"))
    assert ref.returncode in (0, 1) and dev.returncode == ref.returncode, dev.stderr[-2000:]
    a = (tmp_path / "ref" / "grasps.jsonl").read_bytes()
    b = (tmp_path / "dev" / "grasps.jsonl").read_bytes()
    assert len(a) > 0 and a == b
    pa = json.loads((tmp_path / "ref" / "profile.json").read_text())
    pb = json.loads((tmp_path / "dev" / "profile.json").read_text())
    for k in ("candidates", "placements_accepted", "contact_sets_balanced", "ik_finite",
              "penetration_free", "ik_converged", "stable", "valid"):
        assert pa[k] == pb[k], k
    # RunResult.loads and RunResult.index (patches, boxes, memory_bytes, cache)
    assert (tmp_path / "ref" / "load_report.json").read_bytes() == \
        (tmp_path / "dev" / "load_report.json").read_bytes()

    def stage(out, tag):
        return [ln for ln in out.stdout.splitlines() if ln.startswith("[stage] " + tag)]
    for tag in ("load", "field"):
        assert stage(ref, tag) and stage(ref, tag) == stage(dev, tag), tag


def test_reference_cli_build_index_on_the_device(tmp_path):
    """`graspgen build-index` (build_field -> ContactFieldIndex::build on the
    device): the same GGCF file and the same per-patch report."""
    args = ["build-index", "--hand", os.path.join(ASSETS, "hands", "four_finger.urdf"),
            "--config", os.path.join(ASSETS, "configs", "four_finger.cfg"), "--seed", "3"]
    ref = _run("graspgen", *args, "--out", str(tmp_path / "ref"))
    dev = _run("graspgen_b200", *args, "--out", str(tmp_path / "dev"))
    assert ref.returncode == 0 and dev.returncode == 0, dev.stderr[-2000:]
    a = (tmp_path / "ref" / "index_cache.bin").read_bytes()
    b = (tmp_path / "dev" / "index_cache.bin").read_bytes()
    assert len(a) > 0 and a == b
    strip = lambda out: [ln.replace(str(tmp_path / "dev"), "OUT").replace(str(tmp_path / "ref"), "OUT")
                         for ln in out.stdout.splitlines()]
    assert strip(ref) == strip(dev)


def test_reference_cli_validate_on_the_device(tmp_path):
    """`graspgen validate` (validate_dataset on the device) on a dataset the
    reference synthesized, and on a tampered copy: the same issue lines."""
    common = ["--hand", os.path.join(ASSETS, "hands", "four_finger.urdf"),
              "--object", os.path.join(ASSETS, "objects", "sphere_r030.obj"),
              "--config", os.path.join(ASSETS, "configs", "four_finger.cfg"), "--seed", "0"]
    syn = _run("graspgen", "synthesize", *common, "--batch", "256", "--workers", "0",
               "--out", str(tmp_path / "syn"))
    assert syn.returncode == 0, syn.stderr[-2000:]
    ds = tmp_path / "syn" / "grasps.jsonl"
    lines = ds.read_text().splitlines()
    bad = []
    for i, ln in enumerate(lines):
        g = json.loads(ln)
        if i % 3 == 1:
            g["q"][0] += 3.0  # out of limits
        if i % 3 == 2 and g.get("contacts"):
            g["contacts"][0]["p"][0] += 0.01  # off the surfaces
        bad.append(json.dumps(g))
    tampered = tmp_path / "tampered.jsonl"
    tampered.write_text("\n".join(bad) + "\n")
    for path in (ds, tampered):
        ref = _run("graspgen", "validate", *common, "--dataset", str(path))
        dev = _run("graspgen_b200", "validate", *common, "--dataset", str(path))
        assert ref.returncode == dev.returncode, dev.stderr[-2000:]
        assert ref.stdout == dev.stdout and "[result]" in ref.stdout
    assert "issues=0" not in _run("graspgen", "validate", *common, "--dataset", str(tampered)).stdout
