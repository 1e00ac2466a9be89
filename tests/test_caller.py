"""Host side of the boundary (CPU, no device compute):

* the product library loads, exports every symbol include/lg.h declares and
  nothing of the caller side (no loaders in libgraspgen_b200.so);
* the stand-in caller (caller/) reproduces the reference's own caller-side
  steps bit for bit — compared with the compiled reference (oracle/_ref):
  hand fixtures == load_hand, sample_surface, decompose_patches, parse_config,
  index_cache_key, write_dataset;
* the reference's structural expectations (test_hand.cpp, test_mesh.cpp)."""
import ctypes
import json
import os
import re
import struct

import numpy as np
import pytest

import caller as lc
import paper_2511_07418_b200 as lg
from paper_2511_07418_b200 import api
from oracle import orc_py as orc
from oracle import ref_py as R
from conftest import ROOT, asset

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "lg.h")).read()
    names = sorted(set(re.findall(r"\b(lg_[a-z0-9_]+)\s*\(", header)))
    assert len(names) > 25
    so = ctypes.CDLL(api.LIB_PATH)
    missing = [n for n in names if not hasattr(so, n)]
    assert missing == []


def test_product_exports_no_loaders():
    """The product's C-ABI is the device path plus flat descriptors: no URDF,
    mesh, sampling, config or dataset functions (they are the caller's)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", api.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted(re.findall(r" T (lg_[a-z0-9_]+)", out))
    for bad in ("load", "mesh", "sample_surface", "config_parse", "write_dataset", "hull"):
        assert not [n for n in exported if bad in n and n not in ("lg_field_load",)], bad
    header = open(os.path.join(ROOT, "include", "lg.h")).read()
    assert sorted(set(re.findall(r"\b(lg_[a-z0-9_]+)\s*\(", header))) == exported


def test_no_cpu_fallback_without_device():
    if lg.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(lg.CudaError):
        lg.Context(0)


def test_result_accessors_reject_null_handles():
    """The result accessors check their arguments (no device needed)."""
    import ctypes as C
    from paper_2511_07418_b200 import lgabi as A
    L = C.CDLL(lg.api.LIB_PATH)
    L.lg_result_profile.restype = C.c_int
    L.lg_result_profile.argtypes = [C.c_void_p, C.c_void_p]
    prof = A.Profile()
    assert L.lg_result_profile(None, C.byref(prof)) == -1  # LG_ERR_INVALID_ARGUMENT
    L.lg_result_num_grasps.restype = C.c_longlong
    L.lg_result_num_grasps.argtypes = [C.c_void_p]
    assert L.lg_result_num_grasps(None) == 0
    L.lg_result_grasps.restype = C.c_void_p
    L.lg_result_grasps.argtypes = [C.c_void_p]
    assert L.lg_result_grasps(None) is None


def test_four_finger_structure(four_finger):  # test_hand.cpp:31-105
    d = four_finger.desc
    assert (d.n_links, d.dof, d.n_parts) == (13, 12, 13)
    assert four_finger.link_name(0) == "palm" and d.root == 0
    g, n = four_finger.groups()
    assert n == 4 and g[0] == -1
    assert all(g[1 + 3 * i:4 + 3 * i].tolist() == [i] * 3 for i in range(4))
    assert np.allclose(four_finger.mid_config(), 0.1)


def test_two_finger_hull_parts(two_finger):
    d = two_finger.desc
    assert (d.n_links, d.dof, d.n_parts) == (7, 6, 7)
    planes = np.ctypeslib.as_array(d.part_plane_off, shape=(d.n_parts + 1,))
    assert (np.diff(planes) == 6).all()  # box hulls merge coplanar triangles into 6 planes


HANDS = ["four_finger", "two_finger", "allegro_like", "leap_like", "shadow_like"]


@needs_ref
@pytest.mark.parametrize("name", HANDS)
def test_hand_fixture_is_the_references_load_hand(name):
    """assets/prepared/<hand>.hand.npz == the reference's load_hand +
    dependency_groups on the URDF today (tools/prepare_hands.py)."""
    want = R.load_hand_arrays(asset("hands", f"{name}.urdf"))
    got = np.load(os.path.join(ROOT, "assets", "prepared", f"{name}.hand.npz"))
    for k, v in want.items():
        if isinstance(v, np.ndarray) and v.dtype.kind in "fiu":
            assert np.asarray(got[k]).tobytes() == v.tobytes(), k
        else:
            assert np.array_equal(np.asarray(got[k]), np.asarray(v)), k


def test_mesh_loading_and_stl_weld(tmp_path):  # test_mesh.cpp
    m = lc.load_mesh(asset("objects", "sphere_r030.obj"))
    assert m.info()[:2] == (642, 1280)
    assert m.report["triangles_kept"] == 1280
    v, t = lc.Mesh.box((0.04, 0.04, 0.04)).arrays()
    stl = tmp_path / "b.stl"
    with open(stl, "wb") as f:
        f.write(b"\0" * 80 + struct.pack("<I", len(t)))
        for tri in t:
            f.write(struct.pack("<12fH", 0, 0, 0, *v[tri].ravel(), 0))
    ms = lc.load_mesh(str(stl))
    assert ms.info()[:2] == (8, 12)
    with pytest.raises(RuntimeError):
        lc.load_mesh(str(tmp_path / "missing.obj"))


def test_sample_surface_matches_oracle():  # mesh.cpp:297-339
    m = lc.load_mesh(asset("objects", "sphere_r030.obj"))
    v, t = m.arrays()
    a = lc.sample_surface(m, 30.0, lg.mix_seed(0, 0x6F626A73))
    b = orc.sample_surface(v, t, 30.0, lg.mix_seed(0, 0x6F626A73))
    assert a.shape == (3377, 6) and a.tobytes() == b.tobytes()


@needs_ref
@pytest.mark.parametrize("cfg,hand,obj", [
    ("four_finger.cfg", "four_finger", "sphere_r030.obj"),
    ("two_finger.cfg", "two_finger", "box_040.obj"),
    ("allegro.cfg", "allegro_like", "cylinder_r025_l100.obj"),
    ("leap.cfg", "leap_like", "drill.obj"),
])
def test_caller_inputs_equal_the_references(cfg, hand, obj):
    """parse_config, the hand's patches and the object's samples from the
    caller are the reference's own (pipeline.cpp:273-331)."""
    ref = R.RefInputs(config=asset("configs", cfg), hand=asset("hands", f"{hand}.urdf"),
                      object=asset("objects", obj), batch=16)
    p = lc.parse_config(asset("configs", cfg), hand=asset("hands", f"{hand}.urdf"),
                        object=asset("objects", obj), batch=16)
    for name, _ in p._fields_:
        a, b = getattr(p, name), getattr(ref.params, name)
        a = bytes(a) if hasattr(a, "_length_") else a
        b = bytes(b) if hasattr(b, "_length_") else b
        if name not in ("out", "workers"):
            assert a == b, name
    h, patches, raw, _ = lc.prepare_inputs(p)
    assert raw.tobytes() == ref.raw.tobytes()
    a, b = patches.desc, ref.patches_desc
    P = a.n_patches
    assert P == b.n_patches
    arr = np.ctypeslib.as_array
    for f, n in (("link", P), ("point_off", P + 1), ("fp_off", P + 1)):
        assert np.array_equal(arr(getattr(a, f), shape=(n,)), arr(getattr(b, f), shape=(n,)))
    npts, nfp = arr(a.point_off, shape=(P + 1,))[-1], arr(a.fp_off, shape=(P + 1,))[-1]
    for f in ("points", "normals"):
        assert arr(getattr(a, f), shape=(3 * npts,)).tobytes() == \
            arr(getattr(b, f), shape=(3 * npts,)).tobytes()
    assert np.array_equal(arr(a.field_points, shape=(nfp,)), arr(b.field_points, shape=(nfp,)))
    assert lc.index_cache_key(p) == lg.index_cache_key(p) == ref.cache_key()


def test_patches_match_oracle_decomposition(four_finger):  # contact_field.cpp:26-99
    d = four_finger.desc
    spc, radius, seed = 30.0, 0.014, 0
    per = []
    for l in range(d.n_links):
        vv, tt = four_finger.link_visual(l)
        per.append(orc.sample_surface(vv, tt, spc, lg.mix_seed(seed, 0x686E6473, l)) if len(tt)
                   else np.zeros((0, 6)))
    op = orc.OrcPatches(d, per, radius, seed, 8)
    hp = lc.hand_patches(four_finger, spc, radius, seed, 8)
    a, b = hp.desc, op.desc
    assert a.n_patches == b.n_patches == 767
    P = a.n_patches
    arr = np.ctypeslib.as_array
    for f, n in (("link", P), ("point_off", P + 1), ("fp_off", P + 1)):
        assert np.array_equal(arr(getattr(a, f), shape=(n,)), arr(getattr(b, f), shape=(n,)))
    npts = arr(a.point_off, shape=(P + 1,))[-1]
    assert arr(a.points, shape=(3 * npts,)).tobytes() == arr(b.points, shape=(3 * npts,)).tobytes()
    nfp = arr(a.fp_off, shape=(P + 1,))[-1]
    assert np.array_equal(arr(a.field_points, shape=(nfp,)), arr(b.field_points, shape=(nfp,)))


def test_config_parse_and_errors(tmp_path):  # config.cpp:69-401
    d = lc.default_config()
    assert (d.batch, d.k_contacts, d.field_configs, d.theta_hit) == (1024, 3, 4096, 0.9397)
    p = lc.parse_config(asset("configs", "four_finger.cfg"), batch=7, seed=3)
    assert (p.k_contacts, p.field_configs, p.passes, p.batch, p.seed) == (2, 256, 6, 7, 3)
    assert tuple(p.canonical_center) == (0.0, 0.0, 0.055)
    c = tmp_path / "c.cfg"
    c.write_text("[run]\nbatch = 12 # comment\n")
    assert lc.parse_config(str(c)).batch == 12
    for bad in ("nope = 1", "batch = 0", "mu = x", "k_contacts = 9", "batch 3", "[oops"):
        c.write_text(bad + "\n")
        with pytest.raises(RuntimeError):
            lc.parse_config(str(c))
    with pytest.raises(RuntimeError, match="not found"):
        lc.parse_config(None, hand=str(tmp_path / "none.urdf"))


def test_cache_key(tmp_path):  # config.cpp:403-417
    p = lc.parse_config(asset("configs", "four_finger.cfg"), hand=asset("hands", "four_finger.urdf"))
    k = lg.index_cache_key(p)
    assert k == lg.index_cache_key(p)
    p.seed = 1
    assert lg.index_cache_key(p) != k


def test_jsonl_result_format(tmp_path):  # dataset.cpp:23-56
    from paper_2511_07418_b200 import lgabi as A
    g = np.zeros(1, dtype=A.grasp_dtype())
    g["pose_R"][0] = np.diag([1.0, -1.0, -1.0]).ravel()  # 180 deg about x: w = 0
    g["pose_t"][0] = [0.1, 1e-5, 2.0]
    g["dof"] = 2
    g["q"][0, :2] = [0.5, -1.25]
    g["n_contacts"] = 1
    g["contact_p"][0, 0] = [1, 2, 3]
    g["contact_n"][0, 0] = [0, 0, 1]
    g["contact_link"][0, 0] = 4
    g["objective"] = 0.001
    g["stable"] = 1
    path = tmp_path / "g.jsonl"
    lc.write_dataset(str(path), g)
    line = path.read_text().strip()
    assert line.startswith('{"contacts":[{"link":4,"n":[0.0,0.0,1.0],"p":[1.0,2.0,3.0]}],'
                           '"flags":{"ik_converged":false,"penetration_free":false,"stable":true},'
                           '"objective":0.001,"pose":[')
    rec = json.loads(line)
    assert rec["pose"][4:] == [0.1, 1e-5, 2.0] and rec["q"] == [0.5, -1.25]
    assert rec["pose"][0] >= 0.0 and abs(abs(rec["pose"][1]) - 1.0) < 1e-15
    assert "1e-05" in line
