"""Host side of the boundary (CPU): the C-ABI library loads and exports every
symbol include/lg.h declares, the caller-side loaders match the reference's
structural tests and the oracle's restatements, config/JSONL behave like the
reference.  No device compute here."""
import ctypes
import json
import os
import re
import struct

import numpy as np
import pytest

import paper_2511_07418_b200 as lg
from paper_2511_07418_b200 import api
from oracle import orc_py as orc
from conftest import ROOT, asset


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "lg.h")).read()
    names = sorted(set(re.findall(r"\b(lg_[a-z0-9_]+)\s*\(", header)))
    assert len(names) > 40
    so = ctypes.CDLL(api.LIB_PATH)
    missing = [n for n in names if not hasattr(so, n)]
    assert missing == []


def test_no_cpu_fallback_without_device():
    if lg.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(lg.CudaError):
        lg.Context(0)


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


@pytest.mark.parametrize("body,msg", [
    ('<link name="a"/><link name="a"/>', "duplicate link"),
    ('<link name="a"/><link name="b"/><joint name="j" type="ball"><parent link="a"/>'
     '<child link="b"/></joint>', "unsupported joint type"),
    ('<link name="a"/><joint name="j" type="fixed"><parent link="a"/><child link="x"/></joint>',
     "unknown link"),
])
def test_urdf_errors(tmp_path, body, msg):
    p = tmp_path / "bad.urdf"
    p.write_text(f'<?xml version="1.0"?><robot name="r">{body}</robot>')
    with pytest.raises(RuntimeError, match=msg):
        lg.load_hand(str(p))


def test_mesh_loading_and_stl_weld(tmp_path):  # test_mesh.cpp
    m = lg.load_mesh(asset("objects", "sphere_r030.obj"))
    assert m.info()[:2] == (642, 1280)
    assert m.report["triangles_kept"] == 1280
    v, t = lg.Mesh.box((0.04, 0.04, 0.04)).arrays()
    stl = tmp_path / "b.stl"
    with open(stl, "wb") as f:
        f.write(b"\0" * 80 + struct.pack("<I", len(t)))
        for tri in t:
            f.write(struct.pack("<12fH", 0, 0, 0, *v[tri].ravel(), 0))
    ms = lg.load_mesh(str(stl))
    assert ms.info()[:2] == (8, 12)
    with pytest.raises(RuntimeError):
        lg.load_mesh(str(tmp_path / "missing.obj"))


def test_sample_surface_matches_oracle():  # mesh.cpp:297-339
    m = lg.load_mesh(asset("objects", "sphere_r030.obj"))
    v, t = m.arrays()
    a = lg.sample_surface(m, 30.0, lg.mix_seed(0, 0x6F626A73))
    b = orc.sample_surface(v, t, 30.0, lg.mix_seed(0, 0x6F626A73))
    assert a.shape == (3377, 6) and a.tobytes() == b.tobytes()


def test_patches_match_oracle_decomposition(four_finger):  # contact_field.cpp:26-99
    d = four_finger.desc
    spc, radius, seed = 30.0, 0.014, 0
    per = []
    for l in range(d.n_links):
        vis = four_finger.link_visual(l)
        vv, tt = vis.arrays()
        per.append(orc.sample_surface(vv, tt, spc, lg.mix_seed(seed, 0x686E6473, l)) if len(tt)
                   else np.zeros((0, 6)))
    op = orc.OrcPatches(d, per, radius, seed, 8)
    hp = lg.hand_patches(four_finger, spc, radius, seed, 8)
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
    d = lg.default_config()
    assert (d.batch, d.k_contacts, d.field_configs, d.theta_hit) == (1024, 3, 4096, 0.9397)
    p = lg.parse_config(asset("configs", "four_finger.cfg"), batch=7, seed=3)
    assert (p.k_contacts, p.field_configs, p.passes, p.batch, p.seed) == (2, 256, 6, 7, 3)
    assert tuple(p.canonical_center) == (0.0, 0.0, 0.055)
    c = tmp_path / "c.cfg"
    c.write_text("[run]\nbatch = 12 # comment\n")
    assert lg.parse_config(str(c)).batch == 12
    for bad in ("nope = 1", "batch = 0", "mu = x", "k_contacts = 9", "batch 3", "[oops"):
        c.write_text(bad + "\n")
        with pytest.raises(RuntimeError):
            lg.parse_config(str(c))
    with pytest.raises(RuntimeError, match="not found"):
        lg.parse_config(None, hand=str(tmp_path / "none.urdf"))


def test_cache_key(tmp_path):  # config.cpp:403-417
    p = lg.parse_config(asset("configs", "four_finger.cfg"), hand=asset("hands", "four_finger.urdf"))
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
    lg.write_dataset(str(path), g)
    line = path.read_text().strip()
    assert line.startswith('{"contacts":[{"link":4,"n":[0.0,0.0,1.0],"p":[1.0,2.0,3.0]}],'
                           '"flags":{"ik_converged":false,"penetration_free":false,"stable":true},'
                           '"objective":0.001,"pose":[')
    rec = json.loads(line)
    assert rec["pose"][4:] == [0.1, 1e-5, 2.0] and rec["q"] == [0.5, -1.25]
    assert rec["pose"][0] >= 0.0 and abs(abs(rec["pose"][1]) - 1.0) < 1e-15
    assert "1e-05" in line
