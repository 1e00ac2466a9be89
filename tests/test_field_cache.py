"""Contact-field cache in the reference's GGCF v1 format
(contact_field.cpp:507-655) and the run_batch cache mode (pipeline.cpp:286-304).

CPU: the oracle's writer against a restated reader (tests/ggcf.py) - stream
layout, BVH shape, key / truncation rejection.  GPU: the device writer is
byte-identical to the oracle's, the loader round-trips, and run_batch with
cache=1 builds+saves, then loads, with bit-identical grasps."""
import os

import numpy as np
import pytest

import caller as lc
import paper_2511_07418_b200 as lg
from oracle import orc_py as orc
from conftest import cfg1, mismatched_fields
import ggcf


def _oracle_field(p, N=64, C=64):
    hand, patches, _, _ = lc.prepare_inputs(p)
    return hand, patches, orc.OrcField(hand.desc, patches.desc, N, p.box_width, p.seed, C)


def test_oracle_file_layout(tmp_path):
    p = cfg1()
    _, _, fo = _oracle_field(p)
    key = lg.index_cache_key(p)
    path = tmp_path / "index_cache.bin"
    fo.save(path, key)
    d = ggcf.read(path, key)
    assert d is not None and d["trailing"] == 0
    ex = fo.export()
    assert d["box_width"] == ex["box_width"]
    assert np.array_equal(np.array(d["codebook"]), ex["codebook"])
    assert len(d["patches"]) == len(ex["patch_link"])
    q = 0
    b_all = 0
    for i, P in enumerate(d["patches"]):
        assert P["patch_id"] == i and P["link"] == ex["patch_link"][i]
        nb = len(P["boxes"])
        assert nb == ex["patch_box_off"][i + 1] - ex["patch_box_off"][i]
        # median-split BVH (contact_field.cpp:190-224): 2n-1 nodes, root last,
        # leaves cover every box once
        assert len(P["nodes"]) == 2 * nb - 1 and P["root"] == len(P["nodes"]) - 1
        leaves = sorted(n["leaf"] for n in P["nodes"] if n["leaf"] >= 0)
        assert leaves == list(range(nb))
        for bi, B in enumerate(P["boxes"]):
            assert tuple(B["cell"]) == tuple(ex["box_cell"][b_all])
            for code, rl, pt, nm in B["reps"]:
                assert code == ex["codes"][q] and rl == ex["rep_link"][q]
                assert np.array_equal(pt, ex["rep_point"][q])
                assert np.array_equal(nm, ex["rep_normal"][q])
                q += 1
            b_all += 1
        for n in P["nodes"]:
            if n["leaf"] >= 0:
                c = np.array(P["boxes"][n["leaf"]]["cell"], dtype=float)
                w = d["box_width"]
                assert np.array_equal(n["min"], c * w - 1e-9)
                assert np.array_equal(n["max"], (c + 1) * w + 1e-9)
    assert q == len(ex["codes"])
    assert len(d["top_nodes"]) == 2 * len(d["patches"]) - 1
    # rejected like the reference's std::nullopt
    assert ggcf.read(path, key ^ 1) is None
    raw = open(path, "rb").read()
    (tmp_path / "trunc.bin").write_bytes(raw[: len(raw) // 2])
    assert ggcf.read(tmp_path / "trunc.bin", key) is None
    (tmp_path / "bad.bin").write_bytes(b"GGCX" + raw[4:])
    assert ggcf.read(tmp_path / "bad.bin", key) is None


def test_cache_key_tracks_config():  # config.cpp:403-417
    p = cfg1()
    k0 = lg.index_cache_key(p)
    assert k0 == lg.index_cache_key(cfg1())
    p.box_width = p.box_width * 2
    assert lg.index_cache_key(p) != k0
    p2 = cfg1()
    p2.batch = 999  # not part of the index key
    assert lg.index_cache_key(p2) == k0


@pytest.mark.gpu
@pytest.mark.parametrize("hand_name,N,C", [("four_finger", 256, 256), ("two_finger", 64, 64)])
def test_device_file_bytes_equal_oracle(ctx, tmp_path, hand_name, N, C):
    p = cfg1(hand=hand_name)
    hand, patches, _, _ = lc.prepare_inputs(p)
    key = lg.index_cache_key(p)
    fd = lg.ContactFieldIndex.build(ctx, hand, patches, N, p.box_width, p.seed, C)
    fo = orc.OrcField(hand.desc, patches.desc, N, p.box_width, p.seed, C)
    fd.save(tmp_path / "dev.bin", key)
    fo.save(tmp_path / "orc.bin", key)
    assert (tmp_path / "dev.bin").read_bytes() == (tmp_path / "orc.bin").read_bytes()
    # load -> export reproduces the built index; wrong key / missing / truncated -> None
    ld = lg.ContactFieldIndex.load(ctx, hand, tmp_path / "orc.bin", key)
    assert ld is not None
    a, b = ld.export(), fd.export()
    for k in a:
        if k != "n_vectors":
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    assert lg.ContactFieldIndex.load(ctx, hand, tmp_path / "orc.bin", key + 1) is None
    assert lg.ContactFieldIndex.load(ctx, hand, tmp_path / "missing.bin", key) is None
    raw = (tmp_path / "orc.bin").read_bytes()
    (tmp_path / "t.bin").write_bytes(raw[:-3])
    assert lg.ContactFieldIndex.load(ctx, hand, tmp_path / "t.bin", key) is None
    # a loaded index answers queries exactly like the built one
    gl, _ = hand.groups()
    gop = gl[patches.link_of_patch()]
    _, _, raw_s, _ = lc.prepare_inputs(p)
    poses = np.tile(np.concatenate([np.eye(3).ravel(), [0, 0, 0.05]]), (4, 1))
    poses[:, 9:] += np.random.default_rng(3).normal(scale=0.01, size=(4, 3))
    assert np.array_equal(lg.query_domains_batch(ctx, ld, gop, raw_s, poses, p.theta_hit),
                          lg.query_domains_batch(ctx, fd, gop, raw_s, poses, p.theta_hit))


@pytest.mark.gpu
def test_run_batch_cache_mode(tmp_path):
    p = cfg1(batch=96)
    p.cache = 1
    p.out = os.fsencode(str(tmp_path / "out"))
    hand, patches, raw, _ = lc.prepare_inputs(p)
    ctx = lg.Context(0)
    first = lg.run_batch(ctx, hand, patches, raw, p)
    assert first.profile["index_from_cache"] == 0
    assert (tmp_path / "out" / "index_cache.bin").exists()
    second = lg.run_batch(ctx, hand, patches, raw, p)
    ctx.close()
    assert second.profile["index_from_cache"] == 1
    ref = orc.run_batch(hand.desc, patches.desc, raw, cfg1(batch=96), workers=0)
    assert mismatched_fields(second.traces, ref.traces) == {}
    assert mismatched_fields(second.grasps, first.grasps) == {}
    d = ggcf.read(tmp_path / "out" / "index_cache.bin", lg.index_cache_key(p))
    assert d is not None and d["trailing"] == 0
