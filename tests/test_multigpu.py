"""Multi-GPU path on one B200: seed shards run on the device
reproduce the unsharded run exactly, and the NCCL gather behind the C-ABI
(lg_comm_*) returns the kept grasps in run_batch's order with the summed
funnel.  (Only one GPU is available to the tests; the host-side sharding and
merge logic is also covered with a world-size-2 gloo group in
test_sharding.py.)"""
import numpy as np
import pytest

import caller as lc
import paper_2511_07418_b200 as lg
from paper_2511_07418_b200 import dist as ldist
from conftest import cfg1, mismatched_fields

FUNNEL = ("candidates", "placements_accepted", "contact_sets_balanced", "ik_finite",
          "penetration_free", "ik_converged", "stable", "valid")


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_device_seed_shards_merge_to_the_full_run(ctx, world):
    p = cfg1(batch=96, passes=2)
    p.want_trace = 0
    hand, patches, raw, _ = lc.prepare_inputs(p)
    full = lg.run_batch(ctx, hand, patches, raw, p)
    parts, funnel = [], {k: 0 for k in FUNNEL}
    for r in range(world):
        res = lg.run_batch(ctx, hand, patches, raw, ldist.shard_params(p, r, world))
        parts.append(res.grasps)
        for k in FUNNEL:
            funnel[k] += res.profile[k]
    merged = ldist.merge_grasps(np.concatenate(parts))
    assert full.profile["valid"] > 0
    assert funnel == {k: full.profile[k] for k in FUNNEL}
    assert mismatched_fields(merged, full.grasps) == {}


@pytest.mark.gpu
def test_nccl_gather_single_rank(ctx):
    p = cfg1(batch=64, passes=1)
    p.want_trace = 0
    hand, patches, raw, _ = lc.prepare_inputs(p)
    res = lg.run_batch(ctx, hand, patches, raw, p)
    comm = ldist.Comm(ctx, 0, 1, ldist.Comm.unique_id())
    g, prof = comm.gather(res)
    comm.close()
    assert len(g) == len(res.grasps) > 0
    assert mismatched_fields(g, res.grasps) == {}
    assert {k: prof[k] for k in FUNNEL} == {k: res.profile[k] for k in FUNNEL}
    assert prof["device_seconds"] == res.profile["device_seconds"]
