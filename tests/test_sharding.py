"""Seed sharding with a world-size-2 gloo group on CPU:
each rank runs its candidate shard (through the oracle here: no device on
this host) and the final gather reproduces the single-rank result exactly."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT, cfg1, mismatched_fields


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def gather_records(records):
    """All-gather a structured array over the process group (gloo here; the
    device path gathers over NCCL behind the C-ABI, lg_comm_gather)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    raw = np.ascontiguousarray(records).view(np.uint8).reshape(-1)
    n = torch.tensor([raw.size], dtype=torch.int64)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    cap = int(max(s.item() for s in sizes))
    buf = torch.zeros(max(cap, 1), dtype=torch.uint8)
    if raw.size:
        buf[:raw.size] = torch.from_numpy(raw.copy())
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    parts = [o[:int(s.item())].numpy() for o, s in zip(outs, sizes)]
    return np.concatenate(parts).view(records.dtype)


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    import caller as lc
    import paper_2511_07418_b200 as lg
    from paper_2511_07418_b200 import dist as ldist
    from oracle import orc_py as orc
    from conftest import cfg1 as mk

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = mk(batch=20, passes=2, field_configs=40)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    sp = ldist.shard_params(p, rank, world)
    r = orc.run_batch(hand.desc, patches.desc, raw, sp, workers=1)
    g = ldist.merge_grasps(gather_records(r.grasps))
    t = gather_records(r.traces)
    if rank == 0:
        np.save(os.path.join(outdir, "grasps.npy"), g)
        np.save(os.path.join(outdir, "traces.npy"), t)
    dist.destroy_process_group()


def test_seed_sharding_is_result_invariant(tmp_path):
    import torch.multiprocessing as mp
    import caller as lc
    import paper_2511_07418_b200 as lg
    from oracle import orc_py as orc

    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    g = np.load(tmp_path / "grasps.npy")
    t = np.load(tmp_path / "traces.npy")
    p = cfg1(batch=20, passes=2, field_configs=40)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    full = orc.run_batch(hand.desc, patches.desc, raw, p, workers=2)
    # traces: rank order = (rank, pass, c); reorder by (pass, c) before comparing
    order = np.lexsort((t["c"], t["pass_"]))
    assert mismatched_fields(t[order], full.traces) == {}
    assert len(g) == len(full.grasps)
    assert mismatched_fields(g, full.grasps) == {}
