"""Seed sharding across GPUs and the final gather of valid grasps
(SURVEY.md 8(e)).

Rank r of R owns candidates c in [r*B/R, (r+1)*B/R) for every pass; every
per-candidate RNG stream depends only on (seed, tag, c or g), so the union of
the shards is the single-GPU result.  The only collective is the final
gather: per-rank grasp records as byte tensors, padded to the largest rank,
all-gathered once (NCCL on GPUs, gloo in the CPU tests), then sorted by
g = pass*batch + c to reproduce run_batch's `kept` order (pipeline.cpp:607-614).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import lgabi as A


def shard_params(params, rank, world):
    p = A.RunParams()
    C.pointer(p)[0] = params
    p.shard_rank = int(rank)
    p.shard_count = int(world)
    return p


def shard_range(batch, rank, world):
    return batch * rank // world, batch * (rank + 1) // world


def gather_records(records, device=None, group=None):
    """All-gather a structured numpy array from every rank; returns the
    concatenation in rank order (every rank receives it)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    raw = np.ascontiguousarray(records).view(np.uint8).reshape(-1)
    n = torch.tensor([raw.size], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    cap = int(max(s.item() for s in sizes))
    buf = torch.zeros(max(cap, 1), dtype=torch.uint8, device=device)
    if raw.size:
        buf[:raw.size] = torch.from_numpy(raw.copy()).to(buf.device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    parts = [o[:int(s.item())].cpu().numpy() for o, s in zip(outs, sizes)]
    cat = np.concatenate(parts) if parts else np.zeros(0, np.uint8)
    return cat.view(records.dtype)


def merge_grasps(grasps):
    """Order gathered grasps by candidate id g (pipeline.cpp:607-614)."""
    if len(grasps) == 0:
        return grasps
    return grasps[np.argsort(grasps["g"], kind="stable")]


def sum_profiles(profiles):
    """Funnel counts add across shards; stage times are the max over ranks."""
    out = dict(profiles[0])
    for p in profiles[1:]:
        for k, v in p.items():
            if k in ("placement_domains", "contact_optimization", "kinematics_optimization",
                     "postprocessing", "total", "field_build"):
                out[k] = max(out[k], v)
            elif k in ("patches", "boxes", "field_vectors", "object_samples", "field_samples"):
                out[k] = v
            else:
                out[k] = out[k] + v
    out["grasps_per_second"] = out["valid"] / out["total"] if out["total"] > 0 else 0.0
    return out
