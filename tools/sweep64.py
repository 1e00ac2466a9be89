"""BASELINE config 5: a 64-object sweep with one contact field per GPU
(built once from the hand, reused for every object through
lg_run_batch_field), objects sharded round-robin over ranks (object o ->
rank o mod R), in the "performance-optimized low-diversity mode" SURVEY 8(d)
defines as config overrides (restarts=1, lookup_attempts=1,
unused_attempts=4).  Not the bench line; prints one JSON line.

  python tools/sweep64.py [--objects 64] [--batch 2000]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/sweep64.py
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import caller as lc  # noqa: E402
import paper_2511_07418_b200 as lg  # noqa: E402

LOW_DIVERSITY = dict(restarts=1, lookup_attempts=1, unused_attempts=4)


def make_object(o):
    """Primitive with randomised dimensions, seed = object id."""
    rng = np.random.default_rng(o)
    kind = o % 3
    if kind == 0:
        return "box", lc.Mesh.box(tuple(rng.uniform(0.03, 0.07, size=3)))
    if kind == 1:
        return "cylinder", lc.Mesh.cylinder(float(rng.uniform(0.015, 0.03)),
                                            float(rng.uniform(0.06, 0.12)), 24)
    return "sphere", lc.Mesh.icosphere(float(rng.uniform(0.02, 0.035)), 3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--objects", type=int, default=64)
    ap.add_argument("--batch", type=int, default=2000)
    ap.add_argument("--full-diversity", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    a = os.path.join(ROOT, "assets")
    p = lc.parse_config(os.path.join(a, "configs", "allegro.cfg"),
                        hand=os.path.join(a, "hands", "allegro_like.urdf"),
                        object=os.path.join(a, "objects", "box_050.obj"), batch=args.batch)
    p.want_trace = 0
    if not args.full_diversity:
        for k, v in LOW_DIVERSITY.items():
            setattr(p, k, v)
    hand, patches, _, _ = lc.prepare_inputs(p)
    ctx = lg.Context(local)
    field = lg.ContactFieldIndex.build(ctx, hand, patches, p.field_configs, p.box_width, p.seed,
                                       p.codebook_size)
    mine = [o for o in range(args.objects) if o % world == rank]
    dev_s, valid, cand, t0 = 0.0, 0, 0, time.perf_counter()
    for o in mine:
        _, mesh = make_object(o)
        raw = lc.sample_surface(mesh, p.samples_per_cm2, lg.mix_seed(p.seed, 0x6f626a73))
        r = lg.run_batch(ctx, hand, patches, raw, p, field=field)
        dev_s += r.profile["device_seconds"]
        valid += int(r.profile["valid"])
        cand += int(r.profile["candidates"])
    wall = time.perf_counter() - t0
    if world > 1:
        import torch
        t = torch.tensor([dev_s, wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        c = torch.tensor([valid, cand], dtype=torch.float64, device="cuda")
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        dev_s, wall = float(t[0]), float(t[1])
        valid, cand = int(c[0]), int(c[1])
    if rank == 0:
        print(json.dumps(dict(workload="sweep64", objects=args.objects, n_gpus=world,
                              batch_per_object=args.batch, mode="full" if args.full_diversity
                              else "low-diversity " + json.dumps(LOW_DIVERSITY),
                              candidates=cand, valid=valid,
                              valid_per_s_device=valid / dev_s if dev_s else 0.0,
                              device_seconds_max_rank=dev_s, wall_seconds_max_rank=wall,
                              field="one per GPU, reused across objects")))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
