"""Benchmark: valid grasps/s of the Lightning Grasp forward pass (BASELINE.json
metric) on the Allegro-class config (BASELINE configs[1]).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (seed-sharded, NCCL gather)

A step is one run_batch forward pass over the full candidate batch: field
build, preprocess, placement + domains, contact search, realisation +
collision filter, postprocess.  `value` uses the pass's device time (CUDA
events on the library stream, inputs resident); `e2e` is the same pass
through the public C-ABI call with host buffers (H2D of the hand, patches and
object samples, D2H of the results) timed with CUDA events around the call.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE configs[1]: Allegro-class 16-DoF hand on a box mesh, 10k seeds.
    "allegro_box": dict(hand="hands/allegro_like.urdf", obj="objects/box_050.obj",
                        cfg="configs/allegro.cfg"),
    "allegro_cylinder": dict(hand="hands/allegro_like.urdf", obj="objects/cylinder_r025_l100.obj",
                             cfg="configs/allegro.cfg"),
    # configs[2]: LEAP-class hand on tool-like primitive unions (100k seeds, 8 GPUs)
    "leap_mug": dict(hand="hands/leap_like.urdf", obj="objects/mug.obj", cfg="configs/leap.cfg"),
    "leap_hammer": dict(hand="hands/leap_like.urdf", obj="objects/hammer.obj",
                        cfg="configs/leap.cfg"),
    "leap_drill": dict(hand="hands/leap_like.urdf", obj="objects/drill.obj", cfg="configs/leap.cfg"),
    # configs[3]: Shadow-class 22-DoF hand, high-poly object (~113k samples)
    "shadow_icosphere": dict(hand="hands/shadow_like.urdf", obj="objects/icosphere_r030_s6.obj",
                             cfg="configs/shadow.cfg"),
    # configs[0]: the reference's bundled CPU-runnable case
    "four_finger_sphere": dict(hand="hands/four_finger.urdf", obj="objects/sphere_r030.obj",
                               cfg="configs/four_finger.cfg"),
}
METRIC = "valid grasps/sec per object at 1/2/4/8 B200; forward-pass seconds"
UNIT = "valid grasps/s"


def params_for(workload, batch=None):
    import caller as lc
    import paper_2511_07418_b200 as lg
    w = WORKLOADS[workload]
    a = os.path.join(ROOT, "assets")
    p = lc.parse_config(os.path.join(a, w["cfg"]), hand=os.path.join(a, w["hand"]),
                        object=os.path.join(a, w["obj"]), batch=batch)
    p.want_trace = 0
    return p


# ------------------------------------------------------------ clock sampling
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.proc = None
        self.gpu = gpu
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------- roofline model
# Algorithmic FP64 work per counted unit; n = contacts per
# wrench problem, dof / links / chain depth from the hand.
def flop_model(prof, k, n_static_frac, mu, dof, links, depth):
    n = k + n_static_frac
    fr = 1 if mu > 0 else 0
    wrench = prof["wrench_evals"] * (36 * n + 12) + \
        prof["wrench_grads"] * (36 * n + 12 * n * (1 + 2 * fr) + 3)
    proj = prof["proj_evals"] * 8
    ik = prof["ik_iterations"] * (2 * k * depth * 12 + 2 * 6 * k * dof * dof + dof ** 3 / 3) + \
        prof["fk_evals"] * (60 * links + 20 * k)
    return dict(contact_opt=wrench + proj, realize=ik)


def kernel_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    summary of the default bench workload (tools/ncu_summary.py)."""
    path = os.path.join(ROOT, "profiles", "r01", "ncu_full_summary.json")
    try:
        with open(path) as f:
            rows = json.load(f)
    except (OSError, ValueError):
        return None, None
    names = {"k_contact_opt": "k_contact_opt2", "k_realize": "k_realize_warp"}
    want = names.get(kernel, kernel)
    for r in rows:
        if r["kernel"].startswith(want) and "dram_bytes" in r:
            return r["dram_bytes"], os.path.relpath(path, ROOT)
    return None, None


def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["fp64_tflops"]), "measured (profiles/fp64_peak.json, DFMA loop)"
    except (OSError, KeyError, ValueError):
        # 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
        return 148 * 64 * 2 * 1.965e9 / 1e12, "derived (148 SM x 64 DFMA/clk x 2 x 1.965 GHz)"


# ------------------------------------------------------------ CPU baseline
def cpu_baseline(workload, batch, sample_frac, hand, patches, raw, p):
    """The oracle (CPU restatement of the reference) on the box's host cores:
    field build once (single-threaded, as in the reference), then a bounded
    sample = one 1/sample_frac shard of the batch on all cores; grasps/s is
    extrapolated to the full batch with the field build amortised over it."""
    from oracle import orc_py as orc
    from paper_2511_07418_b200 import dist as ldist
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    field = orc.OrcField(hand.desc, patches.desc, p.field_configs, p.box_width, p.seed,
                         p.codebook_size)
    t_field = time.perf_counter() - t0
    sp = ldist.shard_params(p, 0, sample_frac)
    t0 = time.perf_counter()
    r = orc.run_batch_field(field, hand.desc, patches.desc, raw, sp, workers=cores)
    t_sample = time.perf_counter() - t0
    scale = batch / max(1, ldist.shard_range(batch, 0, sample_frac)[1])
    valid_full = r.profile["valid"] * scale
    total = t_field + t_sample * scale
    return dict(value=valid_full / total, unit=UNIT, cores=cores, kind="port",
                sample=(f"oracle/ CPU restatement: field build ({t_field:.1f}s, 1 thread) + "
                        f"candidates [0,{ldist.shard_range(batch, 0, sample_frac)[1]}) of {batch} "
                        f"({t_sample:.1f}s on {cores} threads, {r.profile['valid']} valid), "
                        f"stage time and valid count scaled x{scale:.0f} to the batch"),
                seconds=t_field + t_sample, forward_seconds_extrapolated=total)


# ---------------------------------------------------------------- arms
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import caller as lc
    import paper_2511_07418_b200 as lg
    p = params_for(args.workload, args.batch)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(cpu_baseline(args.workload, p.batch, args.sample_frac, hand, patches, raw, p))
    timed = vals[args.warmup:]
    v = float(np.mean([x["value"] for x in timed]))
    cb = dict(timed[-1])
    cb["value"] = v
    line = dict(metric=METRIC, value=v, unit=UNIT, impl="reference", n_gpus=args.gpus,
                steps=args.steps, warmup=args.warmup,
                ms_per_step=1e3 * float(np.mean([x["forward_seconds_extrapolated"] for x in timed])),
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64",
                data="synthetic assets (tools/make_assets.py), reference CPU path = oracle port",
                config=dict(workload=args.workload, batch=p.batch, passes=p.passes,
                            k_contacts=p.k_contacts, field_configs=p.field_configs),
                cpu_baseline=cb,
                e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line))
    return 0


def run_b200(args):
    import torch
    import torch.distributed as dist
    import caller as lc
    import paper_2511_07418_b200 as lg
    from paper_2511_07418_b200 import dist as ldist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    p = params_for(args.workload, args.batch)
    hand, patches, raw, _ = lc.prepare_inputs(p)
    sp = ldist.shard_params(p, rank, world) if world > 1 else p
    ctx = lg.Context(local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        r = lg.run_batch(ctx, hand, patches, raw, sp)
        grasps = r.grasps
        if world > 1:
            grasps = ldist.merge_grasps(ldist.gather_records(grasps, device=dev))
        return r, grasps

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(local) if not args.no_clocks else None
    if clocks:
        time.sleep(1.0)  # let nvidia-smi finish NVML start-up before the timed steps
        step()
    e2e_ms, dev_s, valid, launches, h2d, d2h, profs = [], [], [], [], [], [], []
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict L2 (126 MB) between timed steps
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r, grasps = step()
        b.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_ms.append(a.elapsed_time(b))
        dev_s.append(r.profile["device_seconds"])
        valid.append(r.profile["valid"])
        launches.append(r.profile["gpu_launches"])
        h2d.append(r.profile["h2d_bytes"])
        d2h.append(r.profile["d2h_bytes"])
        profs.append(r.profile)
    clk = clocks.stop() if clocks else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled"]}
    # the same metric with a cached field (built once, reused),
    # the multi-object / multi-pass operating point
    field = lg.ContactFieldIndex.build(ctx, hand, patches, sp.field_configs, sp.box_width, sp.seed,
                                       sp.codebook_size)
    lg.run_batch(ctx, hand, patches, raw, sp, field=field)
    cached_s, cached_valid = [], []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        rc = lg.run_batch(ctx, hand, patches, raw, sp, field=field)
        cached_s.append(rc.profile["device_seconds"])
        cached_valid.append(rc.profile["valid"])
    del field
    if args.verbose:
        print("per-step device ms:", [round(1e3 * x, 1) for x in dev_s], file=sys.stderr)

    def reduce(x, op):
        t = torch.tensor(x, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=op)
        return t.cpu().numpy()

    MAX, SUM = (dist.ReduceOp.MAX, dist.ReduceOp.SUM) if world > 1 else (None, None)
    e2e_ms = reduce(e2e_ms, MAX)
    dev_s = reduce(dev_s, MAX)
    cached_s = reduce(cached_s, MAX)
    cached_valid = reduce(cached_valid, SUM)
    valid = reduce(valid, SUM)
    h2d_t = reduce(h2d, SUM)
    d2h_t = reduce(d2h, SUM)
    launches_t = reduce(launches, SUM)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    value = float(valid.sum() / dev_s.sum())
    e2e_v = float(valid.sum() / (e2e_ms.sum() / 1e3))
    prof = profs[-1]
    # roofline of the dominant kernel (device time per launch from CUDA events)
    groups = hand.groups()
    depth = 0
    d = hand.desc
    for l in range(d.n_links):
        dd, x = 0, l
        while x >= 0:
            dd += d.joint_index[x] >= 0
            x = d.parent[x]
        depth = max(depth, dd)
    fl = flop_model(prof, p.k_contacts, p.static_contact_prob, p.mu, d.dof, d.n_links, depth)
    kern = {"k_realize": (fl["realize"], prof["realize_seconds"]),
            "k_contact_opt": (fl["contact_opt"], prof["contact_opt_seconds"])}
    dom = max(kern, key=lambda n: kern[n][1])
    flops, secs = kern[dom]
    peak, peak_src = fp64_peak()
    achieved = flops / secs / 1e12 if secs > 0 else 0.0
    traffic, traffic_src = kernel_traffic(dom) if args.workload == "allegro_box" else (None, None)
    roof = dict(bound="fp64", kernel=dom, achieved=achieved, peak=peak, unit="TFLOP/s",
                frac=achieved / peak, traffic=traffic, traffic_source=traffic_src,
                peak_source=peak_src,
                kernel_share_of_step=secs / prof["device_seconds"],
                note="SIMT FP64 kernel (no HBM- or tensor-bound stage); algorithmic FLOPs from "
                     "device work counters x SURVEY 8(d) per-unit model")
    line = dict(
        metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps,
        warmup=args.warmup, ms_per_step=float(dev_s.mean() * 1e3), higher_is_better=True,
        scaling="weak" if world > 1 else "weak", vs_baseline=None, dtype="f64",
        data="synthetic assets (tools/make_assets.py; BASELINE configs[1])",
        config=dict(workload=args.workload, batch=p.batch, passes=p.passes,
                    k_contacts=p.k_contacts, field_configs=p.field_configs,
                    object_samples=int(prof["object_samples"]), patches=int(prof["patches"]),
                    parallelism=f"seed-shard x{world}", l2="flushed (256 MB write) between steps",
                    forward_seconds=float(dev_s.mean())),
        e2e=dict(value=e2e_v, unit=UNIT, h2d_bytes_per_step=int(h2d_t.mean()),
                 d2h_bytes_per_step=int(d2h_t.mean()), ms_per_step=float(e2e_ms.mean())),
        cached_field=dict(value=float(cached_valid.sum() / cached_s.sum()), unit=UNIT,
                          ms_per_step=float(cached_s.mean() * 1e3),
                          note="field built once and reused (run_batch with a prebuilt index)"),
        gpu_launches=int(launches_t.sum()),
        clocks=clk, roofline=roof,
        funnel={k: int(prof[k]) for k in ("candidates", "placements_accepted",
                                           "contact_sets_balanced", "ik_finite",
                                           "penetration_free", "ik_converged", "stable", "valid")},
        work={k: int(prof[k]) for k in ("ik_iterations", "fk_evals", "wrench_evals", "wrench_grads",
                                        "proj_evals", "realize_calls", "collision_calls")},
        stage_seconds={k: float(prof[k]) for k in ("field_build", "placement_domains",
                                                    "contact_optimization",
                                                    "kinematics_optimization", "postprocessing")},
    )
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.workload, p.batch, args.sample_frac, hand,
                                            patches, raw, p)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="allegro_box", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--sample-frac", type=int, default=40,
                    help="CPU legs time one 1/N shard of the batch")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
