"""Benchmark: valid grasps/s of the Lightning Grasp forward pass (BASELINE.json
metric) on the Allegro-class config (BASELINE configs[1]).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]

With --gpus N > 1 and no WORLD_SIZE in the environment the script relaunches
itself under torch.distributed.run with N ranks (one per GPU, 127.0.0.1).

A step is one run_batch forward pass of the workload: field build,
preprocess, placement + domains, contact search, realisation + collision
filter, postprocess — the reference's `total` (pipeline.cpp:308-625) — on
every rank, followed (N > 1) by the NCCL gather of the kept grasps to rank 0
behind the C-ABI (lg_comm_gather).  Scaling is weak: every rank owns a seed
shard of B candidates of one object (global batch N x B, rank r owns
candidates [rB, (r+1)B)), the per-object throughput the north star asks for.

  value  valid grasps / device seconds of the pass (CUDA events on the
         library stream, inputs resident), max over ranks;
  e2e    the same through the public C-ABI call with HOST buffers: the call
         uploads the hand, patches and object samples (H2D), downloads the
         kept grasps (D2H) and, for N > 1, gathers them to rank 0; timed with
         CUDA events around the call, max over ranks.

--impl reference runs THE REFERENCE ITSELF (oracle/_ref: /root/reference/proj
compiled unmodified) — its run_batch on the same workload, all host threads —
on a bounded sample per step (see run_reference).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
    # configs[2]: LEAP-class hand on tool-like primitive unions
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
REF_SAMPLE = 320  # candidates per reference step (bounded CPU sample, ~9 s on 16 cores)


def asset(*p):
    return os.path.join(ROOT, "assets", *p)


def workload_paths(workload):
    w = WORKLOADS[workload]
    return asset(w["cfg"]), asset(w["hand"]), asset(w["obj"])


def config_keys(workload, p, world):
    """The `config` object both arms print (same keys, same values)."""
    return dict(workload=workload, hand=WORKLOADS[workload]["hand"],
                object=WORKLOADS[workload]["obj"], batch_per_gpu=int(p.batch),
                global_batch=int(p.batch) * world, passes=int(p.passes),
                k_contacts=int(p.k_contacts), field_configs=int(p.field_configs),
                samples_per_cm2=float(p.samples_per_cm2), seed=int(p.seed),
                parallelism=f"seed-shard x{world}",
                l2="flushed (256 MB write) between steps")


# ------------------------------------------------------------ clock sampling
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.proc = None
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
    """DRAM bytes per launch of `kernel` from the newest committed ncu
    --set full summary of the default bench workload (tools/ncu_summary.py)."""
    names = {"k_contact_opt": "k_contact_opt2", "k_realize": "k_realize_warp"}
    want = names.get(kernel, kernel)
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", rnd, "ncu_full_summary.json")
        try:
            with open(path) as f:
                rows = json.load(f)
        except (OSError, ValueError):
            continue
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


# ------------------------------------------- the reference on the host cores
def reference_step(workload, sample, workers, out_dir):
    """One run of THE REFERENCE's run_batch (oracle/_ref) on `sample`
    candidates of the workload with `workers` threads, in the reference's
    cache mode (cache = true: the contact-field index is loaded from the GGCF
    file under out_dir after the first call builds it).  Returns (valid,
    seconds, profile)."""
    from oracle import ref_py as R
    cfg, hand, obj = workload_paths(workload)
    inp = R.RefInputs(config=cfg, extra="cache = true\n", hand=hand, object=obj, out=out_dir,
                      batch=sample, workers=workers)
    t0 = time.perf_counter()
    res = inp.run_batch()
    dt = time.perf_counter() - t0
    inp.close()
    return res.profile["valid"], dt, res.profile


def cpu_baseline(workload, sample=REF_SAMPLE):
    cores = os.cpu_count() or 1
    out_dir = f"/tmp/lg_ref_cache_{os.getpid()}"
    reference_step(workload, sample, cores, out_dir)  # builds + saves the field index
    valid, dt, prof = reference_step(workload, sample, cores, out_dir)
    return dict(value=valid / dt, unit=UNIT, cores=cores, kind="reference",
                sample=(f"oracle/_ref run_batch (the reference compiled from /root/reference) on "
                        f"candidates [0,{sample}) of the workload, {cores} threads, cache mode "
                        f"(field index loaded from its GGCF file): {valid} valid in {dt:.2f} s"),
                seconds=dt, funnel={k: int(prof[k]) for k in ("candidates", "placements_accepted",
                                                               "contact_sets_balanced", "valid")})


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref_py as R  # the reference only: no product or caller library
    cfg, hand, obj = workload_paths(args.workload)
    p = R.RefInputs(config=cfg, hand=hand, object=obj, batch=args.batch).params
    cores = os.cpu_count() or 1
    out_dir = f"/tmp/lg_ref_cache_{os.getpid()}"
    sample = min(args.ref_sample, p.batch)
    steps = []
    for i in range(args.warmup + args.steps):
        steps.append(reference_step(args.workload, sample, cores, out_dir))
    timed = steps[args.warmup:]
    valid = sum(v for v, _, _ in timed)
    secs = sum(t for _, t, _ in timed)
    v = valid / secs
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    cb = dict(value=v, unit=UNIT, cores=cores, kind="reference",
              sample=(f"each step = the reference's run_batch (oracle/_ref, compiled unmodified "
                      f"from /root/reference) on candidates [0,{sample}) of the {p.batch}-candidate "
                      f"workload with {cores} threads, cache mode (contact-field index built once "
                      f"in warm-up, loaded from its GGCF file each step)"))
    line = dict(metric=METRIC, value=v, unit=UNIT, impl="reference", n_gpus=world,
                steps=args.steps, warmup=args.warmup, ms_per_step=1e3 * secs / len(timed),
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64",
                data="synthetic assets (tools/make_assets.py); host CPU",
                config=config_keys(args.workload, p, world),
                cpu_baseline=cb,
                e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                per_step_seconds=[round(t, 3) for _, t, _ in timed],
                valid_per_step=[int(x) for x, _, _ in timed])
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist
    import caller as lc
    import paper_2511_07418_b200 as lg
    from paper_2511_07418_b200 import dist as ldist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    cfg, hand_path, obj = workload_paths(args.workload)
    p = lc.parse_config(cfg, hand=hand_path, object=obj, batch=args.batch)
    p.want_trace = 0
    B = p.batch
    # weak scaling: global batch world x B, rank r owns [rB, (r+1)B)
    pg = ldist.shard_params(p, rank, world)
    pg.batch = B * world
    hand, patches, raw, _ = lc.prepare_inputs(p)
    ctx = lg.Context(local)
    comm = None
    if world > 1:
        uid = [ldist.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ldist.Comm(ctx, rank, world, uid[0])
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        r = lg.run_batch(ctx, hand, patches, raw, pg)
        if comm is not None:
            g, prof = comm.gather(r)
            return r, g, prof
        return r, r.grasps, r.profile

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
        r, grasps, merged = step()
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
        if rank == 0 and merged["valid"] != len(grasps):
            raise RuntimeError("gather lost grasps")
    clk = clocks.stop() if clocks else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled"]}
    # the same metric with a cached field (built once, reused)
    field = lg.ContactFieldIndex.build(ctx, hand, patches, pg.field_configs, pg.box_width, pg.seed,
                                       pg.codebook_size)
    lg.run_batch(ctx, hand, patches, raw, pg, field=field)
    cached_s, cached_valid = [], []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        rc = lg.run_batch(ctx, hand, patches, raw, pg, field=field)
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
    if comm is not None:
        comm.close()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    value = float(valid.sum() / dev_s.sum())
    e2e_v = float(valid.sum() / (e2e_ms.sum() / 1e3))
    prof = profs[-1]
    # roofline of the dominant kernel (device time per launch from CUDA events)
    d = hand.desc
    depth = 0
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
    # the same config keys as the reference arm; measured workload sizes
    # go beside it
    config = config_keys(args.workload, p, world)
    workload_stats = dict(object_samples=int(prof["object_samples"]), patches=int(prof["patches"]),
                          forward_seconds=float(dev_s.mean()))
    line = dict(
        metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps,
        warmup=args.warmup, ms_per_step=float(dev_s.mean() * 1e3), higher_is_better=True,
        scaling="weak", vs_baseline=None, dtype="f64",
        data="synthetic assets (tools/make_assets.py; BASELINE configs[1])",
        config=config,
        workload_stats=workload_stats,
        e2e=dict(value=e2e_v, unit=UNIT, h2d_bytes_per_step=int(h2d_t.mean()),
                 d2h_bytes_per_step=int(d2h_t.mean()), ms_per_step=float(e2e_ms.mean()),
                 includes="H2D inputs, the pass, D2H of the kept grasps" +
                          (", NCCL gather to rank 0" if world > 1 else "")),
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
        from oracle import ref_py as R
        if R.available():
            line["cpu_baseline"] = cpu_baseline(args.workload)
    print(json.dumps(line))
    sys.stdout.flush()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args_list, n):
    """--gpus N without a launcher: run N ranks under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + args_list
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="allegro_box", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None, help="candidates per GPU")
    ap.add_argument("--ref-sample", type=int, default=REF_SAMPLE,
                    help="candidates per reference step (bounded CPU sample)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(sys.argv[1:], args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
