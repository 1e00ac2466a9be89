"""Funnel + device time of each bench workload at a reduced batch (tuning
aid for the synthetic configs; not a bench line)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import caller as lc  # noqa: E402
import paper_2511_07418_b200 as lg  # noqa: E402


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else sorted(bench.WORKLOADS)
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    ctx = lg.Context(0)
    for name in names:
        p = bench.params_for(name, batch)
        t0 = time.perf_counter()
        hand, patches, raw, _ = lc.prepare_inputs(p)
        t_prep = time.perf_counter() - t0
        r = lg.run_batch(ctx, hand, patches, raw, p)
        r = lg.run_batch(ctx, hand, patches, raw, p)
        pr = r.profile
        print(json.dumps(dict(workload=name, batch=batch, prep_s=round(t_prep, 2),
                              device_ms=round(1e3 * pr["device_seconds"], 1),
                              field_build_ms=round(1e3 * pr["field_build"], 1),
                              samples=int(pr["object_samples"]), field_samples=int(pr["field_samples"]),
                              patches=int(pr["patches"]), boxes=int(pr["boxes"]),
                              funnel={k: int(pr[k]) for k in ("placements_accepted",
                                      "contact_sets_balanced", "penetration_free", "ik_converged",
                                      "stable", "valid")})), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
