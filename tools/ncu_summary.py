"""Per-kernel summary of an `ncu --set full` report (JSON + markdown).

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [OUT.md]
Per captured launch: duration, DRAM bytes read/written (the roofline
`traffic`), FP64-pipe and warp-slot utilisation, IPC, registers, executed
instructions and the dominant warp-stall reasons.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "ipc": ("sm__inst_executed.avg.per_cycle_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "grid_size": ("launch__grid_size", 1.0),
    "block_size": ("launch__block_size", 1.0),
}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
STALLS = ["smsp__pcsamp_warps_issue_stalled_" + s for s in (
    "wait", "no_instructions", "short_scoreboard", "long_scoreboard", "barrier", "selected",
    "not_selected", "branch_resolving", "math_pipe_throttle", "mio_throttle", "lg_throttle",
    "dispatch_stall", "membar", "sleeping", "drain", "imc_miss", "misc", "tex_throttle")]


def main():
    rep, out_json = sys.argv[1], sys.argv[2]
    out_md = sys.argv[3] if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, (m, scale) in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if scale is None:
                v *= BYTES.get(units[i], 1.0)
            d[k] = v
        st = {}
        for m in STALLS:
            if m in hdr:
                try:
                    st[m.rsplit("stalled_", 1)[1]] = float(r[hdr.index(m)].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        d["stalls_pct"] = {k: round(100 * v / tot, 1)
                           for k, v in sorted(st.items(), key=lambda x: -x[1])[:5]}
        if "dram_read_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)
        res.append(d)
    with open(out_json, "w") as f:
        json.dump(res, f, indent=1)
    if out_md:
        with open(out_md, "w") as f:
            f.write("| kernel | ms | DRAM MB | FP64 pipe % | warps active % | IPC | regs | top stalls |\n")
            f.write("|---|---|---|---|---|---|---|---|\n")
            for d in res:
                f.write(f"| {d['kernel']} | {d.get('duration_ms', 0):.2f} | "
                        f"{d.get('dram_bytes', 0) / 1e6:.1f} | {d.get('fp64_pipe_active_pct', 0):.1f} | "
                        f"{d.get('warps_active_pct', 0):.1f} | {d.get('ipc', 0):.2f} | "
                        f"{int(d.get('registers', 0))} | "
                        + ", ".join(f"{k} {v}%" for k, v in d["stalls_pct"].items()) + " |\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
