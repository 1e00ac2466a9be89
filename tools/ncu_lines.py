"""Per-source-line stall samples from an ncu report (needs -lineinfo).

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP] [stall|inst]
Runs `ncu -i REPORT --page source --csv --print-source cuda,sass -k KERNEL`
and prints the TOP source lines by warp-stall samples with their dominant
stall reasons.
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    by = sys.argv[4] if len(sys.argv) > 4 else "stall"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", kern], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr = "?", None
    lines = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        lines.append((fname, r))
    if not hdr:
        print("no source rows")
        return
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    stall = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    tot = sum(f(r[si]) for _, r in lines) or 1.0
    itot = sum(f(r[ie]) for _, r in lines) or 1.0
    col = ie if by == "inst" else si
    ranked = sorted(lines, key=lambda x: -f(x[1][col]))[:top]
    for fn, r in ranked:
        reasons = sorted(((f(r[i]), h[6:]) for i, h in stall), reverse=True)[:3]
        rs = " ".join(f"{h}:{100 * v / max(f(r[si]), 1):.0f}%" for v, h in reasons if v > 0)
        print(f"{100 * f(r[si]) / tot:5.1f}% {fn}:{r[0]:>4s} inst={100 * f(r[ie]) / itot:5.1f}% "
              f"{r[1].strip()[:70]:70s} {rs}")


if __name__ == "__main__":
    main()
