"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    if len(r) <= vi or r[vi] == "":
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "")
    name = name if len(name) < 60 else name[:57] + "..."
    tot[name] += v
    cnt[name] += 1
# steps = launches of a once-per-pass kernel unless given
steps = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, cnt.get("lgd::k_place_pose", 1))
T = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms/step':>9s} {'share':>6s}")
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{n:60s} {cnt[n] // steps:8d} {v / steps:9.3f} {100 * v / T:5.1f}%")
print(f"{'total':60s} {'':8s} {T / steps:9.3f}")
