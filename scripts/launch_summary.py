"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel totals, and
per-grid totals for the kernels named on the command line.
Usage: python scripts/launch_summary.py launches.csv [kernel-substring ...]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hd = rows[h]
ki, vi, gi, ui = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Grid Size"), hd.index("Metric Unit")
mi = hd.index("Metric Name")
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
agg = collections.defaultdict(lambda: [0, 0.0])
grids = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    k = r[ki].split("(")[0][:60]
    agg[k][0] += 1
    agg[k][1] += ms
    if any(s in r[ki] for s in sys.argv[2:]):
        grids[(k, r[gi])][0] += 1
        grids[(k, r[gi])][1] += ms
tot = sum(v for _, v in agg.values())
print(f"total {tot:.2f} ms, {sum(n for n, _ in agg.values())} launches")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{v:8.2f} ms {n:5d} {100 * v / tot:5.1f}%  {k}")
for (k, g), (n, v) in sorted(grids.items(), key=lambda x: -x[1][1])[:20]:
    print(f"  {k[:30]:30s} grid {g:16s} x{n:4d} {v:8.3f} ms ({1e3 * v / n:.1f} us each)")
