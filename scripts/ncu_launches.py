"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel.

python scripts/ncu_launches.py launches.csv   -> per-kernel count, total ms, share
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows:
    v = float(r[vi].replace(",", "")) * SCALE[r[ui]]
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"{len(rows)} launches, {tot:.1f} ms total (cold-cache, serialised)")
print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    if t / tot < 0.001:
        continue
    print(f"{t:10.2f} {100 * t / tot:5.1f}% {n:8d}  {k[:90]}")
