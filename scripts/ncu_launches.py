"""Summarise an ncu launch list by kernel.

python scripts/ncu_launches.py launches.csv [top]

The CSV is `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv --log-file ...`; prints per kernel: launches,
total device ms, share of all launches, DRAM bytes and their rate.
"""
import collections
import csv
import re
import sys

TIME = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name):
    name = re.sub(r"^void ", "", name).replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    name = name.split("(")[0]
    return re.sub(r"<.*", "", name) if not name.startswith("slk::tc") else name.split("<")[0]


rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h, rows = rows[0], rows[1:]
ki, vi, ui, mi, idi = (h.index(c) for c in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name", "ID"))
launch = collections.OrderedDict()
for r in rows:
    d = launch.setdefault(r[idi], {"name": short(r[ki]), "t": 0.0, "b": 0.0})
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        d["t"] = v * TIME[r[ui]]
    elif r[mi].startswith("dram__bytes"):
        d["b"] += v * BYTES[r[ui]]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in launch.values():
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d["t"]
    a[2] += d["b"]
tot = sum(a[1] for a in agg.values())
print(f"{len(launch)} launches, {tot:.2f} ms device time")
for name, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    rate = b / 1e9 / (t / 1e3) if t else 0.0
    print(f"{name[:48]:48s} {c:5d} {t:9.3f} ms {100 * t / tot:5.1f}%  {b / 1e9:8.3f} GB {rate:7.0f} GB/s")
