"""Summarise an ncu report's SASS page: hottest instructions and stall mix.

python scripts/ncu_hot.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
data = [dict(zip(h, r)) for r in rows[1:] if len(r) == len(h)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
print(f"{len(data)} SASS instructions, {tot} samples")
for i, d in enumerate(data):
    d["_i"] = i
hot = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top]
for d in sorted(hot, key=lambda d: d["_i"]):
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    st = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{d['_i']:5d} {100*s/tot:5.1f}% {d['Source'].strip()[:60]:60s} "
          + " ".join(f"{n}:{v}" for v, n in st if v))
# cumulative by region of 50 instructions
print("--- by 100-instruction window")
for w in range(0, len(data), 100):
    s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data[w:w + 100])
    if s:
        print(f"{w:5d}-{w+99:5d} {100*s/tot:5.1f}%")
