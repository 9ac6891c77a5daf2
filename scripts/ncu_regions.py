"""Executed warp-instructions per SASS window with the window's signature
opcodes (to attribute work to warp roles).  python scripts/ncu_regions.py REP [win]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]
data = [dict(zip(h, r)) for r in rows[1:] if len(r) == len(h)]
ie = "Instructions Executed"
tot = sum(int(d[ie] or 0) for d in data)
print(f"total executed warp-instructions {tot:.4g}")
for w in range(0, len(data), win):
    seg = data[w:w + win]
    s = sum(int(d[ie] or 0) for d in seg)
    if s < 0.005 * tot:
        continue
    ops = collections.Counter()
    for d in seg:
        op = d["Source"].strip().split()[0]
        if op.startswith("@"):
            op = d["Source"].strip().split()[1]
        ops[op.split(".")[0]] += int(d[ie] or 0)
    sig = " ".join(f"{k}:{v / s:.0%}" for k, v in ops.most_common(5))
    print(f"{w:5d}-{w + win - 1:5d} {100 * s / tot:5.1f}%  {sig}")
