"""Summarise a tc_scan timeline dump (build variant "timeline", SLK_TIMELINE=<file>).

python scripts/timeline.py FILE
Per launch: median cycles per tile between the warp roles' hand-offs
(tc_scan.cu TL events), over CTAs 0..15, tiles 8..end (steady state).
"""
import sys

import numpy as np

EV = ["P.wait_empty", "P.got_empty", "P.issued", "C.raw_landed", "C.converted", "M.wait_full",
      "M.got_full", "M.got_tempty", "M.committed", "E.wait_full", "E.got_full", "E.released"]
PAIRS = [("TMA landed - issued", 3, 2), ("convert", 4, 3), ("MMA waits B", 6, 5), ("MMA waits tempty", 7, 6),
         ("MMA issue", 8, 7), ("epi waits acc", 10, 9), ("epi works", 11, 10), ("P waits empty", 1, 0),
         ("P visitor", 0, 12)]
raw = open(sys.argv[1], "rb").read()
off = 0
while off < len(raw):
    mode, rows, ctas, nev, nit = np.frombuffer(raw, np.int64, 5, off)
    off += 40
    n = int(ctas * nev * nit)
    t = np.frombuffer(raw, np.uint64, n, off).astype(np.int64).reshape(ctas, nev, nit)
    off += n * 8
    out = []
    for c in range(ctas):
        valid = (t[c, :12] > 0).all(axis=0)
        idx = np.nonzero(valid)[0]
        idx = idx[idx >= 8]
        if len(idx) < 8:
            continue
        per = {name: np.median(t[c, a, idx] - t[c, b, idx]) for name, a, b in PAIRS
               if (t[c, a, idx] > 0).all() and (t[c, b, idx] > 0).all()}
        commits = t[c, 8, idx]
        per["tile interval"] = np.median(np.diff(commits))
        per["P interval"] = np.median(np.diff(t[c, 2, idx]))
        per["E interval"] = np.median(np.diff(t[c, 11, idx]))
        per["tiles"] = len(idx)
        out.append(per)
    if not out:
        print(f"mode {mode} rows {rows}: no complete tiles")
        continue
    keys = [k for k in out[0].keys() if all(k in o for o in out)]
    print(f"mode {mode} rows {rows}: " + ", ".join(f"{k} {np.median([o[k] for o in out]):.0f}" for k in keys))
