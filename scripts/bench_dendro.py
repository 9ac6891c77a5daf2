"""Time build_dendrogram on large synthetic trees: python scripts/bench_dendro.py [n]."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_16354_b200 as slk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(0)
for shape in ("random", "chain", "star"):
    src = np.arange(1, n)
    if shape == "chain":
        dst = src - 1
    elif shape == "star":
        dst = np.zeros(n - 1, dtype=np.int64)
    else:
        dst = (rng.random(n - 1) * src).astype(np.int64)
    perm = rng.permutation(n)
    e = slk.EdgeList(n, perm[src], perm[dst], rng.random(n - 1) + 0.5)
    for rep in range(3):
        t0 = time.perf_counter()
        slk.build_dendrogram(e, n)
        print(shape, n, f"{(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
