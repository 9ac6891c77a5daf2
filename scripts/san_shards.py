"""compute-sanitizer driver: the in-process multi-shard pipeline alone."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_16354_b200 as slk  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2306_16354_b200.synthetic import make_blobs  # noqa: E402

u = make_blobs(np.random.default_rng(5), 3100, 64, 9).astype(np.float32)
ref = orc.single_linkage(u, 9, k=3, seed=0)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    res = slk.single_linkage_result(u, slk.LinkageConfig(n_clusters=9, k=3, seed=0), n_gpus=3)
    assert np.array_equal(res.dendrogram.merges, ref["merges"])
    print("rep", rep, "ok", flush=True)
