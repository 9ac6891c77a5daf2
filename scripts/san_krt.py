"""compute-sanitizer driver for the device merge table alone (dendro.cu:krt_kernel)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_16354_b200 as slk  # noqa: E402
from oracle import oracle as orc  # noqa: E402

for nt in [int(v) for v in sys.argv[1:]] or [40, 100, 6000]:
    ts = np.arange(1, nt)
    td = (np.random.default_rng(6).random(nt - 1) * ts).astype(np.int64)
    tw = np.random.default_rng(7).random(nt - 1) + 0.5
    t0 = time.time()
    d = slk.build_dendrogram(slk.EdgeList(nt, ts, td, tw), nt)
    assert np.array_equal(d.merges, orc.build_dendrogram(ts, td, tw, nt))
    print("ok", nt, f"{time.time() - t0:.1f}s", flush=True)
