"""Quick tensor-core scan check vs the oracle (and the FFMA path)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2306_16354_b200 import _lib  # noqa: E402
from paper_2306_16354_b200.neighbors import DevicePoints, knn_device  # noqa: E402
from paper_2306_16354_b200.synthetic import bench_points  # noqa: E402

for (n, d, c, k) in [(3000, 16, 10, 15), (20000, 64, 20, 15), (8000, 128, 8, 32), (5000, 32, None, 8)]:
    x = bench_points(n, d, c)
    pts = DevicePoints.from_tensors(torch.from_numpy(x).cuda())
    t0 = time.time()
    idx, dist = knn_device(pts, k)
    torch.cuda.synchronize()
    st = _lib.scan_stats()
    oi, od = orc.fused_knn(x, k, rows=(0, min(n, 1024)))
    gi, gd = idx.cpu().numpy()[: len(oi)], dist.cpu().numpy()[: len(oi)]
    print(n, d, c, k, "match idx", np.array_equal(gi, oi), "dist", np.array_equal(gd, od), st,
          f"{time.time() - t0:.3f}s", flush=True)
print(_lib.profile())
