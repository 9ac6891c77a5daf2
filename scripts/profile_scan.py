"""Run one neighbour search for ncu: python scripts/profile_scan.py [knn|cc] N d c k."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2306_16354_b200 import _lib  # noqa: E402
from paper_2306_16354_b200.neighbors import DevicePoints, knn_device, nn1_device  # noqa: E402
from paper_2306_16354_b200.synthetic import bench_points  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "knn"
n, d, c, k = (int(v) for v in (sys.argv[2:6] if len(sys.argv) > 5 else (200000, 64, 10, 15)))
x = bench_points(n, d, c if c > 0 else None)
pts = DevicePoints.from_tensors(torch.from_numpy(x).cuda())
if mode == "knn":
    knn_device(pts, k)
else:
    counts = np.full(c, n // c)
    counts[: n % c] += 1
    col = np.repeat(np.concatenate([[0], np.cumsum(counts)[:-1]]), counts).astype(np.int32)
    dcol = torch.from_numpy(col).cuda()
    nn1_device(pts, pts, mode=2, qcolor=dcol, xcolor=dcol)
torch.cuda.synchronize()
print(mode, n, d, c, k, _lib.scan_stats(), _lib.profile())
