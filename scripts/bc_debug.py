"""Raw output of the block-centred scan (SLK_DEBUG_BC=1) against float64 math."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

os.environ["SLK_DEBUG_BC"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2306_16354_b200 import _lib  # noqa: E402
from paper_2306_16354_b200.synthetic import bench_points  # noqa: E402

lib = _lib.load()
fn = lib.slk_debug_tc_scan
n, d, k = int(sys.argv[1]), int(sys.argv[2]), 15
x = bench_points(n, d, 4)
xd = torch.from_numpy(x).cuda()
cand = torch.full((n, 64), -7, dtype=torch.int32, device="cuda")
kth = torch.full((n, 2), -7.0, dtype=torch.float32, device="cuda")
qhat = torch.zeros(n, dtype=torch.float32, device="cuda")
sc = ctypes.c_float()
st = fn(_lib.ptr(xd), n, d, k, _lib.ptr(cand), _lib.ptr(kth), _lib.ptr(qhat), ctypes.byref(sc),
        _lib.stream_handle())
torch.cuda.synchronize()
print("status", st, lib.slk_last_error(), "scale", sc.value)
cand, kth, qhat = cand.cpu().numpy(), kth.cpu().numpy(), qhat.cpu().numpy()
s = sc.value
x64 = x.astype(np.float64)
for r in [0, 1, 5, 127, 128, 300, n - 1]:
    d2 = ((x64 - x64[r]) ** 2).sum(1) * s * s
    d2[r] = np.inf
    order = np.argsort(d2)
    for h in range(2):
        ids = cand[r, h * 32:(h + 1) * 32]
        ids = ids[ids >= 0]
        print(f"row {r} half {h}: kth {kth[r, h]:.6g} rho {qhat[r]:.6g}  listed {len(ids)} "
              f"max listed d2 {d2[ids].max() if len(ids) else -1:.6g} min {d2[ids].min() if len(ids) else -1:.6g}")
    print(f"   true 15th {d2[order[14]]:.6g} 16th {d2[order[15]]:.6g} 32nd {d2[order[31]]:.6g}; ids0 {cand[r, :6]}")
