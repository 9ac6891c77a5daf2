"""Inspect the raw tensor-core scan output against direct fp32 math."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2306_16354_b200 import _lib  # noqa: E402
from paper_2306_16354_b200.synthetic import bench_points  # noqa: E402

lib = _lib.load()
fn = lib.slk_debug_tc_scan
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
               ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.c_void_p]
n, d, k = int(sys.argv[1]), int(sys.argv[2]), 15
x = bench_points(n, d, 4)
xd = torch.from_numpy(x).cuda()
cand = torch.empty((n, 32), dtype=torch.int32, device="cuda")
kth = torch.empty(n, dtype=torch.float32, device="cuda")
qhat = torch.empty(n, dtype=torch.float32, device="cuda")
sc = ctypes.c_float()
st = fn(_lib.ptr(xd), n, d, k, _lib.ptr(cand), _lib.ptr(kth), _lib.ptr(qhat), ctypes.byref(sc),
        _lib.stream_handle())
print("status", st, lib.slk_last_error(), "scale", sc.value)
cand, kth, qhat = cand.cpu().numpy(), kth.cpu().numpy(), qhat.cpu().numpy()
s = sc.value
# reference: centred by the query block centroid (mean of block rows, float)
for r in [0, 1, 5, 127, 128, 300]:
    if r >= n:
        continue
    b = r // 128
    blk = x[b * 128: min(n, (b + 1) * 128)].astype(np.float64)
    c = blk.mean(axis=0).astype(np.float32)
    qh = ((x[r] - c) * s).astype(np.float16).astype(np.float64)
    d2 = ((x.astype(np.float64) - x[r]) ** 2).sum(1)
    d2[r] = np.inf
    true_top = np.argsort(d2)[:32]
    got = cand[r]
    print(f"row {r}: qhat {qhat[r]:.4f} vs {np.sum(qh**2):.4f}; kth {kth[r]:.4f} (/s2 {kth[r]/s/s:.4f}); "
          f"true 32nd {np.sort(d2)[31]:.4f}; overlap {len(set(got) & set(true_top))}/32; first ids {got[:6]} true {true_top[:6]}")

# ---- certificate diagnosis over all rows (python restatement of certified_floor_tc)
import math
x64 = x.astype(np.float64)
norms = (x64 ** 2).sum(1)
maxn = norms.max()
R = cand.shape[1]
fails = []
for r in range(n):
    ids = cand[r][cand[r] >= 0]
    v = ((x64[ids] - x64[r]) ** 2).sum(1)
    vk = np.sort(v)[k - 1] if len(v) >= k else np.inf
    A, q2 = float(kth[r]), float(qhat[r])
    rr = math.sqrt(q2)
    g = (2 * d + 8) * 2**-23
    ca, cb, cc = 1 + g, 4 * g * rr, 4 * g * rr * rr - A
    disc = cb * cb - 4 * ca * cc
    sh = (-cb + math.sqrt(disc)) / (2 * ca) if disc > 0 else -1
    eta = 2**-11 * 1.01
    etap = eta * (1 + 2 * eta)
    sd = (sh * (1 - etap) - 2 * etap * rr - 2 * math.sqrt(d) * 2**-25) / s
    dlo = sd * sd
    ev = (d + 4) * 2**-52 * (norms[r] + maxn) * 1.01
    ok = (dlo - ev) > vk
    if not ok:
        fails.append((r, A / s / s, vk, dlo, rr / s, len(ids)))
print("failing rows", len(fails), "of", n)
for f in fails[:10]:
    print("row %d approxK'=%.4f vk=%.4f floor=%.4f |q'|=%.3f ncand=%d" % f)
