"""k-NN-graph-only sweep (BASELINE.json configs[3]: N=1M, d in {32,128,512},
k in {8,32,64}; N(0,1) points, no cluster structure, so pruning skips little).

    python scripts/bench_knn.py [--n 1000000] [--cases 32:8,128:8,...] [--steps 2]

One JSON line per (d, k): seconds per k-NN graph (CUDA events, points resident
in HBM, warm-up first), the scan engine the library chose (tcgen05 tensor
cores for k <= 127 and d <= 512 — the chunked kernel above d = 128 — else the
exact-fp32 FFMA scan), the
computed-tile work and its rate against the matching peak.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16354_b200 import _lib  # noqa: E402
from paper_2306_16354_b200.neighbors import DevicePoints, knn_device  # noqa: E402
from paper_2306_16354_b200.synthetic import bench_points  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--cases", default="32:8,32:32,32:64,128:8,128:32,128:64,512:8,512:32,512:64")
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args()
peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {"bf16_tflops": 1590.0}
torch.cuda.set_device(0)
for case in args.cases.split(","):
    d, k = (int(v) for v in case.split(":"))
    x = bench_points(args.n, d, None)
    pts = DevicePoints.from_tensors(torch.from_numpy(x).cuda())
    knn_device(pts, k)  # warm-up
    torch.cuda.synchronize()
    _lib.profile(reset=True)
    times = []
    for _ in range(args.steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        knn_device(pts, k)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) / 1e3)
    prof = _lib.profile(reset=True)
    tc = prof["tc_ms"] > 0
    ms = prof["tc_ms"] if tc else prof["scan_ms"]
    flops = prof["tc_flops_done"] if tc else prof["scan_flops_done"]
    rate = flops / (ms / 1e3) / 1e12 if ms else None
    peak = float(peaks["bf16_tflops"]) if tc else 148 * 128 * 2 * 1.965e9 / 1e12
    print(json.dumps({
        "config": f"knn-only N={args.n} d={d} k={k} N(0,1)", "seconds": float(np.mean(times)),
        "engine": "tcgen05" if tc else "ffma", "computed_tile_tflops": rate,
        "peak_tflops": peak, "frac": rate / peak if rate else None,
        "tiles_computed_frac": prof["scan_tiles"] / max(prof["scan_tiles_total"], 1),
        "rows_uncertified_per_call": prof["tc_uncertified"] / args.steps,
        "brute_force_tflop_per_call": prof["scan_flops"] / args.steps / 1e12,
    }), flush=True)
    del pts
    torch.cuda.empty_cache()
