"""General-graph MST benchmark on road-network-shaped graphs (SURVEY §8f rank 4,
the paper's Table 3: DIMACS road networks).

    python scripts/bench_mst.py [--graphs nyc,fl,usa] [--steps 3] [--cpu]

The DIMACS files are not available offline, so each graph is synthetic with
the paper's node and edge counts: a W x H lattice whose horizontal / vertical
links are kept at the rate that gives the same undirected edge count (about
1.22 per node, above the square-lattice percolation threshold, so one giant
component plus small pieces, like a road map), with integer link lengths in
[1, 100000] (DIMACS-style integer weights: many ties, so the seeded weight
alteration decides the order).  The CSR is built once on the device; each
timed step is one `slk_solve_mst` on it (validation + symmetry check + weight
alteration + Boruvka), CUDA events on the library stream, after warm-up.

Prints one JSON line per graph: solve time, the Boruvka round loop's
algorithmic bytes (12 B per directed entry + 16 B per vertex per
round) and rate against the measured HBM peak, the paper's A100 time for the
same-size road graph as context, and with --cpu the oracle port's
(single-threaded C restatement of the reference solver) time on the same
graph for the smallest size.
"""
import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16354_b200 import _lib  # noqa: E402
from paper_2306_16354_b200.core import EdgeList, edge_list_to_csr  # noqa: E402
from paper_2306_16354_b200.mst import _DeviceCsr  # noqa: E402

# name: (nodes, undirected edges, cuSLINK A100 ms from PAPER.md Table 3; the
# paper's edge column counts arcs, i.e. both directions)
GRAPHS = {
    "nyc": (263_346, 733_846 // 2, 20.217),
    "fl": (1_070_376, 2_712_798 // 2, 35.552),
    "east": (3_598_623, 8_778_114 // 2, 96.100),
    "usa": (23_947_347, 58_333_344 // 2, 478.898),
}


def road_graph(n_target, m_target, seed=0):
    rng = np.random.default_rng(seed)
    w_ = int(np.sqrt(n_target))
    h_ = (n_target + w_ - 1) // w_
    n = w_ * h_
    keep = m_target / (2.0 * n - w_ - h_)
    v = np.arange(n, dtype=np.int64)
    right = v[(v % w_) < w_ - 1]
    down = v[v < n - w_]
    right = right[rng.random(len(right)) < keep]
    down = down[rng.random(len(down)) < keep]
    src = np.concatenate([right, down])
    dst = np.concatenate([right + 1, down + w_])
    wt = rng.integers(1, 100_001, size=len(src)).astype(np.float64)
    return n, src, dst, wt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graphs", default="nyc,fl,east,usa")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--cpu", action="store_true", help="time the oracle port on the smallest graph")
    args = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm = float(peaks["hbm_gbs"])
    torch.cuda.set_device(0)
    for name in args.graphs.split(","):
        nodes, edges, paper_ms = GRAPHS[name]
        n, src, dst, wt = road_graph(nodes, edges)
        g = edge_list_to_csr(EdgeList(n, src, dst, wt))
        dev = _DeviceCsr(g)
        cap = max(n - 1, 1)
        o_src, o_dst = _lib.empty(cap, np.int32), _lib.empty(cap, np.int32)
        o_w, col = _lib.empty(cap, np.float64), _lib.empty(n, np.int32)
        ne, nc = ctypes.c_int64(), ctypes.c_int64()
        stream = torch.cuda.current_stream()

        def solve():
            _lib.call("slk_solve_mst", n, _lib.ptr(dev.offs), _lib.ptr(dev.cols), _lib.ptr(dev.w), 0, 0,
                      _lib.ptr(o_src), _lib.ptr(o_dst), _lib.ptr(o_w), _lib.ptr(col), ctypes.byref(ne),
                      ctypes.byref(nc), _lib.stream_handle())

        for _ in range(args.warmup):
            solve()
        torch.cuda.synchronize()
        _lib.profile(reset=True)
        times = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            solve()
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        prof = _lib.profile(reset=True)
        ms = float(np.mean(times))
        loop_ms = prof["mst_ms"] / args.steps
        nbytes = prof["mst_bytes"] / args.steps
        total_w = float(o_w[: ne.value].sum().item())
        line = {
            "graph": f"road-like lattice '{name}': {n} nodes, {len(src)} undirected edges "
                     f"({2 * len(src)} directed), integer weights 1..1e5",
            "solve_ms": ms, "steps_ms": [round(t, 3) for t in times],
            "round_loop_ms": loop_ms, "rounds": prof["mst_rounds"] / args.steps,
            "algorithmic_bytes": nbytes,
            "round_loop_gbs": nbytes / (loop_ms / 1e3) / 1e9 if loop_ms else None,
            "round_loop_frac_of_hbm": (nbytes / (loop_ms / 1e3) / 1e9) / hbm if loop_ms else None,
            "hbm_peak_gbs": hbm,
            "tree_edges": ne.value, "components": nc.value, "total_weight": total_w,
            "paper_a100_ms_same_size_road_graph": paper_ms,
        }
        if args.cpu and name == args.graphs.split(",")[0]:
            from oracle import oracle as orc

            t0 = time.perf_counter()
            _, _, ow, _, ncomp = orc.solve_mst(n, g.row_offsets, g.col_indices, g.weights)
            line["cpu_baseline"] = {"value_ms": (time.perf_counter() - t0) * 1e3, "cores": 1, "kind": "port",
                                    "sample": "oracle port (C restatement of ref mst.py:292-344), same graph",
                                    "same_total_weight": bool(abs(ow.sum() - total_w) <= 1e-9 * total_w),
                                    "same_components": ncomp == nc.value}
        print(json.dumps(line), flush=True)
        del dev, g


if __name__ == "__main__":
    main()
