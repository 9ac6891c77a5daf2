"""Configuration-scale golden digests (TEST INFRASTRUCTURE, build container only).

    python oracle/gen_config_golden.py C1 --impl reference   # parlink itself
    python oracle/gen_config_golden.py C3 --impl oracle      # the C restatement

Runs single linkage on BASELINE.json's configurations at their FULL size, on
exactly the inputs ``bench.py`` times (``synthetic.bench_points``, seed 0,
float32 points handed to the reference as float64), and writes
``tests/golden/configs/<C>_<impl>.json``: sha256 digests of every output array
in a canonical dtype (tree src/dst int64, tree weights float64 squared L2,
merges float64 (n-1)x4, labels int64), the connect-iteration count, the MST
total weight and a few merge rows for diagnosis.  ``tests/test_configs_gpu.py``
recomputes the digests of the CUDA pipeline's outputs on the B200 and requires
equality: a bit-exact end-to-end comparison at 10k / 100k / 500k / 1M points
without shipping 100 MB fixtures.

``--impl reference`` imports parlink from /root/reference/pkg/src (numba JIT
cache redirected to /tmp); it is how the C restatement is pinned at C1 and C2
(both digests must agree).  ``--impl oracle`` runs oracle/slink_oracle.c with
OpenMP (C3 takes about an hour on 8 cores; the reference itself ~4.6 h).
With ``--save-npz DIR`` the full arrays are also written there (not tracked).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:] = [str(ROOT)] + [p for p in sys.path if Path(p or ".").resolve() != Path(__file__).resolve().parent]

CONFIGS = {  # = bench.py CONFIGS (BASELINE.json configs[0,1,2,4])
    "C1": dict(n=10_000, d=16, c=10, k=15, n_clusters=10),
    "C2": dict(n=100_000, d=128, c=50, k=15, n_clusters=50),
    "C3": dict(n=1_000_000, d=64, c=50, k=15, n_clusters=50),
    "C5": dict(n=500_000, d=32, c=1000, k=2, n_clusters=1000),
}
OUT = ROOT / "tests" / "golden" / "configs"


def digest(a, dtype) -> str:
    a = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    return hashlib.sha256(a.tobytes()).hexdigest()


def summarise(name, impl, c, x, tree_src, tree_dst, tree_w, merges, labels, iters, seconds):
    order = np.argsort(merges[:, 2], kind="stable")
    return {
        "config": name, "impl": impl, **c, "metric": "euclidean", "seed": 0,
        "x_sha256": digest(x, np.float32),
        "tree_src_sha256": digest(tree_src, np.int64),
        "tree_dst_sha256": digest(tree_dst, np.int64),
        "tree_w_sha256": digest(tree_w, np.float64),
        "merges_sha256": digest(merges, np.float64),
        "labels_sha256": digest(labels, np.int64),
        "connect_iters": int(iters),
        "mst_total_weight_sq": float(np.sum(tree_w)),
        "mst_total_weight": float(np.sum(np.sqrt(tree_w))),
        "merges_first": merges[:3].tolist(),
        "merges_last": merges[-3:].tolist(),
        "label_sizes_top": np.sort(np.bincount(labels))[::-1][:5].tolist(),
        "max_height_row": int(order[-1]),
        "seconds": round(seconds, 1),
    }


def run_reference(c, x):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    import parlink
    from parlink import LinkageConfig, connect_graph, edge_list_to_csr, fused_knn, solve_mst

    x64 = x.astype(np.float64)
    cfg = LinkageConfig(n_clusters=c["n_clusters"], k=c["k"], seed=0)
    # the tree and the iteration count: the reference's own building blocks in
    # single_linkage's order (linkage.py:287-293), counting cross-colour passes
    knn = fused_knn(x64, c["k"])
    forest = solve_mst(edge_list_to_csr(knn.to_edge_list()), seed=0)
    calls = {"n": 0}
    orig = parlink.linkage.cross_color_1nn

    def counted(*a, **kw):
        calls["n"] += 1
        return orig(*a, **kw)

    parlink.linkage.cross_color_1nn = counted
    try:
        tree = connect_graph(x64, forest.edges, forest.colors, cfg)
    finally:
        parlink.linkage.cross_color_1nn = orig
    dendro, labels = parlink.single_linkage(x64, cfg)
    return tree.src, tree.dst, tree.weight, dendro.merges, labels.labels, calls["n"]


def run_oracle(c, x, threads):
    from oracle import oracle as orc

    orc.build()
    r = orc.single_linkage(x.astype(np.float64), c["n_clusters"], k=c["k"], seed=0, threads=threads)
    return r["tree_src"], r["tree_dst"], r["tree_w"], r["merges"], r["labels"], r["connect_iters"]


def main():
    from paper_2306_16354_b200.synthetic import bench_points

    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--impl", choices=["reference", "oracle"], default="oracle")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--save-npz", default=None)
    args = ap.parse_args()
    c = CONFIGS[args.config]
    x = bench_points(c["n"], c["d"], c["c"], seed=0)
    t0 = time.time()
    if args.impl == "reference":
        out = run_reference(c, x)
    else:
        out = run_oracle(c, x, args.threads)
    secs = time.time() - t0
    s = summarise(args.config, args.impl, c, x, *out, secs)
    OUT.mkdir(parents=True, exist_ok=True)
    path = OUT / f"{args.config}_{args.impl}.json"
    path.write_text(json.dumps(s, indent=1) + "\n")
    print(path, json.dumps({k: s[k] for k in ("connect_iters", "mst_total_weight", "seconds")}))
    if args.save_npz:
        Path(args.save_npz).mkdir(parents=True, exist_ok=True)
        np.savez(Path(args.save_npz) / f"{args.config}_{args.impl}.npz", tree_src=out[0], tree_dst=out[1],
                 tree_w=out[2], merges=out[3], labels=out[4])


if __name__ == "__main__":
    main()
