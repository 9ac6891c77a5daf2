"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python scripts/sanitize_run.py

Drives every kernel family of libslink.so once at a size where the sanitizer
finishes in minutes: the full single-linkage pipeline on 3,000 blob points
(tcgen05 k-NN and cross-colour scans, the block-centred scan with its split
index and the multi-GPU shard driver, refine, visit order, Boruvka rounds,
connect loop, dendrogram sort + device merge table (krt_kernel, both the
one-sort and the two-sort paths) + cut), the chunked large-d tensor kernel
(d = 192), the exact-fp32/float64 fallbacks (integer grid with ties), the
colour-blocked and pivot-blocked scans, and a general-graph MST with maximize.
Each result is checked against the CPU oracle so a sanitizer run that
perturbs timing still has to produce the reference's answer.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2306_16354_b200 as slk  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2306_16354_b200.synthetic import make_blobs, random_connected_graph  # noqa: E402


def step(msg):
    print("step:", msg, flush=True)


def main():
    x = make_blobs(np.random.default_rng(0), 3000, 16, 12).astype(np.float32)
    res = slk.single_linkage_result(x, slk.LinkageConfig(n_clusters=12, k=15, seed=0))
    ref = orc.single_linkage(x, 12, k=15, seed=0)
    assert np.array_equal(res.dendrogram.merges, ref["merges"])
    assert np.array_equal(res.labels.labels, ref["labels"])

    step("pipeline 3000x16")
    # small k: connect loop with several iterations, colour-aligned blocks
    y = make_blobs(np.random.default_rng(1), 2500, 24, 60).astype(np.float32)
    res = slk.single_linkage_result(y, slk.LinkageConfig(n_clusters=60, k=2, seed=1))
    ref = orc.single_linkage(y, 60, k=2, seed=1)
    assert np.array_equal(res.tree.src, ref["tree_src"]) and np.array_equal(res.labels.labels, ref["labels"])

    step("pipeline 2500x24 k=2")
    # block-centred kernel (cross-colour passes at d >= 64) with a split
    # index (clusters unaligned to 128-point blocks), the k-NN pass on it too
    # (SLK_TC_BC=2), and the in-process multi-GPU driver (3 shards)
    u = make_blobs(np.random.default_rng(5), 3100, 64, 9).astype(np.float32)
    ref = orc.single_linkage(u, 9, k=3, seed=0)
    for env, shards in (("1", 1), ("2", 1), ("1", 3)):
        os.environ["SLK_TC_BC"] = env
        res = slk.single_linkage_result(u, slk.LinkageConfig(n_clusters=9, k=3, seed=0), n_gpus=shards)
        assert np.array_equal(res.dendrogram.merges, ref["merges"]), (env, shards)
        assert np.array_equal(res.labels.labels, ref["labels"]), (env, shards)
        step(f"block-centred SLK_TC_BC={env} shards={shards}")
    os.environ["SLK_TC_BC"] = "1"

    # chunked tcgen05 kernel (d > 128)
    z = np.random.default_rng(2).standard_normal((1500, 192)).astype(np.float32)
    g = slk.fused_knn(z, 8)
    oi, od = orc.fused_knn(z, 8, rows=(0, 300))
    assert np.array_equal(g.indices[:300], oi) and np.array_equal(g.distances[:300], od)

    step("chunked d=192")
    # exact fallbacks: ties on an integer grid, k beyond the fused lists
    t = np.random.default_rng(3).integers(0, 5, size=(1200, 3)).astype(np.float32)
    t += np.arange(1200, dtype=np.float32)[:, None] * 1e-3
    g = slk.fused_knn(t, 130)
    oi, od = orc.fused_knn(t, 130, rows=(0, 100))
    assert np.array_equal(g.indices[:100], oi) and np.array_equal(g.distances[:100], od)

    step("exact fallbacks")
    # the device merge table on its own: a random tree deep enough for
    # several grid-wide levels, heights with long tied runs (two-sort path)
    nt = 6000
    ts = np.arange(1, nt)
    td = (np.random.default_rng(6).random(nt - 1) * ts).astype(np.int64)
    for tw in (np.random.default_rng(7).random(nt - 1) + 0.5, np.floor(np.random.default_rng(8).random(nt - 1) * 3)
               + 1.0):
        d = slk.build_dendrogram(slk.EdgeList(nt, ts, td, tw), nt)
        assert np.array_equal(d.merges, orc.build_dendrogram(ts, td, tw, nt))

    step("device merge table")
    # general-graph MST incl. maximize
    src, dst, w = random_connected_graph(np.random.default_rng(4), 400, 1500, weights="ties")
    csr = slk.edge_list_to_csr(slk.EdgeList(400, src, dst, w))
    for maximize in (False, True):
        r = slk.solve_mst(csr, maximize=maximize, seed=3)
        o = orc.solve_mst(400, csr.row_offsets, csr.col_indices, csr.weights, maximize=maximize, seed=3)
        assert np.array_equal(r.edges.src, o[0]) and np.array_equal(r.edges.weight, o[2])
    print("SANITIZE_RUN_OK")


if __name__ == "__main__":
    main()
