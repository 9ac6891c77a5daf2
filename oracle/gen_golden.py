"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):

    python oracle/gen_golden.py

It imports ``parlink`` straight from /root/reference/pkg/src (numba JIT cache
redirected to /tmp so nothing is written into the read-only reference tree),
runs the reference's own public functions on seeded inputs, and writes the
results to ``tests/golden/*.npz``.  The fixtures travel with the repo; the GPU
box never needs /root/reference.  ``tests/test_oracle.py`` pins the CPU oracle
against these files and ``tests/test_parity_gpu.py`` checks the CUDA path
against both.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import parlink  # noqa: E402
from parlink import (  # noqa: E402
    ColorArray,
    EdgeList,
    LinkageConfig,
    ValidationError,
    build_dendrogram,
    connect_graph,
    cross_color_1nn,
    edge_list_to_csr,
    extract_clusters,
    fused_1nn,
    fused_knn,
    single_linkage,
    solve_mst,
    weight_alteration,
)

from paper_2306_16354_b200.synthetic import (  # noqa: E402
    make_blobs,
    random_connected_graph,
    tiny_blob_dataset,
)

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def pipeline(x, n_clusters, k, seed=0, metric="euclidean"):
    """single_linkage plus the intermediate tree (ref linkage.py:257-311)."""
    cfg = LinkageConfig(n_clusters=n_clusters, k=k, seed=seed, metric=metric)
    knn = fused_knn(x, k)
    forest = solve_mst(edge_list_to_csr(knn.to_edge_list()), seed=seed)
    iters = {"n": 0}
    orig = parlink.linkage.cross_color_1nn

    def counted(*a, **kw):
        iters["n"] += 1
        return orig(*a, **kw)

    parlink.linkage.cross_color_1nn = counted
    try:
        tree = connect_graph(x, forest.edges, forest.colors, cfg)
        dendro, labels = single_linkage(x, cfg)
    finally:
        parlink.linkage.cross_color_1nn = orig
    return dict(
        x=np.asarray(x), k=k, n_clusters=n_clusters, seed=seed,
        knn_idx=knn.indices.astype(np.int64), knn_dist=knn.distances,
        forest_src=forest.edges.src, forest_dst=forest.edges.dst, forest_w=forest.edges.weight,
        forest_colors=forest.colors.colors, forest_ncomp=forest.n_components,
        tree_src=tree.src, tree_dst=tree.dst, tree_w=tree.weight,
        merges=dendro.merges, labels=labels.labels, connect_iters=iters["n"] // 2,
    )


def save(name, **arrays):
    path = OUT / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"{path.name}: {path.stat().st_size / 1024:.0f} KiB")


def main():
    OUT.mkdir(parents=True, exist_ok=True)

    # --- end-to-end pipelines -------------------------------------------------
    # C1 geometry (BASELINE configs[0]) at 3k points, float32 inputs
    x = make_blobs(np.random.default_rng(0), 3000, 16, 10).astype(np.float32)
    save("slink_blobs_3k_d16", **pipeline(x.astype(np.float64), 10, 15))
    # d=64 blobs: large norms (the C3 geometry), exercises the error bound
    x = make_blobs(np.random.default_rng(1), 2000, 64, 8).astype(np.float32)
    save("slink_blobs_2k_d64", **pipeline(x.astype(np.float64), 8, 15, seed=3))
    # small-k stress (C5 geometry): many components, connect loop iterations
    x = make_blobs(np.random.default_rng(2), 2000, 32, 100).astype(np.float32)
    save("slink_blobs_2k_d32_k2", **pipeline(x.astype(np.float64), 100, 2, seed=1))
    # float64 inputs that are not float32-representable, sqeuclidean metric
    x = np.random.default_rng(3).standard_normal((600, 8))
    save("slink_normal_600_d8_f64", **pipeline(x, 5, 7, seed=2, metric="sqeuclidean"))
    # tiny blobs, k=2 (ref tests/test_acceptance.py:129-157 geometry)
    x = tiny_blob_dataset(np.random.default_rng(3005), 6)
    save("slink_tiny_k2", **pipeline(x, 2, 2, seed=5))

    # --- neighbours -----------------------------------------------------------
    rng = np.random.default_rng(12345)
    x = rng.standard_normal((300, 5))
    knn = fused_knn(x, 32)
    reps = np.sort(rng.choice(300, size=3, replace=False))
    reps[0] = 0
    colors = reps[rng.integers(0, 3, size=300)]
    colors[reps] = reps
    cc = cross_color_1nn(x, ColorArray(colors))
    q = rng.standard_normal((40, 4))
    xi = rng.standard_normal((60, 4))
    mask = rng.random((40, 60)) < 0.4
    mask[:, 0] = True
    nn = fused_1nn(q, xi, mask)
    # integer grid + duplicates: exact ties on every path (ref test_acceptance.py:174-194)
    grid = np.array([[i % 5, i // 5] for i in range(25)], dtype=np.float64)
    dup = np.concatenate([grid, grid[:10]])
    tie = fused_knn(dup, 6)
    dcol = np.zeros(len(dup), dtype=np.int64)
    dcol[len(grid):] = len(grid)
    tie_cc = cross_color_1nn(dup, ColorArray(dcol))
    save("neighbors", x=x, knn_idx=knn.indices, knn_dist=knn.distances, colors=colors,
         cc_dst=cc.dst, cc_w=cc.weight, q=q, xi=xi, mask=mask,
         nn_idx=np.array([p.index for p in nn]), nn_dist=np.array([p.distance for p in nn]),
         dup=dup, tie_idx=tie.indices, tie_dist=tie.distances, dup_colors=dcol,
         tie_cc_dst=tie_cc.dst, tie_cc_w=tie_cc.weight)

    # --- spanning forest ------------------------------------------------------
    rng = np.random.default_rng(4242)
    graphs = {}
    for trial in range(12):
        v = int(rng.integers(4, 300))
        e = int(rng.integers(0, 2000))
        mode = ("uniform", "ties", "equal")[trial % 3]
        src, dst, w = random_connected_graph(rng, v, e, weights=mode)
        if trial % 4 == 3:
            w = w - 5.0
            w[w == 0.0] = 0.5
        g = edge_list_to_csr(EdgeList(v, src, dst, w))
        maximize = trial % 5 == 4
        res = solve_mst(g, maximize=maximize, seed=trial)
        alt = weight_alteration(g if not maximize else parlink.CsrGraph(
            v, g.row_offsets, g.col_indices, -g.weights), seed=trial)
        graphs[f"g{trial}_n"] = v
        graphs[f"g{trial}_src"], graphs[f"g{trial}_dst"], graphs[f"g{trial}_w"] = src, dst, w
        graphs[f"g{trial}_offs"] = g.row_offsets
        graphs[f"g{trial}_cols"] = g.col_indices
        graphs[f"g{trial}_csrw"] = g.weights
        graphs[f"g{trial}_max"] = maximize
        graphs[f"g{trial}_alt"] = alt.graph.weights
        graphs[f"g{trial}_theta"] = alt.theta
        graphs[f"g{trial}_msrc"] = res.edges.src
        graphs[f"g{trial}_mdst"] = res.edges.dst
        graphs[f"g{trial}_mw"] = res.edges.weight
        graphs[f"g{trial}_colors"] = res.colors.colors
        graphs[f"g{trial}_ncomp"] = res.n_components
    # disconnected forest (ref tests/test_acceptance.py:105-126 geometry)
    src_all, dst_all, w_all, off = [], [], [], 0
    for _ in range(4):
        cv = int(rng.integers(2, 40))
        s, d, w = random_connected_graph(rng, cv, int(rng.integers(0, 60)))
        src_all.append(s + off)
        dst_all.append(d + off)
        w_all.append(w)
        off += cv
    g = edge_list_to_csr(EdgeList(off, np.concatenate(src_all), np.concatenate(dst_all),
                                  np.concatenate(w_all)))
    res = solve_mst(g, seed=7)
    graphs.update(dict(f_n=off, f_offs=g.row_offsets, f_cols=g.col_indices, f_w=g.weights,
                       f_msrc=res.edges.src, f_mdst=res.edges.dst, f_mw=res.edges.weight,
                       f_colors=res.colors.colors, f_ncomp=res.n_components))
    save("mst", n_graphs=12, **graphs)

    # --- dendrogram / cut -----------------------------------------------------
    rng = np.random.default_rng(777)
    den = {}
    for trial in range(6):
        n = int(rng.integers(3, 150))
        dst = np.array([int(rng.integers(0, v)) for v in range(1, n)])
        src = np.arange(1, n)
        w = rng.uniform(0.1, 9.0, size=n - 1)
        if trial % 2:
            w = np.round(w)  # weight ties → (a, b) tie-break
            w[w == 0] = 1.0
        d = build_dendrogram(EdgeList(n, src, dst, w), n)
        c = int(rng.integers(1, n + 1))
        labels = extract_clusters(d, c)
        den.update({f"t{trial}_n": n, f"t{trial}_src": src, f"t{trial}_dst": dst,
                    f"t{trial}_w": w, f"t{trial}_merges": d.merges, f"t{trial}_c": c,
                    f"t{trial}_labels": labels.labels})
    save("dendrogram", n_trees=6, **den)

    # error behaviour on duplicates (zero-weight edge)
    try:
        single_linkage(dup, LinkageConfig(n_clusters=2, k=3))
        raise SystemExit("expected ValidationError on duplicate points")
    except ValidationError as exc:
        print("duplicates ->", exc)


if __name__ == "__main__":
    main()
