"""Parity at BASELINE.json's configurations, full size, on the bench inputs.

C1 10k x 16 k15 c10, C2 100k x 128 k15 c50, C3 1M x 64 k15 c50 (the headline)
and C5 500k x 32 k2 c1000 run through the CUDA pipeline exactly as bench.py
times them (``synthetic.bench_points``, seed 0).  Two layers of evidence:

* ``test_pipeline_digest``: the spanning tree, merge table and labels of
  ``single_linkage_result`` are hashed (sha256 of canonical int64 / float64
  bytes) and compared with ``tests/golden/configs/<C>_*.json``, which
  ``oracle/gen_config_golden.py`` wrote by running the REFERENCE itself
  (parlink, C1 and C2) and the C restatement (oracle, C1, C2, C3, C5; equal to
  parlink wherever both ran).  Equal digests = bit-identical outputs.
* ``test_stagewise_matches_oracle``: every stage of the path checked on its
  own against the oracle, so a mismatch names the stage: k-NN rows (one
  contiguous and three random 1024-row samples), the symmetrised CSR and the
  spanning forest of the full k-NN graph, every connect iteration's
  cross-colour bridges (same samples, that iteration's real colours) and its
  union forest, then the merge table and cut of the GPU tree.

The k-NN-only sweep C4 (1M N(0,1) points) is covered by
``test_c4_knn_rows_match_oracle`` at one k per d.
All comparisons are bit-exact.  Reference: linkage.py:257-311.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CONFIGS = {
    "C1": dict(n=10_000, d=16, c=10, k=15, n_clusters=10),
    "C2": dict(n=100_000, d=128, c=50, k=15, n_clusters=50),
    "C3": dict(n=1_000_000, d=64, c=50, k=15, n_clusters=50),
    "C5": dict(n=500_000, d=32, c=1000, k=2, n_clusters=1000),
}
DIGEST_KEYS = ("tree_src_sha256", "tree_dst_sha256", "tree_w_sha256", "merges_sha256", "labels_sha256")


def _digest(a, dtype):
    """sha256 of the canonical bytes (as oracle/gen_config_golden.py:digest)."""
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(np.asarray(a), dtype=dtype).tobytes()).hexdigest()


def _golden(name):
    """The digests of every implementation that ran this config; they must agree."""
    files = sorted((GOLDEN / "configs").glob(f"{name}_*.json"))
    assert files, f"no golden digests for {name}"
    docs = [json.loads(f.read_text()) for f in files]
    for d in docs[1:]:
        for key in DIGEST_KEYS + ("x_sha256", "connect_iters"):
            assert d[key] == docs[0][key], f"{files[0].name} and {d['impl']} disagree on {key}"
    return docs[0], [d["impl"] for d in docs]


_POINTS = {}


def _points(name):
    from paper_2306_16354_b200.synthetic import bench_points

    if name not in _POINTS:
        c = CONFIGS[name]
        _POINTS.clear()  # one config resident at a time (C3: 256 MB + float64 copy)
        _POINTS[name] = bench_points(c["n"], c["d"], c["c"], seed=0)
    return _POINTS[name]


def _sample_rows(n, seed):
    rng = np.random.default_rng(seed)
    rows = [np.arange(min(n, 1024))]
    for _ in range(3):
        rows.append(np.sort(rng.choice(n, size=min(n, 1024), replace=False)))
    return np.unique(np.concatenate(rows))


@pytest.fixture(scope="module")
def slk():
    import paper_2306_16354_b200 as slk

    return slk


@pytest.mark.parametrize("name", ["C1", "C2", "C5", "C3"])
def test_pipeline_digest(slk, name):
    g, impls = _golden(name)
    c = CONFIGS[name]
    x = _points(name)
    assert _digest(x, np.float32) == g["x_sha256"], "bench inputs differ from the golden run's"
    cfg = slk.LinkageConfig(n_clusters=c["n_clusters"], k=c["k"], seed=0)
    res = slk.single_linkage_result(x, cfg)
    got = {
        "tree_src_sha256": _digest(res.tree.src, np.int64),
        "tree_dst_sha256": _digest(res.tree.dst, np.int64),
        "tree_w_sha256": _digest(res.tree.weight, np.float64),
        "merges_sha256": _digest(res.dendrogram.merges, np.float64),
        "labels_sha256": _digest(res.labels.labels, np.int64),
    }
    bad = [k for k in DIGEST_KEYS if got[k] != g[k]]
    assert not bad, (f"{name}: {bad} differ from {impls}; MST weight {np.sum(np.sqrt(res.tree.weight))!r} "
                     f"vs {g['mst_total_weight']!r}, first merges {res.dendrogram.merges[:3].tolist()} "
                     f"vs {g['merges_first']}")
    assert res.connect_iters == g["connect_iters"]
    if name == "C1":
        # the drop-in entry point (ref linkage.py:257) returns the same arrays
        dendro, labels = slk.single_linkage(x, cfg)
        assert _digest(dendro.merges, np.float64) == g["merges_sha256"]
        assert _digest(labels.labels, np.int64) == g["labels_sha256"]


def _forest_equal(res, o):
    s, d, w, col, nc = o
    assert res.n_components == nc
    assert np.array_equal(res.edges.src, s) and np.array_equal(res.edges.dst, d)
    assert np.array_equal(res.edges.weight, w)
    assert np.array_equal(res.colors.colors, col)


@pytest.mark.parametrize("name", ["C2", "C5", "C3"])
def test_stagewise_matches_oracle(slk, oracle, name):
    c = CONFIGS[name]
    n, k = c["n"], c["k"]
    x = _points(name)
    x64 = x.astype(np.float64)
    rows = _sample_rows(n, seed=len(name) + n)

    # (i) k-NN rows (neighbors.py:246-298)
    knn = slk.fused_knn(x, k)
    oi, od = oracle.knn_rows(x64, k, rows)
    assert np.array_equal(knn.indices[rows], oi), f"{name}: k-NN indices differ"
    assert np.array_equal(knn.distances[rows], od), f"{name}: k-NN distances differ"

    # (iii) symmetrised CSR and forest of the full GPU k-NN graph (core.py:264-286, mst.py:292-344)
    el = knn.to_edge_list()
    csr = slk.edge_list_to_csr(el)
    offs, cols, ws = oracle.edge_list_to_csr(n, el.src, el.dst, el.weight)
    assert np.array_equal(csr.row_offsets, offs) and np.array_equal(csr.col_indices, cols)
    assert np.array_equal(csr.weights, ws)
    res = slk.solve_mst(csr, seed=0)
    _forest_equal(res, oracle.solve_mst(n, offs, cols, ws, seed=0))

    # (ii) + (iii) every connect iteration (linkage.py:222-254) with its real colours
    iters = 0
    while res.n_components > 1:
        colors = res.colors
        bridges = slk.cross_color_1nn(x, colors)
        bi, bw = oracle.cross_color_1nn_rows(x64, colors.colors, rows)
        assert np.array_equal(bridges.dst[rows], bi), f"{name} iteration {iters}: bridges differ"
        assert np.array_equal(bridges.weight[rows], bw), f"{name} iteration {iters}: bridge weights differ"
        union = slk.EdgeList(n, np.concatenate([res.edges.src, bridges.src]),
                             np.concatenate([res.edges.dst, bridges.dst]),
                             np.concatenate([res.edges.weight, bridges.weight]))
        csr = slk.edge_list_to_csr(union)
        res = slk.solve_mst(csr, seed=0)
        _forest_equal(res, oracle.solve_mst(n, csr.row_offsets, csr.col_indices, csr.weights, seed=0))
        iters += 1
    tree = res.edges

    # the one-call pipeline reproduces the stage-by-stage tree
    cfg = slk.LinkageConfig(n_clusters=c["n_clusters"], k=k, seed=0)
    full = slk.single_linkage_result(x, cfg)
    assert full.connect_iters == iters
    assert np.array_equal(full.tree.src, tree.src) and np.array_equal(full.tree.dst, tree.dst)
    assert np.array_equal(full.tree.weight, tree.weight)

    # (iv) dendrogram and cut of the GPU tree (linkage.py:160-213)
    merges = oracle.build_dendrogram(tree.src, tree.dst, np.sqrt(tree.weight), n)
    assert np.array_equal(full.dendrogram.merges, merges), f"{name}: merge table differs"
    labels = oracle.extract_clusters(merges, n, c["n_clusters"])
    assert np.array_equal(full.labels.labels, labels), f"{name}: labels differ"


@pytest.mark.parametrize("d,k", [(32, 64), (128, 32), (512, 8)])
def test_c4_knn_rows_match_oracle(slk, oracle, d, k):
    """configs[3]: k-NN graph of 1M N(0,1) points (nothing prunes; every
    tile is computed), sampled rows against the oracle."""
    from paper_2306_16354_b200.synthetic import bench_points

    _POINTS.clear()
    x = bench_points(1_000_000, d, None, seed=0)
    knn = slk.fused_knn(x, k)
    rows = _sample_rows(len(x), seed=d * 1000 + k)[:: 2 if d == 512 else 1]
    oi, od = oracle.knn_rows(x.astype(np.float64), k, rows)
    assert np.array_equal(knn.indices[rows], oi) and np.array_equal(knn.distances[rows], od)
