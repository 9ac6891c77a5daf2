"""Pin the CPU oracle (oracle/slink_oracle.c) to the reference's own outputs.

The fixtures in tests/golden were produced by running the reference package
(oracle/gen_golden.py).  Every comparison here is bit-exact: the oracle
restates the reference's float64 operation order.
"""

import numpy as np
import pytest

from conftest import load_golden

PIPELINES = ["slink_blobs_3k_d16", "slink_blobs_2k_d64", "slink_blobs_2k_d32_k2",
             "slink_normal_600_d8_f64", "slink_tiny_k2"]


@pytest.mark.parametrize("name", PIPELINES)
def test_knn_matches_reference(oracle, name):
    g = load_golden(name)
    idx, dist = oracle.fused_knn(g["x"], int(g["k"]))
    assert np.array_equal(idx, g["knn_idx"])
    assert np.array_equal(dist, g["knn_dist"])


@pytest.mark.parametrize("name", PIPELINES)
def test_forest_matches_reference(oracle, name):
    g = load_golden(name)
    n, k = len(g["x"]), int(g["k"])
    src = np.repeat(np.arange(n), k)
    offs, cols, w = oracle.edge_list_to_csr(n, src, g["knn_idx"].ravel(), g["knn_dist"].ravel())
    s, d, ww, colors, nc = oracle.solve_mst(n, offs, cols, w, seed=int(g["seed"]))
    assert np.array_equal(s, g["forest_src"]) and np.array_equal(d, g["forest_dst"])
    assert np.array_equal(ww, g["forest_w"])
    assert np.array_equal(colors, g["forest_colors"]) and nc == int(g["forest_ncomp"])


@pytest.mark.parametrize("name", PIPELINES)
def test_single_linkage_matches_reference(oracle, name):
    g = load_golden(name)
    metric = "sqeuclidean" if "sqeuclid" in name or "f64" in name else "euclidean"
    out = oracle.single_linkage(g["x"], int(g["n_clusters"]), k=int(g["k"]), seed=int(g["seed"]),
                                metric=metric)
    assert np.array_equal(out["tree_src"], g["tree_src"])
    assert np.array_equal(out["tree_dst"], g["tree_dst"])
    assert np.array_equal(out["tree_w"], g["tree_w"])
    assert np.array_equal(out["merges"], g["merges"])
    assert np.array_equal(out["labels"], g["labels"])
    assert out["connect_iters"] == int(g["connect_iters"])


def test_neighbors_known_answers(oracle):
    g = load_golden("neighbors")
    idx, dist = oracle.fused_knn(g["x"], 32)
    assert np.array_equal(idx, g["knn_idx"]) and np.array_equal(dist, g["knn_dist"])
    dst, w = oracle.cross_color_1nn(g["x"], g["colors"])
    assert np.array_equal(dst, g["cc_dst"]) and np.array_equal(w, g["cc_w"])
    i, d = oracle.nn1(g["q"], g["xi"], mask=g["mask"])
    assert np.array_equal(i, g["nn_idx"]) and np.array_equal(d, g["nn_dist"])
    i, d = oracle.fused_knn(g["dup"], 6)
    assert np.array_equal(i, g["tie_idx"]) and np.array_equal(d, g["tie_dist"])
    dst, w = oracle.cross_color_1nn(g["dup"], g["dup_colors"])
    assert np.array_equal(dst, g["tie_cc_dst"]) and np.array_equal(w, g["tie_cc_w"])


def test_neighbors_line_example(oracle):
    # ref tests/test_neighbors.py:46-52
    idx, dist = oracle.fused_knn(np.array([[0.0], [1.0], [3.0]]), 1)
    assert idx.ravel().tolist() == [1, 0, 1] and dist.ravel().tolist() == [1.0, 1.0, 4.0]
    # ref tests/test_neighbors.py:165-168
    dst, w = oracle.cross_color_1nn(np.array([[0.0], [2.0]]), np.array([0, 1]))
    assert dst.tolist() == [1, 0] and w.tolist() == [4.0, 4.0]


def test_mst_matches_reference(oracle):
    g = load_golden("mst")
    for t in range(int(g["n_graphs"])):
        n = int(g[f"g{t}_n"])
        offs, cols, w = oracle.edge_list_to_csr(n, g[f"g{t}_src"], g[f"g{t}_dst"], g[f"g{t}_w"])
        assert np.array_equal(offs, g[f"g{t}_offs"]) and np.array_equal(cols, g[f"g{t}_cols"])
        assert np.array_equal(w, g[f"g{t}_csrw"])
        maximize = bool(g[f"g{t}_max"])
        alt, theta = oracle.weight_alteration(n, offs, cols, -w if maximize else w, seed=t)
        assert theta == float(g[f"g{t}_theta"]) and np.array_equal(alt, g[f"g{t}_alt"])
        s, d, ww, colors, nc = oracle.solve_mst(n, offs, cols, w, maximize=maximize, seed=t)
        assert np.array_equal(s, g[f"g{t}_msrc"]) and np.array_equal(d, g[f"g{t}_mdst"])
        assert np.array_equal(ww, g[f"g{t}_mw"]) and np.array_equal(colors, g[f"g{t}_colors"])
        assert nc == int(g[f"g{t}_ncomp"])
    n = int(g["f_n"])
    s, d, ww, colors, nc = oracle.solve_mst(n, g["f_offs"], g["f_cols"], g["f_w"], seed=7)
    assert np.array_equal(s, g["f_msrc"]) and np.array_equal(ww, g["f_mw"])
    assert np.array_equal(colors, g["f_colors"]) and nc == int(g["f_ncomp"])


def test_dendrogram_matches_reference(oracle):
    g = load_golden("dendrogram")
    for t in range(int(g["n_trees"])):
        n = int(g[f"t{t}_n"])
        merges = oracle.build_dendrogram(g[f"t{t}_src"], g[f"t{t}_dst"], g[f"t{t}_w"], n)
        assert np.array_equal(merges, g[f"t{t}_merges"])
        labels = oracle.extract_clusters(merges, n, int(g[f"t{t}_c"]))
        assert np.array_equal(labels, g[f"t{t}_labels"])


def test_zero_weight_rejected(oracle):
    g = load_golden("neighbors")
    with pytest.raises(oracle.OracleError, match="zero-weight"):
        oracle.single_linkage(g["dup"], 2, k=3)


def test_hash_unit_known_values(oracle):
    # symmetric in the canonical key and seeded
    assert 0.0 <= oracle.hash_unit(3, 7, 0) < 1.0
    assert oracle.hash_unit(3, 7, 0) != oracle.hash_unit(3, 7, 1)
