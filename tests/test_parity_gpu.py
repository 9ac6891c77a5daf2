"""Parity of the CUDA path with the reference (golden fixtures) and the oracle.

Every comparison is bit-exact (np.array_equal on float64 values) unless the
north-star tolerance is named: MST total weight / dendrogram heights within
1e-5 relative, labels ARI == 1.0.  All tests need a B200.
"""

from pathlib import Path

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

PIPELINES = ["slink_blobs_3k_d16", "slink_blobs_2k_d64", "slink_blobs_2k_d32_k2",
             "slink_normal_600_d8_f64", "slink_tiny_k2"]


@pytest.fixture(scope="module")
def slk():
    import paper_2306_16354_b200 as slk

    return slk


def _points(g):
    x = g["x"]
    x32 = x.astype(np.float32)
    return x32 if np.array_equal(x32.astype(np.float64), x) else x


@pytest.mark.parametrize("name", PIPELINES)
def test_knn_golden(slk, name):
    g = load_golden(name)
    knn = slk.fused_knn(_points(g), int(g["k"]))
    assert np.array_equal(knn.indices, g["knn_idx"])
    assert np.array_equal(knn.distances, g["knn_dist"])


@pytest.mark.parametrize("name", PIPELINES)
def test_forest_golden(slk, name):
    g = load_golden(name)
    knn = slk.KnnGraph(g["knn_idx"], g["knn_dist"])
    res = slk.solve_mst(slk.edge_list_to_csr(knn.to_edge_list()), seed=int(g["seed"]))
    assert np.array_equal(res.edges.src, g["forest_src"])
    assert np.array_equal(res.edges.dst, g["forest_dst"])
    assert np.array_equal(res.edges.weight, g["forest_w"])
    assert np.array_equal(res.colors.colors, g["forest_colors"])
    assert res.n_components == int(g["forest_ncomp"])


@pytest.mark.parametrize("name", PIPELINES)
def test_single_linkage_golden(slk, name):
    g = load_golden(name)
    metric = "sqeuclidean" if "f64" in name else "euclidean"
    cfg = slk.LinkageConfig(n_clusters=int(g["n_clusters"]), k=int(g["k"]), seed=int(g["seed"]),
                            metric=metric)
    res = slk.single_linkage_result(_points(g), cfg)
    assert np.array_equal(res.tree.src, g["tree_src"])
    assert np.array_equal(res.tree.dst, g["tree_dst"])
    assert np.array_equal(res.tree.weight, g["tree_w"])
    assert np.array_equal(res.dendrogram.merges, g["merges"])
    assert np.array_equal(res.labels.labels, g["labels"])
    assert res.connect_iters == int(g["connect_iters"])
    # the public drop-in entry point returns the same
    dendro, labels = slk.single_linkage(_points(g), cfg)
    assert np.array_equal(dendro.merges, g["merges"]) and np.array_equal(labels.labels, g["labels"])


@pytest.mark.parametrize("name", ["slink_blobs_2k_d32_k2", "slink_tiny_k2"])
def test_connect_graph_golden(slk, name):
    g = load_golden(name)
    cfg = slk.LinkageConfig(n_clusters=int(g["n_clusters"]), k=int(g["k"]), seed=int(g["seed"]))
    forest = slk.EdgeList(len(g["x"]), g["forest_src"], g["forest_dst"], g["forest_w"])
    tree = slk.connect_graph(_points(g), forest, slk.ColorArray(g["forest_colors"]), cfg)
    assert np.array_equal(tree.src, g["tree_src"]) and np.array_equal(tree.weight, g["tree_w"])


def test_neighbors_golden(slk):
    g = load_golden("neighbors")
    knn = slk.fused_knn(g["x"], 32)  # float64 data, not float32-representable
    assert np.array_equal(knn.indices, g["knn_idx"]) and np.array_equal(knn.distances, g["knn_dist"])
    cc = slk.cross_color_1nn(g["x"], slk.ColorArray(g["colors"]))
    assert np.array_equal(cc.dst, g["cc_dst"]) and np.array_equal(cc.weight, g["cc_w"])
    nn = slk.fused_1nn(g["q"], g["xi"], g["mask"])
    assert [p.index for p in nn] == g["nn_idx"].tolist()
    assert [p.distance for p in nn] == g["nn_dist"].tolist()
    tie = slk.fused_knn(g["dup"], 6)  # exact ties and duplicates: certificate must fall back
    assert np.array_equal(tie.indices, g["tie_idx"]) and np.array_equal(tie.distances, g["tie_dist"])
    tcc = slk.cross_color_1nn(g["dup"], slk.ColorArray(g["dup_colors"]))
    assert np.array_equal(tcc.dst, g["tie_cc_dst"]) and np.array_equal(tcc.weight, g["tie_cc_w"])


def test_known_answers(slk):
    # ref tests/test_neighbors.py:46-52, :165-175, :53-59
    g = slk.fused_knn(np.array([[0.0], [1.0], [3.0]]), 1)
    assert g.indices.ravel().tolist() == [1, 0, 1]
    assert g.distances.ravel().tolist() == [1.0, 1.0, 4.0]
    assert slk.fused_knn(np.array([[0.0], [1.0], [3.0]]), 1, squared=False).distances.ravel().tolist() == [1.0, 1.0, 2.0]
    e = slk.cross_color_1nn(np.array([[0.0], [2.0]]), slk.ColorArray(np.array([0, 1])))
    assert list(e.iter_edges()) == [(0, 1, 4.0), (1, 0, 4.0)]
    e = slk.cross_color_1nn(np.array([[0.0], [0.1], [10.0]]), slk.ColorArray(np.array([0, 0, 2])),
                            squared=False)
    assert e.dst[2] == 1 and e.weight[2] == pytest.approx(9.9)
    x = np.array([[1.0, 1.0]] * 3 + [[5.0, 5.0]])
    g = slk.fused_knn(x, 2)
    assert g.indices.tolist() == [[1, 2], [0, 2], [0, 1], [0, 1]]
    assert slk.fused_1nn(np.array([[0.0, 0.0]]), np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]]))[0].index == 0
    row = np.array([[1.5, -2.0, 3.0]])
    assert slk.pairwise_l2_tile(row, row)[0, 0] == 0.0
    assert slk.pairwise_l2_tile(np.array([[0.0, 0.0]]), np.array([[3.0, 4.0]]), squared=False)[0, 0] == pytest.approx(5.0)


def test_k_full_sort_matches_oracle(slk, oracle, rng):
    x = rng.standard_normal((30, 4))
    g = slk.fused_knn(x, 29)
    oi, od = oracle.fused_knn(x, 29)
    assert np.array_equal(g.indices, oi) and np.array_equal(g.distances, od)


def test_mst_golden(slk):
    g = load_golden("mst")
    for t in range(int(g["n_graphs"])):
        n = int(g[f"g{t}_n"])
        csr = slk.edge_list_to_csr(slk.EdgeList(n, g[f"g{t}_src"], g[f"g{t}_dst"], g[f"g{t}_w"]))
        assert np.array_equal(csr.row_offsets, g[f"g{t}_offs"])
        assert np.array_equal(csr.col_indices, g[f"g{t}_cols"])
        assert np.array_equal(csr.weights, g[f"g{t}_csrw"])
        maximize = bool(g[f"g{t}_max"])
        work = slk.CsrGraph(n, csr.row_offsets, csr.col_indices, -csr.weights) if maximize else csr
        alt = slk.weight_alteration(work, seed=t)
        assert alt.theta == float(g[f"g{t}_theta"])
        assert np.array_equal(alt.graph.weights, g[f"g{t}_alt"])
        res = slk.solve_mst(csr, maximize=maximize, seed=t)
        assert np.array_equal(res.edges.src, g[f"g{t}_msrc"])
        assert np.array_equal(res.edges.dst, g[f"g{t}_mdst"])
        assert np.array_equal(res.edges.weight, g[f"g{t}_mw"])
        assert np.array_equal(res.colors.colors, g[f"g{t}_colors"])
        assert res.n_components == int(g[f"g{t}_ncomp"])
    n = int(g["f_n"])
    res = slk.solve_mst(slk.CsrGraph(n, g["f_offs"], g["f_cols"], g["f_w"]), seed=7)
    assert np.array_equal(res.edges.src, g["f_msrc"]) and np.array_equal(res.edges.weight, g["f_mw"])
    assert np.array_equal(res.colors.colors, g["f_colors"]) and res.n_components == int(g["f_ncomp"])


def test_mst_step_functions_match_oracle(slk, oracle, rng):
    from paper_2306_16354_b200.synthetic import random_connected_graph

    src, dst, w = random_connected_graph(rng, 60, 240, weights="ties")
    csr = slk.edge_list_to_csr(slk.EdgeList(60, src, dst, w))
    alt = slk.weight_alteration(csr, seed=4)
    reps = np.array([0, 17, 33])
    colors = reps[rng.integers(0, 3, size=60)]
    colors[reps] = reps
    cand = slk.min_edge_per_vertex(alt, slk.ColorArray(colors))
    pos = oracle.min_edge_scan(60, csr.row_offsets, csr.col_indices, alt.graph.weights, colors)
    assert np.array_equal(cand.position, pos)
    batch = slk.min_edge_per_supervertex(cand, slk.ColorArray(colors))
    a, b, ww = oracle.reconcile(60, cand.position, np.where(cand.position >= 0, cand.dst, -1),
                                cand.altered_weight, cand.original_weight, colors)
    assert np.array_equal(batch.src, a) and np.array_equal(batch.dst, b)
    assert np.array_equal(batch.weight, ww)
    new = slk.label_propagation(batch, slk.ColorArray(colors))
    assert np.array_equal(new.colors, oracle.propagate_colors(colors, a, b))


def test_dendrogram_golden(slk):
    g = load_golden("dendrogram")
    for t in range(int(g["n_trees"])):
        n = int(g[f"t{t}_n"])
        d = slk.build_dendrogram(slk.EdgeList(n, g[f"t{t}_src"], g[f"t{t}_dst"], g[f"t{t}_w"]), n)
        assert np.array_equal(d.merges, g[f"t{t}_merges"])
        labels = slk.extract_clusters(d, int(g[f"t{t}_c"]))
        assert np.array_equal(labels.labels, g[f"t{t}_labels"])


def test_errors(slk, rng):
    g = load_golden("neighbors")
    with pytest.raises(slk.ValidationError, match="zero"):
        slk.single_linkage(g["dup"], slk.LinkageConfig(n_clusters=2, k=3))
    q, x = rng.standard_normal((3, 2)), rng.standard_normal((4, 2))
    mask = np.ones((3, 4), dtype=bool)
    mask[1] = False
    with pytest.raises(slk.ValidationError, match="row 1"):
        slk.fused_1nn(q, x, mask)
    with pytest.raises(slk.ValidationError, match="already connected"):
        slk.cross_color_1nn(rng.standard_normal((4, 2)), slk.ColorArray(np.zeros(4, dtype=np.int64)))
    x = np.concatenate([rng.standard_normal((10, 2)), rng.standard_normal((10, 2)) + 50.0])
    knn = slk.fused_knn(x, 1)
    res = slk.solve_mst(slk.edge_list_to_csr(knn.to_edge_list()), seed=0)
    with pytest.raises(slk.ConvergenceError, match="components"):
        slk.connect_graph(x, res.edges, res.colors, slk.LinkageConfig(n_clusters=2, k=1, max_connect_iters=0))
    with pytest.raises(slk.ValidationError, match="symmetric"):
        slk.solve_mst(slk.CsrGraph(2, np.array([0, 1, 1]), np.array([1]), np.array([2.0])))
    with pytest.raises(slk.ValidationError, match="finite"):
        slk.solve_mst(slk.CsrGraph(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([np.inf, np.inf])))
    with pytest.raises(slk.ValidationError, match="empty"):
        slk.solve_mst(slk.edge_list_to_csr(slk.EdgeList.from_pairs(0, [])))
    with pytest.raises(slk.ValidationError, match="cycle"):
        slk.build_dendrogram(slk.EdgeList.from_pairs(4, [(0, 1, 1.0), (1, 2, 2.0), (2, 0, 3.0)]), 4)
    # float32 input: finiteness is checked on the device (knn.cu:make_pointset)
    for bad in (np.nan, np.inf, -np.inf):
        xf = rng.standard_normal((300, 8)).astype(np.float32)
        xf[123, 5] = bad
        with pytest.raises(slk.ValidationError, match="non-finite"):
            slk.single_linkage(xf, slk.LinkageConfig(n_clusters=2, k=3))


@pytest.mark.parametrize("n,d,k,c", [(20000, 64, 15, 20), (6000, 128, 32, 6), (5000, 32, 64, 5),
                                     (4000, 512, 8, 4), (3000, 7, 3, 3)])
def test_knn_blobs_match_oracle(slk, oracle, n, d, k, c):
    from paper_2306_16354_b200.synthetic import make_blobs

    x = make_blobs(np.random.default_rng(n + d), n, d, c).astype(np.float32)
    g = slk.fused_knn(x, k)
    rows = (0, min(n, 2048))
    oi, od = oracle.fused_knn(x, k, rows=rows)
    assert np.array_equal(g.indices[rows[0]:rows[1]], oi)
    assert np.array_equal(g.distances[rows[0]:rows[1]], od)


@pytest.mark.parametrize("n,d,k", [(8000, 32, 8), (8000, 128, 32)])
def test_knn_normal_match_oracle(slk, oracle, n, d, k):
    x = np.random.default_rng(7).standard_normal((n, d), dtype=np.float32)
    g = slk.fused_knn(x, k)
    oi, od = oracle.fused_knn(x, k, rows=(0, 1024))
    assert np.array_equal(g.indices[:1024], oi) and np.array_equal(g.distances[:1024], od)


def test_single_linkage_blobs_match_oracle(slk, oracle):
    from paper_2306_16354_b200.synthetic import make_blobs

    x = make_blobs(np.random.default_rng(11), 12000, 24, 30).astype(np.float32)
    cfg = slk.LinkageConfig(n_clusters=30, k=5, seed=2)
    res = slk.single_linkage_result(x, cfg)
    ref = oracle.single_linkage(x, 30, k=5, seed=2)
    assert np.array_equal(res.tree.src, ref["tree_src"]) and np.array_equal(res.tree.weight, ref["tree_w"])
    assert np.array_equal(res.dendrogram.merges, ref["merges"])
    assert np.array_equal(res.labels.labels, ref["labels"])
    assert res.connect_iters == ref["connect_iters"]


def test_distributed_two_ranks_one_gpu(slk):
    """The multi-GPU path (parallel.py) end to end on the device engine: two
    torchrun ranks share cuda:0 over gloo (host-staged collectives) and rank 0
    must reproduce the single-process result bit for bit."""
    import subprocess
    import sys

    worker = Path(__file__).resolve().parent / "dist_gpu_worker.py"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29561", str(worker)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "DIST_OK" in out.stdout, out.stdout[-2000:]


@pytest.mark.parametrize("qb,k", [("2", 5), ("1", 5), ("2", 1)])
def test_single_linkage_grouping_modes_match_oracle(slk, oracle, monkeypatch, qb, k):
    """Query-block pairs (two blocks per CTA sharing each converted index
    tile; at scale chosen by knn.cu:pairs_are_tight) and forced single blocks
    must both reproduce the oracle exactly, including ragged last groups."""
    from paper_2306_16354_b200.synthetic import make_blobs

    monkeypatch.setenv("SLK_TC_QB", qb)
    x = make_blobs(np.random.default_rng(5), 9000 + 77, 20, 12).astype(np.float32)
    cfg = slk.LinkageConfig(n_clusters=12, k=k, seed=1)
    res = slk.single_linkage_result(x, cfg)
    ref = oracle.single_linkage(x, 12, k=k, seed=1)
    assert np.array_equal(res.tree.src, ref["tree_src"]) and np.array_equal(res.tree.weight, ref["tree_w"])
    assert np.array_equal(res.dendrogram.merges, ref["merges"])
    assert np.array_equal(res.labels.labels, ref["labels"])


@pytest.mark.parametrize("k", [32, 48, 64])
def test_knn_large_k_tensor_path_matches_oracle(slk, oracle, k):
    """k >= 32 on the tensor path: the index is dealt over several CTAs per
    query block whose top-32 lists the refine unites (knn.cu:tc_pass)."""
    rng = np.random.default_rng(k)
    x = rng.standard_normal((6000, 40)).astype(np.float32)
    g = slk.fused_knn(x, k)
    oi, od = oracle.fused_knn(x.astype(np.float64), k, rows=(0, 1500))
    assert np.array_equal(g.indices[:1500], oi) and np.array_equal(g.distances[:1500], od)


@pytest.mark.parametrize("d,k", [(136, 8), (256, 15), (512, 8), (512, 40), (300, 1)])
def test_knn_large_d_chunked_tensor_path_matches_oracle(slk, oracle, d, k):
    """d > 128 runs the chunked tcgen05 kernel (query hi term in TMEM, index
    blocks streamed in 32-dim stages, tc_scan.cu CK); it must be the engine
    that ran (tensor-core time recorded) and match the oracle exactly."""
    from paper_2306_16354_b200 import _lib

    x = np.random.default_rng(d + k).standard_normal((5000, d), dtype=np.float32)
    _lib.profile(reset=True)
    g = slk.fused_knn(x, k)
    assert _lib.profile()["tc_ms"] > 0.0
    oi, od = oracle.fused_knn(x, k, rows=(0, 1024))
    assert np.array_equal(g.indices[:1024], oi) and np.array_equal(g.distances[:1024], od)


def test_single_linkage_large_d_matches_oracle(slk, oracle):
    """Cross-colour passes through the chunked kernel (d = 192)."""
    from paper_2306_16354_b200.synthetic import make_blobs

    x = make_blobs(np.random.default_rng(192), 6000 + 33, 192, 9).astype(np.float32)
    cfg = slk.LinkageConfig(n_clusters=9, k=4, seed=3)
    res = slk.single_linkage_result(x, cfg)
    ref = oracle.single_linkage(x, 9, k=4, seed=3)
    assert np.array_equal(res.tree.src, ref["tree_src"]) and np.array_equal(res.tree.weight, ref["tree_w"])
    assert np.array_equal(res.dendrogram.merges, ref["merges"])
    assert np.array_equal(res.labels.labels, ref["labels"])


@pytest.mark.parametrize("n_clusters", [1, 30, 5000])
def test_device_fold_matches_host_folds(slk, monkeypatch, n_clusters):
    """The merge table is built on the device (dendro.cu:krt_kernel); the
    host fold (SLK_HOST_FOLD=1: parallel per forest component, or one thread
    in order) must give the same merge table and cut bit for bit."""
    from paper_2306_16354_b200.synthetic import make_blobs

    x = make_blobs(np.random.default_rng(3), 300_000, 8, 30).astype(np.float32)
    cfg = slk.LinkageConfig(n_clusters=n_clusters, k=5)
    dev = slk.single_linkage_result(x, cfg)
    monkeypatch.setenv("SLK_HOST_FOLD", "1")
    monkeypatch.setenv("SLK_FOLD_THREADS", "1")
    seq = slk.single_linkage_result(x, cfg)
    monkeypatch.setenv("SLK_FOLD_THREADS", "8")
    par = slk.single_linkage_result(x, cfg)
    for other in (seq, par):
        assert np.array_equal(dev.dendrogram.merges, other.dendrogram.merges)
        assert np.array_equal(dev.labels.labels, other.labels.labels)
    monkeypatch.delenv("SLK_HOST_FOLD")
    d = slk.build_dendrogram(par.tree, len(x))  # standalone entry (no cut), squared weights
    assert d.merges.shape == (len(x) - 1, 4)


def _random_tree(rng, n, shape):
    if shape == "chain":
        src = np.arange(1, n)
        dst = src - 1
    elif shape == "star":
        src = np.arange(1, n)
        dst = np.zeros(n - 1, dtype=np.int64)
    elif shape == "caterpillar":
        src = np.arange(1, n)
        dst = np.where(src % 2 == 1, np.maximum(src - 2, 0), src - 1)
    else:  # random attachment
        src = np.arange(1, n)
        dst = (rng.random(n - 1) * src).astype(np.int64)
    perm = rng.permutation(n)  # random vertex ids
    return perm[src], perm[dst]


@pytest.mark.parametrize("n", [2, 3, 33, 34, 65, 1025, 4097, 200_001])
@pytest.mark.parametrize("shape", ["chain", "star", "caterpillar", "random"])
def test_dendrogram_shapes_match_oracle(slk, oracle, n, shape):
    """Device merge table vs the oracle's in-order fold on trees whose
    dendrograms are as deep (chain, caterpillar) or as flat (star) as they
    get, at sizes around the leaf windows (32) and not powers of two, with
    many tied heights (ties resolve by the canonical (a, b) key)."""
    rng = np.random.default_rng(n + len(shape))
    src, dst = _random_tree(rng, n, shape)
    w = rng.integers(0, max(2, n // 8), size=n - 1).astype(np.float64) + 0.5
    d = slk.build_dendrogram(slk.EdgeList(n, src, dst, w), n)
    assert np.array_equal(d.merges, oracle.build_dendrogram(src, dst, w, n))


@pytest.mark.parametrize("levels", [1, 3, 50])
def test_dendrogram_long_ties_match_oracle(slk, oracle, levels):
    """Heights with runs of equal values far longer than the sort's in-place
    run fix-up handles (dendro.cu:RUN_MAX): the (a, b) order inside a run
    comes from the two-sort fallback and must still match the reference."""
    rng = np.random.default_rng(levels)
    n = 5000
    src, dst = _random_tree(rng, n, "random")
    w = rng.integers(0, levels, size=n - 1).astype(np.float64) + 1.0
    d = slk.build_dendrogram(slk.EdgeList(n, src, dst, w), n)
    assert np.array_equal(d.merges, oracle.build_dendrogram(src, dst, w, n))


def test_dendrogram_cycle_large(slk):
    """A cycle in a large edge list raises the reference's error."""
    n = 100_000
    src = np.arange(1, n)
    dst = src - 1
    dst[-1] = 5  # edge (n-1, 5) closes nothing...
    src[-2], dst[-2] = 7, 3  # ...(7, 3) closes the cycle 3-4-5-6-7 and leaves n-2 disconnected
    w = np.arange(n - 1, dtype=np.float64) + 1.0
    with pytest.raises(slk.ValidationError, match="cycle"):
        slk.build_dendrogram(slk.EdgeList(n, src, dst, w), n)


def _ref_is_symmetric(g):
    """core.py:165-174 restated in numpy (stable orders, numeric weight equality)."""
    src = np.repeat(np.arange(g.n_vertices), np.diff(g.row_offsets))
    fwd = np.lexsort((g.col_indices, src))
    rev = np.lexsort((src, g.col_indices))
    return (np.array_equal(src[fwd], g.col_indices[rev]) and np.array_equal(g.col_indices[fwd], src[rev])
            and np.array_equal(g.weights[fwd], g.weights[rev]))


def test_csr_symmetry_check_sorted_unsorted_and_duplicates(slk):
    """Strictly sorted rows take the binary-search mirror check, other rows
    the reference's pairing of the two stable orders (graph.cu:csr_symmetric);
    both must agree with core.py:165-174, duplicates included."""
    from paper_2306_16354_b200.synthetic import random_connected_graph

    rng = np.random.default_rng(8)
    g = slk.edge_list_to_csr(slk.EdgeList(300, *random_connected_graph(rng, 300, 900)))
    cases = [g]
    # same graph with every row's entries shuffled (unsorted rows)
    perm = np.concatenate([g.row_offsets[i] + rng.permutation(g.row_offsets[i + 1] - g.row_offsets[i])
                           for i in range(g.n_vertices)])
    cases.append(slk.CsrGraph(g.n_vertices, g.row_offsets, g.col_indices[perm], g.weights[perm]))
    # one asymmetric weight, sorted rows
    w = g.weights.copy()
    w[5] += 1.0
    cases.append(slk.CsrGraph(g.n_vertices, g.row_offsets, g.col_indices, w))
    # duplicates: (0,1,w1),(0,1,w2) vs (1,0,w2),(1,0,w1) -- the stable orders disagree
    cases.append(slk.CsrGraph(2, np.array([0, 2, 4]), np.array([1, 1, 0, 0]), np.array([1.0, 2.0, 2.0, 1.0])))
    cases.append(slk.CsrGraph(2, np.array([0, 2, 4]), np.array([1, 1, 0, 0]), np.array([1.0, 2.0, 1.0, 2.0])))
    for c in cases:
        assert c.is_symmetric() == _ref_is_symmetric(c)
    assert [c.is_symmetric() for c in cases] == [True, True, False, False, True]
    # unsorted rows still give the same forest as the canonical CSR
    a = slk.solve_mst(cases[0], seed=4)
    b = slk.solve_mst(cases[1], seed=4)
    assert np.array_equal(a.edges.src, b.edges.src) and np.array_equal(a.edges.weight, b.edges.weight)


def test_road_lattice_mst_matches_oracle(slk, oracle):
    """Road-network-shaped graph with integer weights (many ties), as in
    scripts/bench_mst.py: the forest, its weights and the components match
    the oracle's restatement of the reference solver."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mst", Path(__file__).resolve().parents[1] / "scripts" / "bench_mst.py")
    bm = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bm)
    n, src, dst, wt = bm.road_graph(40_000, 49_000, seed=5)
    g = slk.edge_list_to_csr(slk.EdgeList(n, src, dst, wt))
    for maximize in (False, True):
        r = slk.solve_mst(g, maximize=maximize, seed=2)
        os_, od, ow, ocol, onc = oracle.solve_mst(n, g.row_offsets, g.col_indices, g.weights, maximize=maximize, seed=2)
        assert r.n_components == onc
        assert np.array_equal(r.edges.src, os_) and np.array_equal(r.edges.dst, od)
        assert np.array_equal(r.edges.weight, ow) and np.array_equal(r.colors.colors, ocol)


def test_exact_fallback_split_over_warps_matches_oracle(slk, oracle):
    """Rows the certificate rejects (exact distance ties on an integer grid)
    and k beyond the fused lists go to the float64 re-scan, whose index is
    dealt over several warps per row and merged (knn.cu:launch_exact)."""
    from paper_2306_16354_b200 import _lib

    rng = np.random.default_rng(4)
    x = rng.integers(0, 6, size=(6000, 3)).astype(np.float32)
    x += np.arange(6000, dtype=np.float32)[:, None] * 1e-3  # distinct points, many near-ties
    colors = slk.ColorArray(np.repeat(np.arange(6), 1000))
    got = slk.cross_color_1nn(x, colors)
    ref = oracle.cross_color_1nn(x.astype(np.float64), colors.colors)
    assert np.array_equal(got.dst, ref[0]) and np.array_equal(got.weight, ref[1])
    y = rng.standard_normal((3000, 16)).astype(np.float32)
    _lib.scan_stats()
    g = slk.fused_knn(y, 200)
    assert _lib.scan_stats()["rows_rescanned"] > 0
    oi, od = oracle.fused_knn(y, 200, rows=(0, 300))
    assert np.array_equal(g.indices[:300], oi) and np.array_equal(g.distances[:300], od)


@pytest.mark.parametrize("layout", ["clusters", "interleaved", "mixed_sizes"])
def test_cross_colour_colour_blocked_matches_oracle(slk, oracle, monkeypatch, layout):
    """When colour segments straddle the 128-point blocks, the cross-colour
    pass scans a colour-sorted, block-aligned copy (knn.cu:plan_colour_blocks)
    and maps candidates back; results must equal the oracle's (and the
    unblocked scan's) exactly."""
    from paper_2306_16354_b200.synthetic import make_blobs

    rng = np.random.default_rng(len(layout))
    if layout == "clusters":
        x = make_blobs(rng, 60 * 333, 16, 60).astype(np.float32)
        col = np.repeat(np.arange(60), 333)
    elif layout == "interleaved":
        x = rng.standard_normal((9000, 8)).astype(np.float32)
        col = rng.integers(0, 7, size=9000)
    else:  # clusters of 3 .. 700 points: small segments pack without padding
        sizes = rng.integers(3, 700, size=40)
        x = make_blobs(rng, int(sizes.sum()), 12, 40).astype(np.float32)
        col = np.repeat(np.arange(40), sizes)[: len(x)]
    colors = slk.ColorArray(col)
    got = slk.cross_color_1nn(x, colors)
    ref = oracle.cross_color_1nn(x.astype(np.float64), col)
    assert np.array_equal(got.dst, ref[0]) and np.array_equal(got.weight, ref[1])
    monkeypatch.setenv("SLK_NO_COLOUR_REBLOCK", "1")
    plain = slk.cross_color_1nn(x, colors)
    assert np.array_equal(plain.dst, got.dst) and np.array_equal(plain.weight, got.weight)


def test_single_linkage_unaligned_clusters_matches_oracle(slk, oracle):
    """C5-shaped (many clusters not aligned to blocks, k = 2): the connect
    passes take the colour-blocked scan."""
    from paper_2306_16354_b200.synthetic import make_blobs

    x = make_blobs(np.random.default_rng(55), 150 * 200 + 7, 24, 150).astype(np.float32)
    cfg = slk.LinkageConfig(n_clusters=150, k=2, seed=5)
    res = slk.single_linkage_result(x, cfg)
    ref = oracle.single_linkage(x, 150, k=2, seed=5)
    assert np.array_equal(res.tree.src, ref["tree_src"]) and np.array_equal(res.tree.weight, ref["tree_w"])
    assert np.array_equal(res.dendrogram.merges, ref["merges"])
    assert np.array_equal(res.labels.labels, ref["labels"])


@pytest.mark.parametrize("k", [2, 15])
def test_knn_pivot_blocked_matches_oracle(slk, oracle, monkeypatch, k):
    """Clusters that straddle the 128-point blocks: the k-NN pass scans a
    pivot-ordered copy (knn.cu:plan_pivot_blocks, self excluded by position,
    candidates mapped back); identical to the oracle and to the plain scan."""
    from paper_2306_16354_b200 import _lib
    from paper_2306_16354_b200.synthetic import make_blobs

    x = make_blobs(np.random.default_rng(k), 90 * 210, 20, 90).astype(np.float32)
    _lib.profile(reset=True)
    g = slk.fused_knn(x, k)
    oi, od = oracle.fused_knn(x, k, rows=(0, 2500))
    assert np.array_equal(g.indices[:2500], oi) and np.array_equal(g.distances[:2500], od)
    monkeypatch.setenv("SLK_NO_PIVOT_REBLOCK", "1")
    p = slk.fused_knn(x, k)
    assert np.array_equal(p.indices, g.indices) and np.array_equal(p.distances, g.distances)


def test_huge_float64_points_match_oracle(slk, oracle):
    """Finite float64 values beyond float32 range (ref PointMatrix accepts any
    finite float64): the device computes on x * 2^-e and every distance,
    weight and height scales back exactly (core.py:PointMatrix)."""
    from paper_2306_16354_b200.synthetic import make_blobs

    x = make_blobs(np.random.default_rng(21), 3000, 12, 6) * 3e38
    for metric in ("euclidean", "sqeuclidean"):
        cfg = slk.LinkageConfig(n_clusters=6, k=5, seed=1, metric=metric)
        res = slk.single_linkage_result(x, cfg)
        ref = oracle.single_linkage(x, 6, k=5, seed=1, metric=metric)
        assert np.array_equal(res.tree.src, ref["tree_src"]) and np.array_equal(res.tree.weight, ref["tree_w"])
        assert np.array_equal(res.dendrogram.merges, ref["merges"])
        assert np.array_equal(res.labels.labels, ref["labels"])
    g = slk.fused_knn(x, 7)
    oi, od = oracle.fused_knn(x, 7, rows=(0, 500))
    assert np.array_equal(g.indices[:500], oi) and np.array_equal(g.distances[:500], od)
    colors = slk.ColorArray(np.repeat(np.arange(6), 500))
    e = slk.cross_color_1nn(x, colors)
    ci, cd = oracle.cross_color_1nn(x, colors.colors, rows=(0, 500))
    assert np.array_equal(e.dst[:500], ci) and np.array_equal(e.weight[:500], cd)


@pytest.mark.parametrize("two_sorts", ["0", "1"])
def test_single_linkage_tied_distances_match_oracle(slk, oracle, monkeypatch, two_sorts):
    """Points on a small integer lattice (with a few duplicates removed):
    thousands of exactly equal squared distances, so the forest solver's
    (w_alt, a, b) order comes from long runs of equal weights.  The pipeline's
    one-sort path must fall back (or fix up) to exactly the reference's
    order; SLK_MSF_TWO_SORTS=1 forces the two-sort path for comparison.
    Reference: mst.py:198-222,292-344."""
    if two_sorts == "1":
        monkeypatch.setenv("SLK_MSF_TWO_SORTS", "1")
    else:
        monkeypatch.delenv("SLK_MSF_TWO_SORTS", raising=False)
    rng = np.random.default_rng(21)
    pts = np.unique(rng.integers(0, 9, size=(2600, 3)), axis=0).astype(np.float32)
    pts = pts[rng.permutation(len(pts))][:700]
    cfg = slk.LinkageConfig(n_clusters=5, k=6, seed=3)
    res = slk.single_linkage_result(pts, cfg)
    ref = oracle.single_linkage(pts, 5, k=6, seed=3)
    assert np.array_equal(res.tree.src, ref["tree_src"]) and np.array_equal(res.tree.dst, ref["tree_dst"])
    assert np.array_equal(res.tree.weight, ref["tree_w"])
    assert np.array_equal(res.dendrogram.merges, ref["merges"])
    assert np.array_equal(res.labels.labels, ref["labels"])
