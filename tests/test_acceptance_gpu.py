"""The reference's acceptance battery, run against the CUDA path.

Restates /root/reference/pkg/tests/test_acceptance.py criteria c01-c07 and
c09 (c08 is the CLI determinism check, covered by tests/test_cli_gpu.py; c10
is CPU thread scaling, not applicable) on the same seeded grids.  Every case
must meet the reference's own acceptance criterion (ARI = 1 against a naive
single-linkage partition, Kruskal weight within 1e-9, V - c edges, ...) AND
match the C oracle (oracle/slink_oracle.c, pinned to the reference) bit for
bit.  These random shapes are where tiling edge cases live: n < 128, d = 1,
k close to n - 1, many tiny components, ragged last blocks.
"""

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slk():
    import paper_2306_16354_b200 as slk

    return slk


def _scipy_partition(x, c):
    """Naive single linkage of the complete graph (stands in for ref
    oracles.naive_single_linkage in the ARI criterion)."""
    from scipy.cluster.hierarchy import fcluster, linkage

    return fcluster(linkage(np.asarray(x, dtype=np.float64), method="single"), t=c, criterion="maxclust")


def test_c01_single_linkage_oracle_equivalence(slk, oracle):
    """ref test_acceptance.py:56-77: 50 blob datasets, n in {50..2000}, d in {2,8,32}, k in {3,10,25}."""
    from paper_2306_16354_b200.checkers import adjusted_rand_index
    from paper_2306_16354_b200.synthetic import make_blobs

    grid = list(itertools.product([50, 200, 1000, 2000], [2, 8, 32], [2, 5, 10], [3, 10, 25]))
    picks = np.random.default_rng(20260810).permutation(len(grid))[:50]
    failures = []
    for i, (n, d, c, k) in enumerate(grid[j] for j in picks):
        x = make_blobs(np.random.default_rng(777 + i), n, d, c)
        res = slk.single_linkage_result(x, slk.LinkageConfig(n_clusters=c, k=k, seed=i))
        ref = oracle.single_linkage(x, c, k=k, seed=i)
        exact = (np.array_equal(res.dendrogram.merges, ref["merges"])
                 and np.array_equal(res.labels.labels, ref["labels"])
                 and np.array_equal(res.tree.weight, ref["tree_w"]))
        ari = adjusted_rand_index(res.labels.labels, _scipy_partition(x, c))
        if not exact or ari != 1.0:
            failures.append((i, n, d, c, k, exact, ari))
    assert not failures, failures


def test_c02_mst_optimality(slk, oracle):
    """ref test_acceptance.py:80-102: 100 random connected graphs vs Kruskal."""
    from paper_2306_16354_b200.checkers import kruskal_forest, partition_of
    from paper_2306_16354_b200.synthetic import random_connected_graph

    rng = np.random.default_rng(4242)
    failures = []
    for trial in range(100):
        v = int(rng.integers(4, 501))
        e_extra = int(rng.integers(0, 10_000 - (v - 1)))
        mode = "equal" if trial == 50 else ("ties" if trial % 3 == 0 else "uniform")
        src, dst, w = random_connected_graph(rng, v, e_extra, weights=mode)
        g = slk.edge_list_to_csr(slk.EdgeList(v, src, dst, w))
        res = slk.solve_mst(g, seed=trial)
        us, ud, uw = g.undirected_edges()
        _, _, kw = kruskal_forest(v, us, ud, uw)
        acyclic = len(np.unique(partition_of(v, res.edges.src, res.edges.dst))) == 1
        ok = (len(res.edges) == v - 1 and acyclic
              and abs(res.edges.weight.sum() - kw.sum()) <= 1e-9 * max(1.0, abs(kw.sum())))
        os_, od, ow, ocol, onc = oracle.solve_mst(v, g.row_offsets, g.col_indices, g.weights, seed=trial)
        ok &= (np.array_equal(res.edges.src, os_) and np.array_equal(res.edges.dst, od)
               and np.array_equal(res.edges.weight, ow) and np.array_equal(res.colors.colors, ocol))
        if not ok:
            failures.append(trial)
    assert not failures, failures


def test_c03_msf_law(slk, oracle):
    """ref test_acceptance.py:105-126: 50 disconnected graphs -> V - c edges, c colours."""
    from paper_2306_16354_b200.synthetic import random_connected_graph

    rng = np.random.default_rng(99)
    failures = []
    for trial in range(50):
        comps = int(rng.integers(2, 8))
        src_all, dst_all, w_all, off = [], [], [], 0
        for _ in range(comps):
            cv = int(rng.integers(2, 60))
            s, d, w = random_connected_graph(rng, cv, int(rng.integers(0, 120)))
            src_all.append(s + off)
            dst_all.append(d + off)
            w_all.append(w)
            off += cv
        g = slk.edge_list_to_csr(slk.EdgeList(off, np.concatenate(src_all), np.concatenate(dst_all),
                                              np.concatenate(w_all)))
        res = slk.solve_mst(g, seed=trial)
        ok = (len(res.edges) == off - comps and res.n_components == comps
              and len(np.unique(res.colors.colors)) == comps)
        os_, _, ow, ocol, _ = oracle.solve_mst(off, g.row_offsets, g.col_indices, g.weights, seed=trial)
        ok &= np.array_equal(res.edges.src, os_) and np.array_equal(res.edges.weight, ow)
        ok &= np.array_equal(res.colors.colors, ocol)
        if not ok:
            failures.append(trial)
    assert not failures, failures


def test_c04_reconnection(slk, oracle):
    """ref test_acceptance.py:129-157: k = 2 graphs of 3-6 tiny blobs reconnect."""
    from paper_2306_16354_b200.checkers import full_sq_dists, kruskal_forest
    from paper_2306_16354_b200.synthetic import tiny_blob_dataset

    failures = []
    for trial in range(12):
        rng = np.random.default_rng(3000 + trial)
        x = tiny_blob_dataset(rng, int(rng.integers(3, 7)))
        n = len(x)
        knn = slk.fused_knn(x, 2)
        forest = slk.solve_mst(slk.edge_list_to_csr(knn.to_edge_list()), seed=trial)
        if forest.n_components < 3:
            failures.append((trial, "not >= 3 components"))
            continue
        cfg = slk.LinkageConfig(n_clusters=2, k=2, seed=trial)
        spanning = slk.connect_graph(x, forest.edges, forest.colors, cfg)
        dendro = slk.build_dendrogram(slk.EdgeList(n, spanning.src, spanning.dst, np.sqrt(spanning.weight)), n)
        # naive: Kruskal over the complete graph, same merge heights and sizes
        d2 = full_sq_dists(x, x)
        iu, ju = np.triu_indices(n, 1)
        ks, kd, kw = kruskal_forest(n, iu, ju, np.sqrt(d2[iu, ju]))
        naive = oracle.build_dendrogram(ks, kd, kw, n)
        ok = (len(spanning) == n - 1
              and np.allclose(dendro.distances, naive[:, 2], rtol=1e-9, atol=0)
              and np.array_equal(np.sort(dendro.merges[:, :2], axis=1), np.sort(naive[:, :2], axis=1))
              and np.array_equal(dendro.sizes, naive[:, 3].astype(np.int64)))
        ref = oracle.single_linkage(x, 2, k=2, seed=trial)
        ok &= np.array_equal(spanning.src, ref["tree_src"]) and np.array_equal(spanning.weight, ref["tree_w"])
        if not ok:
            failures.append((trial, "mismatch"))
    assert not failures, failures


def test_c05_fused_neighbor_exactness(slk, oracle):
    """ref test_acceptance.py:160-208: 50 random k-NN cases (n 10-500, d 1-16,
    k up to 64) plus exact-tie grids on the k-NN, 1-NN and cross-colour paths."""
    from paper_2306_16354_b200.checkers import full_sq_dists, sorted_knn

    rng = np.random.default_rng(555)
    failures = []
    for trial in range(50):
        n = int(rng.integers(10, 501))
        d = int(rng.integers(1, 17))
        k = int(rng.integers(1, min(n - 1, 64) + 1))
        x = rng.standard_normal((n, d))
        rng.integers(1, 128), rng.integers(1, 256)  # the reference draws a tile shape here
        g = slk.fused_knn(x, k)
        si, sd = sorted_knn(x, k)
        oi, od = oracle.fused_knn(x, k)
        if not (np.array_equal(g.indices, si) and np.allclose(g.distances, sd, rtol=1e-6, atol=1e-12)
                and np.array_equal(g.indices, oi) and np.array_equal(g.distances, od)):
            failures.append(("knn", trial, n, d, k))
    # k = n - 1 (full sort) and tiny n, d = 1
    for n, d in [(2, 1), (3, 1), (17, 1), (129, 2), (200, 1), (257, 3)]:
        x = np.random.default_rng(n * 10 + d).standard_normal((n, d))
        for k in sorted({1, n - 1, max(1, min(n - 1, 64))}):
            g = slk.fused_knn(x, k)
            oi, od = oracle.fused_knn(x, k)
            if not (np.array_equal(g.indices, oi) and np.array_equal(g.distances, od)):
                failures.append(("knn-edge", n, d, k))
    grid = np.array([[i % 5, i // 5] for i in range(25)], dtype=np.float64)
    dup = np.concatenate([grid, grid[:10]])
    tie = slk.fused_knn(dup, 6)
    ti, td = oracle.fused_knn(dup, 6)
    if not (np.array_equal(tie.indices, ti) and np.array_equal(tie.distances, td)):
        failures.append("knn ties")
    eye = ~np.eye(len(dup), dtype=bool)
    pairs = slk.fused_1nn(dup, dup, eye)
    qi, qd = oracle.nn1(dup, dup, mask=eye)
    if [p.index for p in pairs] != qi.tolist() or [p.distance for p in pairs] != qd.tolist():
        failures.append("1nn ties")
    colors = np.zeros(len(dup), dtype=np.int64)
    colors[len(grid):] = len(grid)
    edges = slk.cross_color_1nn(dup, slk.ColorArray(colors))
    d2 = full_sq_dists(dup, dup)
    d2[colors[:, None] == colors[None, :]] = np.inf
    ci = np.argmin(d2, axis=1)  # first minimum = smallest id on ties
    ref_i, ref_d = oracle.cross_color_1nn(dup, colors)
    if not (np.array_equal(edges.dst, ci) and np.array_equal(edges.dst, ref_i)
            and np.array_equal(edges.weight, ref_d)):
        failures.append("cross-colour ties")
    rng2 = np.random.default_rng(556)
    q, xs = rng2.standard_normal((80, 6)), rng2.standard_normal((200, 6))
    pairs = slk.fused_1nn(q, xs)
    oi2, od2 = oracle.nn1(q, xs)
    if [p.index for p in pairs] != oi2.tolist() or [p.distance for p in pairs] != od2.tolist():
        failures.append("1nn random")
    assert not failures, failures


def test_c06_alteration_properties(slk, oracle):
    """ref test_acceptance.py:211-250: alteration keeps order, is distinct and symmetric."""
    from paper_2306_16354_b200.synthetic import random_connected_graph

    rng = np.random.default_rng(66)
    failures = []
    for trial in range(50):
        v = int(rng.integers(4, 120))
        e_extra = int(rng.integers(0, max(2, min(2000 - v, 900))))
        mode = ("uniform", "ties", "equal")[trial % 3]
        src, dst, w = random_connected_graph(rng, v, e_extra, weights=mode)
        g = slk.edge_list_to_csr(slk.EdgeList(v, src, dst, w))
        alt = slk.weight_alteration(g, seed=trial)
        oalt, otheta = oracle.weight_alteration(v, g.row_offsets, g.col_indices, g.weights, seed=trial)
        aw = alt.graph.weights
        s = g.row_sources()
        a, b = np.minimum(s, g.col_indices), np.maximum(s, g.col_indices)
        _, first, inv = np.unique(a * v + b, return_index=True, return_inverse=True)
        uw, uo = aw[first], g.weights[first]
        sym = np.array_equal(aw, uw[inv])  # both directions carry one altered value
        # order kept: a strictly smaller original weight stays strictly smaller
        o = np.argsort(uo, kind="stable")
        so, sw = uo[o], uw[o]
        step = np.nonzero(np.diff(so) > 0)[0] + 1
        prefix_max = np.maximum.accumulate(sw)
        suffix_min = np.minimum.accumulate(sw[::-1])[::-1]
        kept = bool(np.all(prefix_max[step - 1] < suffix_min[step]))
        ok = np.array_equal(aw, oalt) and alt.theta == otheta and sym and kept
        if not ok:
            failures.append(trial)
    assert not failures, failures


def test_c07_formula_conformance(slk):
    """ref test_acceptance.py:253-283: cut level, parent ids n + i, monotone heights, sizes."""
    from paper_2306_16354_b200.synthetic import make_blobs

    assert all(slk.compute_cut_level(n, c) == (n - 1) - (c - 1) for n in range(1, 65) for c in range(1, n + 1))
    rng = np.random.default_rng(77)
    for trial in range(10):
        n = int(rng.integers(3, 200))
        x = make_blobs(rng, n, 3, min(3, n))
        dendro, _ = slk.single_linkage(x, slk.LinkageConfig(n_clusters=1, k=min(5, n - 1), seed=trial))
        ch = dendro.merges[:, :2].astype(np.int64)
        assert np.all((ch >= 0) & (ch < (n + np.arange(n - 1))[:, None]))
        assert np.all(np.diff(dendro.distances) >= 0)
        sizes = np.concatenate([np.ones(n), dendro.merges[:, 3]])
        assert np.array_equal(dendro.merges[:, 3], sizes[ch[:, 0]] + sizes[ch[:, 1]])


def test_c09_max_tree_duality(slk, oracle):
    """ref test_acceptance.py:315-335: maximize == negate-minimize-negate."""
    from paper_2306_16354_b200.synthetic import random_connected_graph

    rng = np.random.default_rng(909)
    failures = []
    for trial in range(20):
        v = int(rng.integers(4, 200))
        src, dst, w = random_connected_graph(rng, v, int(rng.integers(0, 1500)))
        if trial % 4 == 0:
            w = w - 5.0
            w[w == 0.0] = 0.5
        g = slk.edge_list_to_csr(slk.EdgeList(v, src, dst, w))
        res_max = slk.solve_mst(g, maximize=True, seed=trial)
        res_neg = slk.solve_mst(slk.CsrGraph(g.n_vertices, g.row_offsets, g.col_indices, -g.weights), seed=trial)
        om = oracle.solve_mst(v, g.row_offsets, g.col_indices, g.weights, maximize=True, seed=trial)
        if not (np.array_equal(res_max.edges.src, res_neg.edges.src)
                and np.array_equal(res_max.edges.dst, res_neg.edges.dst)
                and np.array_equal(res_max.edges.weight, -res_neg.edges.weight)
                and np.array_equal(res_max.edges.src, om[0]) and np.array_equal(res_max.edges.weight, om[2])):
            failures.append(trial)
    assert not failures, failures
