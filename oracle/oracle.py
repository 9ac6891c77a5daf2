"""numpy-level wrapper around the CPU oracle (``oracle/slink_oracle.c``).

TEST INFRASTRUCTURE ONLY — the parity checker, never the thing measured or
shipped.  Imported by ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``; nothing in
``paper_2306_16354_b200`` imports it.

Every function restates the reference ``parlink`` function named in its
docstring (file:line into /root/reference/pkg/src/parlink) with the same
float64 operation order; the C code does the arithmetic.  The oracle is pinned
against the reference's own outputs by ``tests/test_oracle.py`` using the
fixtures that ``oracle/gen_golden.py`` produced by importing the reference.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "lib" / "liboracle.so"
_lib = None

OK, INTERNAL, INVALID, CONVERGENCE = 0, 1, 2, 3


class OracleError(Exception):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def build() -> Path:
    """Compile the oracle shared library (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build()
    lib = ctypes.CDLL(str(_LIB_PATH))
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    I = ctypes.c_int
    D = ctypes.c_double
    sig = {
        "orc_last_error": (ctypes.c_char_p, []),
        "orc_max_threads": (I, []),
        "orc_row_sq_norms": (None, [P, I64, I, P]),
        "orc_pairwise_l2": (None, [P, I64, P, I64, I, I, P]),
        "orc_knn": (I, [P, P, I64, I, I, I64, I64, P, P, I]),
        "orc_nn1": (I, [P, P, I64, P, P, I64, I, I, P, P, P, I64, I64, P, P, I]),
        "orc_knn_rows": (I, [P, P, I64, I, I, P, I64, P, P, I]),
        "orc_nn1_rows": (I, [P, P, I64, P, P, I64, I, I, P, P, P, P, I64, P, P, I]),
        "orc_edge_list_to_csr": (I64, [I64, P, P, P, I64, P, P, P]),
        "orc_csr_is_symmetric": (I, [I64, P, P, P]),
        "orc_hash_unit": (D, [I64, I64, I64]),
        "orc_weight_alteration": (I, [I64, P, P, P, I64, P, P]),
        "orc_min_edge_scan": (None, [I64, P, P, P, P, P]),
        "orc_reconcile": (I64, [I64, P, P, P, P, P, P, P, P]),
        "orc_propagate_colors": (None, [I64, P, P, P, I64]),
        "orc_solve_mst": (I, [I64, P, P, P, I, I64, P, P, P, P, P, P]),
        "orc_build_dendrogram": (I, [P, P, P, I64, P]),
        "orc_extract_clusters": (I, [P, I64, I64, P]),
        "orc_single_linkage": (I, [P, I64, I, I, I64, I, I64, I64, I, P, P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(status: int):
    if status != OK:
        raise OracleError(status, _load().orc_last_error().decode())


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int64)


def max_threads() -> int:
    return int(_load().orc_max_threads())


def row_sq_norms(x) -> np.ndarray:
    """ref neighbors.py:80-89 (_row_sq_norms)."""
    x = _f64(x)
    out = np.empty(len(x))
    _load().orc_row_sq_norms(_p(x), len(x), x.shape[1], _p(out))
    return out


def pairwise_l2_tile(q, x, squared=True) -> np.ndarray:
    """ref neighbors.py:229-243 (pairwise_l2_tile)."""
    q, x = _f64(q), _f64(x)
    out = np.empty((len(q), len(x)))
    _load().orc_pairwise_l2(_p(q), len(q), _p(x), len(x), q.shape[1], int(squared), _p(out))
    return out


def fused_knn(x, k, *, squared=True, rows=None, threads=0):
    """ref neighbors.py:246-298 (fused_knn) → (indices, distances).

    rows=(q0, q1) restricts the query rows (bounded CPU-baseline samples).
    """
    x = _f64(x)
    n, d = x.shape
    q0, q1 = rows if rows is not None else (0, n)
    norms = row_sq_norms(x)
    idx = np.empty((q1 - q0, k), dtype=np.int64)
    dist = np.empty((q1 - q0, k))
    _check(_load().orc_knn(_p(x), _p(norms), n, d, k, q0, q1, _p(idx), _p(dist), threads))
    if not squared:
        dist = np.sqrt(dist)
    return idx, dist


def knn_rows(x, k, rows, *, threads=0):
    """fused_knn (ref neighbors.py:246-298) for an explicit list of query rows
    → (indices, distances), one output row per entry of ``rows``."""
    x = _f64(x)
    n, d = x.shape
    rows = _i64(rows)
    norms = row_sq_norms(x)
    idx = np.empty((len(rows), k), dtype=np.int64)
    dist = np.empty((len(rows), k))
    _check(_load().orc_knn_rows(_p(x), _p(norms), n, d, k, _p(rows), len(rows), _p(idx), _p(dist),
                                threads))
    return idx, dist


def cross_color_1nn_rows(x, colors, rows, *, threads=0):
    """cross_color_1nn (ref neighbors.py:375-391) for an explicit list of
    query rows → (dst, squared weight) per entry of ``rows``."""
    x = _f64(x)
    n, d = x.shape
    rows, col = _i64(rows), _i64(colors)
    norms = row_sq_norms(x)
    idx = np.empty(len(rows), dtype=np.int64)
    dist = np.empty(len(rows))
    _check(_load().orc_nn1_rows(_p(x), _p(norms), n, _p(x), _p(norms), n, d, 2, _p(np.zeros(1, np.uint8)),
                                _p(col), _p(col), _p(rows), len(rows), _p(idx), _p(dist), threads))
    return idx, dist


def nn1(q, x, *, mask=None, qcolor=None, xcolor=None, squared=True, rows=None, threads=0):
    """ref neighbors.py:301-348 (_fused_1nn_arrays) → (indices, distances)."""
    q, x = _f64(q), _f64(x)
    nq, d = q.shape
    q0, q1 = rows if rows is not None else (0, nq)
    qn, xn = row_sq_norms(q), row_sq_norms(x)
    mode, m, qc, xc = 0, np.zeros(1, np.uint8), np.zeros(1, np.int64), np.zeros(1, np.int64)
    if mask is not None:
        mode, m = 1, np.ascontiguousarray(mask, dtype=np.uint8)
    elif qcolor is not None:
        mode, qc, xc = 2, _i64(qcolor), _i64(xcolor)
    idx = np.empty(q1 - q0, dtype=np.int64)
    dist = np.empty(q1 - q0)
    _check(_load().orc_nn1(_p(q), _p(qn), nq, _p(x), _p(xn), len(x), d, mode, _p(m), _p(qc), _p(xc),
                           q0, q1, _p(idx), _p(dist), threads))
    if not squared:
        dist = np.sqrt(dist)
    return idx, dist


def cross_color_1nn(x, colors, *, squared=True, rows=None, threads=0):
    """ref neighbors.py:375-391 (cross_color_1nn) → (dst, weight)."""
    return nn1(x, x, qcolor=colors, xcolor=colors, squared=squared, rows=rows, threads=threads)


def edge_list_to_csr(n, src, dst, w):
    """ref core.py:264-286 (edge_list_to_csr) → (offsets, cols, weights)."""
    src, dst, w = _i64(src), _i64(dst), _f64(w)
    m = len(src)
    offs = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(max(2 * m, 1), dtype=np.int64)
    ws = np.empty(max(2 * m, 1))
    nnz = _load().orc_edge_list_to_csr(n, _p(src), _p(dst), _p(w), m, _p(offs), _p(cols), _p(ws))
    return offs, cols[:nnz].copy(), ws[:nnz].copy()


def csr_is_symmetric(n, offs, cols, w) -> bool:
    """ref core.py:165-174 (CsrGraph.is_symmetric)."""
    offs, cols, w = _i64(offs), _i64(cols), _f64(w)
    return bool(_load().orc_csr_is_symmetric(n, _p(offs), _p(cols), _p(w)))


def hash_unit(a, b, seed) -> float:
    """ref mst.py:82-91 (_hash_unit)."""
    return float(_load().orc_hash_unit(int(a), int(b), int(seed)))


def weight_alteration(n, offs, cols, w, seed=0):
    """ref mst.py:198-222 (weight_alteration) → (altered weights, theta)."""
    offs, cols, w = _i64(offs), _i64(cols), _f64(w)
    alt = np.empty(max(len(w), 1))
    theta = ctypes.c_double()
    _check(_load().orc_weight_alteration(n, _p(offs), _p(cols), _p(w), seed, _p(alt),
                                         ctypes.byref(theta)))
    return alt[: len(w)].copy(), theta.value


def min_edge_scan(n, offs, cols, alt, colors) -> np.ndarray:
    """ref mst.py:108-128 (_min_edge_scan) → CSR position per vertex (-1 none)."""
    offs, cols, alt, colors = _i64(offs), _i64(cols), _f64(alt), _i64(colors)
    pos = np.empty(n, dtype=np.int64)
    _load().orc_min_edge_scan(n, _p(offs), _p(cols), _p(alt), _p(colors), _p(pos))
    return pos


def reconcile(n, position, cdst, calt, corig, colors):
    """ref mst.py:257-280 (min_edge_per_supervertex) → (a, b, w)."""
    args = [_i64(position), _i64(cdst), _f64(calt), _f64(corig), _i64(colors)]
    a = np.empty(max(n, 1), np.int64)
    b = np.empty(max(n, 1), np.int64)
    w = np.empty(max(n, 1))
    m = _load().orc_reconcile(n, *[_p(v) for v in args], _p(a), _p(b), _p(w))
    return a[:m].copy(), b[:m].copy(), w[:m].copy()


def propagate_colors(colors, us, vs) -> np.ndarray:
    """ref mst.py:283-289 (label_propagation) / _propagate_colors (:154-186)."""
    out = _i64(colors).copy()
    us, vs = _i64(us), _i64(vs)
    _load().orc_propagate_colors(len(out), _p(out), _p(us), _p(vs), len(us))
    return out


def solve_mst(n, offs, cols, w, maximize=False, seed=0):
    """ref mst.py:292-344 (solve_mst) → (src, dst, w, colors, n_components)."""
    offs, cols, w = _i64(offs), _i64(cols), _f64(w)
    src = np.empty(max(n - 1, 1), np.int64)
    dst = np.empty(max(n - 1, 1), np.int64)
    ow = np.empty(max(n - 1, 1))
    colors = np.empty(max(n, 1), np.int64)
    ne, nc = ctypes.c_int64(), ctypes.c_int64()
    _check(_load().orc_solve_mst(n, _p(offs), _p(cols), _p(w), int(maximize), seed, _p(src), _p(dst),
                                 _p(ow), ctypes.byref(ne), _p(colors), ctypes.byref(nc)))
    m = ne.value
    return src[:m].copy(), dst[:m].copy(), ow[:m].copy(), colors[:n].copy(), nc.value


def build_dendrogram(src, dst, w, n) -> np.ndarray:
    """ref linkage.py:160-181 (build_dendrogram) → merges (n-1, 4)."""
    src, dst, w = _i64(src), _i64(dst), _f64(w)
    merges = np.empty((max(n - 1, 1), 4))
    _check(_load().orc_build_dendrogram(_p(src), _p(dst), _p(w), n, _p(merges)))
    return merges[: n - 1].copy()


def extract_clusters(merges, n, n_clusters) -> np.ndarray:
    """ref linkage.py:184-213 (extract_clusters) → labels."""
    merges = _f64(merges).reshape(-1, 4) if n > 1 else np.zeros((1, 4))
    labels = np.empty(n, np.int64)
    _check(_load().orc_extract_clusters(_p(merges), n, n_clusters, _p(labels)))
    return labels


def single_linkage(x, n_clusters, k=15, metric="euclidean", seed=0, max_connect_iters=None,
                   threads=0):
    """ref linkage.py:257-311 (single_linkage).

    Returns dict(merges, labels, tree_src, tree_dst, tree_w (squared L2),
    connect_iters).
    """
    x = _f64(x)
    n, d = x.shape
    merges = np.empty((max(n - 1, 1), 4))
    labels = np.empty(n, np.int64)
    ts = np.empty(max(n - 1, 1), np.int64)
    td = np.empty(max(n - 1, 1), np.int64)
    tw = np.empty(max(n - 1, 1))
    iters = ctypes.c_int64()
    budget = -1 if max_connect_iters is None else int(max_connect_iters)
    _check(_load().orc_single_linkage(_p(x), n, d, k, n_clusters, int(metric == "euclidean"), seed,
                                      budget, threads, _p(merges), _p(labels), _p(ts), _p(td),
                                      _p(tw), ctypes.byref(iters)))
    return dict(merges=merges[: n - 1].copy(), labels=labels, tree_src=ts[: n - 1].copy(),
                tree_dst=td[: n - 1].copy(), tree_w=tw[: n - 1].copy(), connect_iters=iters.value)


def connect_budget(n: int) -> int:
    """ref linkage.py:216-219 (_resolve_connect_budget) default."""
    return math.ceil(math.log2(max(n, 2))) + 8


def adjusted_rand_index(labels_a, labels_b) -> float:
    """Adjusted Rand index (restates ref oracles.py:168-194)."""
    a = np.asarray(labels_a).ravel()
    b = np.asarray(labels_b).ravel()
    n = len(a)
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    na, nb = int(ai.max()) + 1, int(bi.max()) + 1
    cont = np.bincount(ai * nb + bi, minlength=na * nb).reshape(na, nb)
    c2 = lambda v: v * (v - 1) // 2  # noqa: E731
    cells = int(c2(cont).sum())
    rows = int(c2(cont.sum(axis=1)).sum())
    cols = int(c2(cont.sum(axis=0)).sum())
    total = c2(n)
    if total == 0:
        return 1.0
    expected = rows * cols / total
    mx = (rows + cols) / 2
    if mx == expected:
        return 1.0
    return (cells - expected) / (mx - expected)


def kruskal_mst(n, src, dst, w):
    """Kruskal forest by (w, a, b) (restates ref oracles.py:62-99) → (a, b, w)."""
    src, dst, w = _i64(src), _i64(dst), _f64(w)
    a, b = np.minimum(src, dst), np.maximum(src, dst)
    order = np.lexsort((b, a, w))
    a, b, w = a[order], b[order], w[order]
    parent = np.arange(n)

    def find(v):
        while parent[v] != v:
            parent[v] = parent[parent[v]]
            v = parent[v]
        return v

    keep = np.zeros(len(a), bool)
    for e in range(len(a)):
        ra, rb = find(a[e]), find(b[e])
        if ra != rb:
            parent[rb] = ra
            keep[e] = True
    return a[keep], b[keep], w[keep]


if os.environ.get("SLK_ORACLE_BUILD_ON_IMPORT"):
    build()
