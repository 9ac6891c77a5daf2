"""Independent CPU checkers behind ``parlink verify`` and ``parlink mst --verify``.

The reference's CLI cross-checks library results against brute-force
restatements (cli.py:196-266 calling oracles.py).  These are this package's
own small numpy versions of the same checks: a full-matrix sorted k-NN, a
Kruskal spanning forest, a naive single-linkage partition and the adjusted
Rand index.  They only ever judge results the CUDA path produced — no
compute entry point of the package calls them, and they are sized for the
verification instances (hundreds of points, up to a few million edges).
"""

from __future__ import annotations

import numpy as np


def full_sq_dists(a, b, rows: int = 256) -> np.ndarray:
    """Squared distances by summing squared coordinate differences (no expansion)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    out = np.empty((len(a), len(b)))
    for r0 in range(0, len(a), rows):
        diff = a[r0:r0 + rows, None, :] - b[None, :, :]
        out[r0:r0 + rows] = (diff * diff).sum(axis=2)
    return out


def sorted_knn(x, k: int, squared: bool = True):
    """(indices, distances): the k nearest other rows, ordered by (distance, id)."""
    d2 = full_sq_dists(x, x)
    np.fill_diagonal(d2, np.inf)
    # a stable sort on distance keeps equal distances in id order
    order = np.argsort(d2, axis=1, kind="stable")[:, :k]
    dist = np.take_along_axis(d2, order, axis=1)
    return order.astype(np.int64), (dist if squared else np.sqrt(dist))


def kruskal_forest(n: int, src, dst, weight):
    """Spanning forest over edges taken in (weight, min id, max id) order.

    Returns the accepted (src, dst, weight) with src < dst, in merge order.
    """
    lo = np.minimum(src, dst).astype(np.int64)
    hi = np.maximum(src, dst).astype(np.int64)
    w = np.asarray(weight, dtype=np.float64)
    order = np.lexsort((hi, lo, w))
    parent = list(range(n))

    def root(v):
        while parent[v] != v:
            parent[v] = parent[parent[v]]
            v = parent[v]
        return v

    keep = []
    for e in order.tolist():
        ra, rb = root(int(lo[e])), root(int(hi[e]))
        if ra != rb:
            parent[rb] = ra
            keep.append(e)
            if len(keep) == n - 1:
                break
    keep = np.asarray(keep, dtype=np.int64)
    return lo[keep], hi[keep], w[keep]


def partition_of(n: int, src, dst) -> np.ndarray:
    """Dense labels 0..c-1 of the connected components of (n, edges)."""
    parent = np.arange(n)
    for a, b in zip(np.asarray(src).tolist(), np.asarray(dst).tolist()):
        while parent[a] != a:
            a = parent[a]
        while parent[b] != b:
            b = parent[b]
        if a != b:
            parent[b] = a
    roots = np.array([_top(parent, v) for v in range(n)])
    return np.unique(roots, return_inverse=True)[1]


def _top(parent, v):
    while parent[v] != v:
        v = parent[v]
    return v


def naive_partition(x, n_clusters: int, metric: str = "euclidean") -> np.ndarray:
    """Flat single-linkage labels from the complete graph: Kruskal, drop the top merges."""
    x = np.asarray(x, dtype=np.float64)
    n = len(x)
    d2 = full_sq_dists(x, x)
    iu, ju = np.triu_indices(n, 1)
    w = d2[iu, ju]
    if metric == "euclidean":
        w = np.sqrt(w)
    s, d, _ = kruskal_forest(n, iu, ju, w)
    keep = n - n_clusters
    return partition_of(n, s[:keep], d[:keep])


def adjusted_rand_index(a, b) -> float:
    """Adjusted Rand index of two labelings; 1.0 exactly when the partitions agree."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    if len(a) != len(b):
        raise ValueError("partitions must label the same points")
    _, ia = np.unique(a, return_inverse=True)
    _, ib = np.unique(b, return_inverse=True)
    table = np.zeros((ia.max() + 1 if len(a) else 0, ib.max() + 1 if len(b) else 0), np.int64)
    np.add.at(table, (ia, ib), 1)

    def pairs(v):
        v = np.asarray(v, dtype=np.int64)
        return int((v * (v - 1) // 2).sum())

    n_pairs = len(a) * (len(a) - 1) // 2
    if n_pairs == 0:
        return 1.0
    both = pairs(table)
    ra, rb = pairs(table.sum(axis=1)), pairs(table.sum(axis=0))
    chance = ra * rb / n_pairs
    top = (ra + rb) / 2
    if top == chance:
        return 1.0
    return (both - chance) / (top - chance)
