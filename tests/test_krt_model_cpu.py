"""CPU model of the device merge table's time-split recursion
(paper_2306_16354_b200/csrc/dendro.cu:krt_kernel), checked against the
oracle's sequential fold (oracle.build_dendrogram, ref linkage.py:103-129).

The model mirrors the kernel's phases with plain Python containers (no
concurrency): per level, the union-find of the left halves' edges over node
ids shared by every window, the largest edge and the size of each component,
and the relabelling of the right halves; then the in-order fold of the leaf
windows.  It pins the ALGORITHM (including the claim that one union-find may
serve all windows of a level) on many tree shapes at several leaf sizes; the
CUDA kernel itself is compared with the oracle in tests/test_parity_gpu.py.
"""

import numpy as np
import pytest


def krt_model(a, b, w, n, leaf_log):
    m = n - 1
    top = 0
    while (1 << top) < m:
        top += 1
    levels = max(0, top - leaf_log)
    la, lb = list(a), list(b)
    size = {v: 1 for v in range(n)}
    for D in range(levels):
        sh = top - D - 1
        left = [i for i in range(m) if not (i >> sh) & 1]
        uf = {}

        def find(x):
            while uf.get(x, x) != x:
                x = uf[x]
            return x

        for i in left:
            u, v = find(la[i]), find(lb[i])
            if u != v:
                uf[min(u, v)] = max(u, v)  # the smaller root hooks under the larger
        cmax, acc, seen = {}, {}, set()
        for i in left:
            r = find(la[i])
            cmax[r] = max(cmax.get(r, -1), i)
            for x in (la[i], lb[i]):
                if x not in seen:
                    seen.add(x)
                    acc[r] = acc.get(r, 0) + size[x]
        new_la, new_lb = list(la), list(lb)
        for i in range(m):
            if not (i >> sh) & 1:
                r = find(la[i])
                if cmax[r] == i:
                    size[n + i] = acc[r]
            else:
                if la[i] in seen:
                    new_la[i] = n + cmax[find(la[i])]
                if lb[i] in seen:
                    new_lb[i] = n + cmax[find(lb[i])]
        la, lb = new_la, new_lb
    L = 1 << (top - levels)
    rows = np.zeros((m, 4))
    for i0 in range(0, m, L):
        par, cid, sz = {}, {}, {}

        def root(q):
            while par[q] != q:
                q = par[q]
            return q

        for i in range(i0, min(m, i0 + L)):
            r = []
            for x in (la[i], lb[i]):
                if x not in par:
                    par[x], cid[x], sz[x] = x, x, size[x]
                r.append(root(x))
            if r[0] == r[1]:
                raise ValueError("cycle")
            ca, cb, tot = cid[r[0]], cid[r[1]], sz[r[0]] + sz[r[1]]
            rows[i] = (min(ca, cb), max(ca, cb), w[i], tot)
            par[r[1]] = r[0]
            cid[r[0]] = n + i
            sz[r[0]] = tot
    return rows


def _tree(rng, n, shape):
    src = np.arange(1, n)
    if shape == "chain":
        dst = src - 1
    elif shape == "star":
        dst = np.zeros(n - 1, dtype=np.int64)
    else:
        dst = (rng.random(n - 1) * src).astype(np.int64)
    perm = rng.permutation(n)
    return perm[src], perm[dst]


@pytest.mark.parametrize("leaf_log", [0, 1, 2, 5])
@pytest.mark.parametrize("shape", ["chain", "star", "random"])
def test_krt_model_matches_oracle_fold(oracle, shape, leaf_log):
    rng = np.random.default_rng(leaf_log * 7 + len(shape))
    for n in [2, 3, 5, 17, 33, 64, 65, 130, 257, 700]:
        src, dst = _tree(rng, n, shape)
        # merge order = the order the oracle sorts into: distinct heights
        w = rng.permutation(n - 1).astype(np.float64) + 1.0
        ref = oracle.build_dendrogram(src, dst, w, n)
        lo, hi = np.minimum(src, dst), np.maximum(src, dst)
        order = np.lexsort((hi, lo, w))
        got = krt_model(lo[order], hi[order], w[order], n, leaf_log)
        assert np.array_equal(got, ref), (shape, n, leaf_log)
