"""CPU model of the device segment blocking (knn.cu:segment_blocks) used by
the colour and pivot re-blocking of the neighbour searches: the scan over
segments with the step  x -> (len >= 64 ? align(x + a) : x) + b  must place
every point and pad row exactly where the sequential planner of round 1 put
them (each segment of >= 64 points after the first starts a fresh 128-row
block; the gap repeats the previous segment's first point, query id -1)."""

import numpy as np
import pytest

BM = 128


def sequential(keys, ids):
    src, qid, prev, i, n = [], [], ids[0], 0, len(keys)
    while i < n:
        j = i + 1
        while j < n and keys[j] == keys[i]:
            j += 1
        if j - i >= BM // 2 and src:
            while len(src) % BM:
                src.append(prev)
                qid.append(-1)
        src += list(ids[i:j])
        qid += list(ids[i:j])
        prev, i = ids[i], j
    return src, qid


def align(x):
    return (x + BM - 1) // BM * BM


def compose(l, r):  # apply l, then r (knn.cu:SegStepCompose)
    if not r[0]:
        return (l[0], l[1], l[2] + r[2])
    if not l[0]:
        return (1, l[2] + r[1], r[2])
    return (1, l[1], align(l[2] + r[1]) + r[2])


def scanned(keys, ids):
    n = len(keys)
    flag = np.r_[1, (keys[1:] != keys[:-1]).astype(int)]
    segid = np.cumsum(flag) - 1
    start = np.flatnonzero(flag)
    nseg = len(start)
    lens = np.diff(np.r_[start, n])
    step = [(1 if (lens[g] >= BM // 2 and g > 0) else 0, 0, int(lens[g])) for g in range(nseg)]
    excl = [(0, 0, 0)]
    for g in range(1, nseg):
        excl.append(compose(excl[-1], step[g - 1]))
    off = []
    for g in range(nseg):
        e = excl[g]
        x = 0 if g == 0 else (align(e[1]) + e[2] if e[0] else e[2])
        off.append(align(x) if step[g][0] else x)
    nout = off[-1] + (n - start[-1])
    src, qid = [None] * nout, [None] * nout
    for i in range(n):
        p = off[segid[i]] + i - start[segid[i]]
        src[p] = qid[p] = ids[i]
    for g in range(1, nseg):
        for p in range(off[g - 1] + start[g] - start[g - 1], off[g]):
            src[p], qid[p] = ids[start[g - 1]], -1
    return src, qid


@pytest.mark.parametrize("seed", range(6))
def test_segment_scan_matches_sequential_planner(seed):
    rng = np.random.default_rng(seed)
    for _ in range(40):
        n = int(rng.integers(1, 2500))
        keys = np.sort(rng.integers(0, int(rng.integers(1, 80)), size=n))
        ids = rng.permutation(n)
        assert scanned(keys, ids) == sequential(keys, ids)
