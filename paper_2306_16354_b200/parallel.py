"""Multi-GPU single linkage: query-row sharding of the two neighbour searches.

One process per GPU (torchrun), ``torch.distributed`` over NCCL.  Following
the north star, only the brute-force k-NN scan and the cross-colour 1-NN
scans shard: every rank holds the full point matrix (the index is
replicated), scans its round-robin chunks of query rows (``shard_chunks``),
and rank 0 gathers the per-chunk results (the only consumer).  Boruvka, the dendrogram and the cut run
on rank 0; the colours rank 0 produces are broadcast before each connect
pass.  The reference has no distributed path (its parallelism is the thread
pool of /root/reference/pkg/src/parlink/parallel.py:36-48 over the same
query-row blocks, neighbors.py:273-294).

The orchestration is engine-agnostic: ``DeviceEngine`` runs the CUDA kernels
(the product); the CPU ``gloo`` tests inject a checker engine to exercise the
sharding and collective logic without a GPU.
"""

from __future__ import annotations

import math
import os

import numpy as np

from .core import (ConvergenceError, Dendrogram, EdgeList, LinkageError, ValidationError, as_point_matrix,
                   unscale_sq)
from .linkage import STAGES, LabelArray, LinkageConfig, SingleLinkageResult

ROW_ALIGN = 128  # query-block granularity of the scan kernel
THREADS_ENV_VAR = "PARLINK_THREADS"


def resolve_threads(threads: int | None = None) -> int:
    """Host worker count: the argument, else $PARLINK_THREADS, else the CPU count.

    Same rule and error as /root/reference/pkg/src/parlink/parallel.py:16-26.
    The CUDA path does not use host threads for compute; the count is
    validated and recorded (run manifests, bench CSV) for compatibility.
    """
    if threads is None:
        env = os.environ.get(THREADS_ENV_VAR)
        threads = int(env) if env is not None else (os.cpu_count() or 1)
    if threads < 1:
        raise ValueError(f"thread count must be >= 1, got {threads}")
    return threads


CHUNKS_PER_RANK = 4  # round-robin chunks per rank (balances clusters of unequal pruning cost)


def shard_chunks(n: int, world: int, rank: int, per_rank: int = CHUNKS_PER_RANK,
                 align: int = ROW_ALIGN) -> list[tuple[int, int]]:
    """Block-aligned query-row chunks of one rank: [0, n) is cut into
    min(blocks, per_rank * world) near-equal chunks and chunk j goes to rank
    j % world, so every rank samples the whole row order (pruning makes the
    cost of a query block depend on its cluster; contiguous shards would
    inherit that imbalance).  The same rule as the single-process driver
    (slink_api.cu:ShardSet)."""
    blocks = max(1, math.ceil(n / align))
    c = max(1, min(blocks, per_rank * world))
    chunks = [(min(n, blocks * j // c * align), min(n, blocks * (j + 1) // c * align)) for j in range(c)]
    return [chunks[j] for j in range(rank, c, world)]


class DeviceEngine:
    """CUDA kernels of libslink.so on the current device."""

    def __init__(self):
        from . import _lib

        self._lib = _lib
        self.torch = _lib.torch_cuda()
        self.device = _lib.device()

    def upload(self, x):
        from .neighbors import DevicePoints

        if isinstance(x, DevicePoints):
            return x
        return DevicePoints(as_point_matrix(x))

    def n_points(self, pts) -> int:
        return pts.n

    # both searches go through the points' persistent handle: one PointSet
    # (spheres, operand packs, split index) per rank for the k-NN chunks and
    # every connect pass
    def knn_shard(self, pts, k, rows):
        from .neighbors import knn_device

        return knn_device(pts, k, rows, reuse=True)

    def nn1_shard(self, pts, colors, rows):
        from .neighbors import nn1_colour_device

        return nn1_colour_device(pts, colors, rows)

    def msf(self, n, src, dst, w, m, seed):
        from .linkage import msf_of_edges

        return msf_of_edges(n, src, dst, w, m, seed)

    def scale_exp(self, pts) -> int:
        return getattr(pts, "scale_exp", 0)

    def finish(self, n, t_src, t_dst, t_w, cfg, scale_exp=0):
        """Dendrogram + cut of the device tree in one native call (slk_finish_tree:
        the single-process pipeline's own tail, no host round trip of the tree
        before the fold); the library's outputs skip re-validation."""
        import ctypes

        from .core import _trusted

        merges = np.empty((max(n - 1, 1), 4))
        labels = np.empty(n, dtype=np.int64)
        ts = np.empty(max(n - 1, 1), dtype=np.int64)
        td = np.empty(max(n - 1, 1), dtype=np.int64)
        tw = np.empty(max(n - 1, 1))
        p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        metric = 0 if cfg.metric == "euclidean" else 1
        self._lib.call("slk_finish_tree", self._lib.ptr(t_src), self._lib.ptr(t_dst), self._lib.ptr(t_w), n,
                       metric, cfg.n_clusters, p(merges), p(labels), p(ts), p(td), p(tw), None,
                       self._lib.stream_handle())
        if scale_exp:  # back from the device's power-of-two scaled units (exact)
            tw[: n - 1] = np.ldexp(tw[: n - 1], 2 * scale_exp)
            merges[: n - 1, 2] = np.ldexp(merges[: n - 1, 2], scale_exp if metric == 0 else 2 * scale_exp)
        tree = _trusted(EdgeList, n_vertices=n, src=ts[: n - 1], dst=td[: n - 1], weight=tw[: n - 1])
        dendro = _trusted(Dendrogram, n_points=n, merges=merges[: n - 1])
        return tree, dendro, _trusted(LabelArray, labels=labels, n_clusters=cfg.n_clusters)

    def sync(self):
        self.torch.cuda.synchronize()


def _host_staged(dist, group, t) -> bool:
    """gloo moves host tensors only: device tensors are staged through the host
    (lets the orchestration run with several ranks on one GPU, e.g. in tests)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _gather_chunks(torch, dist, group, parts, n, world, rank, row_shape, dtype, dev):
    """Rank 0 receives every rank's chunk results (row blocks, concatenated in
    chunk order, padded to the largest rank) and reassembles rows [0, n);
    other ranks only send (a rank may hold no chunk when n is small).
    Returns the full tensor on rank 0, None elsewhere."""
    per_rank = [sum(b - a for a, b in shard_chunks(n, world, r)) for r in range(world)]
    cap = max(per_rank)
    t = torch.cat([p for _, p in parts]) if parts else torch.empty((0,) + tuple(row_shape), dtype=dtype, device=dev)
    if _host_staged(dist, group, t):
        t = t.cpu()
    pad = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    out = torch.empty((n,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    for r in range(world):
        at = 0
        for a, b in shard_chunks(n, world, r):
            out[a:b] = bufs[r][at: at + (b - a)]
            at += b - a
    return out.to(dev)


def _broadcast(dist, group, t):
    """In-place broadcast from rank 0 (host-staged under gloo)."""
    if _host_staged(dist, group, t):
        h = t.cpu()
        dist.broadcast(h, 0, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, 0, group=group)


_ERRORS = (ValidationError, ConvergenceError, LinkageError)  # status -1, -2, -3


def _rank0_step(dist, group, rank, ncomp_t, fn):
    """Runs ``fn`` (rank-0-only work returning the new component count) on rank
    0 and broadcasts the count; a failure there is broadcast as a negative
    status plus its message so EVERY rank raises the same exception class
    instead of waiting in the next collective."""
    err = None
    if rank == 0:
        try:
            ncomp_t.fill_(int(fn()))
        except _ERRORS as exc:
            err = exc
            code = next(i for i, cls in enumerate(_ERRORS) if isinstance(exc, cls))
            ncomp_t.fill_(-1 - code)
    _broadcast(dist, group, ncomp_t)
    status = int(ncomp_t.item())
    if status < 0:
        msg = [str(err) if err is not None else None]
        dist.broadcast_object_list(msg, src=0, group=group)
        if err is not None:
            raise err
        raise _ERRORS[-1 - status](msg[0])
    return status


def single_linkage_distributed(x, cfg: LinkageConfig, *, engine=None, group=None):
    """single_linkage over all ranks of ``group``; returns the result on rank 0, None elsewhere.

    Every rank must pass the same points (host array or its DevicePoints).
    """
    import time

    import torch
    import torch.distributed as dist

    engine = engine or DeviceEngine()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    pts = engine.upload(x)
    n = engine.n_points(pts)
    if n < 2:
        raise ValidationError(f"need at least 2 points, got {n}")
    if cfg.n_clusters > n:
        raise ValidationError(f"n_clusters={cfg.n_clusters} exceeds {n} points")
    if cfg.k > n - 1:
        raise ValidationError(f"k={cfg.k} exceeds N-1={n - 1}")
    chunks = shard_chunks(n, world, rank)
    marks = [time.perf_counter()]

    # --- sharded k-NN (round-robin chunks), gathered on rank 0 only
    dev = getattr(engine, "device", torch.device("cpu"))
    res = [engine.knn_shard(pts, cfg.k, c) for c in chunks]
    idx_all = _gather_chunks(torch, dist, group, [(c, r[0]) for c, r in zip(chunks, res)], n, world, rank,
                             (cfg.k,), torch.int32, dev)
    dst_all = _gather_chunks(torch, dist, group, [(c, r[1]) for c, r in zip(chunks, res)], n, world, rank,
                             (cfg.k,), torch.float64, dev)
    engine.sync()
    marks.append(time.perf_counter())
    del res
    ncomp_t = torch.zeros(1, dtype=torch.int64, device=dev)
    colors = torch.empty(n, dtype=torch.int32, device=dev)
    state = None

    def first_forest():
        nonlocal state
        src = torch.arange(n, dtype=torch.int32, device=dev).repeat_interleave(cfg.k)
        state = engine.msf(n, src, idx_all.reshape(-1), dst_all.reshape(-1), n * cfg.k, cfg.seed)
        colors.copy_(state[3][:n])
        return state[5]

    ncomp = _rank0_step(dist, group, rank, ncomp_t, first_forest)
    del idx_all, dst_all
    marks.append(time.perf_counter())

    # --- connect loop: colours broadcast, sharded cross-colour 1-NN, gather bridges
    budget = cfg.max_connect_iters if cfg.max_connect_iters is not None else \
        math.ceil(math.log2(max(n, 2))) + 8
    iters = 0
    iota = torch.arange(n, dtype=torch.int32, device=dev)
    while ncomp > 1:
        if iters >= budget:
            raise ConvergenceError(
                f"reconnection did not converge within {budget} iterations: "
                f"{ncomp} components remain")
        _broadcast(dist, group, colors)
        res = [engine.nn1_shard(pts, colors, c) for c in chunks]
        bidx_all = _gather_chunks(torch, dist, group, [(c, r[0]) for c, r in zip(chunks, res)], n, world, rank,
                                  (), torch.int32, dev)
        bw_all = _gather_chunks(torch, dist, group, [(c, r[1]) for c, r in zip(chunks, res)], n, world, rank,
                                (), torch.float64, dev)
        del res

        def resolve():
            nonlocal state
            ne = state[4]
            u_src = torch.cat([state[0][:ne], iota])
            u_dst = torch.cat([state[1][:ne], bidx_all])
            u_w = torch.cat([state[2][:ne], bw_all])
            state = engine.msf(n, u_src, u_dst, u_w, ne + n, cfg.seed)
            colors.copy_(state[3][:n])
            return state[5]

        ncomp = _rank0_step(dist, group, rank, ncomp_t, resolve)
        iters += 1
    engine.sync()
    marks.append(time.perf_counter())
    if rank != 0:
        return None

    # --- dendrogram + cut on rank 0
    ne = state[4]
    tree, dendro, labels = engine.finish(n, state[0][:ne], state[1][:ne], state[2][:ne], cfg,
                                         engine.scale_exp(pts))
    marks.append(time.perf_counter())
    timings = {STAGES[i]: (marks[i + 1] - marks[i]) * 1e3 for i in range(4)}
    timings["extract"] = 0.0
    return SingleLinkageResult(dendro, labels, tree, iters, timings)


def knn_distributed(x, k: int, *, engine=None, group=None, to_host: bool = False):
    """fused_knn over all ranks of ``group`` (BASELINE configs[3] sharded):
    each rank scans its query-row shard against the replicated index, rank 0
    gathers the lists.  Returns (idx, dist) on rank 0 (device tensors, or a
    KnnGraph with ``to_host``), None elsewhere."""
    import torch
    import torch.distributed as dist

    engine = engine or DeviceEngine()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    pts = engine.upload(x)
    n = engine.n_points(pts)
    chunks = shard_chunks(n, world, rank)
    dev = getattr(engine, "device", torch.device("cpu"))
    res = [engine.knn_shard(pts, k, c) for c in chunks]
    idx_all = _gather_chunks(torch, dist, group, [(c, r[0]) for c, r in zip(chunks, res)], n, world, rank,
                             (k,), torch.int32, dev)
    dst_all = _gather_chunks(torch, dist, group, [(c, r[1]) for c, r in zip(chunks, res)], n, world, rank,
                             (k,), torch.float64, dev)
    engine.sync()
    if rank != 0:
        return None
    if not to_host:
        return idx_all, dst_all
    from .neighbors import KnnGraph

    return KnnGraph(idx_all.cpu().numpy().astype(np.int64),
                    unscale_sq(dst_all.cpu().numpy(), engine.scale_exp(pts)))


__all__ = ["DeviceEngine", "knn_distributed", "shard_chunks", "single_linkage_distributed", "Dendrogram",
           "LabelArray"]
