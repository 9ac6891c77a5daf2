"""Multi-GPU single linkage: query-row sharding of the two neighbour searches.

One process per GPU (torchrun), ``torch.distributed`` over NCCL.  Following
the north star, only the brute-force k-NN scan and the cross-colour 1-NN
scans shard: every rank holds the full point matrix (the index is
replicated), scans the query rows ``[q0, q1)`` of its shard, and the
per-shard results are all-gathered.  Boruvka, the dendrogram and the cut run
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


def shard_rows(n: int, world: int, rank: int, align: int = ROW_ALIGN) -> tuple[int, int]:
    """Contiguous, block-aligned query-row range of one rank (covers [0, n) exactly)."""
    blocks = math.ceil(n / align)
    per = math.ceil(blocks / world)
    q0 = min(n, rank * per * align)
    q1 = min(n, (rank + 1) * per * align)
    return q0, q1


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

    def knn_shard(self, pts, k, rows):
        from .neighbors import knn_device

        return knn_device(pts, k, rows)

    def nn1_shard(self, pts, colors, rows):
        from .neighbors import nn1_device

        return nn1_device(pts, pts, mode=2, qcolor=colors, xcolor=colors, rows=rows)

    def msf(self, n, src, dst, w, m, seed):
        from .linkage import msf_of_edges

        return msf_of_edges(n, src, dst, w, m, seed)

    def scale_exp(self, pts) -> int:
        return getattr(pts, "scale_exp", 0)

    def finish(self, n, t_src, t_dst, t_w, cfg, scale_exp=0):
        from .linkage import build_dendrogram, extract_clusters

        tree = EdgeList(n, self._lib.to_host(t_src).astype(np.int64),
                        self._lib.to_host(t_dst).astype(np.int64),
                        unscale_sq(self._lib.to_host(t_w), scale_exp))
        w = np.sqrt(tree.weight) if cfg.metric == "euclidean" else tree.weight
        dendro = build_dendrogram(EdgeList(n, tree.src, tree.dst, w), n)
        return tree, dendro, extract_clusters(dendro, cfg.n_clusters)

    def sync(self):
        self.torch.cuda.synchronize()


def _host_staged(dist, group, t) -> bool:
    """gloo moves host tensors only: device tensors are staged through the host
    (lets the orchestration run with several ranks on one GPU, e.g. in tests)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _gather_rows(torch, dist, group, t, rows_per_rank, world):
    """All-gather variable-length row shards (padded to the largest) → concatenated."""
    cap = max(rows_per_rank)
    dev = t.device
    if _host_staged(dist, group, t):
        t = t.cpu()
    shape = (cap,) + tuple(t.shape[1:])
    pad = torch.zeros(shape, dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    out = torch.empty((world * cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * cap: r * cap + rows_per_rank[r]] for r in range(world)]
    return torch.cat(parts).to(dev)


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
    ranges = [shard_rows(n, world, r) for r in range(world)]
    rows_per_rank = [b - a for a, b in ranges]
    marks = [time.perf_counter()]

    # --- sharded k-NN, gathered on every rank (rank 0 consumes it)
    idx, dst = engine.knn_shard(pts, cfg.k, ranges[rank])
    idx_all = _gather_rows(torch, dist, group, idx, rows_per_rank, world)
    dst_all = _gather_rows(torch, dist, group, dst, rows_per_rank, world)
    engine.sync()
    marks.append(time.perf_counter())

    dev = idx.device
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
        bidx, bw = engine.nn1_shard(pts, colors, ranges[rank])
        bidx_all = _gather_rows(torch, dist, group, bidx, rows_per_rank, world)
        bw_all = _gather_rows(torch, dist, group, bw, rows_per_rank, world)

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
    ranges = [shard_rows(n, world, r) for r in range(world)]
    rows_per_rank = [b - a for a, b in ranges]
    idx, dst = engine.knn_shard(pts, k, ranges[rank])
    idx_all = _gather_rows(torch, dist, group, idx, rows_per_rank, world)
    dst_all = _gather_rows(torch, dist, group, dst, rows_per_rank, world)
    engine.sync()
    if rank != 0:
        return None
    if not to_host:
        return idx_all, dst_all
    from .neighbors import KnnGraph

    return KnnGraph(idx_all.cpu().numpy().astype(np.int64),
                    unscale_sq(dst_all.cpu().numpy(), engine.scale_exp(pts)))


__all__ = ["DeviceEngine", "knn_distributed", "shard_rows", "single_linkage_distributed", "Dendrogram",
           "LabelArray"]
