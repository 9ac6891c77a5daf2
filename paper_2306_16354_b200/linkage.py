"""Single-linkage pipeline on the GPU (mirrors ``parlink.linkage``).

Public names follow /root/reference/pkg/src/parlink/linkage.py:37-311.
``single_linkage`` makes ONE call into libslink.so (``slk_single_linkage``):
k-NN graph → symmetrise → Boruvka forest → connect loop (cross-colour 1-NN +
re-solve) → device-sorted dendrogram → flat cut, all on one GPU with host
buffers in and out.  ``single_linkage_result`` returns the same plus the
spanning tree, the connect-iteration count and stage timings.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import (
    ColorArray,
    ConvergenceError,
    Dendrogram,
    EdgeList,
    PointMatrix,
    ValidationError,
    _trusted,
    as_point_matrix,
    unscale_sq,
)
from .neighbors import DevicePoints, TileSpec, nn1_device

METRICS = ("euclidean", "sqeuclidean")
STAGES = ("knn", "mst", "connect", "dendrogram", "extract")


@dataclass(frozen=True)
class LinkageConfig:
    """Run configuration (linkage.py:37-65); k > 64 needs ``allow_large_k``."""

    n_clusters: int
    k: int = 15
    metric: str = "euclidean"
    seed: int = 0
    max_connect_iters: int | None = None
    allow_large_k: bool = False

    def __post_init__(self):
        if self.n_clusters < 1:
            raise ValidationError(f"n_clusters must be >= 1, got {self.n_clusters}")
        if self.k < 1:
            raise ValidationError(f"k must be >= 1, got {self.k}")
        if self.k > 64 and not self.allow_large_k:
            raise ValidationError(f"k={self.k} exceeds 64; set allow_large_k=True to permit it")
        if self.metric not in METRICS:
            raise ValidationError(f"metric must be one of {METRICS}, got {self.metric!r}")
        if self.max_connect_iters is not None and self.max_connect_iters < 0:
            raise ValidationError("max_connect_iters must be >= 0")


@dataclass(frozen=True)
class LabelArray:
    """One label in [0, n_clusters) per point, every label used (linkage.py:68-88)."""

    labels: np.ndarray
    n_clusters: int

    def __post_init__(self):
        arr = np.asarray(self.labels, dtype=np.int64).ravel()
        distinct = np.unique(arr)
        if len(distinct) != self.n_clusters or (
            len(distinct) and (distinct[0] < 0 or distinct[-1] >= self.n_clusters)
        ):
            raise ValidationError(f"labels must cover exactly {self.n_clusters} values in range")
        arr.setflags(write=False)
        object.__setattr__(self, "labels", arr)

    def __len__(self) -> int:
        return len(self.labels)


@dataclass(frozen=True)
class SingleLinkageResult:
    """Everything one pipeline run produces (north-star output arrays).

    tree_*: the spanning tree (squared-L2 weights, sorted (src, dst));
    dendrogram: children / deltas / sizes; labels: flat cut.
    """

    dendrogram: Dendrogram
    labels: LabelArray
    tree: EdgeList
    connect_iters: int
    timings: dict = field(default_factory=dict)


def compute_cut_level(n_points: int, n_clusters: int) -> int:
    """Number of merges kept below the cut for n_clusters labels (linkage.py:151-157)."""
    if not 1 <= n_clusters <= n_points:
        raise ValidationError(f"n_clusters must be in [1, {n_points}], got {n_clusters}")
    return (n_points - 1) - (n_clusters - 1)


def build_dendrogram(mst_edges: EdgeList, n_points: int) -> Dendrogram:
    """Merge table of a spanning tree (linkage.py:160-181).

    Device radix sort by (weight, a, b), then the union-find fold (union by
    rank, path compression): row i joins the current clusters of its two
    endpoints and creates node n_points + i.
    """
    if n_points < 2:
        raise ValidationError("dendrogram needs at least 2 points")
    if len(mst_edges) != n_points - 1:
        raise ValidationError(
            f"spanning tree over {n_points} points needs {n_points - 1} edges, "
            f"got {len(mst_edges)}")
    src, dst = _lib.ids_to_device(mst_edges.src), _lib.ids_to_device(mst_edges.dst)
    w = _lib.to_device(mst_edges.weight, np.float64)
    merges = np.empty((n_points - 1, 4))
    _lib.call("slk_build_dendrogram", _lib.ptr(src), _lib.ptr(dst), _lib.ptr(w), n_points,
              merges.ctypes.data_as(ctypes.c_void_p), _lib.stream_handle())
    return Dendrogram(n_points, merges)


def extract_clusters(dendrogram: Dendrogram, n_clusters: int) -> LabelArray:
    """Flat labels from cutting the dendrogram at n_clusters (linkage.py:184-213).

    Roots are the ids below the cut never consumed as children, labelled in
    ascending id order; every point inherits its nearest labelled ancestor.
    """
    n = dendrogram.n_points
    compute_cut_level(n, n_clusters)
    merges = np.ascontiguousarray(dendrogram.merges, dtype=np.float64)
    if n < 2:
        merges = np.zeros((1, 4))
    labels = np.empty(n, dtype=np.int64)
    _lib.check(_lib.load().slk_extract_clusters(merges.ctypes.data_as(ctypes.c_void_p), n,
                                                n_clusters, labels.ctypes.data_as(ctypes.c_void_p)))
    return LabelArray(labels, n_clusters)


def _connect_budget(cfg: LinkageConfig, n_points: int) -> int:
    if cfg.max_connect_iters is not None:
        return cfg.max_connect_iters
    return math.ceil(math.log2(max(n_points, 2))) + 8


def _component_sizes(colors: np.ndarray) -> list:
    counts = np.bincount(colors)
    return np.sort(counts[counts > 0])[::-1][:8].tolist()


def msf_of_edges(n: int, src, dst, w, m: int, seed: int):
    """Device spanning forest of an edge-list union → (src, dst, w, colors, n_edges, n_comp)."""
    out_s, out_d = _lib.empty(max(n, 1), np.int32), _lib.empty(max(n, 1), np.int32)
    out_w, colors = _lib.empty(max(n, 1), np.float64), _lib.empty(max(n, 1), np.int32)
    ne, nc = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("slk_msf_edges", n, _lib.ptr(src), _lib.ptr(dst), _lib.ptr(w), m, int(seed),
              _lib.ptr(out_s), _lib.ptr(out_d), _lib.ptr(out_w), _lib.ptr(colors),
              ctypes.byref(ne), ctypes.byref(nc), _lib.stream_handle())
    return out_s, out_d, out_w, colors, ne.value, nc.value


def connect_graph(x, mst_edges: EdgeList, colors: ColorArray, cfg: LinkageConfig, *,
                  tile: TileSpec | None = None, threads: int | None = None) -> EdgeList:
    """Grow a spanning forest into a spanning tree (linkage.py:222-254).

    While more than one colour remains: one cross-colour 1-NN bridge per point,
    union with the current forest, re-solve the forest.  Squared-L2 weights.
    """
    pm = as_point_matrix(x)
    n = pm.n_rows
    budget = _connect_budget(cfg, n)
    if colors.n_components <= 1:
        return mst_edges
    torch = _lib.torch_cuda()
    pts = DevicePoints(pm)
    t_src, t_dst = _lib.ids_to_device(mst_edges.src), _lib.ids_to_device(mst_edges.dst)
    # forest weights in the device's (possibly power-of-two scaled) units: exact
    t_w = _lib.to_device(np.ldexp(mst_edges.weight, -2 * pm.scale_exp), np.float64)
    col = _lib.ids_to_device(colors.colors)
    ncomp, iters, ne = colors.n_components, 0, len(mst_edges)
    iota = torch.arange(n, dtype=torch.int32, device=_lib.device())
    while ncomp > 1:
        if iters >= budget:
            sizes = _component_sizes(_lib.to_host(col).astype(np.int64))
            raise ConvergenceError(
                f"reconnection did not converge within {budget} iterations: "
                f"{ncomp} components remain (largest sizes {sizes})")
        bdst, bw = nn1_device(pts, pts, mode=2, qcolor=col, xcolor=col)
        u_src = torch.cat([t_src[:ne], iota])
        u_dst = torch.cat([t_dst[:ne], bdst])
        u_w = torch.cat([t_w[:ne], bw])
        t_src, t_dst, t_w, col, ne, ncomp = msf_of_edges(n, u_src, u_dst, u_w, ne + n, cfg.seed)
        iters += 1
    return EdgeList(n, _lib.to_host(t_src[:ne]).astype(np.int64),
                    _lib.to_host(t_dst[:ne]).astype(np.int64),
                    unscale_sq(_lib.to_host(t_w[:ne]), pm.scale_exp))


MAX_POINTS = (1 << 30) - 1  # int32 node ids of the merge table (n + i < 2^31)


def _validate_run(pm, cfg: LinkageConfig):
    n = pm.n_rows
    if n > MAX_POINTS:
        raise ValidationError(f"n={n} exceeds the {MAX_POINTS} point limit")
    if n < 2:
        raise ValidationError(f"need at least 2 points, got {n}")
    if cfg.n_clusters > n:
        raise ValidationError(f"n_clusters={cfg.n_clusters} exceeds {n} points")
    if cfg.k > n - 1:
        raise ValidationError(f"k={cfg.k} exceeds N-1={n - 1}")


def _check_gpus(n_gpus) -> int:
    g = 1 if n_gpus is None else n_gpus
    if isinstance(g, bool) or not isinstance(g, (int, np.integer)) or not 1 <= g <= 64:
        raise ValidationError(f"n_gpus must be an integer in [1, 64], got {n_gpus!r}")
    return int(g)


def _run(pm, cfg: LinkageConfig, device_points=None, n_gpus: int = 1) -> SingleLinkageResult:
    n, d = pm.n_rows if pm is not None else device_points.n, (
        pm.n_cols if pm is not None else device_points.d)
    merges = np.empty((max(n - 1, 1), 4))
    labels = np.empty(n, dtype=np.int64)
    ts = np.empty(max(n - 1, 1), dtype=np.int64)
    td = np.empty(max(n - 1, 1), dtype=np.int64)
    tw = np.empty(max(n - 1, 1))
    iters = ctypes.c_int64()
    tim = np.zeros(5)
    budget = -1 if cfg.max_connect_iters is None else int(cfg.max_connect_iters)
    metric = 0 if cfg.metric == "euclidean" else 1
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    if device_points is None:
        x32 = np.ascontiguousarray(pm.float32)
        x64 = None if pm.exact_f32 else np.ascontiguousarray(pm.device_f64)
        _lib.torch_cuda()
        _lib.call("slk_single_linkage", p(x32), None if x64 is None else p(x64), n, d, cfg.k,
                  cfg.n_clusters, metric, int(cfg.seed), budget, n_gpus, p(merges), p(labels),
                  p(ts), p(td), p(tw), ctypes.byref(iters), p(tim))
    else:
        dp = device_points
        _lib.call("slk_single_linkage_device", _lib.ptr(dp.x32), _lib.ptr(dp.x64), n, d, cfg.k,
                  cfg.n_clusters, metric, int(cfg.seed), budget, n_gpus, p(merges), p(labels),
                  p(ts), p(td), p(tw), ctypes.byref(iters), p(tim), _lib.stream_handle())
    e = pm.scale_exp if pm is not None else 0
    if e:  # back from the device's power-of-two scaled units (exact)
        tw[: n - 1] = np.ldexp(tw[: n - 1], 2 * e)
        merges[: n - 1, 2] = np.ldexp(merges[: n - 1, 2], e if metric == 0 else 2 * e)
    # outputs of the library itself: skip re-validating 1M-row arrays
    dendro = _trusted(Dendrogram, n_points=n, merges=merges[: n - 1])
    lab = _trusted(LabelArray, labels=labels, n_clusters=cfg.n_clusters)
    tree = _trusted(EdgeList, n_vertices=n, src=ts[: n - 1], dst=td[: n - 1], weight=tw[: n - 1])
    return SingleLinkageResult(dendro, lab, tree, int(iters.value), dict(zip(STAGES, tim.tolist())))


def single_linkage_result(x, cfg: LinkageConfig, *, n_gpus: int | None = None) -> SingleLinkageResult:
    """single_linkage plus the spanning tree, connect iterations and stage timings."""
    g = _check_gpus(n_gpus)
    if isinstance(x, np.ndarray) and x.dtype == np.float32 and x.ndim == 2:
        pm = PointMatrix._float32_device_checked(x)  # finiteness checked on the GPU
    else:
        pm = as_point_matrix(x)
    _validate_run(pm, cfg)
    return _run(pm, cfg, n_gpus=g)


def single_linkage_on_device(points: DevicePoints, cfg: LinkageConfig, *,
                             n_gpus: int | None = None) -> SingleLinkageResult:
    """Pipeline over points already resident on the GPU (bench ``value`` leg)."""
    g = _check_gpus(n_gpus)
    if points.n > MAX_POINTS:
        raise ValidationError(f"n={points.n} exceeds the {MAX_POINTS} point limit")
    if points.n < 2:
        raise ValidationError(f"need at least 2 points, got {points.n}")
    if cfg.n_clusters > points.n:
        raise ValidationError(f"n_clusters={cfg.n_clusters} exceeds {points.n} points")
    if cfg.k > points.n - 1:
        raise ValidationError(f"k={cfg.k} exceeds N-1={points.n - 1}")
    return _run(None, cfg, device_points=points, n_gpus=g)


def single_linkage(x, cfg: LinkageConfig, *, tile: TileSpec | None = None,
                   threads: int | None = None, timings: dict | None = None,
                   n_gpus: int | None = None) -> tuple[Dendrogram, LabelArray]:
    """End-to-end single-linkage clustering (linkage.py:257-311).

    Returns the full dendrogram and the flat labels for cfg.n_clusters.
    ``timings`` (optional dict) receives per-stage milliseconds under the
    reference's keys.  ``tile`` / ``threads`` are accepted and ignored.
    ``n_gpus`` (extension; the GPU counterpart of ``threads``, parallel.py:16-48)
    shards the neighbour searches over that many devices of this process
    (include/slink.h: slk_single_linkage); results do not depend on it.
    """
    res = single_linkage_result(x, cfg, n_gpus=n_gpus)
    if timings is not None:
        timings.update(res.timings)
    return res.dendrogram, res.labels
