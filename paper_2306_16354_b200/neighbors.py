"""Brute-force neighbour search on the GPU (mirrors ``parlink.neighbors``).

Public names and signatures follow /root/reference/pkg/src/parlink/
neighbors.py:32-391.  The work happens in libslink.so (csrc/knn.cu): an
exact-fp32 fused distance+top-K' scan, a float64 refine that reproduces the
reference's values bit for bit, a per-row certificate and an exact re-scan
for rows it cannot certify.  ``tile`` and ``threads`` are accepted for
signature compatibility; the result never depends on them (as in the
reference, test_neighbors.py:88-95).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import (ColorArray, EdgeList, NeighborPair, PointMatrix, ValidationError, as_point_matrix,
                   common_scale, unscale_sq)


@dataclass(frozen=True)
class TileSpec:
    """Scan tile shape of the reference (neighbors.py:32-41).

    Kept for API compatibility; the GPU kernel's tiling is fixed (128 query
    rows x 128 index points per CTA step) and results do not depend on it.
    """

    batch_m: int = 256
    batch_n: int = 2048

    def __post_init__(self):
        if self.batch_m < 1 or self.batch_n < 1:
            raise ValidationError("tile sizes must be >= 1")


@dataclass(frozen=True)
class KnnGraph:
    """k nearest neighbours per row, ascending by (distance, id), self excluded."""

    indices: np.ndarray
    distances: np.ndarray

    def __post_init__(self):
        idx = np.asarray(self.indices, dtype=np.int64)
        dist = np.asarray(self.distances, dtype=np.float64)
        if idx.ndim != 2 or idx.shape != dist.shape:
            raise ValidationError("indices and distances must be 2-d with equal shape")
        idx.setflags(write=False)
        dist.setflags(write=False)
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "distances", dist)

    @property
    def n_rows(self) -> int:
        return self.indices.shape[0]

    @property
    def k(self) -> int:
        return self.indices.shape[1]

    def to_edge_list(self) -> EdgeList:
        """Directed edges (i, indices[i, j], distances[i, j])."""
        n, k = self.indices.shape
        return EdgeList(n, np.repeat(np.arange(n, dtype=np.int64), k), self.indices.ravel(),
                        self.distances.ravel())


class DevicePoints:
    """A PointMatrix resident on the current CUDA device.

    ``x32`` always; ``x64`` only when the values are not exactly float32
    (then the refine reads the float64 originals).
    """

    def __init__(self, pm: PointMatrix):
        self.n, self.d = pm.n_rows, pm.n_cols
        self.scale_exp = pm.scale_exp
        self.x32 = _lib.to_device(pm.float32, np.float32)
        self.x64 = None if pm.exact_f32 else _lib.to_device(pm.device_f64, np.float64)

    @classmethod
    def from_tensors(cls, x32, x64=None):
        self = cls.__new__(cls)
        self.n, self.d = int(x32.shape[0]), int(x32.shape[1])
        self.x32, self.x64 = x32, x64
        self.scale_exp = 0
        return self

    def handle(self):
        """The library's search state over these points (slk_pointset_create),
        built on first use and reused by every later search on them."""
        h = getattr(self, "_handle", None)
        if h is None:
            import ctypes

            out = ctypes.c_void_p()
            _lib.call("slk_pointset_create", _lib.ptr(self.x32), _lib.ptr(self.x64), self.n, self.d,
                      ctypes.byref(out), _lib.stream_handle())
            h = self._handle = out
        return h

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib is not None:
            try:
                _lib.load().slk_pointset_destroy(h)
            except Exception:  # interpreter shutdown
                pass


def _check_k(n: int, k: int):
    if not 1 <= k <= n - 1:
        raise ValidationError(f"k must be in [1, {n - 1}] for {n} points, got {k}")


def knn_device(pts: DevicePoints, k: int, rows=None, *, reuse: bool = False):
    """Device tensors (idx int32, dist float64) of rows [q0, q1).

    ``reuse``: search through the points' persistent handle (DevicePoints.handle)
    instead of building the search state for this call only."""
    _check_k(pts.n, k)
    q0, q1 = rows if rows is not None else (0, pts.n)
    idx = _lib.empty((q1 - q0, k), np.int32)
    dist = _lib.empty((q1 - q0, k), np.float64)
    if reuse:
        _lib.call("slk_knn_ps", pts.handle(), k, q0, q1, _lib.ptr(idx), _lib.ptr(dist), _lib.stream_handle())
    else:
        _lib.call("slk_knn", _lib.ptr(pts.x32), _lib.ptr(pts.x64), pts.n, pts.d, k, q0, q1,
                  _lib.ptr(idx), _lib.ptr(dist), _lib.stream_handle())
    return idx, dist


def nn1_colour_device(pts: DevicePoints, colors, rows=None):
    """cross_color_1nn rows [q0, q1) through the points' persistent handle."""
    q0, q1 = rows if rows is not None else (0, pts.n)
    idx = _lib.empty(q1 - q0, np.int32)
    dist = _lib.empty(q1 - q0, np.float64)
    _lib.call("slk_nn1_colour_ps", pts.handle(), _lib.ptr(colors), q0, q1, _lib.ptr(idx), _lib.ptr(dist),
              _lib.stream_handle())
    return idx, dist


def nn1_device(q: DevicePoints, x: DevicePoints, *, mode=0, mask=None, qcolor=None, xcolor=None,
               rows=None):
    """Device tensors (idx int32, dist float64) of the admissible 1-NN of rows [q0, q1)."""
    q0, q1 = rows if rows is not None else (0, q.n)
    idx = _lib.empty(q1 - q0, np.int32)
    dist = _lib.empty(q1 - q0, np.float64)
    _lib.call("slk_nn1", _lib.ptr(q.x32), _lib.ptr(q.x64), q.n, _lib.ptr(x.x32), _lib.ptr(x.x64),
              x.n, q.d, mode, _lib.ptr(mask), _lib.ptr(qcolor), _lib.ptr(xcolor), q0, q1,
              _lib.ptr(idx), _lib.ptr(dist), _lib.stream_handle())
    return idx, dist


def pairwise_l2_tile(queries, index, squared: bool = True) -> np.ndarray:
    """Dense distance tile in the expanded form, clamped at 0 (neighbors.py:229-243)."""
    q = as_point_matrix(queries).data
    x = as_point_matrix(index).data
    if q.shape[1] != x.shape[1]:
        raise ValidationError(f"feature dimensions differ: {q.shape[1]} vs {x.shape[1]}")
    dq, dx = _lib.to_device(q, np.float64), _lib.to_device(x, np.float64)
    out = _lib.empty((len(q), len(x)), np.float64)
    _lib.call("slk_pairwise_l2", _lib.ptr(dq), len(q), _lib.ptr(dx), len(x), q.shape[1],
              int(squared), _lib.ptr(out), _lib.stream_handle())
    return _lib.to_host(out)


def fused_knn(x, k: int, tile: TileSpec | None = None, *, squared: bool = True,
              threads: int | None = None) -> KnnGraph:
    """Exact k nearest neighbours of every row among the other rows (neighbors.py:246-298).

    Rows are sorted by (squared distance, id); distances are bit-identical to
    the reference's float64 expanded-form values.
    """
    pm = as_point_matrix(x)
    _check_k(pm.n_rows, k)
    idx, dist = knn_device(DevicePoints(pm), k)
    out_d = unscale_sq(_lib.to_host(dist), pm.scale_exp)
    if not squared:
        out_d = np.sqrt(out_d)
    return KnnGraph(_lib.to_host(idx).astype(np.int64), out_d)


def fused_1nn(queries, index, mask: np.ndarray | None = None, *, squared: bool = True,
              tile: TileSpec | None = None, threads: int | None = None) -> list[NeighborPair]:
    """Nearest admissible candidate per query row, ties to the smaller id (neighbors.py:351-372)."""
    qm, xm = as_point_matrix(queries), as_point_matrix(index)
    if qm.n_cols != xm.n_cols:
        raise ValidationError(f"feature dimensions differ: {qm.n_cols} vs {xm.n_cols}")
    if mask is not None and mask.shape != (qm.n_rows, xm.n_rows):
        raise ValidationError(
            f"mask shape {mask.shape} does not match ({qm.n_rows}, {xm.n_rows})")
    qm, xm = common_scale(qm, xm)
    q, xx = DevicePoints(qm), DevicePoints(xm)
    dmask = None if mask is None else _lib.to_device(np.asarray(mask, dtype=bool), np.uint8)
    idx, dist = nn1_device(q, xx, mode=0 if mask is None else 1, mask=dmask)
    d = unscale_sq(_lib.to_host(dist), qm.scale_exp)
    if not squared:
        d = np.sqrt(d)
    return [NeighborPair(int(i), float(v)) for i, v in zip(_lib.to_host(idx), d)]


def cross_color_1nn(x, colors: ColorArray, *, squared: bool = True, tile: TileSpec | None = None,
                    threads: int | None = None) -> EdgeList:
    """Per point, the nearest point of another colour: one directed edge each (neighbors.py:375-391)."""
    pm = as_point_matrix(x)
    labels = colors.colors
    if len(labels) != pm.n_rows:
        raise ValidationError("colors length must match point count")
    if len(np.unique(labels)) < 2:
        raise ValidationError("graph is already connected: only one color present")
    pts = DevicePoints(pm)
    dcol = _lib.ids_to_device(labels)
    idx, dist = nn1_device(pts, pts, mode=2, qcolor=dcol, xcolor=dcol)
    d = unscale_sq(_lib.to_host(dist), pm.scale_exp)
    if not squared:
        d = np.sqrt(d)
    return EdgeList(pm.n_rows, np.arange(pm.n_rows, dtype=np.int64),
                    _lib.to_host(idx).astype(np.int64), d)
