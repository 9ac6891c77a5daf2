"""Deterministic Boruvka spanning forest on the GPU (mirrors ``parlink.mst``).

Public names follow /root/reference/pkg/src/parlink/mst.py:36-344.  The
seeded weight alteration reproduces the reference's altered values bit for
bit (_hash_unit :82-91, _alter_weights :94-105); the solver's strict total
order (altered weight, a, b) is turned into 32-bit ranks by one device radix
sort and Boruvka runs on ranks (csrc/graph.cu), so the forest is the unique
minimum spanning forest under that order — the reference's forest.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import ColorArray, CsrGraph, EdgeList, NeighborPair, ValidationError


@dataclass(frozen=True)
class AlteredGraph:
    """CSR graph with perturbed weights plus the originals (mst.py:36-50)."""

    graph: CsrGraph
    original_weights: np.ndarray
    theta: float
    seed: int

    def __post_init__(self):
        orig = np.asarray(self.original_weights, dtype=np.float64).ravel()
        if len(orig) != self.graph.n_edges:
            raise ValidationError("original_weights must parallel the CSR entries")
        orig.setflags(write=False)
        object.__setattr__(self, "original_weights", orig)


@dataclass(frozen=True)
class MstResult:
    """Spanning forest edges (original weights), final colours, component count."""

    edges: EdgeList
    colors: ColorArray
    n_components: int


@dataclass(frozen=True)
class VertexCandidates:
    """Per-vertex minimum cross-colour edge; position -1 means none (mst.py:62-79)."""

    src: np.ndarray
    dst: np.ndarray
    position: np.ndarray
    altered_weight: np.ndarray
    original_weight: np.ndarray

    def pair(self, vertex: int) -> NeighborPair | None:
        if self.position[vertex] < 0:
            return None
        return NeighborPair(int(self.dst[vertex]), float(self.altered_weight[vertex]))


class _DeviceCsr:
    def __init__(self, g: CsrGraph, weights=None):
        self.n = g.n_vertices
        self.offs = _lib.to_device(g.row_offsets, np.int64)
        self.cols = _lib.ids_to_device(g.col_indices) if g.n_edges else _lib.empty(1, np.int32)
        w = g.weights if weights is None else weights
        self.w = _lib.to_device(w, np.float64) if g.n_edges else _lib.empty(1, np.float64)


def weight_alteration(g: CsrGraph, seed: int = 0) -> AlteredGraph:
    """Seeded order-preserving perturbation of a symmetric graph's weights (mst.py:198-222).

    theta = smallest gap between distinct weights (fallback max(|w|, 1)*2^-20);
    every undirected edge gets w + hash(a, b, seed) * theta * (1 - 2^-20).
    Rejects empty, non-finite, asymmetric and zero-weight graphs.
    """
    if g.n_vertices == 0:
        raise ValidationError("empty graph: no vertices")
    if g.n_edges == 0:
        return AlteredGraph(g, g.weights, 0.0, seed)
    dev = _DeviceCsr(g)
    alt = _lib.empty(g.n_edges, np.float64)
    theta = ctypes.c_double()
    _lib.call("slk_weight_alteration", g.n_vertices, _lib.ptr(dev.offs), _lib.ptr(dev.cols),
              _lib.ptr(dev.w), int(seed), _lib.ptr(alt), ctypes.byref(theta), _lib.stream_handle())
    altered = CsrGraph(g.n_vertices, g.row_offsets, g.col_indices, _lib.to_host(alt))
    return AlteredGraph(altered, g.weights, theta.value, seed)


def min_edge_per_vertex(g: AlteredGraph, colors: ColorArray, *,
                        threads: int | None = None) -> VertexCandidates:
    """Per vertex, the minimum (altered weight, a, b) edge to another colour (mst.py:225-254)."""
    csr = g.graph
    n = csr.n_vertices
    if len(colors) != n:
        raise ValidationError("colors length must match vertex count")
    if csr.n_edges == 0:
        none = np.full(n, -1, dtype=np.int64)
        return VertexCandidates(np.arange(n, dtype=np.int64), none, none, np.full(n, np.inf),
                                np.full(n, np.inf))
    dev = _DeviceCsr(csr)
    col = _lib.ids_to_device(colors.colors)
    pos = _lib.empty(n, np.int64)
    _lib.call("slk_min_edge_per_vertex", n, _lib.ptr(dev.offs), _lib.ptr(dev.cols),
              _lib.ptr(dev.w), _lib.ptr(col), _lib.ptr(pos), _lib.stream_handle())
    positions = _lib.to_host(pos)
    found = positions >= 0
    safe = np.where(found, positions, 0)
    dst = np.where(found, csr.col_indices[safe], -1)
    alt = np.where(found, csr.weights[safe], np.inf)
    orig = np.where(found, g.original_weights[safe], np.inf)
    return VertexCandidates(np.arange(n, dtype=np.int64), dst, positions, alt, orig)


def min_edge_per_supervertex(candidates: VertexCandidates, colors: ColorArray) -> EdgeList:
    """One minimum candidate per colour, canonical and deduplicated (mst.py:257-280)."""
    n = len(candidates.position)
    if n == 0:
        return EdgeList(0, np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0))
    pos = _lib.to_device(candidates.position, np.int64)
    dst = _lib.ids_to_device(np.where(candidates.position >= 0, candidates.dst, 0))
    alt = _lib.to_device(candidates.altered_weight, np.float64)
    orig = _lib.to_device(candidates.original_weight, np.float64)
    col = _lib.ids_to_device(colors.colors)
    a, b = _lib.empty(n, np.int32), _lib.empty(n, np.int32)
    w = _lib.empty(n, np.float64)
    m = ctypes.c_int64()
    _lib.call("slk_min_edge_per_supervertex", n, _lib.ptr(pos), _lib.ptr(dst), _lib.ptr(alt),
              _lib.ptr(orig), _lib.ptr(col), _lib.ptr(a), _lib.ptr(b), _lib.ptr(w),
              ctypes.byref(m), _lib.stream_handle())
    k = m.value
    return EdgeList(n, _lib.to_host(a[:k]).astype(np.int64), _lib.to_host(b[:k]).astype(np.int64),
                    _lib.to_host(w[:k]))


def label_propagation(new_edges: EdgeList, colors: ColorArray) -> ColorArray:
    """Spread the minimum colour over every group joined by new edges (mst.py:283-289)."""
    if len(new_edges) == 0:
        return ColorArray(colors.colors.copy())
    col = _lib.ids_to_device(colors.colors)
    us, vs = _lib.ids_to_device(new_edges.src), _lib.ids_to_device(new_edges.dst)
    _lib.call("slk_label_propagation", len(colors), _lib.ptr(col), _lib.ptr(us), _lib.ptr(vs),
              len(new_edges), _lib.stream_handle())
    return ColorArray(_lib.to_host(col).astype(np.int64))


def solve_mst(g: CsrGraph, maximize: bool = False, seed: int = 0, *,
              threads: int | None = None) -> MstResult:
    """Minimum (or maximum) spanning tree / forest of a symmetric graph (mst.py:292-344).

    Edges come back with their original weights, sorted by (src, dst), src <
    dst; colours are canonical (smallest vertex id per component).  Fixed
    (graph, seed, maximize) gives a bit-identical result.
    """
    n = g.n_vertices
    if n == 0:
        raise ValidationError("empty graph: no vertices")
    dev = _DeviceCsr(g)
    src, dst = _lib.empty(max(n - 1, 1), np.int32), _lib.empty(max(n - 1, 1), np.int32)
    w = _lib.empty(max(n - 1, 1), np.float64)
    col = _lib.empty(n, np.int32)
    ne, nc = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("slk_solve_mst", n, _lib.ptr(dev.offs), _lib.ptr(dev.cols), _lib.ptr(dev.w),
              int(bool(maximize)), int(seed), _lib.ptr(src), _lib.ptr(dst), _lib.ptr(w),
              _lib.ptr(col), ctypes.byref(ne), ctypes.byref(nc), _lib.stream_handle())
    k = ne.value
    edges = EdgeList(n, _lib.to_host(src[:k]).astype(np.int64),
                     _lib.to_host(dst[:k]).astype(np.int64), _lib.to_host(w[:k]))
    return MstResult(edges, ColorArray(_lib.to_host(col).astype(np.int64)), nc.value)
