"""CPU-side checks: the C-ABI library builds, loads and exports every symbol
include/slink.h declares; the Python mirror exposes the reference's API; the
compute path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "slink.h").read_text()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(slk_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for name in ["slk_knn", "slk_nn1", "slk_solve_mst", "slk_build_dendrogram",
                 "slk_extract_clusters", "slk_single_linkage", "slk_edge_list_to_csr"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2306_16354_b200 import _lib

    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} lacks a ctypes signature"
    assert lib.slk_version() >= 100


def test_library_is_sm100a():
    from paper_2306_16354_b200 import build

    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(build.LIB)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_api_surface_matches_reference():
    import paper_2306_16354_b200 as slk

    reference_all = ["AlteredGraph", "ColorArray", "ConvergenceError", "CsrGraph", "Dendrogram",
                     "EdgeList", "KnnGraph", "LabelArray", "LinkageConfig", "LinkageError",
                     "MstResult", "NeighborPair", "PointMatrix", "TileSpec", "ValidationError",
                     "VertexCandidates", "build_dendrogram", "canonical_edge_key",
                     "compute_cut_level", "connect_graph", "cross_color_1nn", "edge_list_to_csr",
                     "extract_clusters", "fused_1nn", "fused_knn", "label_propagation",
                     "min_edge_per_supervertex", "min_edge_per_vertex", "pairwise_l2_tile",
                     "single_linkage", "solve_mst", "weight_alteration"]
    for name in reference_all:
        assert name in slk.__all__ and hasattr(slk, name), name


def test_no_cpu_fallback():
    import torch

    import paper_2306_16354_b200 as slk

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(slk.LinkageError, match="CUDA"):
        slk.fused_knn(np.random.default_rng(0).standard_normal((10, 2)), 3)


def test_config_and_containers():
    import paper_2306_16354_b200 as slk

    with pytest.raises(slk.ValidationError, match="64"):
        slk.LinkageConfig(n_clusters=2, k=65)
    assert slk.LinkageConfig(n_clusters=2, k=65, allow_large_k=True).k == 65
    with pytest.raises(slk.ValidationError):
        slk.LinkageConfig(n_clusters=2, metric="cosine")
    assert slk.compute_cut_level(6, 3) == 3
    for n in range(1, 30):
        for c in range(1, n + 1):
            assert slk.compute_cut_level(n, c) == (n - 1) - (c - 1)
    with pytest.raises(slk.ValidationError):
        slk.compute_cut_level(5, 6)
    assert slk.canonical_edge_key(3, 1) == (1, 3)
    with pytest.raises(slk.ValidationError):
        slk.canonical_edge_key(2, 2)
    with pytest.raises(slk.ValidationError):
        slk.EdgeList.from_pairs(2, [(0, 2, 1.0)])
    with pytest.raises(slk.ValidationError):
        slk.EdgeList.from_pairs(3, [(1, 1, 1.0)])
    with pytest.raises(slk.ValidationError):
        slk.PointMatrix(np.array([[0.0, np.nan]]))
    pm = slk.PointMatrix(np.zeros((4, 3), dtype=np.float32))
    assert pm.n_rows == 4 and pm.n_cols == 3 and pm.exact_f32
    assert not slk.PointMatrix(np.array([[0.1, 0.2]])).exact_f32
    with pytest.raises(slk.ValidationError):
        slk.LabelArray(np.array([0, 0, 2]), 2)
    d = slk.Dendrogram(2, np.array([[0.0, 1.0, 0.5, 2.0]]))
    assert d.sizes.tolist() == [2]
    with pytest.raises(slk.ValidationError):
        slk.Dendrogram(3, np.array([[0.0, 1.0, 0.5, 2.0], [0.0, 2.0, 1.0, 3.0]]))


def test_every_exported_symbol_is_declared():
    """No undeclared entry points: the .so's slk_* exports == include/slink.h."""
    import subprocess

    from paper_2306_16354_b200 import _lib, build

    _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(build.LIB)], capture_output=True, text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if ln.split()[-1].startswith("slk_")})
    assert exported == declared_symbols()


def test_huge_float64_points_scale_exactly():
    """float64 inputs beyond float32 range go to the device as x * 2^-e (core.py
    PointMatrix): the float32 copy is finite, the float64 copy is the exact
    power-of-two scaling, and distances scale back exactly."""
    from paper_2306_16354_b200.core import PointMatrix, unscale_sq

    x = np.random.default_rng(0).standard_normal((50, 4)) * 1e40
    pm = PointMatrix(x)
    assert pm.scale_exp > 0 and np.isfinite(pm.float32).all()
    assert np.abs(pm.float32).max() < 2.0 ** 64
    assert np.array_equal(np.ldexp(pm.device_f64, pm.scale_exp), x)
    assert np.array_equal(pm.data, x)
    d2 = ((pm.device_f64[0] - pm.device_f64[1]) ** 2).sum()
    assert unscale_sq(d2, pm.scale_exp) == ((x[0] - x[1]) ** 2).sum()
    small = PointMatrix(np.ones((3, 2)))
    assert small.scale_exp == 0 and small.exact_f32
