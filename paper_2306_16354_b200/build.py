"""Build libslink.so (sm_100a) in-tree: paper_2306_16354_b200/lib/libslink.so.

nvcc cross-compiles without a GPU.  Flags: -gencode arch=compute_100a,
code=sm_100a (tcgen05/TMA need the arch-specific target), -lineinfo for ncu
source correlation, -O3.  No --use_fast_math: the float64 refine relies on
IEEE semantics (it also uses explicit __dadd_rn/__dmul_rn so nothing is
contracted into FMA).
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "lib"
LIB = OUT_DIR / "libslink.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


# Diagnostic variants (never loaded unless SLK_LIB_VARIANT names one):
# "timeline" stamps the scan's warp-role hand-offs (tc_scan.cu, SLK_TIMELINE).
VARIANTS = {"timeline": ["-DSLK_TIMELINE"], "nomma": ["-DSLK_ABL_NOMMA"], "noconv": ["-DSLK_ABL_NOCONV"],
            "noepi": ["-DSLK_ABL_NOEPI"], "ncg2": ["-DSLK_BC_NCG2_MIN_DK=64"]}


def variant_path(name: str) -> Path:
    return OUT_DIR / f"libslink_{name}.so"


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "slink.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, variant: str | None = None) -> Path:
    lib = variant_path(variant) if variant else LIB
    extra = VARIANTS[variant] if variant else []
    if not force and not _stale(lib):
        return lib
    OUT_DIR.mkdir(exist_ok=True)
    objs = []

    def compile_one(src: Path):
        obj = OUT_DIR / (src.stem + (f"_{variant}" if variant else "") + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        o.unlink(missing_ok=True)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    print(build(force="--force" in sys.argv, verbose=True, variant=var))
