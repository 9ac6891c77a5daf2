"""Golden CLI fixtures: run the REFERENCE command line on seeded inputs.

Build container only (needs /root/reference):

    python oracle/gen_golden_cli.py

For every case it writes the input file(s) and the files the reference's
``parlink`` CLI produced (/root/reference/pkg/src/parlink/cli.py) plus its
exit code and stdout (paths replaced by ``<OUT>``) under
``tests/golden/cli/<case>/``.  ``tests/test_cli_gpu.py`` runs this
package's CLI on the same inputs and requires byte-identical output files;
``tests/test_io_cpu.py`` reads the inputs back with this package's readers.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import shutil
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from parlink import io as ref_io  # noqa: E402
from parlink.cli import main as ref_main  # noqa: E402

from paper_2306_16354_b200.synthetic import make_blobs  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "cli"


def write_mtx(path, n, triples, symmetry="general"):
    with open(path, "w") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate real {symmetry}\n")
        fh.write(f"{n} {n} {len(triples)}\n")
        for i, j, w in triples:
            fh.write(f"{i + 1} {j + 1} {w!r}\n")


def lattice(rng, rows, cols, symmetric=False):
    """Road-style grid with random link lengths; symmetric stores the lower triangle."""
    t = []
    for r in range(rows):
        for c in range(cols):
            v = r * cols + c
            for u in ((v + 1) if c + 1 < cols else None, (v + cols) if r + 1 < rows else None):
                if u is not None:
                    w = float(np.round(rng.uniform(0.5, 9.0), 3))
                    t.append((u, v, w) if symmetric else (v, u, w))
    return t


def run_case(name, inputs, argv):
    """inputs: {filename: writer(path)}; argv uses {IN:<file>} and <OUT>."""
    case = OUT / name
    shutil.rmtree(case, ignore_errors=True)
    case.mkdir(parents=True)
    for fname, writer in inputs.items():
        writer(case / fname)
    with tempfile.TemporaryDirectory() as tmp:
        args = [a.replace("<OUT>", tmp) for a in argv]
        args = [str(case / a[3:]) if a.startswith("IN:") else a for a in args]
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = ref_main(args)
        stdout = buf.getvalue().replace(tmp, "<OUT>").replace(str(case), "<CASE>")
        produced = sorted(p.name for p in Path(tmp).iterdir() if p.name != "run_manifest.json")
        for fname in produced:
            shutil.copy(Path(tmp) / fname, case / ("ref_" + fname))
    meta = {"argv": argv, "exit": code, "stdout": stdout, "outputs": produced}
    (case / "case.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    print(f"{name}: exit {code}, outputs {produced}")


def main():
    rng = np.random.default_rng(2306)
    blobs = make_blobs(rng, 400, 5, 4).astype(np.float32).astype(np.float64)
    normal = rng.standard_normal((300, 6))
    tiny = np.array([[0.0], [0.1], [10.0], [10.1]])

    run_case("cluster_csv", {"pts.csv": lambda p: ref_io.write_matrix_csv(p, blobs)},
             ["cluster", "--input", "IN:pts.csv", "--output-dir", "<OUT>",
              "--n-clusters", "4", "--seed", "3"])
    run_case("cluster_slnk_sq", {"pts.slnk": lambda p: ref_io.write_matrix_binary(p, blobs)},
             ["cluster", "--input", "IN:pts.slnk", "--output-dir", "<OUT>",
              "--n-clusters", "7", "--k", "8", "--metric", "sqeuclidean"])
    run_case("cluster_tiny", {"pts.csv": lambda p: ref_io.write_matrix_csv(p, tiny)},
             ["cluster", "--input", "IN:pts.csv", "--output-dir", "<OUT>",
              "--n-clusters", "2", "--k", "2"])
    run_case("knn_csv", {"pts.csv": lambda p: ref_io.write_matrix_csv(p, normal)},
             ["knn", "--input", "IN:pts.csv", "--output-dir", "<OUT>", "--k", "10"])
    run_case("knn_slnk_sq", {"pts.slnk": lambda p: ref_io.write_matrix_binary(p, normal)},
             ["knn", "--input", "IN:pts.slnk", "--output-dir", "<OUT>", "--k", "7",
              "--metric", "sqeuclidean"])
    grid = lattice(rng, 12, 17)
    run_case("mst_grid", {"g.mtx": lambda p: write_mtx(p, 12 * 17, grid)},
             ["mst", "--input", "IN:g.mtx", "--output-dir", "<OUT>", "--verify"])
    run_case("mst_grid_max", {"g.mtx": lambda p: write_mtx(p, 12 * 17, grid)},
             ["mst", "--input", "IN:g.mtx", "--output-dir", "<OUT>", "--maximize"])
    sym = lattice(rng, 9, 11, symmetric=True)
    run_case("mst_symmetric", {"g.mtx": lambda p: write_mtx(p, 99, sym, "symmetric")},
             ["mst", "--input", "IN:g.mtx", "--output-dir", "<OUT>"])
    forest = [(0, 1, 1.0), (2, 3, 2.0), (3, 4, 1.5), (6, 7, 0.25)]
    run_case("mst_forest", {"g.mtx": lambda p: write_mtx(p, 9, forest)},
             ["mst", "--input", "IN:g.mtx", "--output-dir", "<OUT>"])


if __name__ == "__main__":
    main()
