"""GPU tests of the parlink-compatible CLI (python -m paper_2306_16354_b200).

Each case under tests/golden/cli holds an input file and the output files the
REFERENCE CLI wrote for the same argv (oracle/gen_golden_cli.py); this
package's CLI must exit the same way, print the same summary and write
byte-identical labels / dendrogram / k-NN / MST files.  The remaining tests
restate the command-level behaviour of /root/reference/pkg/tests/test_cli.py.
"""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2306_16354_b200 import io as fio
from paper_2306_16354_b200.cli import main

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "tests" / "golden" / "cli"
CASES = sorted(p.name for p in CLI.iterdir() if (p / "case.json").exists())


def run_cli(*argv):
    return main([str(a) for a in argv])


@pytest.mark.parametrize("name", CASES)
def test_outputs_identical_to_reference_cli(name, tmp_path, capsys):
    case = CLI / name
    meta = json.loads((case / "case.json").read_text())
    argv = [str(case / a[3:]) if a.startswith("IN:") else a.replace("<OUT>", str(tmp_path))
            for a in meta["argv"]]
    assert main(argv) == meta["exit"]
    out = capsys.readouterr().out.replace(str(tmp_path), "<OUT>")
    assert out == meta["stdout"]
    produced = sorted(p.name for p in tmp_path.iterdir() if p.name != "run_manifest.json")
    assert produced == meta["outputs"]
    for fname in produced:
        assert (tmp_path / fname).read_bytes() == (case / ("ref_" + fname)).read_bytes(), fname


def test_module_entry_point(tmp_path):
    case = CLI / "cluster_tiny"
    r = subprocess.run([sys.executable, "-m", "paper_2306_16354_b200", "cluster", "--input",
                        str(case / "pts.csv"), "--output-dir", str(tmp_path),
                        "--n-clusters", "2", "--k", "2"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "labels.csv").read_bytes() == (case / "ref_labels.csv").read_bytes()


def test_manifest_contents(tmp_path, rng):
    from paper_2306_16354_b200.synthetic import make_blobs

    inp = tmp_path / "pts.csv"
    x = make_blobs(rng, 50, 3, 2)
    fio.write_matrix_csv(inp, x)
    assert run_cli("cluster", "--input", inp, "--output-dir", tmp_path, "--n-clusters", 3,
                   "--k", 5, "--seed", 7, "--threads", 2) == 0
    dendro = np.loadtxt(tmp_path / "dendrogram.csv", delimiter=",")
    assert dendro.shape == (len(x) - 1, 4)
    m = json.loads((tmp_path / "run_manifest.json").read_text())
    assert m["subcommand"] == "cluster" and m["input"] == str(inp)
    assert m["parameters"] == {"k": 5, "n_clusters": 3, "metric": "euclidean", "seed": 7,
                               "threads": 2}
    assert set(m["timings_ms"]) == {"knn", "mst", "connect", "dendrogram", "extract"}
    assert all(v >= 0 for v in m["timings_ms"].values())
    assert m["stats"] == {"n_points": 50, "n_features": 3}
    assert all(Path(p).exists() for p in m["outputs"])


def test_n_clusters_equals_n_and_range_error(tmp_path, rng):
    inp = tmp_path / "pts.csv"
    fio.write_matrix_csv(inp, rng.standard_normal((12, 3)))
    assert run_cli("cluster", "--input", inp, "--output-dir", tmp_path,
                   "--n-clusters", 12, "--k", 3) == 0
    assert len(np.unique(np.loadtxt(tmp_path / "labels.csv", dtype=np.int64))) == 12
    assert run_cli("cluster", "--input", inp, "--output-dir", tmp_path,
                   "--n-clusters", 13) == 2
    assert run_cli("knn", "--input", inp, "--output-dir", tmp_path, "--k", 12) == 2


def test_csv_and_binary_inputs_give_identical_outputs(tmp_path, rng):
    x = rng.standard_normal((300, 4)).astype(np.float32)
    fio.write_matrix_csv(tmp_path / "p.csv", x.astype(np.float64))
    fio.write_matrix_binary(tmp_path / "p.slnk", x)
    for src, out in (("p.csv", "a"), ("p.slnk", "b")):
        assert run_cli("cluster", "--input", tmp_path / src, "--output-dir", tmp_path / out,
                       "--n-clusters", 3, "--k", 4, "--seed", 1) == 0
    for f in ("labels.csv", "dendrogram.csv"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()


def test_large_k_is_allowed_by_the_cli(tmp_path, rng):
    inp = tmp_path / "pts.slnk"
    fio.write_matrix_binary(inp, rng.standard_normal((200, 3)))
    assert run_cli("cluster", "--input", inp, "--output-dir", tmp_path,
                   "--n-clusters", 2, "--k", 80) == 0


def test_knn_rows_sorted_and_self_free(tmp_path, rng):
    inp = tmp_path / "pts.csv"
    fio.write_matrix_csv(inp, rng.standard_normal((25, 3)))
    assert run_cli("knn", "--input", inp, "--output-dir", tmp_path, "--k", 6) == 0
    idx = np.loadtxt(tmp_path / "knn_indices.csv", delimiter=",", dtype=np.int64)
    dist = np.loadtxt(tmp_path / "knn_distances.csv", delimiter=",")
    assert idx.shape == dist.shape == (25, 6)
    assert (np.diff(dist, axis=1) >= 0).all() and (idx != np.arange(25)[:, None]).all()


def _mtx(path, n, triples, symmetry="general"):
    with open(path, "w") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate real {symmetry}\n{n} {n} {len(triples)}\n")
        fh.writelines(f"{i + 1} {j + 1} {w}\n" for i, j, w in triples)


def test_mst_small_graphs(tmp_path, capsys):
    tri = [(0, 1, 1.0), (1, 2, 2.0), (0, 2, 3.0)]
    _mtx(tmp_path / "t.mtx", 3, tri)
    assert run_cli("mst", "--input", tmp_path / "t.mtx", "--output-dir", tmp_path) == 0
    assert np.loadtxt(tmp_path / "mst.csv", delimiter=",")[:, 2].sum() == 3.0
    assert "components=1" in capsys.readouterr().out
    assert run_cli("mst", "--input", tmp_path / "t.mtx", "--output-dir", tmp_path,
                   "--maximize", "--verify") == 0
    assert np.loadtxt(tmp_path / "mst.csv", delimiter=",")[:, 2].sum() == 5.0
    assert "verify ok" in capsys.readouterr().out
    _mtx(tmp_path / "z.mtx", 3, [(0, 1, 0.0), (1, 2, 2.0)])
    assert run_cli("mst", "--input", tmp_path / "z.mtx", "--output-dir", tmp_path) == 2
    assert "zero-weight" in capsys.readouterr().err


def test_mst_verify_on_larger_lattice(tmp_path, rng, capsys):
    rows, cols = 60, 70
    t = []
    for r in range(rows):
        for c in range(cols):
            v = r * cols + c
            if c + 1 < cols:
                t.append((v, v + 1, float(rng.uniform(0.5, 9.0))))
            if r + 1 < rows:
                t.append((v, v + cols, float(rng.uniform(0.5, 9.0))))
    _mtx(tmp_path / "g.mtx", rows * cols, t)
    assert run_cli("mst", "--input", tmp_path / "g.mtx", "--output-dir", tmp_path,
                   "--verify") == 0
    out = capsys.readouterr().out
    assert f"edges={rows * cols - 1} components=1" in out and "verify ok" in out


def test_verify_subcommand_passes(capsys):
    assert run_cli("verify", "--seed", 3) == 0
    out = capsys.readouterr().out
    assert "FAIL" not in out and "6/6 checks passed" in out


def test_bench_subcommand_writes_csv(tmp_path):
    assert run_cli("bench", "--output-dir", tmp_path, "--sizes", "120", "--dims", "4",
                   "--ks", "5", "--thread-counts", "1,2") == 0
    lines = (tmp_path / "bench.csv").read_text().strip().splitlines()
    assert lines[0] == "stage,n,d,k,threads,ms"
    assert len(lines) == 1 + 5 * 2
