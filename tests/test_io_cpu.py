"""CPU tests of the file formats, the CLI's input-error paths and the checkers.

Mirrors the I/O half of /root/reference/pkg/tests/test_cli.py (binary format,
CSV diagnostics, Matrix Market parsing, thread resolution, exit codes for
bad input) and pins this package's readers/writers to files the reference
itself wrote (tests/golden/cli, made by oracle/gen_golden_cli.py).
"""

import json
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2306_16354_b200 import checkers
from paper_2306_16354_b200 import io as fio
from paper_2306_16354_b200.cli import RunManifest, main
from paper_2306_16354_b200.core import Dendrogram, EdgeList, LinkageError, ValidationError
from paper_2306_16354_b200.neighbors import KnnGraph
from paper_2306_16354_b200.parallel import resolve_threads

CLI = Path(__file__).resolve().parent / "golden" / "cli"


def run_cli(*argv):
    return main([str(a) for a in argv])


# --------------------------------------------------------------------------- SLNK binary

def test_binary_round_trip_is_lossless_at_f32(tmp_path, rng):
    x = rng.standard_normal((13, 5)).astype(np.float32)
    p = tmp_path / "m.slnk"
    fio.write_matrix_binary(p, x)
    back = fio.read_matrix_binary(p)
    assert back.dtype == np.float64 and np.array_equal(back, x.astype(np.float64))
    assert p.stat().st_size == 16 + 13 * 5 * 4
    assert p.read_bytes()[:16] == struct.pack("<4sIII", b"SLNK", 1, 13, 5)


def test_binary_auto_detect(tmp_path, rng):
    x = rng.standard_normal((4, 2)).astype(np.float32)
    p = tmp_path / "m.dat"
    fio.write_matrix_binary(p, x)
    assert np.array_equal(fio.read_matrix_auto(p), x.astype(np.float64))


def test_binary_reads_reference_written_file():
    case = CLI / "cluster_slnk_sq"
    x = fio.read_matrix_binary(case / "pts.slnk")
    assert x.shape == (400, 5)
    # the CSV case was written from the same float32-exact matrix
    assert np.array_equal(x, fio.read_matrix_csv(CLI / "cluster_csv" / "pts.csv"))


def test_binary_writer_matches_reference_bytes(tmp_path):
    src = CLI / "knn_slnk_sq" / "pts.slnk"
    p = tmp_path / "again.slnk"
    fio.write_matrix_binary(p, fio.read_matrix_binary(src))
    assert p.read_bytes() == src.read_bytes()


@pytest.mark.parametrize("cut,match", [(-3, "payload is"), (10, "truncated header at offset 10")])
def test_binary_truncation(tmp_path, rng, cut, match):
    p = tmp_path / "m.slnk"
    fio.write_matrix_binary(p, rng.standard_normal((4, 2)))
    raw = p.read_bytes()
    p.write_bytes(raw[:cut])
    with pytest.raises(ValidationError, match=match):
        fio.read_matrix_binary(p)


def test_binary_trailing_bytes_rejected(tmp_path, rng):
    p = tmp_path / "m.slnk"
    fio.write_matrix_binary(p, rng.standard_normal((4, 2)))
    p.write_bytes(p.read_bytes() + b"xyz")
    with pytest.raises(ValidationError, match=r"payload is 35 bytes at offset 16, expected 32"):
        fio.read_matrix_binary(p)


def test_binary_bad_magic_and_version(tmp_path):
    p = tmp_path / "m.slnk"
    p.write_bytes(struct.pack("<4sIII", b"SLNX", 1, 1, 1) + b"\0" * 4)
    with pytest.raises(ValidationError, match="bad magic b'SLNX' at offset 0"):
        fio.read_matrix_binary(p)
    p.write_bytes(struct.pack("<4sIII", b"SLNK", 2, 1, 1) + b"\0" * 4)
    with pytest.raises(ValidationError, match="unsupported version 2"):
        fio.read_matrix_binary(p)


def test_binary_rejects_non_2d(tmp_path):
    with pytest.raises(ValidationError, match="2-d"):
        fio.write_matrix_binary(tmp_path / "m.slnk", np.zeros(3))


# --------------------------------------------------------------------------- CSV

def test_csv_round_trip_is_exact(tmp_path, rng):
    x = rng.standard_normal((9, 4)) * 1e3
    p = tmp_path / "m.csv"
    fio.write_matrix_csv(p, x)
    assert np.array_equal(fio.read_matrix_csv(p), x)


def test_csv_writer_matches_reference_bytes(tmp_path):
    src = CLI / "knn_csv" / "pts.csv"
    p = tmp_path / "again.csv"
    fio.write_matrix_csv(p, fio.read_matrix_csv(src))
    assert p.read_bytes() == src.read_bytes()


def test_csv_single_column_and_single_row(tmp_path):
    p = tmp_path / "c.csv"
    p.write_text("1.5\n2.5\n")
    assert fio.read_matrix_csv(p).shape == (2, 1)
    p.write_text("1,2,3\n")
    assert fio.read_matrix_csv(p).shape == (1, 3)


@pytest.mark.parametrize("text,match", [
    ("1.0,2.0\n3.0,oops\n", r"line 2, field 2: not a number: 'oops'"),
    ("1,2\n3,4\n5\n", r"line 3 has 1 fields, expected 2"),
    ("1,2\n\n3,4,5\n", r"line 3 has 3 fields, expected 2"),
])
def test_csv_diagnostics_name_the_line(tmp_path, text, match):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(ValidationError, match=match):
        fio.read_matrix_csv(p)


# --------------------------------------------------------------------------- Matrix Market

def test_mtx_general_and_symmetric(tmp_path):
    g = fio.read_mtx_graph(CLI / "mst_grid" / "g.mtx")
    assert g.n_vertices == 12 * 17 and len(g) == 12 * 16 + 11 * 17
    s = fio.read_mtx_graph(CLI / "mst_symmetric" / "g.mtx")
    # symmetric files come back with both triangles
    assert s.n_vertices == 99 and len(s) == 2 * (9 * 10 + 8 * 11)
    assert (s.src > s.dst).sum() == (s.src < s.dst).sum()


def test_mtx_writer_round_trip(tmp_path, rng):
    e = EdgeList(6, np.array([0, 1, 2, 4]), np.array([1, 2, 3, 5]), rng.uniform(0.1, 2, 4))
    for sym in (False, True):
        p = tmp_path / f"g{sym}.mtx"
        fio.write_mtx_graph(p, e, symmetric=sym)
        back = fio.read_mtx_graph(p)
        assert back.n_vertices == 6
        got = {(min(a, b), max(a, b)): w for a, b, w in back.iter_edges()}
        assert got == {(a, b): w for a, b, w in e.iter_edges()}


@pytest.mark.parametrize("text,match", [
    ("this is not matrix market\n", "not a readable Matrix Market file"),
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "expected a coordinate"),
    ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 2 1.0\n", "must be square"),
])
def test_mtx_errors(tmp_path, text, match):
    p = tmp_path / "g.mtx"
    p.write_text(text)
    with pytest.raises(ValidationError, match=match):
        fio.read_mtx_graph(p)


# --------------------------------------------------------------------------- output writers

def test_output_writers_reproduce_reference_files(tmp_path):
    rows = np.loadtxt(CLI / "cluster_csv" / "ref_dendrogram.csv", delimiter=",")
    fio.write_dendrogram_csv(tmp_path / "d.csv", Dendrogram(400, rows))
    assert (tmp_path / "d.csv").read_bytes() == (CLI / "cluster_csv" /
                                                  "ref_dendrogram.csv").read_bytes()
    labels = np.loadtxt(CLI / "cluster_csv" / "ref_labels.csv", dtype=np.int64)
    fio.write_labels_csv(tmp_path / "l.csv", labels)
    assert (tmp_path / "l.csv").read_bytes() == (CLI / "cluster_csv" / "ref_labels.csv").read_bytes()
    case = CLI / "knn_csv"
    knn = KnnGraph(np.loadtxt(case / "ref_knn_indices.csv", delimiter=",", dtype=np.int64),
                   np.loadtxt(case / "ref_knn_distances.csv", delimiter=","))
    fio.write_knn_csvs(tmp_path / "i.csv", tmp_path / "x.csv", knn)
    assert (tmp_path / "i.csv").read_bytes() == (case / "ref_knn_indices.csv").read_bytes()
    assert (tmp_path / "x.csv").read_bytes() == (case / "ref_knn_distances.csv").read_bytes()
    m = np.loadtxt(CLI / "mst_grid" / "ref_mst.csv", delimiter=",")
    fio.write_mst_csv(tmp_path / "m.csv", EdgeList(204, m[:, 0], m[:, 1], m[:, 2]))
    assert (tmp_path / "m.csv").read_bytes() == (CLI / "mst_grid" / "ref_mst.csv").read_bytes()


# --------------------------------------------------------------------------- CLI input errors

def test_cli_malformed_csv_exits_2_with_line(tmp_path, capsys):
    p = tmp_path / "bad.csv"
    p.write_text("1.0,2.0\n3.0,oops\n")
    assert run_cli("cluster", "--input", p, "--output-dir", tmp_path, "--n-clusters", 2) == 2
    assert "line 2" in capsys.readouterr().err


def test_cli_missing_input_exits_2(tmp_path):
    assert run_cli("cluster", "--input", tmp_path / "nope.csv", "--output-dir", tmp_path,
                   "--n-clusters", 2) == 2
    assert run_cli("knn", "--input", tmp_path / "nope.csv", "--output-dir", tmp_path,
                   "--k", 2) == 2
    assert run_cli("mst", "--input", tmp_path / "nope.mtx", "--output-dir", tmp_path) == 2


def test_cli_unparsable_mtx_exits_2(tmp_path, capsys):
    p = tmp_path / "junk.mtx"
    p.write_text("this is not matrix market\n")
    assert run_cli("mst", "--input", p, "--output-dir", tmp_path) == 2
    assert "Matrix Market" in capsys.readouterr().err


def test_cli_bad_config_exits_2(tmp_path):
    p = tmp_path / "pts.csv"
    fio.write_matrix_csv(p, np.arange(20.0).reshape(10, 2))
    assert run_cli("cluster", "--input", p, "--output-dir", tmp_path, "--n-clusters", 0) == 2
    assert run_cli("cluster", "--input", p, "--output-dir", tmp_path, "--n-clusters", 2,
                   "--tile-m", 0) == 2


def test_cli_usage_errors_exit_2(tmp_path):
    with pytest.raises(SystemExit) as exc:
        main(["cluster", "--input", "x.csv"])  # --n-clusters missing
    assert exc.value.code == 2
    with pytest.raises(SystemExit) as exc:
        main(["knn", "--input", "x.csv", "--k", "3", "--metric", "cosine"])
    assert exc.value.code == 2


def test_run_manifest_rejects_negative_timing(tmp_path):
    m = RunManifest("in", "cluster", {}, {"knn": -1.0}, [])
    with pytest.raises(LinkageError):
        m.write(tmp_path / "m.json")
    m = RunManifest("in", "cluster", {"k": 3}, {"knn": 1.0}, ["a"], {"n_points": 4})
    m.write(tmp_path / "m.json")
    text = (tmp_path / "m.json").read_text()
    assert text.endswith("}\n") and json.loads(text)["parameters"] == {"k": 3}
    assert list(json.loads(text)) == sorted(json.loads(text))


# --------------------------------------------------------------------------- threads

def test_threads_env_and_flag(monkeypatch):
    monkeypatch.setenv("PARLINK_THREADS", "3")
    assert resolve_threads(None) == 3
    assert resolve_threads(2) == 2
    monkeypatch.delenv("PARLINK_THREADS")
    assert resolve_threads(None) >= 1
    with pytest.raises(ValueError):
        resolve_threads(0)


# --------------------------------------------------------------------------- checkers

def test_checkers_agree_with_reference_outputs():
    case = CLI / "knn_csv"
    x = fio.read_matrix_csv(case / "pts.csv")
    ids, dist = checkers.sorted_knn(x, 10, squared=False)
    assert np.array_equal(ids, np.loadtxt(case / "ref_knn_indices.csv", delimiter=",", dtype=np.int64))
    np.testing.assert_allclose(dist, np.loadtxt(case / "ref_knn_distances.csv", delimiter=","),
                               rtol=1e-12)
    g = fio.read_mtx_graph(CLI / "mst_grid" / "g.mtx")
    s, d, w = checkers.kruskal_forest(g.n_vertices, g.src, g.dst, g.weight)
    ref = np.loadtxt(CLI / "mst_grid" / "ref_mst.csv", delimiter=",")
    assert len(s) == len(ref)
    assert abs(w.sum() - ref[:, 2].sum()) <= 1e-9 * ref[:, 2].sum()
    x = fio.read_matrix_csv(CLI / "cluster_csv" / "pts.csv")
    labels = np.loadtxt(CLI / "cluster_csv" / "ref_labels.csv", dtype=np.int64)
    assert checkers.adjusted_rand_index(checkers.naive_partition(x, 4), labels) == 1.0


def test_adjusted_rand_index_properties():
    a = np.array([0, 0, 1, 1, 2, 2])
    assert checkers.adjusted_rand_index(a, a + 7) == 1.0
    assert checkers.adjusted_rand_index(a, [0, 1, 0, 1, 0, 1]) < 0.5
    assert checkers.adjusted_rand_index([0], [3]) == 1.0


def test_kruskal_checker_matches_oracle_kruskal(oracle, rng):
    """The CLI's Kruskal checker agrees with the oracle's restatement on
    random graphs with tied integer weights (forest edges and total weight)."""
    from paper_2306_16354_b200.synthetic import random_connected_graph

    for n, extra in ((50, 80), (400, 1500)):
        s, d, w = random_connected_graph(rng, n, extra, weights="ties")
        a, b, kw = checkers.kruskal_forest(n, s, d, w)
        oa, ob, ow = oracle.kruskal_mst(n, s, d, w)
        assert len(a) == len(oa) == n - 1
        assert np.array_equal(np.sort(kw), np.sort(ow)) and kw.sum() == ow.sum()


def test_road_graph_generator_is_deterministic():
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "bench_mst", Path(__file__).resolve().parents[1] / "scripts" / "bench_mst.py")
    bm = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bm)
    n1, s1, d1, w1 = bm.road_graph(10_000, 12_000, seed=3)
    n2, s2, d2, w2 = bm.road_graph(10_000, 12_000, seed=3)
    assert n1 == n2 and np.array_equal(s1, s2) and np.array_equal(d1, d2) and np.array_equal(w1, w2)
    assert abs(len(s1) - 12_000) < 600 and (w1 >= 1).all() and (w1 <= 100_000).all()
    assert (s1 != d1).all() and d1.max() < n1
