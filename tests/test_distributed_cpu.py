"""World-size-2 gloo test of the multi-GPU orchestration (paper_2306_16354_b200/parallel.py).

No GPU here: the sharded compute is delegated to a checker engine built on
the CPU oracle (test infrastructure), so this exercises exactly the product's
sharding, padding, all-gather, colour broadcast and connect-loop control
flow, and compares rank 0's result with the reference's golden fixture.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_golden


class OracleEngine:
    """CPU stand-in for DeviceEngine (same interface), backed by the oracle."""

    def __init__(self):
        from oracle import oracle as orc

        self.orc = orc

    def upload(self, x):
        return np.asarray(x, dtype=np.float64)

    def n_points(self, x):
        return len(x)

    def knn_shard(self, x, k, rows):
        idx, d = self.orc.fused_knn(x, k, rows=rows)
        return torch.from_numpy(idx.astype(np.int32)), torch.from_numpy(d)

    def nn1_shard(self, x, colors, rows):
        idx, d = self.orc.cross_color_1nn(x, colors.numpy().astype(np.int64), rows=rows)
        return torch.from_numpy(idx.astype(np.int32)), torch.from_numpy(d)

    def msf(self, n, src, dst, w, m, seed):
        from paper_2306_16354_b200 import ValidationError

        offs, cols, ww = self.orc.edge_list_to_csr(n, src.numpy()[:m], dst.numpy()[:m], w.numpy()[:m])
        try:
            s, d, wt, colors, nc = self.orc.solve_mst(n, offs, cols, ww, seed=seed)
        except self.orc.OracleError as exc:  # the device engine raises the package's classes
            raise ValidationError(str(exc)) from None
        return (torch.from_numpy(s.astype(np.int32)), torch.from_numpy(d.astype(np.int32)),
                torch.from_numpy(wt), torch.from_numpy(colors.astype(np.int32)), len(s), nc)

    def scale_exp(self, x):
        return 0

    def finish(self, n, t_src, t_dst, t_w, cfg, scale_exp=0):
        from paper_2306_16354_b200 import Dendrogram, EdgeList, LabelArray

        w = t_w.numpy()
        w2 = np.sqrt(w) if cfg.metric == "euclidean" else w
        merges = self.orc.build_dendrogram(t_src.numpy(), t_dst.numpy(), w2, n)
        labels = self.orc.extract_clusters(merges, n, cfg.n_clusters)
        tree = EdgeList(n, t_src.numpy(), t_dst.numpy(), w)
        return tree, Dendrogram(n, merges), LabelArray(labels, cfg.n_clusters)

    def sync(self):
        pass


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, str(ROOT))
        import paper_2306_16354_b200 as slk
        from paper_2306_16354_b200.parallel import single_linkage_distributed

        if name == "duplicates":
            # duplicate points -> zero-weight edge: rank 0's forest solve raises
            # (ref mst.py:209-210); every rank must raise the same class
            x = np.concatenate([np.random.default_rng(0).standard_normal((40, 3))] * 2)
            try:
                single_linkage_distributed(x, slk.LinkageConfig(n_clusters=2, k=3), engine=OracleEngine())
                out.put((rank, "no error", ""))
            except slk.LinkageError as exc:
                out.put((rank, type(exc).__name__, str(exc)))
            return
        g = load_golden(name)
        cfg = slk.LinkageConfig(n_clusters=int(g["n_clusters"]), k=int(g["k"]), seed=int(g["seed"]))
        res = single_linkage_distributed(g["x"], cfg, engine=OracleEngine())
        if rank == 0:
            out.put((res.tree.src, res.tree.weight, res.dendrogram.merges, res.labels.labels,
                     res.connect_iters))
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def _run_ranks(world, name, n_results):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, out)) for r in range(world)]
    for p in procs:
        p.start()
    results = [out.get(timeout=300) for _ in range(n_results)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return results


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_chunks_cover_exactly():
    """Round-robin chunks: disjoint, 128-aligned, covering [0, n), every rank
    holding chunks spread over the whole row order."""
    from paper_2306_16354_b200.parallel import shard_chunks

    for n in (1, 127, 128, 129, 1000, 10_000, 1_000_000):
        for world in (1, 2, 3, 4, 8):
            per = [shard_chunks(n, world, r) for r in range(world)]
            allc = sorted(c for p in per for c in p)
            assert allc[0][0] == 0 and allc[-1][1] == n
            for (a0, a1), (b0, b1) in zip(allc, allc[1:]):
                assert a1 == b0 and a0 <= a1
            assert all(a % 128 == 0 for a, _ in allc if a < n)
            blocks = -(-n // 128)
            if blocks >= 4 * world:
                assert all(len(p) == 4 for p in per)


@pytest.mark.parametrize("world,name", [(2, "slink_blobs_2k_d32_k2"), (2, "slink_tiny_k2"),
                                        (3, "slink_blobs_2k_d32_k2")])
def test_multi_rank_pipeline_matches_reference(oracle, world, name):
    """World sizes 2 and 3 (2000 rows = 16 blocks in 12 round-robin chunks of
    1-2 blocks: ragged per-rank row counts, padded in the gather)."""
    (result,) = _run_ranks(world, name, 1)
    src, w, merges, labels, iters = result
    g = load_golden(name)
    assert np.array_equal(src, g["tree_src"]) and np.array_equal(w, g["tree_w"])
    assert np.array_equal(merges, g["merges"]) and np.array_equal(labels, g["labels"])
    assert iters == int(g["connect_iters"])


def test_rank0_failure_raises_on_every_rank(oracle):
    """A ValidationError in rank 0's forest solve is broadcast: no rank hangs."""
    results = _run_ranks(2, "duplicates", 2)
    assert sorted(r[0] for r in results) == [0, 1]
    assert all(r[1] == "ValidationError" and "zero" in r[2] for r in results), results
