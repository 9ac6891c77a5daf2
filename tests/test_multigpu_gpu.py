"""The single-process multi-GPU driver (include/slink.h: n_gpus on
slk_single_linkage / slk_single_linkage_device).

The k-NN pass and every cross-colour pass are dealt to n_gpus shards in
128-row chunks; shard g runs on device (current + g) % device_count, so on a
one-GPU box several shards share the device (separate host threads and
streams) and the sharding, chunk bookkeeping and row gathers are exercised all
the same.  The outputs must not depend on n_gpus and must equal the oracle's
(the reference's algorithm, linkage.py:257-311) bit for bit.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slk():
    import paper_2306_16354_b200 as m

    return m


@pytest.mark.parametrize("n_gpus", [2, 3])
def test_sharded_pipeline_matches_single_and_oracle(slk, oracle, n_gpus):
    from paper_2306_16354_b200.synthetic import make_blobs

    # 100 clusters of uneven size, unaligned to 128-row chunks, two connect passes
    x = make_blobs(np.random.default_rng(5), 21000, 64, 100).astype(np.float32)
    cfg = slk.LinkageConfig(n_clusters=40, k=4, seed=1)
    one = slk.single_linkage_result(x, cfg)
    many = slk.single_linkage_result(x, cfg, n_gpus=n_gpus)
    for a, b in [(one.tree.src, many.tree.src), (one.tree.dst, many.tree.dst),
                 (one.tree.weight, many.tree.weight), (one.dendrogram.merges, many.dendrogram.merges),
                 (one.labels.labels, many.labels.labels)]:
        assert np.array_equal(a, b)
    assert one.connect_iters == many.connect_iters
    ref = oracle.single_linkage(x, 40, k=4, seed=1)
    assert np.array_equal(many.dendrogram.merges, ref["merges"])
    assert np.array_equal(many.labels.labels, ref["labels"])


def test_sharded_pipeline_c1_digest(slk):
    """BASELINE.json configs[0] (C1) on 4 shards against the digests the
    reference itself produced (tests/golden/configs/C1_reference.json)."""
    import hashlib
    import json

    from conftest import GOLDEN
    from paper_2306_16354_b200.synthetic import bench_points

    ref = json.loads((GOLDEN / "configs" / "C1_reference.json").read_text())
    x = bench_points(10_000, 16, 10, seed=0)
    res = slk.single_linkage_result(x, slk.LinkageConfig(n_clusters=10, k=15, seed=0), n_gpus=4)

    def dig(a, dt):
        return hashlib.sha256(np.ascontiguousarray(np.asarray(a), dtype=dt).tobytes()).hexdigest()

    assert dig(res.dendrogram.merges, np.float64) == ref["merges_sha256"]
    assert dig(res.labels.labels, np.int64) == ref["labels_sha256"]
    assert dig(res.tree.weight, np.float64) == ref["tree_w_sha256"]


@pytest.mark.parametrize("bad", [0, -1, 65, 2.5, True])
def test_n_gpus_validation(slk, bad):
    x = np.random.default_rng(0).standard_normal((300, 4)).astype(np.float32)
    with pytest.raises(slk.ValidationError, match="n_gpus"):
        slk.single_linkage(x, slk.LinkageConfig(n_clusters=3, k=3), n_gpus=bad)
