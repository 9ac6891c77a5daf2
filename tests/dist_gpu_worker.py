"""Worker of tests/test_parity_gpu.py::test_distributed_two_ranks_one_gpu.

Run under torchrun with 2 ranks sharing cuda:0 over gloo (collectives staged
through the host): the product's DeviceEngine does all compute, and rank 0
compares the distributed result with the single-process one.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2306_16354_b200 as slk  # noqa: E402
from paper_2306_16354_b200 import parallel  # noqa: E402
from paper_2306_16354_b200.synthetic import make_blobs  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("gloo")
x = make_blobs(np.random.default_rng(3), 3000, 16, 9).astype(np.float32)
cfg = slk.LinkageConfig(n_clusters=9, k=4, seed=0)
res = parallel.single_linkage_distributed(x, cfg)
if dist.get_rank() == 0:
    ref = slk.single_linkage_result(x, cfg)
    ok = (np.array_equal(res.dendrogram.merges, ref.dendrogram.merges)
          and np.array_equal(res.labels.labels, ref.labels.labels)
          and np.array_equal(res.tree.src, ref.tree.src) and np.array_equal(res.tree.weight, ref.tree.weight)
          and res.connect_iters == ref.connect_iters)
    print("DIST_OK" if ok else "DIST_MISMATCH", res.connect_iters, flush=True)
dist.destroy_process_group()
