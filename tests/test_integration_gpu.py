"""the ctypes stub a reference maintainer would add, executed
verbatim (only its relative imports are pointed at this package, whose
dataclasses and error classes carry the reference's names and fields)."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _stub_source():
    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n(# parlink/_b200\.py.*?)```", text, re.S).group(1)
    lib = ROOT / "paper_2306_16354_b200" / "lib" / "libslink.so"
    return (block.replace("from .core import", "from paper_2306_16354_b200 import")
                 .replace("from .linkage import", "from paper_2306_16354_b200 import")
                 .replace('ctypes.CDLL("libslink.so")', f'ctypes.CDLL("{lib}")'))


def test_stub_signature_matches_the_library_binding():
    """CPU: the documented argtypes are the ones the package binds."""
    from paper_2306_16354_b200 import _lib

    src = _stub_source()
    documented = re.search(r"slk_single_linkage\.argtypes = \[(.*?)\]\n", src, re.S).group(1)
    n_doc = len([a for a in documented.replace("\n", " ").split(",") if a.strip()])
    assert n_doc == len(_lib.SIGNATURES["slk_single_linkage"][1])


@pytest.mark.gpu
@pytest.mark.parametrize("n_gpus", [1, 2])
def test_stub_runs_and_matches_the_package(n_gpus):
    import paper_2306_16354_b200 as slk
    from paper_2306_16354_b200.synthetic import make_blobs

    _ = slk._lib.torch_cuda()  # a CUDA context on the current device
    ns = {}
    exec(compile(_stub_source(), "INTEGRATION.md#stub", "exec"), ns)
    x = make_blobs(np.random.default_rng(3), 6000, 32, 12)  # float64, not float32-exact
    cfg = slk.LinkageConfig(n_clusters=12, k=6, seed=4)
    dendro, labels = ns["single_linkage_b200"](x, cfg, n_gpus=n_gpus)
    d_ref, l_ref = slk.single_linkage(x, cfg)
    assert np.array_equal(dendro.merges, d_ref.merges)
    assert np.array_equal(labels.labels, l_ref.labels)
    with pytest.raises(slk.ValidationError):
        ns["single_linkage_b200"](x[:5], slk.LinkageConfig(n_clusters=2, k=9))
