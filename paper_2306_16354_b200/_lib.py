"""ctypes binding of libslink.so (include/slink.h) and device plumbing.

The CUDA library is the only compute path: there is no CPU fallback.  If the
shared library is missing it is built from ``csrc/`` with nvcc; if no CUDA
device is present every compute entry point raises ``LinkageError``.
PyTorch only provides device memory and the current stream.
"""

from __future__ import annotations

import ctypes
import os
import threading
import warnings

import numpy as np

from . import build as _build
from .core import ConvergenceError, LinkageError, ValidationError

OK, INTERNAL, INVALID, CONVERGENCE, CUDA = 0, 1, 2, 3, 4

_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)
_PI = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); must match include/slink.h
SIGNATURES = {
    "slk_version": (_I, []),
    "slk_last_error": (ctypes.c_char_p, []),
    "slk_kernel_launches": (_I64, []),
    "slk_last_scan_stats": (_I, [_PI64]),
    "slk_profile": (_I, [_PD, _I]),
    "slk_knn": (_I, [_P, _P, _I64, _I, _I, _I64, _I64, _P, _P, _P]),
    "slk_nn1": (_I, [_P, _P, _I64, _P, _P, _I64, _I, _I, _P, _P, _P, _I64, _I64, _P, _P, _P]),
    "slk_pairwise_l2": (_I, [_P, _I64, _P, _I64, _I, _I, _P, _P]),
    "slk_row_norms": (_I, [_P, _P, _I64, _I, _P, _P]),
    "slk_edge_list_to_csr": (_I, [_I64, _P, _P, _P, _I64, _P, _P, _P, _PI64, _P]),
    "slk_csr_is_symmetric": (_I, [_I64, _P, _P, _P, _PI, _P]),
    "slk_weight_alteration": (_I, [_I64, _P, _P, _P, _I64, _P, _PD, _P]),
    "slk_min_edge_per_vertex": (_I, [_I64, _P, _P, _P, _P, _P, _P]),
    "slk_min_edge_per_supervertex": (_I, [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _PI64, _P]),
    "slk_label_propagation": (_I, [_I64, _P, _P, _P, _I64, _P]),
    "slk_solve_mst": (_I, [_I64, _P, _P, _P, _I, _I64, _P, _P, _P, _P, _PI64, _PI64, _P]),
    "slk_build_dendrogram": (_I, [_P, _P, _P, _I64, _P, _P]),
    "slk_extract_clusters": (_I, [_P, _I64, _I64, _P]),
    "slk_single_linkage": (_I, [_P, _P, _I64, _I, _I, _I64, _I, _I64, _I64, _I, _P, _P, _P, _P, _P,
                                _PI64, _P]),
    "slk_single_linkage_device": (_I, [_P, _P, _I64, _I, _I, _I64, _I, _I64, _I64, _I, _P, _P, _P,
                                       _P, _P, _PI64, _P, _P]),
    "slk_msf_edges": (_I, [_I64, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _PI64, _PI64, _P]),
    "slk_pointset_create": (_I, [_P, _P, _I64, _I, ctypes.POINTER(ctypes.c_void_p), _P]),
    "slk_pointset_destroy": (_I, [_P]),
    "slk_knn_ps": (_I, [_P, _I, _I64, _I64, _P, _P, _P]),
    "slk_nn1_colour_ps": (_I, [_P, _P, _I64, _I64, _P, _P, _P]),
    "slk_finish_tree": (_I, [_P, _P, _P, _I64, _I, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "slk_debug_tc_scan": (_I, [_P, _I64, _I, _I, _P, _P, _P, ctypes.POINTER(ctypes.c_float), _P]),
}


def load():
    """Load (building if needed) libslink.so and declare its signatures."""
    global _lib
    with _lock:
        if _lib is None:
            # SLK_LIB_VARIANT=timeline: a diagnostic build (build.py VARIANTS)
            variant = os.environ.get("SLK_LIB_VARIANT") or None
            path = _build.build(variant=variant)
            lib = ctypes.CDLL(str(path))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int) -> None:
    """Raise the reference's exception class for a non-zero status."""
    if status == OK:
        return
    msg = load().slk_last_error().decode(errors="replace")
    if status == INVALID:
        raise ValidationError(msg)
    if status == CONVERGENCE:
        raise ConvergenceError(msg)
    raise LinkageError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


# ------------------------------------------------------------ device plumbing
def torch_cuda():
    """The torch module, after asserting a CUDA device exists (no fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise LinkageError(
            "paper_2306_16354_b200 computes on a CUDA device (sm_100a); none is available "
            "and there is no CPU fallback"
        )
    return torch


def device():
    torch = torch_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    torch = torch_cuda()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def to_device(arr: np.ndarray, dtype):
    """Host array → contiguous device tensor of the given numpy dtype."""
    torch = torch_cuda()
    a = np.ascontiguousarray(arr, dtype=dtype)
    with warnings.catch_warnings():
        # read-only host arrays are fine: the tensor is only read, by the copy below
        warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
        return torch.from_numpy(a).to(device(), non_blocking=False)


def empty(shape, dtype):
    torch = torch_cuda()
    tdt = {np.float32: torch.float32, np.float64: torch.float64, np.int32: torch.int32,
           np.int64: torch.int64, np.uint8: torch.uint8}[np.dtype(dtype).type]
    return torch.empty(shape, dtype=tdt, device=device())


def to_host(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def ids_to_device(ids: np.ndarray):
    """int64 ids → int32 device tensor (ids are < 2^31 on the device)."""
    ids = np.asarray(ids)
    if ids.size and (ids.min() < np.iinfo(np.int32).min or ids.max() > np.iinfo(np.int32).max):
        raise ValidationError("vertex ids must fit in int32 on the device")
    return to_device(ids, np.int32)


def scan_stats() -> dict:
    buf = (ctypes.c_int64 * 5)()
    load().slk_last_scan_stats(buf)
    return dict(rows_refined=buf[0], rows_rescanned=buf[1], tiles_computed=buf[2],
                tiles_skipped=buf[3], rows_uncertified=buf[4])


def profile(reset: bool = False) -> dict:
    """Cumulative scan-kernel profile (CUDA-event timed inside the library)."""
    buf = (ctypes.c_double * 16)()
    load().slk_profile(buf, int(reset))
    keys = ("scan_ms", "scan_launches", "scan_flops", "scan_tiles", "refine_ms", "rescan_rows",
            "order_ms", "scan_flops_done", "scan_tiles_total", "tc_ms", "tc_flops_done",
            "tc_uncertified", "mst_ms", "mst_bytes", "mst_rounds", "msf_ms")
    return dict(zip(keys, list(buf)))


def kernel_launches() -> int:
    return int(load().slk_kernel_launches())
