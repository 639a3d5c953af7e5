"""ctypes binding of libgzb200.so (include/gz_b200.h).

The CUDA library is the only compute path of this package: when it is missing
or no CUDA device is visible, every engine call raises EngineUnavailable --
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GZ_LIB") or os.path.join(HERE, "libgzb200.so")   # GZ_LIB: alternate build (experiments)

GZ_OK, GZ_ERR_GUARD, GZ_ERR_INVALID, GZ_ERR_CUDA, GZ_ERR_EXHAUSTED = 0, 1, 2, 3, 4
ALG = {"polar": 0, "ziggurat": 1, "modified-ziggurat": 2}
SRC = {"lcg48": 0, "splitmix": 1}
SEED = {"lcg_master_plus_id": 0, "sm_output_of_master": 1, "sm_id_xor_master": 2, "sm_master_plus_id": 3}
DEFAULT_GUARD = 1_000_000

EXPORTS = ("gz_version", "gz_last_error", "gz_device_count", "gz_set_kernel_policy", "gz_set_device", "gz_tables_upload",
           "gz_fill_gaussians", "gz_fill_gaussians_host", "gz_fill_u64", "gz_seed_streams",
           "gz_fill_unit_affine", "gz_mutate", "gz_moments_reduce", "gz_xor_reduce", "gz_stream_check",
           "gz_host_alloc", "gz_host_free", "gz_build_tables", "gz_hist_edges", "gz_ks_stat", "gz_lowbits_hist", "gz_libm_eval_device", "gz_libm_exp",
           "gz_libm_log", "gz_moments_buffer", "gz_zig_occupancy",
           "gz_wedge_filter_error", "gz_polar_ops_selftest", "gz_tail_sample", "gz_fill_scripted",
           "gz_tail_scripted")


class EngineUnavailable(RuntimeError):
    """The CUDA engine (libgzb200.so + a CUDA device) is not available."""


class RejectionLoopExceeded(RuntimeError):
    """A rejection loop ran LOOP_GUARD times without accepting (samplers.py:32-33)."""


_lib = None
_lock = threading.Lock()


def load(require_device: bool = True):
    """Load the library (raising EngineUnavailable if absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise EngineUnavailable(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                    " or `make -C paper_2405_19493_b200/csrc`")
            L = ctypes.CDLL(LIB_PATH)
            P, i64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
            L.gz_version.restype = I
            L.gz_last_error.restype = ctypes.c_char_p
            L.gz_device_count.restype = I
            L.gz_set_device.argtypes = [I]
            L.gz_set_kernel_policy.argtypes = [I]
            L.gz_tables_upload.argtypes = [I, I, P, P, P, D]
            L.gz_fill_gaussians.argtypes = [I, I, I, i64, i64, i64, P, P, P, P, P, P, P, P, P, i64, P]
            L.gz_fill_gaussians_host.argtypes = [I, I, I, i64, i64, P, P, P, P, P, P, P, P, i64]
            L.gz_fill_u64.argtypes = [I, i64, i64, i64, P, P, P, P]
            L.gz_seed_streams.argtypes = [I, ctypes.c_uint64, i64, i64, P, P]
            L.gz_fill_unit_affine.argtypes = [I, P, i64, D, D, P, P]
            L.gz_mutate.argtypes = [I, i64, i64, i64, P, P, P, P, I, i64, P]
            L.gz_moments_reduce.argtypes = [P, i64, i64, P, P]
            L.gz_xor_reduce.argtypes = [P, i64, P, P]
            L.gz_stream_check.argtypes = [P]
            L.gz_host_alloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), i64]
            L.gz_host_free.argtypes = [P]
            L.gz_build_tables.argtypes = [I, P, P, P, P, P, P]
            L.gz_libm_eval_device.argtypes = [I, P, P, i64, P]
            L.gz_hist_edges.argtypes = [P, i64, P, I, P, P]
            L.gz_ks_stat.argtypes = [P, i64, P, P]
            L.gz_lowbits_hist.argtypes = [P, i64, I, P, P]
            L.gz_moments_buffer.argtypes = [P, i64, P, P]
            L.gz_zig_occupancy.argtypes = [I, I, I, P, P, i64, P, P, i64, P]
            L.gz_wedge_filter_error.argtypes = [I, i64, ctypes.c_uint64, P, P]
            L.gz_polar_ops_selftest.argtypes = [i64, ctypes.c_uint64, P, P]
            L.gz_tail_sample.argtypes = [I, P, D, i64, P, P]
            L.gz_fill_scripted.argtypes = [I, I, P, i64, P, i64, P, P, P, P, P, i64, P]
            L.gz_tail_scripted.argtypes = [P, i64, P, D, i64, P, P]
            L.gz_libm_exp.argtypes = [D]
            L.gz_libm_exp.restype = D
            L.gz_libm_log.argtypes = [D]
            L.gz_libm_log.restype = D
            _lib = L
    if require_device and _lib.gz_device_count() < 1:
        raise EngineUnavailable("no CUDA device visible: the B200 engine has no CPU fallback")
    return _lib


def check(status: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == GZ_OK:
        return
    msg = _lib.gz_last_error().decode() if _lib is not None else "error"
    if status == GZ_ERR_GUARD:
        raise RejectionLoopExceeded(msg)
    if status == GZ_ERR_INVALID:
        raise ValueError(msg)
    if status == GZ_ERR_EXHAUSTED:
        from .sources import ScriptExhausted

        raise ScriptExhausted(msg)
    raise RuntimeError(f"CUDA error: {msg}")
