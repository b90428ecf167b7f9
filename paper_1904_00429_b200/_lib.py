"""Loader of the in-tree CUDA library (paper_1904_00429_b200/_lib/libmlsk.so).

There is deliberately no fallback: if the shared library is missing or cannot
be loaded, importing the product API raises immediately.  `build()` in
__graft_entry__.py (or `python -m paper_1904_00429_b200.build`) produces it.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _abi as abi

# MLSK_LIB_PATH: an alternative build of the same library (A/B experiments, tools/build_variant.py)
LIB_PATH = os.environ.get("MLSK_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                          "libmlsk.so")

_P = C.POINTER
_lib = None


class MlskRuntimeError(RuntimeError):
    """CUDA / runtime failure inside the library (status MLSK_ERUNTIME)."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    est = [_P(abi.ModelDesc), C.c_int32, C.c_double, _P(abi.Plan), C.c_uint64, _P(abi.ExecOpts),
           _P(abi.Report)]
    L.mlsk_mlmc_inner.argtypes = est
    L.mlsk_mlmc_matmul.argtypes = est
    mc = [_P(abi.ModelDesc), C.c_int32, C.c_double, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
          C.c_uint64, _P(abi.ExecOpts), _P(abi.Report)]
    L.mlsk_mc_inner.argtypes = mc
    L.mlsk_mc_matmul.argtypes = mc
    ref = [_P(abi.ModelDesc), C.c_int32, C.c_double, C.c_int64, C.c_uint64, _P(abi.ExecOpts), _P(C.c_double),
           _P(C.c_double)]
    L.mlsk_reference_inner.argtypes = ref
    L.mlsk_reference_matmul.argtypes = ref
    L.mlsk_session_create.argtypes = [_P(abi.ModelDesc), C.c_int32, C.c_double, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_uint64, _P(abi.ExecOpts), _P(C.c_void_p)]
    L.mlsk_session_run_round.argtypes = [C.c_void_p, _P(C.c_int64)]
    L.mlsk_session_stats.argtypes = [C.c_void_p, _P(abi.Report)]
    L.mlsk_session_level_buffer.argtypes = [C.c_void_p, _P(C.c_void_p), _P(C.c_int64)]
    L.mlsk_session_checkpoint.argtypes = [C.c_void_p, C.c_void_p, _P(C.c_int64)]
    L.mlsk_session_restore.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    L.mlsk_session_synchronize.argtypes = [C.c_void_p]
    L.mlsk_session_destroy.argtypes = [C.c_void_p]
    L.mlsk_sketch_inner.argtypes = [_P(C.c_double), _P(C.c_double), C.c_int64, _P(C.c_uint32),
                                    C.c_int64, _P(C.c_double), _P(C.c_double)]
    L.mlsk_sketch_matmul.argtypes = [_P(C.c_double), _P(C.c_double), C.c_int64, C.c_int64, C.c_int64,
                                     _P(C.c_uint32), C.c_int64, _P(C.c_double), _P(C.c_double)]
    L.mlsk_draw_sample.argtypes = [_P(abi.ModelDesc), C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                                   _P(C.c_uint32), _P(C.c_double), _P(C.c_double)]
    L.mlsk_model_data.argtypes = [_P(abi.ModelDesc), C.c_int32, C.c_void_p, _P(C.c_int64)]
    L.mlsk_derive_seed.restype = C.c_uint64
    L.mlsk_derive_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    L.mlsk_last_error.restype = C.c_char_p
    L.mlsk_version.restype = C.c_char_p
    L.mlsk_device_count.restype = C.c_int
    L.mlsk_kernel_launch_count.restype = C.c_int64
    L.mlsk_contraction_columns.argtypes = [_P(C.c_int64), C.c_int]
    L.mlsk_profile_enable.argtypes = [C.c_int]
    L.mlsk_profile_read.argtypes = [C.c_int, C.c_char_p, C.c_int, _P(C.c_int64), _P(C.c_double)]
    L.mlsk_profile_timeline.argtypes = [C.c_int, C.c_char_p, C.c_int, _P(C.c_double), _P(C.c_double)]
    L.mlsk_measure_fp64_peak.restype = C.c_double
    L.mlsk_measure_fp64_peak.argtypes = [C.c_int]
    L.mlsk_measure_tf32_peak.restype = C.c_double
    L.mlsk_measure_tf32_peak.argtypes = [C.c_int, C.c_int]
    L.mlsk_measure_index_rate.restype = C.c_double
    L.mlsk_measure_index_rate.argtypes = [C.c_int]
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a status code to the reference's exception classes."""
    if rc == abi.OK:
        return
    msg = lib().mlsk_last_error().decode()
    if rc == abi.EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    raise MlskRuntimeError(msg)
