"""ctypes mirror of the C-ABI in include/mlsk.h (layouts and constants only).

The shared library itself is located and loaded by :mod:`._lib`; this module
holds nothing but the ABI description so that the test-side oracle bindings
can describe the same structs without importing the product's loader.
"""
import ctypes as C

VERSION = "mlsk-b200 0.1.0"

OK, EINVAL, ERUNTIME = 0, 1, 3

MODEL_CONSTANT_ONES = 1
MODEL_DETERMINISTIC = 2
MODEL_PAPER_INNER = 3
MODEL_PAPER_MATRIX = 4
MODEL_GAUSS_MEAN = 5
MODEL_RFF = 6
MODEL_STUDENT_T = 7

F64, F32 = 0, 1
STREAM_PHILOX, STREAM_REF = 0, 1
TARGET_IDENTITY, TARGET_F1, TARGET_F2 = 0, 1, 2
ENGINE_AUTO, ENGINE_EXACT, ENGINE_FUSED = 0, 1, 2

TAG_MC = 0xFFFFFFFF


class ModelDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dtype", C.c_int32),
        ("stream_mode", C.c_int32),
        ("reserved0", C.c_int32),
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("p", C.c_int64),
        ("data_seed", C.c_uint64),
        ("sd", C.c_double),
        ("mean_lo", C.c_double),
        ("mean_hi", C.c_double),
        ("nu", C.c_double),
        ("sigma", C.c_double),
        ("rff_dim", C.c_int64),
        ("mean_a", C.c_void_p),
        ("mean_b", C.c_void_p),
    ]


class Plan(C.Structure):
    _fields_ = [
        ("M", C.c_int64),
        ("c0", C.c_int64),
        ("L", C.c_int64),
        ("N", C.POINTER(C.c_int64)),
    ]


class ExecOpts(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("engine", C.c_int32),
        ("stream", C.c_void_p),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("probe_k", C.c_int64),
        ("probe_out", C.POINTER(C.c_uint32)),
        ("n_devices", C.c_int32),
        ("device_ids", C.POINTER(C.c_int32)),
        ("deterministic", C.c_int32),
        ("vshards", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("value", C.POINTER(C.c_double)),
        ("level_estimate", C.POINTER(C.c_double)),
        ("level_sum", C.POINTER(C.c_double)),
        ("level_sumsq", C.POINTER(C.c_double)),
        ("level_mean_sq", C.POINTER(C.c_double)),
        ("level_count", C.POINTER(C.c_int64)),
        ("cost_units", C.POINTER(C.c_int64)),
        ("total_cost_units", C.c_int64),
        ("wall_time_s", C.c_double),
        ("seed", C.c_uint64),
    ]
