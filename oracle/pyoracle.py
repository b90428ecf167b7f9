"""ctypes bindings of the CPU oracle (oracle/_build) and of the reference
harness compiled from /root/reference (oracle/_ref).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_1904_00429_b200 import _abi as abi

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmlsk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmlsk_ref.so")
REF_TREE = "/root/reference/proj"

_P = C.POINTER
_u32p = _P(C.c_uint32)
_u64p = _P(C.c_uint64)
_i64p = _P(C.c_int64)
_f64p = _P(C.c_double)


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference harness when the tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_TREE):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64] * 3
        L.orc_mt64_stream.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.orc_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.orc_log_unit.restype = C.c_double
        L.orc_log_unit.argtypes = [C.c_double]
        L.orc_sincos_turn.argtypes = [C.c_double, _f64p, _f64p]
        L.orc_box_muller.argtypes = [C.c_uint64, C.c_uint64, _f64p, _f64p]
        L.orc_box_muller_f.argtypes = [C.c_uint32, C.c_uint32, _P(C.c_float), _P(C.c_float)]
        L.orc_uniform_cumulative.argtypes = [C.c_int64, _f64p]
        L.orc_index_from_u64.restype = C.c_uint32
        L.orc_index_from_u64.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.orc_sketch_inner.argtypes = [_f64p, _f64p, C.c_int64, _u32p, C.c_int64, _f64p, _f64p]
        L.orc_sketch_matmul.argtypes = [_f64p, _f64p, C.c_int64, C.c_int64, C.c_int64, _u32p,
                                        C.c_int64, _f64p, _f64p]
        L.orc_model_create.argtypes = [_P(abi.ModelDesc), _P(C.c_void_p)]
        L.orc_model_destroy.argtypes = [C.c_void_p]
        L.orc_model_mean_a.restype = _f64p
        L.orc_model_mean_a.argtypes = [C.c_void_p]
        L.orc_model_mean_b.restype = _f64p
        L.orc_model_mean_b.argtypes = [C.c_void_p]
        L.orc_draw_sample.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                                      _u32p, _f64p, _f64p]
        L.orc_mlmc.argtypes = [C.c_void_p, C.c_int32, C.c_double, _P(abi.Plan), C.c_uint64,
                               C.c_int, _P(abi.Report)]
        L.orc_mc.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_int64, C.c_int64, C.c_int64,
                             C.c_int64, C.c_uint64, C.c_int, _P(abi.Report)]
        L.orc_sample_y_subset.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                                          C.c_int64, C.c_int32, C.c_double, _i64p, C.c_int64,
                                          _i64p, C.c_int64, _f64p]
        L.orc_last_error.restype = C.c_char_p
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_TREE)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        L = C.CDLL(REF_SO)
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64] * 3
        L.ref_u64_stream.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.ref_normals.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.ref_indices.argtypes = [C.c_uint64, C.c_int64, C.c_int64, _u32p]
        L.ref_sketch_inner.argtypes = [_f64p, _f64p, C.c_int64, _u32p, C.c_int64, _f64p]
        L.ref_sketch_matmul.argtypes = [_f64p, _f64p, C.c_int64, C.c_int64, C.c_int64, _u32p,
                                        C.c_int64, _f64p]
        L.ref_draw_sample.argtypes = [_P(abi.ModelDesc), C.c_uint64, C.c_uint64, C.c_int64,
                                      C.c_int64, _u32p, _f64p, _f64p]
        for f in (L.ref_mlmc, L.ref_mlmc_native):
            f.argtypes = [_P(abi.ModelDesc), C.c_int32, C.c_double, _P(abi.Plan), C.c_uint64,
                          C.c_int32, _P(abi.Report)]
        L.ref_mc_native.argtypes = [_P(abi.ModelDesc), C.c_int32, C.c_double, C.c_int64, C.c_int64,
                                    C.c_int64, C.c_uint64, C.c_int32, _P(abi.Report)]
        L.ref_throughput.restype = C.c_double
        L.ref_throughput.argtypes = [_P(abi.ModelDesc), C.c_int32, C.c_double, _P(abi.Plan), C.c_uint64,
                                     C.c_int32, _f64p]
        L.ref_time_sketch_matmul.restype = C.c_double
        L.ref_time_sketch_matmul.argtypes = [C.c_int64] * 4 + [C.c_uint64, C.c_int32]
        L.ref_reference_value.argtypes = [_P(abi.ModelDesc), C.c_int32, C.c_double, C.c_int64, C.c_uint64,
                                          C.c_int32, _f64p, _f64p]
        L.ref_make_plan.argtypes = [C.c_double, C.c_int64, C.c_double, C.c_double, C.c_int64, _i64p, _i64p,
                                    C.c_int64, _P(C.c_int32), _i64p]
        L.ref_sweep_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, _i64p, C.c_int32, C.c_double, C.c_double,
                                    C.c_double, C.c_uint64, C.c_int32, C.c_int64, C.c_int32, C.c_char_p,
                                    C.c_int64]
        L.ref_estimate_text.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int64, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.c_int32, C.c_char_p, C.c_int64]
        L.ref_last_error.restype = C.c_char_p
        _ref = L
    return _ref


# ------------------------------------------------------------------ helpers


@dataclass
class Result:
    """Numpy view of an mlsk_report."""

    value: np.ndarray
    level_estimate: np.ndarray
    level_sum: np.ndarray
    level_sumsq: np.ndarray
    level_mean_sq: np.ndarray
    level_count: np.ndarray
    cost_units: np.ndarray
    total_cost_units: int
    seed: int


class ReportBuffers:
    def __init__(self, levels: int, cells: int):
        self.value = np.zeros(cells)
        self.level_estimate = np.zeros((levels, cells))
        self.level_sum = np.zeros((levels, cells))
        self.level_sumsq = np.zeros(levels)
        self.level_mean_sq = np.zeros(levels)
        self.level_count = np.zeros(levels, dtype=np.int64)
        self.cost_units = np.zeros(levels, dtype=np.int64)
        self.c = abi.Report(
            _ptr(self.value, _f64p), _ptr(self.level_estimate, _f64p), _ptr(self.level_sum, _f64p),
            _ptr(self.level_sumsq, _f64p), _ptr(self.level_mean_sq, _f64p),
            _ptr(self.level_count, _i64p), _ptr(self.cost_units, _i64p), 0, 0.0, 0)

    def result(self) -> Result:
        return Result(self.value.copy(), self.level_estimate.copy(), self.level_sum.copy(),
                      self.level_sumsq.copy(), self.level_mean_sq.copy(), self.level_count.copy(),
                      self.cost_units.copy(), int(self.c.total_cost_units), int(self.c.seed))


def model_desc(kind, n, m=0, p=0, dtype=abi.F64, stream=abi.STREAM_PHILOX, data_seed=0, sd=1.0,
               mean_lo=0.0, mean_hi=1.0, nu=3.0, sigma=4.0, rff_dim=0, mean_a=None, mean_b=None):
    d = abi.ModelDesc()
    d.kind, d.dtype, d.stream_mode = kind, dtype, stream
    d.m, d.n, d.p = m, n, p
    d.data_seed, d.sd, d.mean_lo, d.mean_hi, d.nu, d.sigma, d.rff_dim = (
        data_seed, sd, mean_lo, mean_hi, nu, sigma, rff_dim)
    d._keep = (mean_a, mean_b)
    d.mean_a = mean_a.ctypes.data if mean_a is not None else None
    d.mean_b = mean_b.ctypes.data if mean_b is not None else None
    return d


def is_vector(d) -> bool:
    return d.kind == abi.MODEL_PAPER_INNER or (
        d.kind in (abi.MODEL_CONSTANT_ONES, abi.MODEL_DETERMINISTIC, abi.MODEL_GAUSS_MEAN)
        and d.m == 0 and d.p == 0)


def out_shape(d):
    if is_vector(d):
        return 1, 1
    if d.kind == abi.MODEL_PAPER_MATRIX:
        return 10, 10
    if d.kind == abi.MODEL_DETERMINISTIC:
        return 2, 2
    if d.kind == abi.MODEL_RFF:
        return d.m, d.m
    return d.m, d.p


def make_plan(M, c0, N):
    arr = np.ascontiguousarray(N, dtype=np.int64)
    pl = abi.Plan(M, c0, len(arr) - 1, _ptr(arr, _i64p))
    pl._keep = arr
    return pl


class OracleModel:
    """An orc_model plus convenience wrappers."""

    def __init__(self, desc):
        self.L = oracle_lib()
        self.desc = desc
        h = C.c_void_p()
        rc = self.L.orc_model_create(C.byref(desc), C.byref(h))
        if rc:
            raise ValueError(self.L.orc_last_error().decode())
        self.h = h
        self.rows, self.cols = out_shape(desc)

    def __del__(self):
        try:
            self.L.orc_model_destroy(self.h)
        except Exception:
            pass

    def means(self):
        d = self.desc
        if is_vector(d):
            na = nb = d.n
        elif d.kind == abi.MODEL_RFF:
            na, nb = d.m * d.rff_dim, d.rff_dim * d.n
        else:
            na, nb = d.m * d.n, d.n * d.p
        a = np.ctypeslib.as_array(self.L.orc_model_mean_a(self.h), (na,)).copy()
        b = np.ctypeslib.as_array(self.L.orc_model_mean_b(self.h), (nb,)).copy()
        return a, b

    def draw(self, seed, tag, k, c):
        idx = np.zeros(c, dtype=np.uint32)
        a = np.zeros((self.rows, c))
        b = np.zeros((c, self.cols))
        rc = self.L.orc_draw_sample(self.h, seed, tag, k, c, _ptr(idx, _u32p), _ptr(a, _f64p),
                                    _ptr(b, _f64p))
        if rc:
            raise ValueError(self.L.orc_last_error().decode())
        return idx, a, b

    def mlmc(self, M, c0, N, seed, target=abi.TARGET_IDENTITY, tp=1e-12):
        plan = make_plan(M, c0, N)
        rb = ReportBuffers(len(N), self.rows * self.cols)
        rc = self.L.orc_mlmc(self.h, target, tp, C.byref(plan), seed, int(not is_vector(self.desc)),
                             C.byref(rb.c))
        if rc:
            raise ValueError(self.L.orc_last_error().decode())
        return rb.result()

    def mc(self, L, N, M, c0, seed, target=abi.TARGET_IDENTITY, tp=1e-12):
        rb = ReportBuffers(1, self.rows * self.cols)
        rc = self.L.orc_mc(self.h, target, tp, L, N, M, c0, seed, int(not is_vector(self.desc)),
                           C.byref(rb.c))
        if rc:
            raise ValueError(self.L.orc_last_error().decode())
        return rb.result()

    def y_subset(self, seed, tag, k, c, coarse, rows, cols, target=abi.TARGET_IDENTITY, tp=1e-12):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        y = np.zeros((len(rows), len(cols)))
        rc = self.L.orc_sample_y_subset(self.h, seed, tag, k, c, coarse, target, tp,
                                        _ptr(rows, _i64p), len(rows), _ptr(cols, _i64p), len(cols),
                                        _ptr(y, _f64p))
        if rc:
            raise ValueError(self.L.orc_last_error().decode())
        return y


def philox(ctr, key):
    L = oracle_lib()
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    L.orc_philox4x32_10(_ptr(c, _u32p), _ptr(k, _u32p), _ptr(o, _u32p))
    return o


def mt64_stream(seed, count):
    out = np.zeros(count, dtype=np.uint64)
    oracle_lib().orc_mt64_stream(seed, count, _ptr(out, _u64p))
    return out


def ref_mlmc(desc, M, c0, N, seed, target=abi.TARGET_IDENTITY, tp=1e-12, threads=1, native=False):
    L = ref_lib()
    rows, cols = out_shape(desc)
    plan = make_plan(M, c0, N)
    rb = ReportBuffers(len(N), rows * cols)
    f = L.ref_mlmc_native if native else L.ref_mlmc
    rc = f(C.byref(desc), target, tp, C.byref(plan), seed, threads, C.byref(rb.c))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return rb.result()


def ref_mc(desc, L_, N, M, seed, target=abi.TARGET_IDENTITY, tp=1e-12, threads=1):
    L = ref_lib()
    rows, cols = out_shape(desc)
    rb = ReportBuffers(1, rows * cols)
    rc = L.ref_mc_native(C.byref(desc), target, tp, L_, N, M, seed, threads, C.byref(rb.c))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return rb.result()


def ref_draw(desc, seed, tag, k, c):
    L = ref_lib()
    rows, cols = out_shape(desc)
    idx = np.zeros(c, dtype=np.uint32)
    a = np.zeros((rows, c))
    b = np.zeros((c, cols))
    rc = L.ref_draw_sample(C.byref(desc), seed, tag, k, c, _ptr(idx, _u32p), _ptr(a, _f64p),
                           _ptr(b, _f64p))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return idx, a, b


def ref_reference_value(desc, count, seed, target=abi.TARGET_IDENTITY, tp=1e-12, threads=1):
    """reference_inner / reference_matmul of the compiled reference: (mean, se)."""
    L = ref_lib()
    rows, cols = out_shape(desc)
    mean = np.zeros(rows * cols)
    se = np.zeros(1)
    if L.ref_reference_value(C.byref(desc), target, tp, count, seed, threads, _ptr(mean, _f64p), _ptr(se, _f64p)):
        raise ValueError(L.ref_last_error().decode())
    return mean, float(se[0])


def ref_make_plan(eps, M, c1, c2, n):
    """make_plan + plan_N_mc of the compiled reference: (L, N list, n_cap_applied, N_mc)."""
    L = ref_lib()
    Lv = np.zeros(1, dtype=np.int64)
    N = np.zeros(256, dtype=np.int64)
    cap = C.c_int32(0)
    nmc = np.zeros(1, dtype=np.int64)
    if L.ref_make_plan(eps, M, c1, c2, n, _ptr(Lv, _i64p), _ptr(N, _i64p), 256, C.byref(cap), _ptr(nmc, _i64p)):
        raise ValueError(L.ref_last_error().decode())
    return int(Lv[0]), [int(x) for x in N[:int(Lv[0]) + 1]], bool(cap.value), int(nmc[0])


def _text(fn, *args):
    cap = 1 << 20
    while True:
        buf = C.create_string_buffer(cap)
        n = fn(*args, buf, cap)
        if n >= 0:
            return buf.value.decode()
        if n == -1:
            raise ValueError(ref_lib().ref_last_error().decode())
        cap = -n + 1


def ref_sweep_csv(mode, model, target, m_list, eps=0.1, c1=1.0, c2=1.0, seed=1, reps=1, n_ref=100000, threads=1):
    """The reference CLI's `sweep --no-timing` CSV (mlsketch_main.cpp:112-198)."""
    ml = np.ascontiguousarray(m_list, dtype=np.int64)
    return _text(ref_lib().ref_sweep_csv, mode.encode(), model.encode(), target.encode(), _ptr(ml, _i64p), len(ml),
                 eps, c1, c2, seed, reps, n_ref, threads)


def ref_estimate_text(mode, model, target, M=7, eps=0.1, c1=1.0, c2=1.0, seed=1, threads=1):
    """The reference CLI's `estimate` output (mlsketch_main.cpp:250-316), wall_time_s written as 0.000."""
    return _text(ref_lib().ref_estimate_text, mode.encode(), model.encode(), target.encode(), M, eps, c1, c2, seed,
                 threads)
