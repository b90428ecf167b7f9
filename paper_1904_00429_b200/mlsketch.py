"""Host-side mirror of the reference library's public interface (`mlsketch`,
/root/reference/proj/include/mlsketch) on top of the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference so that code
(and tests) written against it read the same:

    reference (C++)                          here (Python)
    ---------------------------------------  -------------------------------------
    RngStream::derive_seed  rng.hpp:31-37     RngStream.derive_seed
    VectorPairModel / MatrixPairModel         VectorPairModel / MatrixPairModel
      (std::function draw, models.hpp:17-31)    (device descriptors, no host lambdas)
    paper_inner_model ... models.cpp:12-97    same factory names
    target_identity / f1 / f2 models.cpp:99   same factory names
    LevelPlan  planner.hpp:12-20              LevelPlan (+ c0, default 1)
    EstimatorOptions estimators.hpp:45-50     EstimatorOptions (+ device, engine, rank, world)
    LevelStatistic / EstimateReport           LevelStatistic / EstimateReport
    mlmc_inner / mlmc_matmul / mc_inner /     same names (estimators.hpp:58-80)
      mc_matmul
    sketch_inner / sketch_matmul sketch.hpp   same names (device evaluation)
    std::invalid_argument                     ValueError
    (no reference analogue)                   MlmcSession: round API for adaptive MLMC

All computation runs in the CUDA library; a missing library raises on import.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi as abi
from ._lib import check, lib

_P = C.POINTER
_f64p = _P(C.c_double)
_i64p = _P(C.c_int64)
_u32p = _P(C.c_uint32)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


# ----------------------------------------------------------------- rng.hpp


class RngStream:
    """Only the seed-derivation part of rng.hpp is host-visible; the streams
    themselves live on the device (reference mt19937_64 or Philox4x32-10)."""

    @staticmethod
    def mix(z: int) -> int:  # rng.hpp:22-27
        z = (z + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    @staticmethod
    def derive_seed(master: int, a: int, b: int) -> int:  # rng.hpp:31-37 (== mlsk_derive_seed)
        mix, u = RngStream.mix, 0xFFFFFFFFFFFFFFFF
        return mix(mix(mix(master & u) ^ ((a + 0x9E3779B97F4A7C15) & u)) ^ ((b + 0xBF58476D1CE4E5B9) & u))


# ------------------------------------------------------------------ models


@dataclass
class _Model:
    kind: int
    n: int
    m: int = 0
    p: int = 0
    label: str = ""
    dtype: int = abi.F64
    stream: int = abi.STREAM_PHILOX
    data_seed: int = 0
    sd: float = 1.0
    mean_lo: float = 0.0
    mean_hi: float = 1.0
    nu: float = 3.0
    sigma: float = 4.0
    rff_dim: int = 0
    mean_a: Optional[np.ndarray] = None
    mean_b: Optional[np.ndarray] = None

    @property
    def d(self) -> int:  # the reference's name for p
        return self.p

    def desc(self) -> abi.ModelDesc:
        d = abi.ModelDesc()
        d.kind, d.dtype, d.stream_mode = self.kind, self.dtype, self.stream
        d.m, d.n, d.p = self.m, self.n, self.p
        d.data_seed, d.sd, d.mean_lo, d.mean_hi = self.data_seed, self.sd, self.mean_lo, self.mean_hi
        d.nu, d.sigma, d.rff_dim = self.nu, self.sigma, self.rff_dim
        dt = np.float32 if self.dtype == abi.F32 else np.float64
        keep = []
        for name in ("mean_a", "mean_b"):
            arr = getattr(self, name)
            if arr is not None:
                arr = np.ascontiguousarray(arr, dtype=dt)
                keep.append(arr)
                setattr(d, name, arr.ctypes.data)
        d._keep = keep
        return d

    def with_stream(self, stream: str | int):
        """Copy of the model on the 'ref' (mt19937_64) or 'philox' stream."""
        import copy
        c = copy.copy(self)
        c.stream = _stream_code(stream)
        return c


def _stream_code(s) -> int:
    if isinstance(s, int):
        return s
    return {"philox": abi.STREAM_PHILOX, "ref": abi.STREAM_REF, "reference": abi.STREAM_REF}[s]


class VectorPairModel(_Model):
    """Random vector pair (a, b) in R^n (models.hpp:17-21)."""


class MatrixPairModel(_Model):
    """Random matrix pair A (m x n), B (n x d) (models.hpp:23-31)."""


def paper_inner_model() -> VectorPairModel:  # models.cpp:12-27
    return VectorPairModel(abi.MODEL_PAPER_INNER, 1000, label="paper-inner", stream=abi.STREAM_REF)


def paper_matrix_model() -> MatrixPairModel:  # models.cpp:29-52
    return MatrixPairModel(abi.MODEL_PAPER_MATRIX, 1000, 10, 10, label="paper-matrix",
                           stream=abi.STREAM_REF)


def constant_ones_model(n: int, stream="ref") -> VectorPairModel:  # models.cpp:54-61
    if n <= 0:
        raise ValueError("constant_ones_model: n must be positive")
    return VectorPairModel(abi.MODEL_CONSTANT_ONES, n, label="constant-ones",
                           stream=_stream_code(stream))


def constant_ones_matrix_model(m: int, n: int, d: int, stream="ref") -> MatrixPairModel:
    if m <= 0 or n <= 0 or d <= 0:  # models.cpp:63-74
        raise ValueError("constant_ones_matrix_model: dimensions must be positive")
    return MatrixPairModel(abi.MODEL_CONSTANT_ONES, n, m, d, label="constant-ones",
                           stream=_stream_code(stream))


def deterministic_model(n: int, stream="ref") -> VectorPairModel:  # models.cpp:76-86
    if n <= 0:
        raise ValueError("deterministic_model: n must be positive")
    return VectorPairModel(abi.MODEL_DETERMINISTIC, n, label="deterministic",
                           stream=_stream_code(stream))


def deterministic_matrix_model(stream="ref") -> MatrixPairModel:  # models.cpp:88-97
    return MatrixPairModel(abi.MODEL_DETERMINISTIC, 2, 2, 2, label="deterministic",
                           stream=_stream_code(stream))


def gaussian_mean_model(n: int, sd: float = 1.0, mean_lo: float = 0.0, mean_hi: float = 1.0,
                        data_seed: int = 0, mean_a=None, mean_b=None, stream="philox",
                        dtype: int = abi.F64) -> VectorPairModel:
    """a_j = mu_j + sd N(0,1), b_j = nu_j + sd N(0,1), mu, nu ~ U(lo, hi) fixed from
    data_seed (BASELINE config 1) unless given explicitly."""
    return VectorPairModel(abi.MODEL_GAUSS_MEAN, n, label="gauss-mean", dtype=dtype,
                           stream=_stream_code(stream), data_seed=data_seed, sd=sd, mean_lo=mean_lo,
                           mean_hi=mean_hi, mean_a=mean_a, mean_b=mean_b)


def gaussian_mean_matrix_model(m: int, n: int, p: int, sd: float = 0.5, mean_lo: float = -1.0,
                               mean_hi: float = 1.0, data_seed: int = 0, mean_a=None, mean_b=None,
                               stream="philox", dtype: int = abi.F64) -> MatrixPairModel:
    """A = M + sd N(0,1), B = P + sd N(0,1), M, P ~ U(lo, hi) fixed from data_seed
    (BASELINE configs 2 (fp64) and 3 (fp32))."""
    return MatrixPairModel(abi.MODEL_GAUSS_MEAN, n, m, p, label="gauss-mean", dtype=dtype,
                           stream=_stream_code(stream), data_seed=data_seed, sd=sd,
                           mean_lo=mean_lo, mean_hi=mean_hi, mean_a=mean_a, mean_b=mean_b)


def student_t_matrix_model(m: int, n: int, p: int, nu: float = 3.0, mean_lo: float = -0.5,
                           mean_hi: float = 0.5, data_seed: int = 0) -> MatrixPairModel:
    """iid Student-t(nu) entries plus U(lo, hi) means (BASELINE config 5, fp32)."""
    return MatrixPairModel(abi.MODEL_STUDENT_T, n, m, p, label="student-t", dtype=abi.F32,
                           data_seed=data_seed, nu=nu, mean_lo=mean_lo, mean_hi=mean_hi)


def rff_gram_model(points: int, features: int, dim: int = 64, sigma: float = 4.0,
                   data_seed: int = 0) -> MatrixPairModel:
    """A = sqrt(2/n) cos(X W + b) (points x features), B = A^T: the sketched
    product estimates the random-feature Gram matrix (BASELINE config 4)."""
    return MatrixPairModel(abi.MODEL_RFF, features, points, points, label="rff", dtype=abi.F32,
                           data_seed=data_seed, sigma=sigma, rff_dim=dim)


def vector_model_by_key(key: str):  # models.cpp:119-124
    return {"paper-inner": paper_inner_model, "constant-ones": lambda: constant_ones_model(1000),
            "deterministic": lambda: deterministic_model(2)}.get(key, lambda: None)()


def matrix_model_by_key(key: str):  # models.cpp:126-131
    return {"paper-matrix": paper_matrix_model,
            "constant-ones": lambda: constant_ones_matrix_model(10, 1000, 10),
            "deterministic": deterministic_matrix_model}.get(key, lambda: None)()


# ----------------------------------------------------------------- targets


@dataclass
class TargetFunction:
    """models.hpp:35-39; evaluated on the device by kind."""

    kind: int
    lipschitz_constant: float
    label: str
    param: float = 1e-12

    def f(self, x):  # host evaluation, for convenience in tests
        x = np.asarray(x, dtype=np.float64)
        if self.kind == abi.TARGET_F1:
            return np.abs(x) * (x - 10.0 >= 0.0)
        if self.kind == abi.TARGET_F2:
            return x * x * np.sin(1.0 / (np.abs(x) + self.param))
        return x


def target_identity() -> TargetFunction:
    return TargetFunction(abi.TARGET_IDENTITY, 1.0, "identity")


def target_f1() -> TargetFunction:
    return TargetFunction(abi.TARGET_F1, 1.0, "f1")


def target_f2(zeta: float = 1e-12) -> TargetFunction:
    if not zeta > 0.0:
        raise ValueError("target_f2: zeta must be positive")
    return TargetFunction(abi.TARGET_F2, 1.0, "f2", zeta)


def target_by_key(key: str):
    return {"identity": target_identity, "f1": target_f1, "f2": target_f2}.get(key, lambda: None)()


# ------------------------------------------------------ plan / options / report


@dataclass
class LevelPlan:
    """planner.hpp:12-20 plus c0 (c_l = c0 M^l; the reference is c0 = 1)."""

    M: int
    L: int
    N: Sequence[int]
    epsilon: float = 0.0
    c1: float = 1.0
    c2: float = 1.0
    n_cap_applied: bool = False
    c0: int = 1

    def level_size(self, l: int) -> int:
        return self.c0 * self.M ** l

    def _c(self):
        if len(self.N) != self.L + 1:  # estimators.cpp:24-26
            raise ValueError("estimator: malformed plan")
        arr = np.ascontiguousarray(self.N, dtype=np.int64)
        pl = abi.Plan(self.M, self.c0, self.L, _ptr(arr, _i64p))
        pl._keep = arr
        return pl


CouplingProbe = Callable[[int, int, List[int], List[int]], None]


@dataclass
class EstimatorOptions:
    """estimators.hpp:45-50.  `threads` is accepted for source compatibility and
    ignored (the device runs all replications); a probe is called in
    (level, replication) order with the fine and coarse index sets of the
    first `probe_count` replications of every level >= 1."""

    threads: int = 1
    probe: Optional[CouplingProbe] = None
    probe_count: int = 64
    device: int = -1
    engine: str = "auto"
    rank: int = 0
    world: int = 1
    stream: Optional[int] = None
    # multi-GPU inside the library (mlsk_exec_opts.n_devices / device_ids):
    # one host thread per device slot, slot sums added in slot order
    devices: Optional[Sequence[int]] = None
    # fixed virtual shards: bit-identical results for any device count dividing vshards
    deterministic: bool = False
    vshards: int = 8

    def _c(self, probe_buf=None, probe_k=0):
        eng = {"auto": abi.ENGINE_AUTO, "exact": abi.ENGINE_EXACT, "fused": abi.ENGINE_FUSED}[self.engine]
        ids = None
        if self.devices is not None:
            self._ids = np.ascontiguousarray(self.devices, dtype=np.int32)  # kept alive with the options
            ids = self._ids.ctypes.data_as(C.POINTER(C.c_int32))
        return abi.ExecOpts(self.device, eng, self.stream, self.rank, self.world, probe_k,
                            _ptr(probe_buf, _u32p) if probe_buf is not None else None,
                            len(self.devices) if self.devices is not None else 0, ids,
                            1 if self.deterministic else 0, self.vshards)


class LevelStatistic:
    """estimators.hpp:20-27.  `estimate` = sum * (1 / replication_count), the
    library's own arithmetic, formed on first access (the per-level sums are
    what crosses the C-ABI; materialising every level's estimate matrix on
    every call would double the report's host memory traffic)."""

    __slots__ = ("level", "_estimate", "replication_count", "sample_mean_of_squares", "cost_units", "sum",
                 "sum_of_squares", "_scalar", "_divisor")

    def __init__(self, level, estimate, replication_count, sample_mean_of_squares, cost_units, sum=None,
                 sum_of_squares=0.0, scalar=False, divisor=None):
        self.level = level
        self._estimate = estimate
        self.replication_count = replication_count
        self.sample_mean_of_squares = sample_mean_of_squares
        self.cost_units = cost_units
        self.sum = sum
        self.sum_of_squares = sum_of_squares
        self._scalar = scalar
        # the plan's N_l for estimators (ranks hold partial sums of the global
        # level), the accumulated count for sessions
        self._divisor = replication_count if divisor is None else divisor

    @property
    def estimate(self):
        if self._estimate is None:
            inv = 1.0 / self._divisor if self._divisor > 0 else 0.0
            e = np.asarray(self.sum, dtype=np.float64) * inv
            self._estimate = float(e) if self._scalar else e
        return self._estimate

    def __repr__(self):
        return (f"LevelStatistic(level={self.level}, replication_count={self.replication_count}, "
                f"sample_mean_of_squares={self.sample_mean_of_squares}, cost_units={self.cost_units})")


@dataclass
class EstimateReport:
    value: object
    per_level: List[LevelStatistic] = field(default_factory=list)
    total_cost_units: int = 0
    wall_time_seconds: float = 0.0
    seed: int = 0


class _Buffers:
    def __init__(self, levels: int, cells: int):
        # every entry is written by the library (np.empty: no memset); the
        # per-level estimates are derived from the sums on access
        self.value = np.empty(cells)
        self.level_estimate = None
        self.level_sum = np.empty((levels, cells))
        self.level_sumsq = np.zeros(levels)
        self.level_mean_sq = np.zeros(levels)
        self.level_count = np.zeros(levels, dtype=np.int64)
        self.cost_units = np.zeros(levels, dtype=np.int64)
        self.c = abi.Report(_ptr(self.value, _f64p), None,
                            _ptr(self.level_sum, _f64p), _ptr(self.level_sumsq, _f64p),
                            _ptr(self.level_mean_sq, _f64p), _ptr(self.level_count, _i64p),
                            _ptr(self.cost_units, _i64p), 0, 0.0, 0)


def _shape(model) -> tuple:
    if isinstance(model, VectorPairModel):
        return (1, 1)
    if model.kind == abi.MODEL_DETERMINISTIC:
        return (2, 2)
    if model.kind == abi.MODEL_PAPER_MATRIX:
        return (10, 10)
    if model.kind == abi.MODEL_RFF:
        return (model.m, model.m)
    return (model.m, model.p)


def _report(buf: _Buffers, model, levels: int, vector: bool, with_levels=True, divisors=None) -> EstimateReport:
    rows, cols = _shape(model)
    conv = (lambda x: float(x[0])) if vector else (lambda x: x.reshape(rows, cols))  # views of per-call buffers
    per = []
    if with_levels:
        for l in range(levels):
            per.append(LevelStatistic(l, None, int(buf.level_count[l]), float(buf.level_mean_sq[l]),
                                      int(buf.cost_units[l]), conv(buf.level_sum[l]), float(buf.level_sumsq[l]),
                                      scalar=vector, divisor=None if divisors is None else int(divisors[l])))
    return EstimateReport(conv(buf.value), per, int(buf.c.total_cost_units),
                          float(buf.c.wall_time_s), int(buf.c.seed))


# -------------------------------------------------------------- estimators


def _mlmc(matrix: bool, model, f: TargetFunction, plan: LevelPlan, seed: int,
          options: Optional[EstimatorOptions]) -> EstimateReport:
    options = options or EstimatorOptions()
    if matrix != isinstance(model, MatrixPairModel):
        raise ValueError("estimator: model kind does not match the estimator")
    rows, cols = _shape(model)
    cpl = plan._c()
    buf = _Buffers(plan.L + 1, rows * cols)
    probe_buf, probe_k = None, 0
    if options.probe is not None:
        probe_k = int(min(options.probe_count, max(plan.N)))
        probe_buf = np.zeros((plan.L + 1, probe_k, plan.level_size(plan.L)), dtype=np.uint32)
    desc = model.desc()
    fn = lib().mlsk_mlmc_matmul if matrix else lib().mlsk_mlmc_inner
    check(fn(C.byref(desc), f.kind, f.param, C.byref(cpl), seed, C.byref(options._c(probe_buf, probe_k)),
             C.byref(buf.c)))
    if options.probe is not None:
        for l in range(1, plan.L + 1):
            c = plan.level_size(l)
            for k in range(min(probe_k, plan.N[l])):
                fine = [int(x) for x in probe_buf[l, k, :c]]
                options.probe(l, k, fine, fine[: c // plan.M])
    return _report(buf, model, plan.L + 1, not matrix, divisors=plan.N)


def mlmc_inner(model: VectorPairModel, f: TargetFunction, plan: LevelPlan, seed: int,
               options: Optional[EstimatorOptions] = None) -> EstimateReport:
    """Multilevel estimate of E[f(a^T b)] (estimators.hpp:52-60)."""
    return _mlmc(False, model, f, plan, seed, options)


def mlmc_matmul(model: MatrixPairModel, f: TargetFunction, plan: LevelPlan, seed: int,
                options: Optional[EstimatorOptions] = None) -> EstimateReport:
    """Multilevel estimate of E[f(AB)] entrywise (estimators.hpp:62-67)."""
    return _mlmc(True, model, f, plan, seed, options)


def _mc(matrix: bool, model, f, L, N, M, seed, options, c0=1):
    options = options or EstimatorOptions()
    if matrix != isinstance(model, MatrixPairModel):
        raise ValueError("estimator: model kind does not match the estimator")
    rows, cols = _shape(model)
    buf = _Buffers(1, rows * cols)
    desc = model.desc()
    fn = lib().mlsk_mc_matmul if matrix else lib().mlsk_mc_inner
    check(fn(C.byref(desc), f.kind, f.param, L, N, M, c0, seed, C.byref(options._c()), C.byref(buf.c)))
    return _report(buf, model, 1, not matrix, with_levels=False)


def mc_inner(model: VectorPairModel, f: TargetFunction, L: int, N: int, M: int, seed: int,
             options: Optional[EstimatorOptions] = None, c0: int = 1) -> EstimateReport:
    """Single-level baseline (estimators.hpp:69-74)."""
    return _mc(False, model, f, L, N, M, seed, options, c0)


def mc_matmul(model: MatrixPairModel, f: TargetFunction, L: int, N: int, M: int, seed: int,
              options: Optional[EstimatorOptions] = None, c0: int = 1) -> EstimateReport:
    """Single-level baseline (estimators.hpp:76-79)."""
    return _mc(True, model, f, L, N, M, seed, options, c0)


@dataclass
class ScalarReference:  # models.hpp ScalarReference
    value: float
    std_error: float
    count: int


@dataclass
class MatrixReference:  # models.hpp MatrixReference
    value: np.ndarray
    std_error: float
    count: int


def _reference(matrix: bool, model, f: TargetFunction, count: int, seed: int, options):
    options = options or EstimatorOptions()
    if matrix != isinstance(model, MatrixPairModel):
        raise ValueError("estimator: model kind does not match the estimator")
    rows, cols = _shape(model)
    mean = np.zeros(rows * cols)
    se = C.c_double(0.0)
    desc = model.desc()
    fn = lib().mlsk_reference_matmul if matrix else lib().mlsk_reference_inner
    check(fn(C.byref(desc), f.kind, f.param, count, seed, C.byref(options._c()), _ptr(mean, _f64p), C.byref(se)))
    return mean, se.value


def reference_inner(model: VectorPairModel, f: TargetFunction, count: int, seed: int,
                    options: Optional[EstimatorOptions] = None) -> ScalarReference:
    """MC reference value of E[f(a^T b)] from `count` full draws keyed
    (seed, 0, k) (models.cpp:140-175), on the device."""
    mean, se = _reference(False, model, f, count, seed, options)
    return ScalarReference(float(mean[0]), se, count)


def reference_matmul(model: MatrixPairModel, f: TargetFunction, count: int, seed: int,
                     options: Optional[EstimatorOptions] = None) -> MatrixReference:
    """MC reference value of E[f(AB)] entrywise (models.cpp:177-227)."""
    mean, se = _reference(True, model, f, count, seed, options)
    return MatrixReference(mean.reshape(model.m, model.p), se, count)


# -------------------------------------------------------------- sketches


def sketch_inner(a, b, indices, inv_probs=None) -> float:
    """(1/s) sum_i a_r b_r / xi_r over a realization (sketch.hpp:17-30), on the device."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("sketch_inner: dimension mismatch")
    idx = np.ascontiguousarray(indices, dtype=np.uint32)
    inv = None if inv_probs is None else np.ascontiguousarray(inv_probs, dtype=np.float64)
    if inv is not None and inv.shape != a.shape:
        raise ValueError("sketch_inner: dimension mismatch")
    out = np.zeros(1)
    check(lib().mlsk_sketch_inner(_ptr(a, _f64p), _ptr(b, _f64p), a.size, _ptr(idx, _u32p), idx.size,
                                  _ptr(inv, _f64p), _ptr(out, _f64p)))
    return float(out[0])


def sketch_matmul(A, B, indices, inv_probs=None) -> np.ndarray:
    """(1/s) sum_i A[:, r_i] B[r_i, :] / xi_r (sketch.hpp:32-41), on the device."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
        raise ValueError("sketch_matmul: dimension mismatch")
    idx = np.ascontiguousarray(indices, dtype=np.uint32)
    inv = None if inv_probs is None else np.ascontiguousarray(inv_probs, dtype=np.float64)
    out = np.zeros((A.shape[0], B.shape[1]))
    check(lib().mlsk_sketch_matmul(_ptr(A, _f64p), _ptr(B, _f64p), A.shape[0], A.shape[1], B.shape[1],
                                   _ptr(idx, _u32p), idx.size, _ptr(inv, _f64p), _ptr(out, _f64p)))
    return out


def draw_sample(model, seed: int, tag: int, k: int, c: int):
    """One level-sample's draw (model.draw + draw_realization,
    estimators.cpp:134-136) restricted to the sampled indices: returns
    (indices, A[:, S] as rows x c, B[S, :] as c x cols)."""
    rows, cols = _shape(model)
    idx = np.zeros(c, dtype=np.uint32)
    a = np.zeros((rows, c))
    b = np.zeros((c, cols))
    desc = model.desc()
    check(lib().mlsk_draw_sample(C.byref(desc), seed, tag, k, c, _ptr(idx, _u32p), _ptr(a, _f64p),
                                 _ptr(b, _f64p)))
    return idx, a, b


# ------------------------------------------------------ model data / truth


def model_data(model, which: int) -> np.ndarray:
    """Fixed model data as generated on the device: which = 0 -> means of A / a
    (RFF: the points X, m x D), 1 -> means of B / b (RFF: W, D x n), 2 -> RFF
    phases b."""
    d = model.desc()
    n = C.c_int64()
    check(lib().mlsk_model_data(C.byref(d), which, None, C.byref(n)))
    dt = np.float32 if model.dtype == abi.F32 else np.float64
    out = np.zeros(n.value, dtype=dt)
    check(lib().mlsk_model_data(C.byref(d), which, out.ctypes.data_as(C.c_void_p), C.byref(n)))
    return out


def ground_truth(model, device: str = "cuda"):
    """The exact target of the estimators for identity f: E[a^T b] / E[A B]
    (gauss-mean and deterministic models: the product of the means, one dense
    fp64 GEMM), or for the RFF model the full-feature Gram matrix K_n = Z Z^T
    together with the exact Gaussian kernel exp(-|x-y|^2 / (2 sigma^2)).
    (reference_inner / reference_matmul estimate this by MC, models.cpp:140-227.)"""
    import torch

    if model.kind == abi.MODEL_CONSTANT_ONES:
        return float(model.n) if isinstance(model, VectorPairModel) else np.full((model.m, model.p), float(model.n))
    if model.kind == abi.MODEL_DETERMINISTIC:
        if isinstance(model, VectorPairModel):
            j = np.arange(1, model.n + 1, dtype=np.float64)
            return float(np.dot(j, model.n + j))
        return np.array([[19.0, 22.0], [43.0, 50.0]])
    if model.kind == abi.MODEL_GAUSS_MEAN:
        a = torch.as_tensor(model_data(model, 0), dtype=torch.float64, device=device)
        b = torch.as_tensor(model_data(model, 1), dtype=torch.float64, device=device)
        if isinstance(model, VectorPairModel):
            return float(torch.dot(a, b))
        return (a.view(model.m, model.n) @ b.view(model.n, model.p)).cpu().numpy()
    if model.kind == abi.MODEL_RFF:
        X = torch.as_tensor(model_data(model, 0), dtype=torch.float64, device=device).view(model.m, model.rff_dim)
        W = torch.as_tensor(model_data(model, 1), dtype=torch.float64, device=device).view(model.rff_dim, model.n)
        bph = torch.as_tensor(model_data(model, 2), dtype=torch.float64, device=device)
        Kn = torch.zeros(model.m, model.m, dtype=torch.float64, device=device)
        step = 8192
        for j0 in range(0, model.n, step):
            Z = torch.cos(X @ W[:, j0:j0 + step] + bph[j0:j0 + step]) * math.sqrt(2.0 / model.n)
            Kn += Z @ Z.T
        d2 = torch.cdist(X, X) ** 2
        K = torch.exp(-d2 / (2.0 * model.sigma ** 2))
        return Kn.cpu().numpy(), K.cpu().numpy()
    raise ValueError("ground_truth: no closed form for this model kind")


# ----------------------------------------------------------- round API


class MlmcSession:
    """Round-based MLMC state on the device (the reference has no analogue:
    its planner is a-priori only).  Replications continue
    where the previous round stopped, so the union of rounds equals one run
    with the summed counts."""

    def __init__(self, model, f: TargetFunction, M: int, L: int, seed: int, c0: int = 1,
                 options: Optional[EstimatorOptions] = None):
        options = options or EstimatorOptions()
        self.model, self.f, self.M, self.L, self.c0, self.seed = model, f, M, L, c0, seed
        self.vector = isinstance(model, VectorPairModel)
        self.rows, self.cols = _shape(model)
        self._desc = model.desc()
        h = C.c_void_p()
        check(lib().mlsk_session_create(C.byref(self._desc), f.kind, f.param, M, c0, L, seed,
                                        C.byref(options._c()), C.byref(h)))
        self._h = h

    def run_round(self, dN: Sequence[int]) -> None:
        arr = np.ascontiguousarray(dN, dtype=np.int64)
        if arr.size != self.L + 1:
            raise ValueError("session: dN must have L+1 entries")
        check(lib().mlsk_session_run_round(self._h, _ptr(arr, _i64p)))

    def stats(self) -> EstimateReport:
        buf = _Buffers(self.L + 1, self.rows * self.cols)
        check(lib().mlsk_session_stats(self._h, C.byref(buf.c)))
        return _report(buf, self.model, self.L + 1, self.vector)

    def level_buffer(self):
        """(device pointer, n_doubles) of the packed per-level (sum, sumsq, count)
        buffer, for an in-place all-reduce across ranks."""
        ptr = C.c_void_p()
        n = C.c_int64()
        check(lib().mlsk_session_level_buffer(self._h, C.byref(ptr), C.byref(n)))
        return int(ptr.value), int(n.value)

    @property
    def cells(self) -> int:
        return self.rows * self.cols

    def packed_stats(self) -> np.ndarray:
        """Host copy of this rank's [(sum Y, sum ||Y||^2, count)] per level."""
        r = self.stats()
        cells = self.cells
        buf = np.zeros((self.L + 1, cells + 2))
        for l, st in enumerate(r.per_level):
            buf[l, :cells] = np.asarray(st.sum, dtype=np.float64).ravel()
            buf[l, cells] = st.sum_of_squares
            buf[l, cells + 1] = st.replication_count
        return buf.ravel()

    def checkpoint(self) -> bytes:
        """The session's accumulators and replication counters as bytes
        (mlsk_session_checkpoint); `restore` them into a session created with
        the same arguments to continue the run bit for bit."""
        n = C.c_int64()
        check(lib().mlsk_session_checkpoint(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().mlsk_session_checkpoint(self._h, buf, C.byref(n)))
        return buf.raw[: n.value]

    def restore(self, image: bytes) -> None:
        check(lib().mlsk_session_restore(self._h, image, len(image)))

    def synchronize(self) -> None:
        check(lib().mlsk_session_synchronize(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            check(lib().mlsk_session_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
