"""The reference's own unit-test assertions (proj/tests/test_sketch.cpp,
test_estimators.cpp, test_sampling.cpp) re-expressed against
  * the CPU oracle  (always; parity anchor), and
  * the CUDA library through the public API (marked gpu).
The reference's doctest suite cannot be compiled here (vendor/doctest absent).
"""
import math

import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi


# ----------------------------------------------------------------- sketch KATs

def _oracle_sketch_inner(oracle, a, b, idx):
    a = np.ascontiguousarray(a, float); b = np.ascontiguousarray(b, float)
    ix = np.ascontiguousarray(idx, np.uint32); out = np.zeros(1)
    rc = oracle.oracle_lib().orc_sketch_inner(a.ctypes.data_as(oracle._f64p), b.ctypes.data_as(oracle._f64p),
                                              a.size, ix.ctypes.data_as(oracle._u32p), ix.size, None,
                                              out.ctypes.data_as(oracle._f64p))
    if rc:
        raise ValueError(oracle.oracle_lib().orc_last_error().decode())
    return out[0]


def _oracle_sketch_matmul(oracle, A, B, idx):
    A = np.ascontiguousarray(A, float); B = np.ascontiguousarray(B, float)
    ix = np.ascontiguousarray(idx, np.uint32); out = np.zeros((A.shape[0], B.shape[1]))
    rc = oracle.oracle_lib().orc_sketch_matmul(A.ctypes.data_as(oracle._f64p), B.ctypes.data_as(oracle._f64p),
                                               A.shape[0], A.shape[1], B.shape[1],
                                               ix.ctypes.data_as(oracle._u32p), ix.size, None,
                                               out.ctypes.data_as(oracle._f64p))
    if rc:
        raise ValueError(oracle.oracle_lib().orc_last_error().decode())
    return out


def sketch_cases(si, sm):
    # test_sketch.cpp:12-32 -- every index contributes 1*1*4
    ones4 = np.ones(4)
    assert si(ones4, ones4, [3]) == 4.0
    assert si(ones4, ones4, [1, 4, 2, 2]) == 4.0
    assert si([1, 2], [3, 4], [2, 2, 1]) == pytest.approx(38.0 / 3.0, rel=1e-15)
    for bad in ([], [3], [0]):
        with pytest.raises(ValueError):
            si([1, 2], [3, 4], bad)
    # test_sketch.cpp:46-75
    A = np.array([[1, 2], [3, 4]], float); B = np.array([[5, 6], [7, 8]], float)
    np.testing.assert_array_equal(sm(A, B, [1]), [[10, 12], [30, 36]])
    np.testing.assert_allclose(sm(A, B, [1, 2]), A @ B, rtol=1e-15)
    ex1 = sm(np.array([[2], [5]], float), np.array([[3, 4]], float), [1, 1])
    assert ex1[0, 0] == 6.0 and ex1[1, 1] == 20.0
    with pytest.raises(ValueError):
        sm(A, B, [3])
    # test_sketch.cpp:77-85 -- 1 x n by n x 1 equals the inner sketch
    a = np.array([1, -2, 3], float); b = np.array([4, 5, -6], float)
    r = [2, 3, 3, 1]
    assert sm(a[None, :], b[:, None], r)[0, 0] == pytest.approx(si(a, b, r), rel=1e-15)
    # test_sketch.cpp:111-124 -- sketch results
    assert si([1, 2], [3, 4], [1, 2, 1]) == pytest.approx((6 + 16 + 6) / 3)
    assert sm(A, B, [2, 2])[0, 0] == pytest.approx(2 * 2 * 7)


def test_sketch_kats_oracle(oracle):
    sketch_cases(lambda a, b, r: _oracle_sketch_inner(oracle, a, b, r),
                 lambda A, B, r: _oracle_sketch_matmul(oracle, A, B, r))


@pytest.mark.gpu
def test_sketch_kats_gpu(gpu):
    sketch_cases(gpu.sketch_inner, gpu.sketch_matmul)


# ------------------------------------------------------------- estimator KATs

class OracleBackend:
    def __init__(self, oracle):
        self.o = oracle

    def mlmc(self, kind, n, m, p, M, N, seed, target=abi.TARGET_IDENTITY, c0=1):
        d = self.o.model_desc(kind, n=n, m=m, p=p, stream=abi.STREAM_REF)
        r = self.o.OracleModel(d).mlmc(M, c0, N, seed, target=target)
        cells = r.value.size
        lv = [(r.level_estimate[l] if cells > 1 else r.level_estimate[l][0], r.level_mean_sq[l],
               int(r.level_count[l]), int(r.cost_units[l])) for l in range(len(N))]
        return (r.value if cells > 1 else r.value[0]), lv, r.total_cost_units

    def mc(self, kind, n, m, p, L, N, M, seed):
        d = self.o.model_desc(kind, n=n, m=m, p=p, stream=abi.STREAM_REF)
        r = self.o.OracleModel(d).mc(L, N, M, 1, seed)
        return (r.value if r.value.size > 1 else r.value[0]), r.total_cost_units


class GpuBackend:
    def __init__(self, g):
        self.g = g

    def _model(self, kind, n, m, p):
        g = self.g
        if kind == abi.MODEL_CONSTANT_ONES:
            return g.constant_ones_model(n) if m == 0 else g.constant_ones_matrix_model(m, n, p)
        if kind == abi.MODEL_DETERMINISTIC:
            return g.deterministic_model(n) if m == 0 else g.deterministic_matrix_model()
        if kind == abi.MODEL_PAPER_INNER:
            return g.paper_inner_model()
        return g.paper_matrix_model()

    def mlmc(self, kind, n, m, p, M, N, seed, target=abi.TARGET_IDENTITY, c0=1):
        g = self.g
        model = self._model(kind, n, m, p)
        f = {abi.TARGET_IDENTITY: g.target_identity(), abi.TARGET_F1: g.target_f1(),
             abi.TARGET_F2: g.target_f2()}[target]
        fn = g.mlmc_matmul if isinstance(model, g.MatrixPairModel) else g.mlmc_inner
        r = fn(model, f, g.LevelPlan(M, len(N) - 1, N, c0=c0), seed)
        lv = [(np.asarray(s.estimate).ravel() if np.ndim(s.estimate) else s.estimate, s.sample_mean_of_squares,
               s.replication_count, s.cost_units) for s in r.per_level]
        val = np.asarray(r.value).ravel() if np.ndim(r.value) else r.value
        return val, lv, r.total_cost_units

    def mc(self, kind, n, m, p, L, N, M, seed):
        g = self.g
        model = self._model(kind, n, m, p)
        fn = g.mc_matmul if isinstance(model, g.MatrixPairModel) else g.mc_inner
        r = fn(model, g.target_identity(), L, N, M, seed)
        val = np.asarray(r.value).ravel() if np.ndim(r.value) else r.value
        return val, r.total_cost_units


def estimator_cases(B):
    C1, DET, PI = abi.MODEL_CONSTANT_ONES, abi.MODEL_DETERMINISTIC, abi.MODEL_PAPER_INNER
    # test_estimators.cpp:39-60 -- constant data collapses every level above zero
    val, lv, _ = B.mlmc(C1, 37, 0, 0, 3, [9, 3, 1], 77)
    assert val == 37.0 and lv[0][0] == 37.0 and lv[1][0] == 0.0 and lv[2][0] == 0.0 and lv[1][1] == 0.0
    val, lv, _ = B.mlmc(C1, 4, 3, 2, 3, [9, 3, 1], 77)
    np.testing.assert_array_equal(val, 4.0)
    assert np.sum(np.asarray(lv[2][0]) ** 2) == 0.0
    # test_estimators.cpp:62-82 -- cost accounting
    _, lv, total = B.mlmc(DET, 2, 0, 0, 10, [800, 80, 8, 1], 5)
    assert [x[3] for x in lv] == [800, 80 * 11, 8 * 110, 1100] and total == 3660
    assert lv[2][2] == 8
    _, lv, total = B.mlmc(DET, 2, 2, 2, 2, [4, 2, 1], 5)
    assert [x[3] for x in lv] == [4 * 1 * 4, 2 * 3 * 4, 1 * 6 * 4] and total == 16 * 4
    # test_estimators.cpp:84-105 -- unbiased, level variances 25 / 12.5 / 6.25
    val, lv, _ = B.mlmc(DET, 2, 0, 0, 2, [100000] * 3, 2024)
    var = [lv[0][1] - lv[0][0] ** 2 if False else None]
    assert lv[0][1] - 121.0 == pytest.approx(25.0, rel=0.05)
    v1 = lv[1][1] - lv[1][0] ** 2
    v2 = lv[2][1] - lv[2][0] ** 2
    assert v1 == pytest.approx(12.5, rel=0.05) and v2 == pytest.approx(6.25, rel=0.05)
    se = math.sqrt(sum(max(0.0, s[1] - s[0] ** 2) / s[2] for s in lv))
    assert abs(val - 11.0) <= 3 * se
    assert val == sum(s[0] for s in lv)
    # test_estimators.cpp:107-121 -- matrix level-0 spread 546
    val, lv, _ = B.mlmc(DET, 2, 2, 2, 2, [20000] * 3, 99)
    exact = np.array([19, 22, 43, 50], float)
    se = math.sqrt(sum(max(0.0, s[1] - float(np.sum(np.asarray(s[0]) ** 2))) / s[2] for s in lv))
    assert np.linalg.norm(np.asarray(val) - exact) <= 3 * se
    assert lv[0][1] - 5194.0 == pytest.approx(546.0, rel=0.1)
    # test_estimators.cpp:236-267 -- single-level baseline
    v, tot = B.mc(C1, 7, 0, 0, 3, 11, 2, 5)
    assert v == 7.0 and tot == 11 * 8
    v, tot = B.mc(DET, 2, 0, 0, 0, 5, 2, 17)
    assert 6.0 <= v <= 16.0 and tot == 5
    v, _ = B.mc(DET, 2, 0, 0, 3, 20000, 2, 41)
    assert abs(v - 11.0) <= 3 * math.sqrt(25.0 / 8.0 / 20000.0)
    v, tot = B.mc(C1, 3, 2, 2, 2, 6, 3, 5)
    np.testing.assert_array_equal(v, 3.0)
    assert tot == 6 * 9 * 4
    # test_estimators.cpp:269-277 -- MC and MLMC substreams do not collide
    val, lv, _ = B.mlmc(PI, 1000, 0, 0, 2, [50, 50], 1234)
    v, _ = B.mc(PI, 1000, 0, 0, 1, 50, 2, 1234)
    assert lv[1][0] != v and val != v


def test_estimator_kats_oracle(oracle):
    estimator_cases(OracleBackend(oracle))


@pytest.mark.gpu
def test_estimator_kats_gpu(gpu):
    estimator_cases(GpuBackend(gpu))


@pytest.mark.gpu
def test_malformed_plans_rejected_gpu(gpu):
    """test_estimators.cpp:222-234: std::invalid_argument -> ValueError."""
    m = gpu.deterministic_model(2)
    with pytest.raises(ValueError):
        gpu.mlmc_inner(m, gpu.target_identity(), gpu.LevelPlan(2, 2, [10, 10]), 1)
    with pytest.raises(ValueError):
        gpu.mlmc_inner(m, gpu.target_identity(), gpu.LevelPlan(2, 1, [10, 0]), 1)
    with pytest.raises(ValueError):
        gpu.mc_inner(m, gpu.target_identity(), 2, 0, 2, 1)
    with pytest.raises(ValueError):
        gpu.mc_inner(m, gpu.target_identity(), 2, 10, 1, 1)
    with pytest.raises(ValueError):
        gpu.target_f2(0.0)


@pytest.mark.gpu
def test_coupling_probe_gpu(gpu):
    """test_estimators.cpp:188-220: coarse = prefix of fine, deterministic order."""
    seen = []
    opt = gpu.EstimatorOptions(threads=8, probe=lambda l, k, f, c: seen.append((l, k, f, c)))
    gpu.mlmc_inner(gpu.deterministic_model(2), gpu.target_identity(), gpu.LevelPlan(3, 2, [5, 4, 3]), 321, opt)
    assert len(seen) == 4 + 3
    assert seen[0][:2] == (1, 0) and seen[3][1] == 3 and seen[4][0] == 2
    for l, k, fine, coarse in seen:
        assert len(fine) == (3 if l == 1 else 9) and coarse == fine[: len(fine) // 3]
    assert seen[4][2] != seen[5][2] or seen[5][2] != seen[6][2]


@pytest.mark.gpu
def test_bit_identical_reruns_gpu(gpu):
    """test_estimators.cpp:162-186: reruns are bit-identical; seeds differ."""
    plan = gpu.LevelPlan(3, 2, [300, 100, 33])
    a = gpu.mlmc_inner(gpu.paper_inner_model(), gpu.target_f1(), plan, 314)
    b = gpu.mlmc_inner(gpu.paper_inner_model(), gpu.target_f1(), plan, 314, gpu.EstimatorOptions(threads=4))
    d = gpu.mlmc_inner(gpu.paper_inner_model(), gpu.target_f1(), plan, 315)
    assert a.value == b.value and a.per_level[2].sample_mean_of_squares == b.per_level[2].sample_mean_of_squares
    assert a.value != d.value
    model = gpu.gaussian_mean_matrix_model(128, 4096, 64, data_seed=3)
    p2 = gpu.LevelPlan(2, 2, [200, 100, 50], c0=32)
    x = gpu.mlmc_matmul(model, gpu.target_identity(), p2, 9)
    y = gpu.mlmc_matmul(model, gpu.target_identity(), p2, 9)
    np.testing.assert_array_equal(x.value, y.value)
