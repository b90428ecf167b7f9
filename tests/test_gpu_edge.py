"""Edge cases of the device path: degenerate shapes, non-power-of-two index
ranges, single-level plans, empty session rounds, NaN inputs, bad options.
Fused results are compared with the exact-order engine (1e-12 fp64 / 1e-5
fp32, Frobenius), the exact engine with the CPU oracle bit for bit."""
import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi

pytestmark = pytest.mark.gpu
MASTER = 20260823


def frob_rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


def close(r1, r2, tol):
    for s1, s2 in zip(r1.per_level, r2.per_level):
        assert s1.replication_count == s2.replication_count
        assert frob_rel(s1.sum, s2.sum) <= tol, (s1.level, frob_rel(s1.sum, s2.sum))
        assert abs(s1.sum_of_squares - s2.sum_of_squares) <= tol * max(s2.sum_of_squares, 1e-300)


def both(gpu, model, plan, seed=MASTER):
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, seed, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, seed, gpu.EstimatorOptions(engine="exact"))
    return rf, re_


@pytest.mark.parametrize("shape", [(1, 512, 1), (1, 512, 300), (300, 512, 1), (129, 1000, 65)])
def test_degenerate_and_odd_shapes_fp64(gpu, shape):
    """1 x p, m x 1 and odd m, p; n = 1000 (not a power of two: index by the
    cumulative-table search, sampling.cpp:107-112)."""
    m, n, p = shape
    model = gpu.gaussian_mean_matrix_model(m, n, p, sd=0.5, data_seed=3)
    rf, re_ = both(gpu, model, gpu.LevelPlan(2, 2, [67, 33, 17], c0=24))
    close(rf, re_, 1e-12)


@pytest.mark.parametrize("shape", [(1, 512, 256), (200, 1000, 72)])
def test_degenerate_and_odd_shapes_fp32(gpu, shape):
    m, n, p = shape
    model = gpu.gaussian_mean_matrix_model(m, n, p, sd=1.0, data_seed=5, dtype=abi.F32)
    rf, re_ = both(gpu, model, gpu.LevelPlan(2, 1, [41, 19], c0=48))
    close(rf, re_, 1e-5)


def test_single_level_plans(gpu, oracle):
    """L = 0: the plain sketch estimator (one level, no coarse term)."""
    model = gpu.gaussian_mean_matrix_model(64, 2048, 64, sd=0.5, data_seed=7)
    plan = gpu.LevelPlan(2, 0, [150], c0=40)
    rf, re_ = both(gpu, model, plan)
    close(rf, re_, 1e-12)
    o = oracle.OracleModel(model.desc()).mlmc(2, 40, [150], MASTER)
    np.testing.assert_array_equal(np.asarray(re_.per_level[0].sum).ravel(), o.level_sum[0])
    vm = gpu.gaussian_mean_model(4096, sd=1.0, data_seed=9)
    rv = gpu.mlmc_inner(vm, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    ov = oracle.OracleModel(vm.desc()).mlmc(2, 40, [150], MASTER)
    assert abs(rv.value - ov.value[0]) <= 1e-12 * abs(ov.value[0])


def test_session_rounds_with_empty_levels(gpu):
    """Rounds that add nothing to some levels leave them untouched; the total
    equals one round with the summed counts."""
    model = gpu.gaussian_mean_matrix_model(128, 4096, 128, sd=0.5, data_seed=11)
    s1 = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, 5, c0=32)
    for dN in ([70, 0, 0], [0, 0, 0], [0, 40, 9], [30, 0, 0]):
        s1.run_round(dN)
    s2 = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, 5, c0=32)
    s2.run_round([100, 40, 9])
    a, b = s1.stats(), s2.stats()
    close(a, b, 1e-12)
    s1.close()
    s2.close()


def test_nan_host_means_rejected(gpu):
    """DenseMatrix rejects NaN entries (tensor.cpp:12-18) -> invalid_argument."""
    ma = np.zeros((8, 64))
    mb = np.zeros((64, 8))
    ma[3, 5] = np.nan
    model = gpu.gaussian_mean_matrix_model(8, 64, 8, sd=1.0, mean_a=ma, mean_b=mb)
    with pytest.raises(ValueError):
        gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 1, [4, 2], c0=8), 1)


def test_bad_device_and_engine_rejected(gpu):
    model = gpu.gaussian_mean_matrix_model(8, 64, 8, sd=1.0, data_seed=1)
    plan = gpu.LevelPlan(2, 1, [4, 2], c0=8)
    from paper_1904_00429_b200._lib import MlskRuntimeError
    with pytest.raises((ValueError, MlskRuntimeError)):
        gpu.mlmc_matmul(model, gpu.target_identity(), plan, 1, gpu.EstimatorOptions(device=4096))
    # the fused engine needs the philox stream; on the fp32 (tcgen05) engine an identity target
    with pytest.raises(ValueError):
        gpu.mlmc_matmul(gpu.paper_matrix_model(), gpu.target_identity(), plan, 1,
                        gpu.EstimatorOptions(engine="fused"))
    m32 = gpu.gaussian_mean_matrix_model(8, 64, 8, sd=1.0, data_seed=1, dtype=1)
    with pytest.raises(ValueError):
        gpu.mlmc_matmul(m32, gpu.target_f2(), plan, 1, gpu.EstimatorOptions(engine="fused"))


def test_large_level0_count(gpu):
    """A million-replication level in one call (chunk bookkeeping, batching)."""
    vm = gpu.gaussian_mean_model(4096, sd=1.0, data_seed=13)
    plan = gpu.LevelPlan(2, 1, [1_000_003, 257], c0=8)
    rf = gpu.mlmc_inner(vm, gpu.target_identity(), plan, 3, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_inner(vm, gpu.target_identity(), plan, 3, gpu.EstimatorOptions(engine="exact"))
    assert rf.per_level[0].replication_count == 1_000_003
    assert abs(rf.value - re_.value) <= 1e-11 * abs(re_.value)
