"""Adaptive MLMC driver and ground truth on the device (config-2 shapes)."""
import numpy as np
import pytest

from paper_1904_00429_b200 import driver

pytestmark = pytest.mark.gpu
MASTER = 20260823


def test_adaptive_mlmc_reaches_target_and_truth(gpu):
    model = gpu.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=gpu.RngStream.derive_seed(MASTER, 0xD47A0002, 0))
    exact = gpu.ground_truth(model)
    eps = 0.05 * np.linalg.norm(exact)
    sess = gpu.MlmcSession(model, gpu.target_identity(), 2, 3, MASTER, c0=32)
    r = driver.adaptive_mlmc(sess, 2, 32, 3, eps=eps, n_pilot=128, max_rounds=8)
    assert r.rmse_estimate <= eps * 1.0001
    err = np.linalg.norm(r.value - exact.ravel())
    assert err <= 5 * r.rmse_estimate, (err, r.rmse_estimate)
    # standard allocation shape: V_l c_l roughly constant for l >= 1 -> N_l halves per level
    V = r.stats.variances
    assert all(V[l + 1] < V[l] for l in range(1, 3))
    sess.close()


def test_two_rank_sharding_in_one_process(gpu):
    """Chunk sharding over world=2 sums to the world=1 statistics."""
    model = gpu.gaussian_mean_matrix_model(128, 4096, 128, sd=0.5, data_seed=1)
    dN = [300, 170, 65]
    full = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, 7, c0=32)
    full.run_round(dN)
    parts = []
    for r in range(2):
        s = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, 7, c0=32,
                            options=gpu.EstimatorOptions(rank=r, world=2))
        s.run_round(dN)
        parts.append(s.packed_stats())
        s.close()
    a = driver.unpack(parts[0] + parts[1], 3)
    b = driver.unpack(full.packed_stats(), 3)
    np.testing.assert_array_equal(a.counts, b.counts)
    np.testing.assert_allclose(a.sums, b.sums, rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(a.sumsq, b.sumsq, rtol=1e-12)
    full.close()


def test_ground_truth_vector_and_rff(gpu):
    vm = gpu.gaussian_mean_model(4096, sd=1.0, data_seed=3)
    mu, nu = gpu.model_data(vm, 0), gpu.model_data(vm, 1)
    assert gpu.ground_truth(vm) == pytest.approx(float(mu @ nu), rel=1e-12)
    rm = gpu.rff_gram_model(64, 1024, dim=8, sigma=4.0, data_seed=2)
    Kn, K = gpu.ground_truth(rm)
    assert Kn.shape == (64, 64) and K.shape == (64, 64)
    np.testing.assert_allclose(np.diag(K), 1.0)
    # n random features approximate the kernel (error ~ 1/sqrt(n))
    assert np.abs(Kn - K).max() < 0.2
