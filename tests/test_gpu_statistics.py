"""Statistical assertions of the reference suite, re-expressed on the device
(VERDICT r01 "missing" #7):

  * desk-scale correctness over 100 seeds at 3 combined standard errors
    (proj/tests/acceptance.cpp:191-207, check 5),
  * coupled-difference variance decay on the random model in >= 8 of 10
    seeds (proj/tests/test_estimators.cpp:123-147),
  * multilevel and single-level estimates agree in expectation
    (proj/tests/test_estimators.cpp:149-160),

plus the same properties on the throughput (fused, Philox) engine at the
BASELINE config-2 shapes, where the target E[A] E[B] = M P is known exactly:
the squared Frobenius error of each estimate against M P is a sum over
65,536 cells, so its ratio to the estimator's own predicted mean square error
sum_l V_l / N_l concentrates near 1 seed by seed.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def combined_se(r):  # acceptance.cpp:55-62
    v = 0.0
    for s in r.per_level:
        var = s.sample_mean_of_squares - s.estimate * s.estimate
        v += max(0.0, var) / s.replication_count
    return math.sqrt(v)


def test_desk_scale_correctness_100_seeds(gpu):
    model = gpu.deterministic_model(2)
    f = gpu.target_identity()
    plan = gpu.LevelPlan(2, 3, [10000, 5000, 2500, 1250], 0.1, 1.0, 1.0, False)
    hits = 0
    for seed in range(1000, 1100):
        r = gpu.mlmc_inner(model, f, plan, seed)
        hits += abs(r.value - 11.0) <= 3.0 * combined_se(r)
    assert hits >= 95, f"{hits} of 100 seeds inside 3 combined standard errors of 11 (need >= 95)"


def test_variance_decays_across_levels_on_random_model(gpu):
    model = gpu.paper_inner_model()
    f1 = gpu.target_f1()
    plan = gpu.LevelPlan(7, 4, [200] * 5)
    monotone = 0
    for seed in range(7000, 7010):
        r = gpu.mlmc_inner(model, f1, plan, seed)
        var = [s.sample_mean_of_squares - s.estimate * s.estimate for s in r.per_level]
        monotone += all(var[l + 1] < var[l] for l in range(1, 4))
    assert monotone >= 8


def test_multilevel_and_single_level_agree(gpu):
    model = gpu.deterministic_model(2)
    idf = gpu.target_identity()
    ml = gpu.mlmc_inner(model, idf, gpu.LevelPlan(2, 2, [40000] * 3), 77)
    mc = gpu.mc_inner(model, idf, 2, 40000, 2, 78)
    mc_se = math.sqrt(25.0 / (4.0 * 40000.0))  # single-draw variance at 4 uniform indices: 25/4
    band = 3.0 * math.sqrt(combined_se(ml) ** 2 + mc_se ** 2)
    assert abs(ml.value - mc.value) <= band


def _config2_model(gpu, seed=20260823):
    return gpu.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, mean_lo=-1.0, mean_hi=1.0,
                                          data_seed=gpu.RngStream.derive_seed(seed, 0xD47A0002, 0))


def _predicted_mse(r):
    """sum_l V_l / N_l with V_l = mean ||Y_l||_F^2 - ||mean Y_l||_F^2 (the
    scalar level variance the reference reports, estimators.cpp:153-184)."""
    out = 0.0
    for s in r.per_level:
        est = np.asarray(s.estimate)
        out += (s.sample_mean_of_squares - float(np.sum(est * est))) / s.replication_count
    return out


def test_fused_engine_error_matches_predicted_rmse_config2(gpu):
    """Throughput engine at config-2 shapes: 12 seeds, fixed N_l; the squared
    Frobenius error against the exact M P over the predicted MSE."""
    model = _config2_model(gpu)
    truth = np.asarray(gpu.ground_truth(model, device="cpu"))
    plan = gpu.LevelPlan(2, 3, [256, 128, 64, 32], c0=32)
    opts = gpu.EstimatorOptions(engine="fused")
    ratios = []
    for seed in range(12):
        r = gpu.mlmc_matmul(model, gpu.target_identity(), plan, 9000 + seed, opts)
        err = np.asarray(r.value) - truth
        ratios.append(float(np.sum(err * err)) / _predicted_mse(r))
    ratios = np.array(ratios)
    # 65,536 cells per estimate: each ratio is a normalised chi-square-like sum
    assert np.all((ratios > 0.8) & (ratios < 1.25)), ratios
    assert abs(ratios.mean() - 1.0) < 0.08, ratios


def test_fused_mlmc_and_mc_agree_config2(gpu):
    """MLMC (levels 0..3) against the single-level estimator at c = c_3 on the
    fused engine: both are unbiased for E[A] E[B], so the squared Frobenius
    norm of their difference concentrates at the sum of their predicted mean
    square errors (65,536 cells); allow 1.3x."""
    model = _config2_model(gpu)
    opts = gpu.EstimatorOptions(engine="fused")
    ml = gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 3, [512, 256, 128, 64], c0=32), 77, opts)
    # mc at c = 32 * 2^3 = 256 indices: mc_matmul(L, N, M) with c0 = 32
    mc = gpu.mc_matmul(model, gpu.target_identity(), 3, 256, 2, 78, opts, c0=32)
    d = np.asarray(ml.value) - np.asarray(mc.value)
    # the MC report carries no level statistics: its MSE is predicted from a
    # single-level run of the same shape (c = 256, N = 256) on another seed
    pilot = gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 0, [256], c0=256), 79, opts)
    mc_var = _predicted_mse(pilot)
    assert float(np.sum(d * d)) <= 1.3 * (_predicted_mse(ml) + mc_var)
