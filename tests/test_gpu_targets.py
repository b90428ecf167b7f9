"""Nonlinear targets f1, f2 (models.cpp:99-117) on the fused engine.

The reference applies f to the fine and the coarse sketch separately, entry
by entry (estimators.cpp:137-147), so Y = f(fine) - f(coarse) can no longer be
one signed contraction.  The fused engines keep the prefix apart: the inner
path (config-1 shapes) accumulates the prefix and suffix sums separately;
the DMMA path (config-2 shapes) pads the coarse prefix to whole K-chunks and
reads f((n/cc) S_prefix) at that chunk boundary, Y = f(acc) - f(coarse) in
the epilogue.  Checked against the exact-order engine and the CPU oracle at
1e-12 relative (fp64, BASELINE.json north_star), including prefixes that are
not a multiple of the K-chunk (M = 3, c0 = 1: the padding path) and target
values on both sides of f1's step at 10."""
import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi

pytestmark = pytest.mark.gpu
MASTER = 20260823
TOL = 1e-12


def frob_rel(a, b):
    a = np.atleast_1d(np.asarray(a, dtype=np.float64)).ravel()
    b = np.atleast_1d(np.asarray(b, dtype=np.float64)).ravel()
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / den if den > 0 else np.linalg.norm(a - b)


def targets(g):
    return {"f1": g.target_f1(), "f2": g.target_f2()}


def compare(rf, ro_sum, ro_sq, tol=TOL):
    for l, st in enumerate(rf.per_level):
        assert frob_rel(st.sum, ro_sum[l]) <= tol, (l, frob_rel(st.sum, ro_sum[l]))
        assert abs(st.sum_of_squares - ro_sq[l]) <= tol * abs(ro_sq[l]), l


@pytest.mark.parametrize("tname", ["f1", "f2"])
@pytest.mark.parametrize("shape", [("inner", 2, 8, 4), ("inner", 3, 1, 4)])
def test_inner_nonlinear_fused_vs_exact_and_oracle(gpu, oracle, tname, shape):
    _, M, c0, L = shape
    # small n, means U(-1, 3): sketch values spread around f1's step at 10
    model = gpu.gaussian_mean_model(64, sd=1.0, mean_lo=-1.0, mean_hi=3.0, data_seed=7)
    f = targets(gpu)[tname]
    N = [400, 200, 120, 64, 40][:L + 1]
    plan = gpu.LevelPlan(M, L, N, c0=c0)
    rf = gpu.mlmc_inner(model, f, plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_inner(model, f, plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    compare(rf, [np.asarray(s.sum) for s in re_.per_level], [s.sum_of_squares for s in re_.per_level])
    o = oracle.OracleModel(model.desc()).mlmc(M, c0, N, MASTER, target=f.kind, tp=f.param)
    compare(rf, o.level_sum, o.level_sumsq)
    # the exact engine is the oracle's arithmetic: bit for bit
    for l, st in enumerate(re_.per_level):
        assert np.array_equal(np.atleast_1d(st.sum).ravel(), o.level_sum[l])


@pytest.mark.parametrize("tname", ["f1", "f2"])
@pytest.mark.parametrize("shape", [(2, 32, 3), (3, 1, 4), (2, 24, 2)])
def test_matrix_nonlinear_fused_vs_exact_and_oracle(gpu, oracle, tname, shape):
    """(M, c0, L): (2, 32) prefix = whole K-chunks; (3, 1) and (2, 24) not."""
    M, c0, L = shape
    model = gpu.gaussian_mean_matrix_model(96, 512, 80, sd=0.5, mean_lo=-0.5, mean_hi=1.5, data_seed=11)
    f = targets(gpu)[tname]
    N = [9, 7, 5, 4, 3][:L + 1]
    plan = gpu.LevelPlan(M, L, N, c0=c0)
    rf = gpu.mlmc_matmul(model, f, plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, f, plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    compare(rf, [np.asarray(s.sum) for s in re_.per_level], [s.sum_of_squares for s in re_.per_level])
    o = oracle.OracleModel(model.desc()).mlmc(M, c0, N, MASTER, target=f.kind, tp=f.param)
    compare(rf, o.level_sum, o.level_sumsq)


def test_config2_f2_all_levels(gpu, oracle):
    """Config 2 (256 x 4096 x 256, c = 32 ... 2048) with target f2, levels 0-6."""
    model = gpu.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, mean_lo=-1.0, mean_hi=1.0,
                                           data_seed=gpu.RngStream.derive_seed(MASTER, 0xD47A0002, 0))
    f = gpu.target_f2()
    N = [4, 3, 3, 2, 2, 2, 2]
    plan = gpu.LevelPlan(2, 6, N, c0=32)
    rf = gpu.mlmc_matmul(model, f, plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 32, N, MASTER, target=f.kind, tp=f.param)
    compare(rf, o.level_sum, o.level_sumsq)


def test_nonlinear_probe_indices_match_exact(gpu):
    """The padded prefix layout keeps the sampled index sets (coupling probe)."""
    model = gpu.gaussian_mean_matrix_model(64, 512, 64, sd=0.5, data_seed=3)
    plan = gpu.LevelPlan(3, 2, [4, 3, 2], c0=5)
    seen = {"fused": [], "exact": []}
    for eng in seen:
        gpu.mlmc_matmul(model, gpu.target_f1(), plan, MASTER,
                        gpu.EstimatorOptions(engine=eng, probe=lambda l, k, fi, co, e=eng: seen[e].append((l, k, fi, co))))
    assert seen["fused"] == seen["exact"] and len(seen["fused"]) == 5


def test_auto_engine_takes_fused_for_f64_nonlinear(gpu):
    """AUTO picks the fused engine for fp64 gauss models with f1 / f2 (identical
    level sums to an explicit fused call)."""
    model = gpu.gaussian_mean_matrix_model(64, 512, 64, sd=0.5, data_seed=3)
    plan = gpu.LevelPlan(2, 1, [6, 3], c0=32)
    ra = gpu.mlmc_matmul(model, gpu.target_f2(), plan, MASTER)
    rf = gpu.mlmc_matmul(model, gpu.target_f2(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    for a, b in zip(ra.per_level, rf.per_level):
        assert np.array_equal(np.asarray(a.sum), np.asarray(b.sum))
