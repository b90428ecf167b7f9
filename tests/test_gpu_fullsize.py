"""BASELINE configs 3-5 at their full shapes (fp32, tcgen05 3xTF32 engine):
the fused engine against the exact-order engine (fp64 arithmetic on the same
fp32 draws, reference order) on a few level-samples of the configs' own
levels, plus size-independent properties -- additivity over replication
shards (the multi-GPU split) and seed reproducibility.  Tolerance as in
BASELINE.json's north_star: 1e-5 relative (Frobenius) for fp32 configs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL32 = 1e-5
MASTER = 20260823


def frob_rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def data_seed(g, config):
    return g.RngStream.derive_seed(MASTER, 0xD47A0000 + config, 0)


def check(rf, re_, tol=TOL32):
    for sf, se in zip(rf.per_level, re_.per_level):
        assert sf.replication_count == se.replication_count
        assert frob_rel(sf.sum, se.sum) <= tol, (sf.level, frob_rel(sf.sum, se.sum))
        assert abs(sf.sum_of_squares - se.sum_of_squares) <= tol * se.sum_of_squares, sf.level


def fused_vs_exact(g, model, plan):
    rf = g.mlmc_matmul(model, g.target_identity(), plan, MASTER, g.EstimatorOptions(engine="fused"))
    re_ = g.mlmc_matmul(model, g.target_identity(), plan, MASTER, g.EstimatorOptions(engine="exact"))
    check(rf, re_)
    return rf


def test_config3_full_shape(gpu):
    """A 1024 x 16384, B 16384 x 1024, N(U(-1,1) means, 1): levels c = 64, 128."""
    model = gpu.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=data_seed(gpu, 3), dtype=1)
    fused_vs_exact(gpu, model, gpu.LevelPlan(2, 1, [3, 2], c0=64))


def test_config4_full_shape(gpu):
    """RFF Gram of 4096 points in R^64, 2^16 features: levels c = 128, 256."""
    model = gpu.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=data_seed(gpu, 4))
    fused_vs_exact(gpu, model, gpu.LevelPlan(2, 1, [2, 1], c0=128))


def test_config5_full_shape(gpu):
    """A 8192 x 2^20, B 2^20 x 8192 Student-t(3) + U(-0.5,0.5) means, level 0
    (c = 256) of the config's hierarchy."""
    model = gpu.student_t_matrix_model(8192, 2 ** 20, 8192, data_seed=data_seed(gpu, 5))
    fused_vs_exact(gpu, model, gpu.LevelPlan(2, 0, [2], c0=256))


def test_config3_shard_additivity_and_reproducibility(gpu):
    """Replication shards (rank r of 2 takes the 64-chunks q = r mod 2) add up
    to the single-rank level sums -- to fp32 rounding: each CTA keeps an fp32
    running sum over up to 32 of its samples, and the shards group the samples
    differently (1e-6, ten times tighter than the north-star bound) -- and a
    rerun with the same seed repeats them bit for bit."""
    model = gpu.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=data_seed(gpu, 3), dtype=1)
    plan = gpu.LevelPlan(2, 1, [160, 70], c0=64)
    one = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    again = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    shards = [gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER,
                              gpu.EstimatorOptions(engine="fused", rank=r, world=2)) for r in range(2)]
    for l, st in enumerate(one.per_level):
        assert np.array_equal(np.asarray(st.sum), np.asarray(again.per_level[l].sum))
        assert st.sum_of_squares == again.per_level[l].sum_of_squares
        tot = sum(np.asarray(s.per_level[l].sum, dtype=np.float64) for s in shards)
        assert sum(s.per_level[l].replication_count for s in shards) == st.replication_count
        assert frob_rel(tot, st.sum) <= 1e-6
        sq = sum(s.per_level[l].sum_of_squares for s in shards)
        assert abs(sq - st.sum_of_squares) <= 1e-6 * st.sum_of_squares
