"""Parity over the configs' FULL level hierarchies:
every level of BASELINE configs 2-5 on the fused engine against the CPU
oracle, and the config-4 / config-5 data models (random Fourier features,
Student-t(3)) against the oracle on both device engines.

Configs 3-5 are far too large for a full oracle run, so the deep levels are
checked through a size-independent property of the estimator: the level sum
of a round of k level-samples is the sum of the k per-sample Y, and any
row / column subset of Y can be formed on the CPU from the sampled rows of
A_S and columns of B_S alone (`OracleModel.y_subset`, oracle/mlsk_oracle.c
orc_sample_y_subset, which follows estimators.cpp:137-147 and
sketch.cpp:45-77).  Each level runs as its own round of a session with
exactly the level's samples, so the kernels take the code paths they take
in production at that level: the K-parallel single-sample path of config 4
(c >= 8192) and the K-split path of config 5 (panels > 8 GiB per sample at
c >= 131072).

Tolerances (BASELINE.json north_star): 1e-12 relative (Frobenius) for fp64,
1e-5 for the fp32 configs."""
import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi

pytestmark = pytest.mark.gpu

MASTER = 20260823
TOL64, TOL32 = 1e-12, 1e-5


def frob_rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def data_seed(g, config):
    return g.RngStream.derive_seed(MASTER, 0xD47A0000 + config, 0)


def subset(extent, count, seed):
    """`count` sorted row (column) numbers: both ends of the range plus random
    ones, so every output tile row / column band can be hit."""
    rng = np.random.default_rng(seed)
    pick = set([0, 1, extent - 2, extent - 1])
    pick.update(rng.choice(extent, size=min(extent, count) - len(pick), replace=False).tolist())
    return np.array(sorted(pick)[:count], dtype=np.int64)


def level_rounds(g, model, c0, L, dN, engine="fused"):
    """One session; level l runs as a round of its own with dN[l] samples."""
    s = g.MlmcSession(model, g.target_identity(), 2, L, MASTER, c0=c0, options=g.EstimatorOptions(engine=engine))
    for l in range(L + 1):
        one = [0] * (L + 1)
        one[l] = dN[l]
        s.run_round(one)
    r = s.stats()
    s.close()
    return r


def check_subsets(oracle, model, r, c0, dN, rows_per, tol, seed0=0):
    om = oracle.OracleModel(model.desc())
    rows_total, cols_total = om.rows, om.cols
    worst = 0.0
    for l, st in enumerate(r.per_level):
        if dN[l] == 0:
            continue
        assert st.replication_count == dN[l]
        c = c0 * 2 ** l
        rows = subset(rows_total, rows_per, seed0 + 2 * l)
        cols = subset(cols_total, rows_per, seed0 + 2 * l + 1)
        want = sum(om.y_subset(MASTER, l, k, c, c // 2 if l > 0 else 0, rows, cols) for k in range(dN[l]))
        got = np.asarray(st.sum, dtype=np.float64)[np.ix_(rows, cols)]
        err = frob_rel(got, want)
        worst = max(worst, err)
        assert err <= tol, (l, c, err)
    return worst


# ------------------------------------------------------------ config 2 (fp64)


def config2(g):
    return g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, mean_lo=-1.0, mean_hi=1.0, data_seed=data_seed(g, 2))


def test_config2_all_levels_fused_vs_exact_and_oracle(gpu, oracle):
    """Levels 0-6 (c = 32 ... 2048), a few samples each, one plan: the fused
    DMMA engine against the exact-order engine and the oracle (whole level
    sums and ||Y||^2 sums, 1e-12)."""
    model = config2(gpu)
    N = [5, 4, 3, 3, 2, 2, 2]
    plan = gpu.LevelPlan(2, 6, N, c0=32)
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 32, N, MASTER)
    for l, (sf, se) in enumerate(zip(rf.per_level, re_.per_level)):
        assert sf.replication_count == se.replication_count == o.level_count[l]
        # the exact engine is the oracle's arithmetic order on the device: bit for bit
        assert np.array_equal(np.asarray(se.sum).ravel(), o.level_sum[l]), l
        assert se.sum_of_squares == o.level_sumsq[l], l
        assert frob_rel(sf.sum, o.level_sum[l]) <= TOL64, (l, frob_rel(sf.sum, o.level_sum[l]))
        assert abs(sf.sum_of_squares - o.level_sumsq[l]) <= TOL64 * o.level_sumsq[l], l
    assert frob_rel(rf.value, o.value) <= TOL64


def test_config2_deep_levels_single_rounds(gpu, oracle):
    """Each level as its own round (the adaptive driver's top-up rounds):
    subsets of the level sums against the per-sample oracle."""
    model = config2(gpu)
    dN = [3, 3, 2, 2, 1, 1, 1]
    r = level_rounds(gpu, model, 32, 6, dN)
    check_subsets(oracle, model, r, 32, dN, 48, TOL64)


# ------------------------------------------------------- configs 3-5 (fp32)


def test_config3_all_levels_vs_oracle(gpu, oracle):
    """A 1024 x 16384, B 16384 x 1024 fp32, levels 0-8 (c = 64 ... 16384)."""
    model = gpu.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=data_seed(gpu, 3), dtype=abi.F32)
    dN = [2] * 9
    r = level_rounds(gpu, model, 64, 8, dN)
    check_subsets(oracle, model, r, 64, dN, 64, TOL32)


def test_config4_all_levels_vs_oracle(gpu, oracle):
    """RFF Gram, 4096 points in R^64, 2^16 features, levels 0-9 (c = 128 ...
    65536); one sample per level: the symmetric-tile, shared-panel and (c >=
    8192) K-parallel paths.  Rows and columns are drawn independently, so both
    the computed upper and the mirrored lower triangle are checked."""
    model = gpu.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=data_seed(gpu, 4))
    dN = [1] * 10
    r = level_rounds(gpu, model, 128, 9, dN)
    check_subsets(oracle, model, r, 128, dN, 48, TOL32)


def test_config4_two_sample_levels_vs_oracle(gpu, oracle):
    """Two samples per level (the ordinary multi-sample path at every c)."""
    model = gpu.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=data_seed(gpu, 4))
    dN = [2, 2, 0, 0, 0, 2, 0, 0, 2, 2]
    r = level_rounds(gpu, model, 128, 9, dN)
    check_subsets(oracle, model, r, 128, dN, 32, TOL32, seed0=100)


def test_config5_all_levels_vs_oracle(gpu, oracle):
    """A 8192 x 2^20, B 2^20 x 8192 Student-t(3) + U(-0.5, 0.5) means,
    levels 0-10 (c = 256 ... 262144), one sample per level; c >= 131072 runs
    as K-segments of up to 8 GiB of panels with the partial Y carried."""
    model = gpu.student_t_matrix_model(8192, 2 ** 20, 8192, data_seed=data_seed(gpu, 5))
    dN = [1] * 11
    r = level_rounds(gpu, model, 256, 10, dN)
    check_subsets(oracle, model, r, 256, dN, 32, TOL32)


# ------------------------------------------- config-4 / config-5 data models


def student_t_small(g):
    return g.student_t_matrix_model(192, 8192, 160, data_seed=data_seed(g, 5))


def rff_small(g):
    return g.rff_gram_model(320, 4096, dim=64, sigma=4.0, data_seed=data_seed(g, 4))


def test_student_t_exact_engine_bitexact_vs_oracle(gpu, oracle):
    """Student-t(3) draws use only correctly rounded fp32 operations and the
    spec's table-driven log / sincos (include/mlsk_stream_spec.h), so the
    device's exact engine reproduces the oracle bit for bit."""
    model = student_t_small(gpu)
    N = [9, 5, 3]
    r = gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 2, N, c0=64), MASTER,
                        gpu.EstimatorOptions(engine="exact"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 64, N, MASTER)
    for l, st in enumerate(r.per_level):
        assert np.array_equal(np.asarray(st.sum).ravel(), o.level_sum[l]), l
        assert st.sum_of_squares == o.level_sumsq[l], l
    idx_g, a_g, b_g = gpu.draw_sample(model, MASTER, 2, 1, 256)
    idx_o, a_o, b_o = oracle.OracleModel(model.desc()).draw(MASTER, 2, 1, 256)
    assert np.array_equal(idx_g, idx_o) and np.array_equal(a_g, a_o) and np.array_equal(b_g, b_o)


def test_student_t_fused_vs_oracle(gpu, oracle):
    model = student_t_small(gpu)
    N = [9, 5, 3]
    r = gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 2, N, c0=64), MASTER,
                        gpu.EstimatorOptions(engine="fused"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 64, N, MASTER)
    for l, st in enumerate(r.per_level):
        assert frob_rel(st.sum, o.level_sum[l]) <= TOL32, l
        assert abs(st.sum_of_squares - o.level_sumsq[l]) <= TOL32 * o.level_sumsq[l], l


def test_rff_exact_engine_bitexact_vs_oracle(gpu, oracle):
    """RFF features sqrt(2/n) cos(w.x + b) on the exact engine: the dot
    product in fp64 in the oracle's order and glibc's cos restated on the
    device (mlsk_libm.cuh), so draws and level sums are the oracle's bit for
    bit."""
    model = rff_small(gpu)
    N = [7, 4, 2]
    r = gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 2, N, c0=128), MASTER,
                        gpu.EstimatorOptions(engine="exact"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 128, N, MASTER)
    for l, st in enumerate(r.per_level):
        assert np.array_equal(np.asarray(st.sum).ravel(), o.level_sum[l]), (l, frob_rel(st.sum, o.level_sum[l]))
        assert st.sum_of_squares == o.level_sumsq[l], l
    idx_g, a_g, b_g = gpu.draw_sample(model, MASTER, 1, 3, 512)
    idx_o, a_o, b_o = oracle.OracleModel(model.desc()).draw(MASTER, 1, 3, 512)
    assert np.array_equal(idx_g, idx_o) and np.array_equal(a_g, a_o) and np.array_equal(b_g, b_o)


def test_rff_fused_vs_oracle(gpu, oracle):
    model = rff_small(gpu)
    N = [7, 4, 2]
    r = gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 2, N, c0=128), MASTER,
                        gpu.EstimatorOptions(engine="fused"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 128, N, MASTER)
    for l, st in enumerate(r.per_level):
        assert frob_rel(st.sum, o.level_sum[l]) <= TOL32, (l, frob_rel(st.sum, o.level_sum[l]))
        assert abs(st.sum_of_squares - o.level_sumsq[l]) <= TOL32 * o.level_sumsq[l], l
