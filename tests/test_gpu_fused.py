"""Fused tensor-core engine vs the exact-order engine and the oracle.

Tolerance (BASELINE.json north_star): per-level estimates within 1e-12
relative in the Frobenius norm for the fp64 configs; indices bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MASTER = 20260823
TOL = 1e-12


def frob_rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / den if den > 0 else np.linalg.norm(a - b)


def compare_reports(rf, re_, tol=TOL):
    assert len(rf.per_level) == len(re_.per_level)
    for sf, se in zip(rf.per_level, re_.per_level):
        assert sf.replication_count == se.replication_count
        assert sf.cost_units == se.cost_units
        assert frob_rel(sf.sum, se.sum) <= tol, (sf.level, frob_rel(sf.sum, se.sum))
        assert abs(sf.sum_of_squares - se.sum_of_squares) <= tol * abs(se.sum_of_squares)
    assert frob_rel(rf.value, re_.value) <= tol


def config2_model(gpu, m=256, n=4096, p=256):
    return gpu.gaussian_mean_matrix_model(m, n, p, sd=0.5, mean_lo=-1.0, mean_hi=1.0,
                                          data_seed=gpu.RngStream.derive_seed(MASTER, 0xD47A0002, 0))


def test_config1_fused_vs_exact(gpu):
    model = gpu.gaussian_mean_model(4096, sd=1.0, data_seed=gpu.RngStream.derive_seed(MASTER, 0xD47A0001, 0))
    plan = gpu.LevelPlan(2, 5, [8192, 4096, 2048, 1024, 512, 256], c0=8)
    rf = gpu.mlmc_inner(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_inner(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    compare_reports(rf, re_)


def test_config2_fused_vs_exact(gpu):
    model = config2_model(gpu)
    plan = gpu.LevelPlan(2, 3, [40, 24, 9, 5], c0=32)
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    compare_reports(rf, re_)


def test_config2_fused_vs_oracle(gpu, oracle):
    model = config2_model(gpu)
    plan = gpu.LevelPlan(2, 2, [3, 2, 2], c0=32)
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 32, list(plan.N), MASTER)
    for l, st in enumerate(rf.per_level):
        assert frob_rel(st.sum, o.level_sum[l]) <= TOL
        assert abs(st.sum_of_squares - o.level_sumsq[l]) <= TOL * o.level_sumsq[l]


@pytest.mark.parametrize("shape", [(100, 1000, 70), (1, 37, 1), (130, 4096, 65)])
def test_fused_padding_shapes(gpu, shape):
    m, n, p = shape
    model = gpu.gaussian_mean_matrix_model(m, n, p, sd=0.5, data_seed=11)
    for M, c0, L in [(3, 1, 3), (2, 5, 2)]:
        plan = gpu.LevelPlan(M, L, [70] + [33] * L, c0=c0)
        rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, 9, gpu.EstimatorOptions(engine="fused"))
        re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, 9, gpu.EstimatorOptions(engine="exact"))
        compare_reports(rf, re_)


def test_fused_probe_indices_match_exact(gpu):
    model = config2_model(gpu, 64, 4096, 64)
    plan = gpu.LevelPlan(2, 2, [5, 4, 3], c0=32)
    seen = {"fused": [], "exact": []}
    for eng in seen:
        probe = lambda l, k, fine, coarse, e=eng: seen[e].append((l, k, fine, coarse))
        gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER,
                        gpu.EstimatorOptions(engine=eng, probe=probe))
    assert seen["fused"] == seen["exact"]
    assert len(seen["fused"]) == 4 + 3
    for l, k, fine, coarse in seen["fused"]:
        assert len(fine) == 32 * 2 ** l and coarse == fine[: len(fine) // 2]


def test_rank_sharding_sums(gpu):
    model = config2_model(gpu, 128, 4096, 64)
    plan = gpu.LevelPlan(2, 2, [300, 150, 70], c0=32)
    full = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER)
    parts = [gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER,
                             gpu.EstimatorOptions(rank=r, world=2)) for r in range(2)]
    for l in range(3):
        s = parts[0].per_level[l].sum + parts[1].per_level[l].sum
        assert frob_rel(s, full.per_level[l].sum) <= 1e-13
        assert parts[0].per_level[l].replication_count + parts[1].per_level[l].replication_count == plan.N[l]


@pytest.mark.parametrize("world", [2, 3])
def test_inner_rank_sharding_sums(gpu, world):
    """Config-1 shape (one launch for all levels, replication lists from
    per-chunk runs when sharded): the shards' level sums add up to the
    unsharded run, counts exactly."""
    model = gpu.gaussian_mean_model(4096, sd=1.0, data_seed=gpu.RngStream.derive_seed(MASTER, 0xD47A0001, 0))
    plan = gpu.LevelPlan(2, 3, [1000, 700, 300, 130], c0=8)
    opts = gpu.EstimatorOptions(engine="fused")
    full = gpu.mlmc_inner(model, gpu.target_identity(), plan, MASTER, opts)
    parts = [gpu.mlmc_inner(model, gpu.target_identity(), plan, MASTER,
                            gpu.EstimatorOptions(engine="fused", rank=r, world=world)) for r in range(world)]
    for l in range(4):
        s = sum(p.per_level[l].sum for p in parts)
        assert abs(s - full.per_level[l].sum) <= 1e-13 * abs(full.per_level[l].sum)
        assert sum(p.per_level[l].replication_count for p in parts) == plan.N[l]


def test_session_rounds_equal_single_run(gpu):
    model = config2_model(gpu, 128, 4096, 64)
    sess = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, MASTER, c0=32)
    sess.run_round([100, 50, 20])
    sess.run_round([60, 30, 13])
    r1 = sess.stats()
    r2 = gpu.mlmc_matmul(model, gpu.target_identity(), gpu.LevelPlan(2, 2, [160, 80, 33], c0=32), MASTER)
    compare_reports(r1, r2, tol=1e-13)
    sess.close()


def test_fused_f64_samples_split_along_k(gpu, monkeypatch):
    """fp64 level-samples larger than a panel batch run as K-segments with the
    partial Y carried in device memory; forced here by a 1 MiB batch budget."""
    model = gpu.gaussian_mean_matrix_model(256, 4096, 192, sd=0.5, data_seed=21)
    plan = gpu.LevelPlan(2, 2, [5, 3, 2], c0=256)  # per-sample panels 2 .. 8 MiB
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, 13, gpu.EstimatorOptions(engine="exact"))
    monkeypatch.setenv("MLSK_PANEL_BUDGET_MB", "1")
    monkeypatch.setenv("MLSK_SPLIT_MB", "1")
    rs = gpu.mlmc_matmul(model, gpu.target_identity(), plan, 13, gpu.EstimatorOptions(engine="fused"))
    compare_reports(rs, re_)
