"""fp32 configurations on the tcgen05 3xTF32 engine vs the exact-order
engine (fp64 arithmetic on the same fp32 draws) and the CPU oracle.
Tolerance (BASELINE.json north_star): 1e-5 relative, Frobenius norm."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL32 = 1e-5
MASTER = 20260823


def frob_rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def check(rf, re_, tol=TOL32):
    for sf, se in zip(rf.per_level, re_.per_level):
        assert sf.replication_count == se.replication_count
        assert frob_rel(sf.sum, se.sum) <= tol, (sf.level, frob_rel(sf.sum, se.sum))
        assert abs(sf.sum_of_squares - se.sum_of_squares) <= tol * se.sum_of_squares


def models(g):
    f32 = 1
    return {
        "gauss_f32": g.gaussian_mean_matrix_model(256, 4096, 384, sd=1.0, mean_lo=-1.0, mean_hi=1.0, data_seed=7,
                                                  dtype=f32),
        # m % 128 == 0 and p % 256 == 0: the generator's mean-prefetch path
        "gauss_f32_aligned": g.gaussian_mean_matrix_model(256, 4096, 512, sd=1.0, mean_lo=-1.0, mean_hi=1.0,
                                                          data_seed=8, dtype=f32),
        "student_t": g.student_t_matrix_model(256, 8192, 128, data_seed=9),
        "rff": g.rff_gram_model(256, 4096, dim=64, sigma=4.0, data_seed=11),
    }


@pytest.mark.parametrize("name", ["gauss_f32", "gauss_f32_aligned", "student_t", "rff"])
def test_tc_engine_vs_exact(gpu, name):
    model = models(gpu)[name]
    plan = gpu.LevelPlan(2, 2, [37, 20, 9], c0=64)
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    check(rf, re_)


def test_tc_gauss_vs_oracle(gpu, oracle):
    model = gpu.gaussian_mean_matrix_model(128, 1024, 128, sd=1.0, mean_lo=-1.0, mean_hi=1.0, data_seed=3, dtype=1)
    plan = gpu.LevelPlan(2, 1, [5, 3], c0=64)
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    o = oracle.OracleModel(model.desc()).mlmc(2, 64, [5, 3], MASTER)
    for l, st in enumerate(rf.per_level):
        assert frob_rel(st.sum, o.level_sum[l]) <= TOL32
        assert abs(st.sum_of_squares - o.level_sumsq[l]) <= TOL32 * o.level_sumsq[l]


def test_tc_probe_indices_match_exact(gpu):
    model = models(gpu)["gauss_f32"]
    plan = gpu.LevelPlan(2, 1, [4, 3], c0=64)
    seen = {"fused": [], "exact": []}
    for eng in seen:
        gpu.mlmc_matmul(model, gpu.target_identity(), plan, 5,
                        gpu.EstimatorOptions(engine=eng, probe=lambda l, k, f, c, e=eng: seen[e].append((l, k, f))))
    assert seen["fused"] == seen["exact"] and len(seen["fused"]) == 3


@pytest.mark.parametrize("name", ["gauss_f32", "gauss_f32_aligned", "student_t", "rff"])
def test_tc_samples_split_along_k(gpu, name, monkeypatch):
    """Level-samples whose panels exceed a batch run as K-segments of one
    sample with the partial Y carried in device memory (BASELINE config 5's
    deep levels: one sample of c = 262144 is 34 GB of panels).  A 1 MiB batch
    budget forces the split at test shapes; the result must match the exact
    engine like the unsplit one does."""
    model = models(gpu)[name]
    plan = gpu.LevelPlan(2, 2, [5, 3, 2], c0=256)  # c = 256, 512, 1024 -> 1 .. 8 segments per sample
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    monkeypatch.setenv("MLSK_PANEL_BUDGET_MB", "1")
    monkeypatch.setenv("MLSK_SPLIT_MB", "1")
    rs = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    check(rs, re_)


def test_tc_direct_accumulation_one_cta_per_tile(gpu):
    """Outputs with >= 148 tiles and tile-aligned shapes (configs 4 and 5) put
    one CTA per tile, which adds its running sums straight into the level
    total (no partial buffer / reduction pass)."""
    model = gpu.gaussian_mean_matrix_model(1536, 2048, 2560, sd=1.0, data_seed=17, dtype=1)  # 12 x 10 tiles
    plan = gpu.LevelPlan(2, 1, [6, 3], c0=32)
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    check(rf, re_)


def test_tc_kparallel_single_sample(gpu):
    """One level-sample over a direct-mode tile grid with a poorly filled last
    CTA wave (160 tiles on 148 SMs) runs as two K-halves on two CTA groups
    whose partial Y are combined afterwards; single-sample levels take that
    path, the multi-sample level the ordinary one."""
    model = gpu.gaussian_mean_matrix_model(1280, 4096, 4096, sd=1.0, data_seed=19, dtype=1)  # 10 x 16 tiles
    plan = gpu.LevelPlan(2, 2, [3, 1, 1], c0=256)  # c = 256 (16 K-chunks), 512, 1024
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    check(rf, re_)


@pytest.mark.parametrize("points", [512, 2560, 384])
def test_tc_symmetric_gram(gpu, points, monkeypatch):
    """RFF Gram estimates are symmetric (B = diag(w) A^T): the engine runs only
    the 256 x 256 blocks on and above the diagonal, counts the off-diagonal
    ones twice in ||Y||^2 and mirrors the level total.  512 points: partial
    buffer + reduction; 2560: one CTA per tile (direct); 384 (not a multiple
    of 256): the full tile grid.  Results match the exact engine and the
    full-grid run (MLSK_TC_SYM=0), and the level sums are exactly symmetric
    (the mirror also copies the upper half of the diagonal blocks)."""
    model = gpu.rff_gram_model(points, 4096, dim=64, sigma=4.0, data_seed=23)
    plan = gpu.LevelPlan(2, 2, [9, 5, 3], c0=128)
    rf = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    re_ = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    check(rf, re_)
    # n / c a power of two: the GEMM reads B from the A panel (negated coarse
    # prefix, Y scaled by |w|) -- the same bits as the separate B panel.  (With
    # merged sampled columns the two differ in how a repeated column enters --
    # scaled by sqrt(reps) vs weighted, tests/test_gpu_merge.py -- so the bit identity is a
    # property of the unmerged contraction.)
    # (and of the TF32 / BF16 operand forms: with FP16 pairs, the default for these bounded
    # features, scaling by |w| moves entries across the fp16 subnormal boundary, so the two
    # panels agree to the fp32 tolerance but not bit for bit)
    monkeypatch.setenv("MLSK_MERGE", "0")
    rsh16 = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    monkeypatch.setenv("MLSK_TC_H16", "0")
    rsh = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    check(rsh16, rsh)
    monkeypatch.setenv("MLSK_TC_SHARED", "0")
    rsep = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    for a, b in zip(rsh.per_level, rsep.per_level):
        assert np.array_equal(np.asarray(a.sum), np.asarray(b.sum))
        assert a.sum_of_squares == b.sum_of_squares
    check(rf, rsh)
    monkeypatch.setenv("MLSK_TC_SYM", "0")
    rfull = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused"))
    check(rsh, rfull, tol=1e-6)
    if points % 256 == 0:
        for st in list(rf.per_level) + list(rsh.per_level):
            s = np.asarray(st.sum)
            assert np.array_equal(s, s.T)
