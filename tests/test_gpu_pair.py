"""The CTA-pair tcgen05 GEMM (cta_group::2, M = 256 over two SMs) against the
single-CTA GEMM (MLSK_TC_PAIR=0) on the same draws: every output element is
the same K-ordered chain of tf32 MMAs into an fp32 accumulator whichever SM
pair computes its tile (with BF16 cross terms, the default, and with three
TF32 MMAs per K-step, MLSK_TC_BF16X=0), so the level sums must agree bit for
bit -- at the
BASELINE configs' full shapes (config 3, the symmetric config-4 Gram, config
5) and on the K-split and K-parallel paths."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MASTER = 20260823


def run(g, model, plan, env, opts=None):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return g.mlmc_matmul(model, g.target_identity(), plan, MASTER, opts or g.EstimatorOptions(engine="fused"))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def same(a, b):
    for sa, sb in zip(a.per_level, b.per_level):
        assert sa.replication_count == sb.replication_count
        assert np.array_equal(np.asarray(sa.sum), np.asarray(sb.sum)), sa.level
        assert sa.sum_of_squares == sb.sum_of_squares, sa.level


def ds(g, c):
    return g.RngStream.derive_seed(MASTER, 0xD47A0000 + c, 0)


@pytest.mark.parametrize("case", ["config3", "config4_sym", "config5", "ksplit", "kpar", "odd_rows"])
def test_pair_equals_single_cta(gpu, case):
    g = gpu
    env = {}
    if case == "config3":
        model = g.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=ds(g, 3), dtype=1)
        plan = g.LevelPlan(2, 1, [6, 3], c0=64)
    elif case == "config4_sym":
        model = g.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=ds(g, 4))
        plan = g.LevelPlan(2, 1, [3, 2], c0=128)
    elif case == "config5":
        model = g.student_t_matrix_model(8192, 2 ** 20, 8192, data_seed=ds(g, 5))
        plan = g.LevelPlan(2, 0, [2], c0=256)
    elif case == "ksplit":  # samples split along K (forced 1 MiB batches)
        model = g.gaussian_mean_matrix_model(512, 4096, 512, sd=1.0, data_seed=7, dtype=1)
        plan = g.LevelPlan(2, 1, [2, 2], c0=512)
        env = {"MLSK_SPLIT_MB": "1"}
    elif case == "kpar":  # one sample over the full 512-tile grid: K split over two CTA groups
        model = g.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=ds(g, 4))
        plan = g.LevelPlan(2, 0, [1], c0=512)
        env = {"MLSK_TC_SYM": "0"}
    else:  # an odd number of 128-row tiles: both settings run single CTAs
        model = g.gaussian_mean_matrix_model(384, 2048, 256, sd=1.0, data_seed=9, dtype=1)
        plan = g.LevelPlan(2, 1, [5, 3], c0=64)
    # default (cross terms a b_lo + a_lo b as BF16 MMAs) and with three TF32 MMAs per K-step
    pair = run(g, model, plan, dict(env))
    single = run(g, model, plan, dict(env, MLSK_TC_PAIR="0"))
    same(pair, single)
    pair3 = run(g, model, plan, dict(env, MLSK_TC_BF16X="0"))
    single3 = run(g, model, plan, dict(env, MLSK_TC_PAIR="0", MLSK_TC_BF16X="0"))
    same(pair3, single3)
    # the two forms: the same sums within the fp32 tolerance, not the same bits
    for sa, sb in zip(pair.per_level, pair3.per_level):
        a = np.asarray(sa.sum, dtype=np.float64).ravel()
        b = np.asarray(sb.sum, dtype=np.float64).ravel()
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b), sa.level
        assert abs(sa.sum_of_squares - sb.sum_of_squares) <= 1e-5 * sb.sum_of_squares
    assert not np.array_equal(np.asarray(pair.per_level[0].sum), np.asarray(pair3.per_level[0].sum))


def test_pair_random_shapes_vs_single_and_exact(gpu):
    """Seeded random shapes (m, p not multiples of the tile, c not a multiple
    of the K-chunk, several samples per CTA group): pair == single bit for bit,
    and both within the fp32 tolerance of the exact fp64-order engine."""
    g = gpu
    rng = np.random.default_rng(20261021)
    for _ in range(8):
        m = int(rng.integers(1, 9)) * 128 - int(rng.integers(0, 40))
        p = int(rng.integers(1, 5)) * 256 - int(rng.integers(0, 60))
        n = 1 << int(rng.integers(9, 13))
        c0 = int(rng.integers(3, 40))
        N = [int(rng.integers(1, 7)), int(rng.integers(1, 5))]
        model = g.gaussian_mean_matrix_model(m, n, p, sd=1.0, data_seed=int(rng.integers(1, 1 << 30)), dtype=1)
        plan = g.LevelPlan(2, 1, N, c0=c0)
        pair = run(g, model, plan, {})
        single = run(g, model, plan, {"MLSK_TC_PAIR": "0"})
        same(pair, single)
        pair3 = run(g, model, plan, {"MLSK_TC_BF16X": "0"})  # three TF32 MMAs per K-step
        same(pair3, run(g, model, plan, {"MLSK_TC_PAIR": "0", "MLSK_TC_BF16X": "0"}))
        ex = run(g, model, plan, {}, g.EstimatorOptions(engine="exact"))
        for r in (pair, pair3):
            for sf, se in zip(r.per_level, ex.per_level):
                a = np.asarray(sf.sum, dtype=np.float64).ravel()
                b = np.asarray(se.sum, dtype=np.float64).ravel()
                assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b), (m, n, p, c0, N, sf.level)
