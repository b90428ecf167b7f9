"""Merged sampled columns (mlsk_internal.h KRange, mlsk_fused.cu pre-pass).

A level-sample's contraction sum_t w_t a_{j_t} b_{j_t}^T runs over the
DISTINCT sampled columns with summed weights (a duplicated index gathers the
same drawn column, sketch.cpp:60-71; for M = 2 a column drawn once in the
coarse prefix and once in the suffix cancels).  The result is the same sum
in another order, so the merged engines must agree with the unmerged ones
and with the exact-order engine within the parity tolerances, on every
engine, both list modes and the K-split path."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi
from paper_1904_00429_b200 import _lib

pytestmark = pytest.mark.gpu

MASTER = 20260823
TOL64, TOL32 = 1e-12, 1e-5


def frob_rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


class env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        for k, v in self.kv.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def profiled_names(fn):
    """Runs fn with the library's per-kernel profile on; returns (result, {name: launches})."""
    L = _lib.lib()
    L.mlsk_profile_reset()
    L.mlsk_profile_enable(1)
    try:
        out = fn()
    finally:
        L.mlsk_profile_enable(0)
    name = C.create_string_buffer(64)
    nl, ms = C.c_int64(), C.c_double()
    names = {}
    n = L.mlsk_profile_read(0, name, 64, C.byref(nl), C.byref(ms))
    for i in range(n):
        L.mlsk_profile_read(i, name, 64, C.byref(nl), C.byref(ms))
        names[name.value.decode()] = nl.value
    return out, names


def run(g, model, M, L, N, c0, engine="fused"):
    return g.mlmc_matmul(model, g.target_identity(), g.LevelPlan(M, L, N, c0=c0), MASTER,
                         g.EstimatorOptions(engine=engine))


def three_way(g, model, M, L, N, c0, tol, extra_env=None, exact=True):
    """merged (every level that qualifies) vs unmerged vs the exact engine"""
    kv = dict(extra_env or {})
    with env(MLSK_MERGE=None, MLSK_MERGE_MIN_DEN=1 << 30, **kv):
        rm, names = profiled_names(lambda: run(g, model, M, L, N, c0))
    assert "merge_columns" in names, names
    with env(MLSK_MERGE=0, **kv):
        ru, names_u = profiled_names(lambda: run(g, model, M, L, N, c0))
    assert "merge_columns" not in names_u
    re_ = run(g, model, M, L, N, c0, engine="exact") if exact else None
    for l in range(L + 1):
        sm, su = rm.per_level[l], ru.per_level[l]
        assert sm.replication_count == su.replication_count == N[l]
        assert frob_rel(sm.sum, su.sum) <= tol, (l, frob_rel(sm.sum, su.sum))
        assert abs(sm.sum_of_squares - su.sum_of_squares) <= tol * su.sum_of_squares, l
        if exact:
            se = re_.per_level[l]
            assert frob_rel(sm.sum, se.sum) <= tol, (l, frob_rel(sm.sum, se.sum))
            assert abs(sm.sum_of_squares - se.sum_of_squares) <= tol * se.sum_of_squares, l
    assert frob_rel(rm.value, ru.value) <= tol
    return rm, ru


def test_merge_fp64_gauss(gpu):
    """fp64 DMMA engine, c up to n (levels 0-4 of c0 = 64 over n = 1024)."""
    model = gpu.gaussian_mean_matrix_model(192, 1024, 160, sd=0.5, data_seed=11)
    three_way(gpu, model, 2, 4, [5, 4, 3, 3, 2], 64, TOL64)


def test_merge_fp64_general_weights(gpu):
    """M = 3 (w_coarse = -2 w_fine: weights cancel only when cnt_f = 2 cnt_c)
    and n not a power of two (cumulative-table index draw)."""
    model = gpu.gaussian_mean_matrix_model(130, 1000, 70, sd=0.5, data_seed=12)
    three_way(gpu, model, 3, 2, [4, 3, 3], 100, TOL64)


def test_merge_fp64_sample_groups(gpu):
    """the count scratch bounded to 1 MiB: the pre-pass runs in groups of samples"""
    model = gpu.gaussian_mean_matrix_model(64, 4096, 64, sd=0.5, data_seed=13)
    three_way(gpu, model, 2, 2, [70, 40, 33], 256, TOL64, extra_env={"MLSK_MERGE_GROUP_MB": 1}, exact=False)


def test_merge_passes(gpu):
    """the lists bounded to 1 MiB: the round runs as several passes over slices of every level's samples"""
    model = gpu.gaussian_mean_matrix_model(64, 4096, 64, sd=0.5, data_seed=13)
    three_way(gpu, model, 2, 2, [150, 90, 77], 256, TOL64, extra_env={"MLSK_MERGE_LIST_MB": 1}, exact=False)
    model32 = gpu.gaussian_mean_matrix_model(256, 2048, 256, sd=1.0, data_seed=14, dtype=abi.F32)
    three_way(gpu, model32, 2, 3, [40, 30, 20, 10], 256, TOL32, extra_env={"MLSK_MERGE_LIST_MB": 1}, exact=False)


def test_merge_fp32_gauss(gpu):
    model = gpu.gaussian_mean_matrix_model(256, 2048, 512, sd=1.0, data_seed=14, dtype=abi.F32)
    three_way(gpu, model, 2, 4, [4, 3, 3, 2, 2], 128, TOL32)


def test_merge_student_t(gpu):
    model = gpu.student_t_matrix_model(256, 4096, 256, data_seed=15)
    three_way(gpu, model, 2, 3, [3, 3, 2, 2], 512, TOL32)


def test_merge_student_t_k_split(gpu):
    """samples split along K (forced at this size): the segments walk the merged list"""
    model = gpu.student_t_matrix_model(256, 4096, 256, data_seed=16)
    three_way(gpu, model, 2, 2, [2, 2, 2], 1024, TOL32, extra_env={"MLSK_SPLIT_MB": 1})


def test_merge_rff_shared_panel(gpu):
    """RFF Gram on the symmetric tile grid with the shared A / B panel (n, c
    powers of two): sign groups of scaled columns (mode 2), the negated
    leading chunks per sample."""
    model = gpu.rff_gram_model(512, 4096, dim=64, sigma=4.0, data_seed=17)
    rm, ru = three_way(gpu, model, 2, 5, [3, 3, 2, 2, 2, 2], 128, TOL32)
    v = np.asarray(rm.value)
    assert np.array_equal(v, v.T)  # the mirrored estimate is exactly symmetric


def test_merge_rff_separate_panels(gpu):
    """the same with a separate B panel (summed weights folded into B, mode 1)"""
    model = gpu.rff_gram_model(512, 4096, dim=64, sigma=4.0, data_seed=17)
    three_way(gpu, model, 2, 5, [2, 2, 2, 2, 2, 2], 128, TOL32, extra_env={"MLSK_TC_SHARED": 0}, exact=False)


def test_merge_rff_full_grid(gpu):
    """320 points: no symmetric grid, no shared panel"""
    model = gpu.rff_gram_model(320, 4096, dim=64, sigma=4.0, data_seed=18)
    # (no exact-engine leg: at c0 = 512 the fp32 feature phases alone put the level-0
    # sum of squares 1.3e-5 from the fp64 engine's, merged or not)
    three_way(gpu, model, 2, 3, [2, 2, 2, 2], 512, TOL32, exact=False)


def test_merge_default_threshold(gpu):
    """default: only the levels where merging saves K-chunks merge (mlsk_fused.cu merge_pays: at
    c = 256 of n = 4096 the ~244 surviving columns still take 16 chunks, at c = 512 the ~467
    take 30-31 of 32); the other levels are untouched bit for bit"""
    model = gpu.gaussian_mean_matrix_model(128, 4096, 128, sd=0.5, data_seed=19)
    N = [3, 3, 2]
    with env(MLSK_MERGE=None, MLSK_MERGE_MIN_DEN=None):
        rm, names = profiled_names(lambda: run(gpu, model, 2, 2, N, 128))  # c = 128, 256, 512: only 512
    assert "merge_columns" in names
    with env(MLSK_MERGE=0):
        ru = run(gpu, model, 2, 2, N, 128)
    for l in (0, 1):
        assert np.array_equal(np.asarray(rm.per_level[l].sum), np.asarray(ru.per_level[l].sum))
    assert frob_rel(rm.per_level[2].sum, ru.per_level[2].sum) <= TOL64
    assert not np.array_equal(np.asarray(rm.per_level[2].sum), np.asarray(ru.per_level[2].sum))


def test_merge_rank_shards_add_up(gpu):
    """64-replication chunk sharding (rank / world) with merged columns: the two ranks'
    level sums add up to the single-rank run (each sample's list depends on (seed, l, k) only)."""
    model = gpu.gaussian_mean_matrix_model(96, 2048, 80, sd=0.5, data_seed=21)
    N = [200, 150, 130]
    plan = gpu.LevelPlan(2, 2, N, c0=256)
    with env(MLSK_MERGE=None, MLSK_MERGE_MIN_DEN=1 << 30):
        one, names = profiled_names(
            lambda: gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="fused")))
        parts = [gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER,
                                 gpu.EstimatorOptions(engine="fused", rank=r, world=2)) for r in range(2)]
    assert "merge_columns" in names
    for l in range(3):
        assert parts[0].per_level[l].replication_count + parts[1].per_level[l].replication_count == N[l]
        s = np.asarray(parts[0].per_level[l].sum) + np.asarray(parts[1].per_level[l].sum)
        assert frob_rel(s, one.per_level[l].sum) <= TOL64
        sq = parts[0].per_level[l].sum_of_squares + parts[1].per_level[l].sum_of_squares
        assert abs(sq - one.per_level[l].sum_of_squares) <= TOL64 * one.per_level[l].sum_of_squares


def test_merge_single_level_mc(gpu):
    """the single-level MC baseline (no coarse prefix: duplicates merge, nothing cancels)"""
    model = gpu.gaussian_mean_matrix_model(128, 1024, 128, sd=0.5, data_seed=22)
    kw = dict(L=3, N=12, M=2, seed=MASTER, c0=128)  # s = 128 * 2^3 = 1024 = n
    with env(MLSK_MERGE=None, MLSK_MERGE_MIN_DEN=None):
        rm, names = profiled_names(lambda: gpu.mc_matmul(model, gpu.target_identity(), options=gpu.EstimatorOptions(engine="fused"), **kw))
    assert "merge_columns" in names
    with env(MLSK_MERGE=0):
        ru = gpu.mc_matmul(model, gpu.target_identity(), options=gpu.EstimatorOptions(engine="fused"), **kw)
    re_ = gpu.mc_matmul(model, gpu.target_identity(), options=gpu.EstimatorOptions(engine="exact"), **kw)
    assert frob_rel(rm.value, ru.value) <= TOL64 and frob_rel(rm.value, re_.value) <= TOL64
    assert not np.array_equal(np.asarray(rm.value), np.asarray(ru.value))


def test_contraction_columns_counter(gpu):
    """mlsk_contraction_columns: executed K-columns (whole chunks) vs sampled indices of this
    thread's GEMMs -- equal to the chunk-padded sampled count when merging is off, the expected
    fraction n (1 - e^-l I_0(l)) / c (here c = n: 0.534) when it is on."""
    L = _lib.lib()
    model = gpu.gaussian_mean_matrix_model(64, 1024, 64, sd=0.5, data_seed=23)
    N, c0 = [0, 0, 0, 0, 6], 64  # only level 4: c = 1024 = n
    cols = (C.c_int64 * 2)()

    def one_round():
        s = gpu.MlmcSession(model, gpu.target_identity(), 2, 4, MASTER, c0=c0,
                            options=gpu.EstimatorOptions(engine="fused"))
        s.run_round(N)
        s.stats()
        s.close()

    with env(MLSK_MERGE=0):
        L.mlsk_contraction_columns(cols, 1)
        one_round()
        L.mlsk_contraction_columns(cols, 1)
    assert cols[0] == cols[1] == 6 * 1024
    with env(MLSK_MERGE=None, MLSK_MERGE_MIN_DEN=None):
        one_round()
        L.mlsk_contraction_columns(cols, 1)
    assert cols[1] == 6 * 1024
    frac = cols[0] / cols[1]
    assert 0.50 < frac < 0.60, frac  # 0.534 expected, + chunk padding and the maximum over 6 samples
