"""Exact-order engine on the device vs the CPU oracle (bit-exact where the
draws are bit-exact: philox stream, and reference stream for models whose
draw needs no libm transcendental)."""
import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi

pytestmark = pytest.mark.gpu

MASTER = 20260823


def _oracle_model(oracle, model):
    d = model.desc()
    return oracle.OracleModel(d)


def _levels_equal(r_gpu, r_orc, exact=True, rtol=0.0):
    for l, st in enumerate(r_gpu.per_level):
        g = np.atleast_1d(np.asarray(st.sum, dtype=np.float64)).ravel()
        o = r_orc.level_sum[l]
        if exact:
            assert np.array_equal(g, o), (l, g[:4], o[:4])
            assert st.sum_of_squares == r_orc.level_sumsq[l], l
        else:
            np.testing.assert_allclose(g, o, rtol=rtol, atol=0)
            np.testing.assert_allclose(st.sum_of_squares, r_orc.level_sumsq[l], rtol=rtol)
        assert st.replication_count == r_orc.level_count[l]
        assert st.cost_units == r_orc.cost_units[l]


def test_config1_philox_exact_bitexact(gpu, oracle):
    model = gpu.gaussian_mean_model(4096, sd=1.0, mean_lo=0.0, mean_hi=1.0,
                                    data_seed=gpu.RngStream.derive_seed(MASTER, 0xD47A0001, 0))
    plan = gpu.LevelPlan(2, 5, [130, 70, 64, 33, 9, 5], c0=8)
    r = gpu.mlmc_inner(model, gpu.target_identity(), plan, MASTER,
                       gpu.EstimatorOptions(engine="exact"))
    o = _oracle_model(oracle, model).mlmc(2, 8, list(plan.N), MASTER)
    _levels_equal(r, o)
    assert r.value == o.value[0]


def test_config1_ref_stream_indices_bitexact(gpu, oracle):
    model = gpu.gaussian_mean_model(4096, sd=1.0, data_seed=77, stream="ref")
    om = _oracle_model(oracle, model)
    for (tag, k, c) in [(0, 0, 8), (3, 5, 64), (5, 63, 256)]:
        i_g, a_g, b_g = gpu.draw_sample(model, MASTER, tag, k, c)
        i_o, a_o, b_o = om.draw(MASTER, tag, k, c)
        assert np.array_equal(i_g, i_o)
        # glibc's log / sin / cos restated on the device (mlsk_libm.cuh): bit for bit
        assert np.array_equal(a_g, a_o) and np.array_equal(b_g, b_o)
    plan = gpu.LevelPlan(2, 3, [100, 64, 40, 10], c0=8)
    r = gpu.mlmc_inner(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    o = om.mlmc(2, 8, list(plan.N), MASTER)
    _levels_equal(r, o)


def test_ref_stream_normals_bitexact_at_scale(gpu, oracle):
    """Reference-stream Box-Muller normals (rng.hpp:55-65: sqrt(-2 log u),
    2 pi u', cos / sin) for ~2 M draws of a config-2-shaped model: every value
    identical to the oracle's glibc-computed one (the fraction of differing
    values and the largest ulp distance are reported on failure)."""
    model = gpu.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=5, stream="ref")
    om = _oracle_model(oracle, model)
    bad, total, worst = 0, 0, 0
    for k in range(2):
        _, a_g, b_g = gpu.draw_sample(model, MASTER, 3, k, 4096)
        _, a_o, b_o = om.draw(MASTER, 3, k, 4096)
        for g_, o_ in ((a_g, a_o), (b_g, b_o)):
            d = g_.view(np.int64) - o_.view(np.int64)
            bad += int(np.count_nonzero(d))
            total += d.size
            worst = max(worst, int(np.max(np.abs(d))))
    assert bad == 0, f"{bad} of {total} draws differ, max {worst} ulp"


@pytest.mark.parametrize("kind", ["constant", "deterministic"])
def test_libm_free_models_ref_stream_bitexact(gpu, oracle, kind):
    if kind == "constant":
        mv, mm = gpu.constant_ones_model(37), gpu.constant_ones_matrix_model(3, 4, 2)
    else:
        mv, mm = gpu.deterministic_model(2), gpu.deterministic_matrix_model()
    plan = gpu.LevelPlan(3, 2, [9, 3, 1])
    for model, fn in ((mv, gpu.mlmc_inner), (mm, gpu.mlmc_matmul)):
        for tgt in (gpu.target_identity(), gpu.target_f1()):
            r = fn(model, tgt, plan, 77, gpu.EstimatorOptions(engine="exact"))
            o = _oracle_model(oracle, model).mlmc(3, 1, [9, 3, 1], 77, target=tgt.kind)
            _levels_equal(r, o)


def test_config2_small_philox_bitexact(gpu, oracle):
    model = gpu.gaussian_mean_matrix_model(32, 512, 16, sd=0.5, data_seed=5)
    plan = gpu.LevelPlan(2, 3, [70, 65, 10, 3], c0=32)
    r = gpu.mlmc_matmul(model, gpu.target_identity(), plan, MASTER, gpu.EstimatorOptions(engine="exact"))
    o = _oracle_model(oracle, model).mlmc(2, 32, list(plan.N), MASTER)
    _levels_equal(r, o)
    np.testing.assert_array_equal(r.value.ravel(), o.value)


def test_paper_models_ref_stream(gpu, oracle):
    """Paper models (models.cpp:12-52: Box-Muller, Poisson, Exp(1), cos, sin)
    with the identity, f1 and f2 targets (f2's sin included): bit for bit."""
    plan = gpu.LevelPlan(3, 2, [300, 100, 33])
    for tgt in (gpu.target_identity(), gpu.target_f1(), gpu.target_f2()):
        r = gpu.mlmc_inner(gpu.paper_inner_model(), tgt, plan, 314, gpu.EstimatorOptions(engine="exact"))
        o = _oracle_model(oracle, gpu.paper_inner_model()).mlmc(3, 1, [300, 100, 33], 314, target=tgt.kind)
        _levels_equal(r, o)
    m = gpu.paper_matrix_model()
    for tgt in (gpu.target_identity(), gpu.target_f1(), gpu.target_f2()):
        r = gpu.mlmc_matmul(m, tgt, gpu.LevelPlan(4, 1, [40, 10]), 11, gpu.EstimatorOptions(engine="exact"))
        o = _oracle_model(oracle, m).mlmc(4, 1, [40, 10], 11, target=tgt.kind)
        _levels_equal(r, o)
    for kind in (abi.MODEL_PAPER_INNER, abi.MODEL_PAPER_MATRIX):
        mod = gpu.paper_inner_model() if kind == abi.MODEL_PAPER_INNER else m
        for k in range(3):
            i_g, a_g, b_g = gpu.draw_sample(mod, 99, 2, k, 64)
            i_o, a_o, b_o = _oracle_model(oracle, mod).draw(99, 2, k, 64)
            assert np.array_equal(i_g, i_o) and np.array_equal(a_g, a_o) and np.array_equal(b_g, b_o)
