"""Checkpoint / resume of a session (mlsk_session_checkpoint / _restore,
SURVEY.md section 5): a run stopped after some rounds and restored into a
fresh session continues with the same bits as an uninterrupted one -- on the
fused fp64 and tcgen05 engines, on the exact engine with open 64-replication
chunks, and on a deterministic multi-slot session; a checkpoint of another
run is rejected."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

S = 20260823


def _models(g):
    return {
        "fused_f64": (g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=2), 32, "fused"),
        "fused_tf32": (g.gaussian_mean_matrix_model(256, 2048, 256, sd=1.0, data_seed=3, dtype=1), 64, "fused"),
        "exact_paper": (g.paper_matrix_model(), 1, "exact"),
    }


def _rounds(g, model, c0, engine, rounds, L=2, restore_after=None, **kw):
    opts = g.EstimatorOptions(engine=engine, **kw)
    sess = g.MlmcSession(model, g.target_identity(), 2, L, S, c0=c0, options=opts)
    for i, dN in enumerate(rounds):
        if restore_after is not None and i == restore_after:
            img = sess.checkpoint()
            sess.close()
            sess = g.MlmcSession(model, g.target_identity(), 2, L, S, c0=c0, options=opts)
            sess.restore(img)
        sess.run_round(dN)
    r = sess.stats()
    sess.close()
    return r


@pytest.mark.parametrize("name", ["fused_f64", "fused_tf32", "exact_paper"])
def test_resume_is_bit_identical(gpu, name):
    model, c0, engine = _models(gpu)[name]
    rounds = [[70, 33, 10], [5, 64, 3], [100, 1, 17]]  # open chunks left at every boundary
    a = _rounds(gpu, model, c0, engine, rounds)
    b = _rounds(gpu, model, c0, engine, rounds, restore_after=2)
    for sa, sb in zip(a.per_level, b.per_level):
        assert sa.replication_count == sb.replication_count
        assert np.array_equal(np.asarray(sa.sum), np.asarray(sb.sum))
        assert sa.sum_of_squares == sb.sum_of_squares
    assert np.array_equal(np.asarray(a.value), np.asarray(b.value))


def test_resume_multi_slot_deterministic(gpu):
    model, c0, engine = _models(gpu)["fused_f64"]
    rounds = [[64, 64, 64], [128, 0, 64]]
    a = _rounds(gpu, model, c0, engine, rounds, devices=[0, 0], deterministic=True)
    b = _rounds(gpu, model, c0, engine, rounds, restore_after=1, devices=[0, 0], deterministic=True)
    assert np.array_equal(np.asarray(a.value), np.asarray(b.value))


def test_restore_rejects_another_run(gpu):
    model, c0, engine = _models(gpu)["fused_f64"]
    opts = gpu.EstimatorOptions(engine=engine)
    s1 = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, S, c0=c0, options=opts)
    s1.run_round([64, 32, 16])
    img = s1.checkpoint()
    s1.close()
    for kw in ({"seed": S + 1}, {"L": 3}, {"c0": 64}):
        args = dict(seed=S, L=2, c0=c0)
        args.update(kw)
        s2 = gpu.MlmcSession(model, gpu.target_identity(), 2, args["L"], args["seed"], c0=args["c0"], options=opts)
        with pytest.raises(ValueError):
            s2.restore(img)
        s2.close()
    s3 = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, S, c0=c0, options=opts)
    with pytest.raises(ValueError):
        s3.restore(img[:100])
    s3.close()


def test_adaptive_driver_resume_on_device(gpu, tmp_path):
    from paper_1904_00429_b200 import driver
    model, c0, engine = _models(gpu)["fused_f64"]
    opts = gpu.EstimatorOptions(engine=engine)

    def sess():
        return gpu.MlmcSession(model, gpu.target_identity(), 2, 2, S, c0=c0, options=opts)

    full = driver.adaptive_mlmc(sess(), 2, c0, 2, eps=2000.0, n_pilot=64, max_rounds=4)
    ck = str(tmp_path / "dev")
    driver.adaptive_mlmc(sess(), 2, c0, 2, eps=2000.0, n_pilot=64, max_rounds=2, checkpoint=ck)
    res = driver.adaptive_mlmc(sess(), 2, c0, 2, eps=2000.0, n_pilot=64, max_rounds=4, checkpoint=ck)
    assert res.N == full.N and res.rounds == full.rounds
    assert np.array_equal(res.value, full.value)
