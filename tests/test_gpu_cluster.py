"""The cluster engine (k_level_cluster_f64: generation and DMMA contraction in
one kernel, four CTAs per cluster exchanging operand blocks over DSMEM) vs
the exact-order engine and vs the panel pipeline (MLSK_CLUSTER=0).

It serves fp64 matrix models with m and p in (128, 256] when MLSK_CLUSTER=1
(opt-in); tolerance 1e-12 relative (Frobenius) as for every
fused fp64 path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MASTER = 20260823
TOL = 1e-12


def frob_rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


def close(r1, r2, tol=TOL):
    for s1, s2 in zip(r1.per_level, r2.per_level):
        assert s1.replication_count == s2.replication_count
        assert frob_rel(s1.sum, s2.sum) <= tol, (s1.level, frob_rel(s1.sum, s2.sum))
        assert abs(s1.sum_of_squares - s2.sum_of_squares) <= tol * max(s2.sum_of_squares, 1e-300)


@pytest.fixture(autouse=True)
def cluster_on(monkeypatch):
    monkeypatch.setenv("MLSK_CLUSTER", "1")


def run(gpu, model, plan, engine, seed=MASTER):
    return gpu.mlmc_matmul(model, gpu.target_identity(), plan, seed, gpu.EstimatorOptions(engine=engine))


@pytest.mark.parametrize("shape", [(256, 4096, 256), (200, 1000, 131), (129, 512, 256), (256, 3000, 255)])
def test_cluster_vs_exact(gpu, shape):
    """Ragged tiles (rows / cols past m, p are zero), c not a multiple of the
    16-wide K-chunk (padding columns), n not a power of two."""
    m, n, p = shape
    model = gpu.gaussian_mean_matrix_model(m, n, p, sd=0.5, data_seed=17)
    plan = gpu.LevelPlan(2, 3, [45, 21, 10, 3], c0=24)
    close(run(gpu, model, plan, "fused"), run(gpu, model, plan, "exact"))


def test_cluster_vs_panel_pipeline(gpu, monkeypatch):
    """Same samples through both fused fp64 engines (they differ only in the
    order the per-group partial sums are added)."""
    model = gpu.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=23)
    plan = gpu.LevelPlan(2, 4, [700, 300, 150, 64, 40], c0=32)
    rc = run(gpu, model, plan, "fused")
    monkeypatch.setenv("MLSK_CLUSTER", "0")  # the panel pipeline
    rp = run(gpu, model, plan, "fused")
    close(rc, rp)


def test_cluster_fewer_samples_than_clusters(gpu):
    """1 and 5 samples: most clusters get none and must contribute zeros."""
    model = gpu.gaussian_mean_matrix_model(256, 2048, 256, sd=1.0, data_seed=29)
    plan = gpu.LevelPlan(2, 1, [1, 5], c0=16)
    close(run(gpu, model, plan, "fused"), run(gpu, model, plan, "exact"))


def test_cluster_session_rounds(gpu):
    """Rounds accumulate: four rounds equal one round with the summed counts."""
    model = gpu.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=31)
    s1 = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, 5, c0=32)
    for dN in ([70, 0, 0], [0, 0, 0], [0, 40, 9], [30, 0, 0]):
        s1.run_round(dN)
    s2 = gpu.MlmcSession(model, gpu.target_identity(), 2, 2, 5, c0=32)
    s2.run_round([100, 40, 9])
    close(s1.stats(), s2.stats())
    s1.close()
    s2.close()
