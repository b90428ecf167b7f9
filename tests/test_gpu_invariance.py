"""GPU-count invariance (the reference's thread-count invariance,
/root/reference/proj/README.md:109-119, tests/test_estimators.cpp:162-186),
checked in one process by running every rank's share of a world-W split on
the one GPU, for W = 1, 2, 4, 8.

* plain rank sharding (64-replication chunk q -> rank q mod W, then one
  all-reduce): counts exact, level sums equal to reassociation -- within
  1e-13 (fp64) / 1e-6 (fp32) relative;
* driver.ShardedSession (8 virtual shards, vshard-ordered sum): bit-identical
  statistics for every W."""
import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi
from paper_1904_00429_b200 import driver

pytestmark = pytest.mark.gpu
MASTER = 20260823
WORLDS = (1, 2, 4, 8)


def models(g):
    return {
        "f64": (g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=g.RngStream.derive_seed(MASTER, 0xD47A0002, 0)),
                32, 1e-13),
        "f32": (g.gaussian_mean_matrix_model(512, 4096, 512, sd=1.0, data_seed=3, dtype=abi.F32), 64, 1e-6),
    }


DN = [700, 333, 129]


def _plain(g, model, c0, world):
    parts = []
    for r in range(world):
        s = g.MlmcSession(model, g.target_identity(), 2, 2, MASTER, c0=c0,
                          options=g.EstimatorOptions(rank=r, world=world, engine="fused"))
        s.run_round(DN)
        parts.append(s.packed_stats())
        s.close()
    return driver.unpack(sum(parts), 3)  # the all-reduce


def _sharded(g, model, c0, world):
    per_v = {}
    for r in range(world):
        sh = driver.ShardedSession(
            lambda v, V: g.MlmcSession(model, g.target_identity(), 2, 2, MASTER, c0=c0,
                                       options=g.EstimatorOptions(rank=v, world=V, engine="fused")),
            r, world, vshards=8)
        sh.run_round(DN)
        for v, buf in zip(sh.owned, sh.packed_parts()):
            per_v[v] = buf
        sh.close()
    return driver.unpack(driver.ordered_sum([per_v[v] for v in range(8)]), 3)  # the all-gather + ordered sum


@pytest.mark.parametrize("kind", ["f64", "f32"])
def test_rank_sharding_matches_single_gpu(gpu, kind):
    model, c0, tol = models(gpu)[kind]
    ref = _plain(gpu, model, c0, 1)
    assert list(ref.counts) == DN
    for w in WORLDS[1:]:
        st = _plain(gpu, model, c0, w)
        np.testing.assert_array_equal(st.counts, ref.counts)
        for l in range(3):
            rel = np.linalg.norm(st.sums[l] - ref.sums[l]) / np.linalg.norm(ref.sums[l])
            assert rel <= tol, (w, l, rel)
            assert abs(st.sumsq[l] - ref.sumsq[l]) <= tol * ref.sumsq[l]


@pytest.mark.parametrize("kind", ["f64", "f32"])
def test_sharded_session_bit_identical_across_gpu_counts(gpu, kind):
    model, c0, _ = models(gpu)[kind]
    ref = _sharded(gpu, model, c0, 1)
    assert list(ref.counts) == DN
    for w in WORLDS[1:]:
        st = _sharded(gpu, model, c0, w)
        assert np.array_equal(st.sums, ref.sums), w
        assert np.array_equal(st.sumsq, ref.sumsq), w
        assert np.array_equal(st.counts, ref.counts), w
    # same samples as the plain split, summed in another order
    plain = _plain(gpu, model, c0, 1)
    for l in range(3):
        assert np.linalg.norm(plain.sums[l] - ref.sums[l]) <= 1e-6 * np.linalg.norm(ref.sums[l])
