"""Multi-GPU inside the C-ABI (mlsk_exec_opts.n_devices / device_ids /
deterministic): the library deals the replications to device slots, one host
thread per slot, and adds the slots' per-level sums on the host in a fixed
order -- the reference parallelises inside the library the same way
(parallel.hpp:18-52).  The test box has one GPU, so the slots repeat device 0
(the host threads then share it); the sharding, the threads and the ordered
combination are the same code a multi-GPU box runs.

Deterministic mode (fixed virtual shards) must give bit-identical results
for every device count dividing the shard count, like the reference's
thread-count invariance (README.md:109-119, test_estimators.cpp:162-186)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MASTER = 20260823


def model(g):
    return g.gaussian_mean_matrix_model(128, 4096, 96, sd=0.5, data_seed=g.RngStream.derive_seed(MASTER, 0xD47A0002, 0))


PLAN = dict(M=2, L=2, N=[300, 170, 65], c0=32)


def run(g, **opts):
    plan = g.LevelPlan(PLAN["M"], PLAN["L"], PLAN["N"], c0=PLAN["c0"])
    return g.mlmc_matmul(model(g), g.target_identity(), plan, MASTER, g.EstimatorOptions(engine="fused", **opts))


def test_two_slots_match_one_device(gpu):
    one = run(gpu)
    two = run(gpu, devices=[0, 0])
    for a, b in zip(one.per_level, two.per_level):
        assert a.replication_count == b.replication_count
        assert np.linalg.norm(np.asarray(a.sum) - np.asarray(b.sum)) <= 1e-13 * np.linalg.norm(np.asarray(a.sum))
        assert abs(a.sum_of_squares - b.sum_of_squares) <= 1e-13 * a.sum_of_squares


def test_deterministic_bit_identical_for_1_2_4_8_devices(gpu):
    ref = run(gpu, devices=[0], deterministic=True)
    for n in (2, 4, 8):
        r = run(gpu, devices=[0] * n, deterministic=True)
        assert np.array_equal(np.asarray(r.value), np.asarray(ref.value)), n
        for a, b in zip(r.per_level, ref.per_level):
            assert np.array_equal(np.asarray(a.sum), np.asarray(b.sum)), n
            assert a.sum_of_squares == b.sum_of_squares and a.replication_count == b.replication_count
    # same samples as the plain call, in another summation order
    plain = run(gpu)
    for a, b in zip(plain.per_level, ref.per_level):
        assert np.linalg.norm(np.asarray(a.sum) - np.asarray(b.sum)) <= 1e-13 * np.linalg.norm(np.asarray(a.sum))


def test_multi_device_session_rounds_and_level_buffer(gpu):
    """Rounds of a multi-device session = one call; the packed level buffer
    (for a cross-process all-reduce) holds the combined sums."""
    def session(n):
        opts = gpu.EstimatorOptions(engine="fused", devices=[0] * n, deterministic=True)
        s = gpu.MlmcSession(model(gpu), gpu.target_identity(), 2, 2, MASTER, c0=32, options=opts)
        s.run_round([100, 70, 15])
        s.run_round([200, 100, 50])
        return s
    s, s1 = session(4), session(1)
    r, r1 = s.stats(), s1.stats()
    one = run(gpu, devices=[0, 0], deterministic=True)
    for a, b, c in zip(r.per_level, r1.per_level, one.per_level):
        assert np.array_equal(np.asarray(a.sum), np.asarray(b.sum))  # same rounds: bit-identical
        assert a.sum_of_squares == b.sum_of_squares
        assert a.replication_count == c.replication_count
        assert np.linalg.norm(np.asarray(a.sum) - np.asarray(c.sum)) <= 1e-13 * np.linalg.norm(np.asarray(c.sum))
    s1.close()
    ptr, n = s.level_buffer()
    import torch

    class _Dev:
        def __init__(self, p, k):
            self.__cuda_array_interface__ = {"shape": (k,), "typestr": "<f8", "data": (p, False), "version": 3,
                                             "stream": None}
    got = torch.as_tensor(_Dev(ptr, n), device="cuda").cpu().numpy()
    assert np.array_equal(got, s.packed_stats())
    s.close()


def test_multi_device_option_errors(gpu):
    with pytest.raises(ValueError):  # deterministic across processes: the driver's ShardedSession
        run(gpu, devices=[0, 0], deterministic=True, rank=0, world=2)
    with pytest.raises(ValueError):  # 3 slots do not divide 8 virtual shards
        run(gpu, devices=[0, 0, 0], deterministic=True)
    with pytest.raises(ValueError):  # unknown device
        run(gpu, devices=[0, 4096])
    plan = gpu.LevelPlan(2, 1, [5, 3], c0=32)
    with pytest.raises(ValueError):  # the coupling probe needs one device
        gpu.mlmc_matmul(model(gpu), gpu.target_identity(), plan, MASTER,
                        gpu.EstimatorOptions(devices=[0, 0], probe=lambda *a: None))
