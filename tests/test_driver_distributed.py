"""The adaptive multi-rank driver (paper_1904_00429_b200/driver.py) on CPU:
world_size 2 over gloo with an oracle-backed session (test infrastructure)
standing in for the GPU session, against a single-process run."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1904_00429_b200 import _abi as abi
from paper_1904_00429_b200 import driver


class OracleSession:
    """run_round / packed_stats / cells over the CPU oracle's philox-mode
    draws; rank r owns the 64-replication chunks q = r (mod world)."""

    def __init__(self, M, c0, L, seed, rank=0, world=1):
        from oracle import pyoracle
        self.om = pyoracle.OracleModel(pyoracle.model_desc(abi.MODEL_GAUSS_MEAN, n=64, m=4, p=3, sd=0.5,
                                                           mean_lo=-1, mean_hi=1, data_seed=5))
        self.M, self.c0, self.L, self.seed, self.rank, self.world = M, c0, L, seed, rank, world
        self.cells = 12
        self.sums = np.zeros((L + 1, 12))
        self.sumsq = np.zeros(L + 1)
        self.counts = np.zeros(L + 1, dtype=np.int64)
        self.next_k = [0] * (L + 1)

    def run_round(self, dN):
        n = 64.0
        for l, d in enumerate(dN):
            c = self.c0 * self.M ** l
            cc = c // self.M if l > 0 else 0
            for k in range(self.next_k[l], self.next_k[l] + d):
                if (k // 64) % self.world != self.rank:
                    continue
                _, a, b = self.om.draw(self.seed, l, k, c)
                y = (n / c) * a @ b
                if cc:
                    y = y - (n / cc) * a[:, :cc] @ b[:cc, :]
                self.sums[l] += y.ravel()
                self.sumsq[l] += float(np.sum(y * y))
                self.counts[l] += 1
            self.next_k[l] += d

    def packed_stats(self):
        return driver.pack(self.sums, self.sumsq, self.counts)

    def checkpoint(self):
        import pickle
        return pickle.dumps((self.sums, self.sumsq, self.counts, self.next_k))

    def restore(self, image):
        import pickle
        self.sums, self.sumsq, self.counts, self.next_k = pickle.loads(image)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sess = OracleSession(2, 4, 3, 99, rank, world)
        r = driver.adaptive_mlmc(sess, 2, 4, 3, eps=0.5, n_pilot=96, max_rounds=6)
        out[rank] = (r.value.tolist(), r.N, r.rounds, r.rmse_estimate, [list(h) for h in r.history])
    finally:
        dist.destroy_process_group()


def test_adaptive_driver_two_ranks_matches_single_process():
    single = driver.adaptive_mlmc(OracleSession(2, 4, 3, 99), 2, 4, 3, eps=0.5, n_pilot=96, max_rounds=6)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        r0, r1 = out[0], out[1]
    # both ranks hold the same global statistics and took the same decisions
    assert r0 == r1
    assert r0[1] == single.N and r0[2] == single.rounds and r0[4] == single.history
    np.testing.assert_allclose(r0[0], single.value, rtol=1e-12, atol=1e-12)
    assert abs(r0[3] - single.rmse_estimate) <= 1e-12 * single.rmse_estimate


def _det_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sess = driver.ShardedSession(lambda v, V: OracleSession(2, 4, 3, 99, v, V), rank, world, vshards=4)
        r = driver.adaptive_mlmc(sess, 2, 4, 3, eps=0.5, n_pilot=96, max_rounds=6)
        out[rank] = (r.value.tobytes(), r.stats.sums.tobytes(), r.stats.sumsq.tobytes(), r.N, r.history)
    finally:
        dist.destroy_process_group()


def _run_ranks(target, world):
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=target, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        return [out[r] for r in range(world)]


def test_deterministic_sharding_bit_identical_across_world_sizes():
    """ShardedSession (fixed virtual shards, all-gather + vshard-ordered sum):
    the world-2 run (gloo) reproduces the single-process run bit for bit --
    every level sum, the estimate and the adaptive decisions."""
    one = driver.ShardedSession(lambda v, V: OracleSession(2, 4, 3, 99, v, V), 0, 1, vshards=4)
    single = driver.adaptive_mlmc(one, 2, 4, 3, eps=0.5, n_pilot=96, max_rounds=6)
    r0, r1 = _run_ranks(_det_worker, 2)
    assert r0 == r1
    assert r0[0] == single.value.tobytes() and r0[1] == single.stats.sums.tobytes()
    assert r0[2] == single.stats.sumsq.tobytes()
    assert r0[3] == single.N and r0[4] == single.history
    # and the virtual shards partition the plain run's samples
    plain = driver.adaptive_mlmc(OracleSession(2, 4, 3, 99), 2, 4, 3, eps=0.5, n_pilot=96, max_rounds=6)
    assert plain.N == single.N
    np.testing.assert_allclose(plain.value, single.value, rtol=1e-12, atol=1e-12)


def test_sharded_session_rejects_bad_split():
    with pytest.raises(ValueError):
        driver.ShardedSession(lambda v, V: OracleSession(2, 4, 3, 99, v, V), 0, 3, vshards=8)
    with pytest.raises(ValueError):
        driver.ShardedSession(lambda v, V: OracleSession(2, 4, 3, 99, v, V), 2, 2, vshards=8)


def test_optimal_allocation_and_costs():
    C = driver.level_costs(2, 32, 2, 4)
    assert C == [32 * 4.0, (64 + 32) * 4.0, (128 + 64) * 4.0]
    N = driver.optimal_allocation([4.0, 1.0, 0.25], C, eps=0.1)
    s = sum(np.sqrt(v * c) for v, c in zip([4.0, 1.0, 0.25], C))
    assert N == [int(np.ceil(np.sqrt(v / c) * s / 0.01)) for v, c in zip([4.0, 1.0, 0.25], C)]
    # the allocation meets the variance target
    assert sum(v / n for v, n in zip([4.0, 1.0, 0.25], N)) <= 0.01 * (1 + 1e-9)


def test_relative_error_matches_reference_definition():
    assert driver.relative_error([3.0], [3.0]) == 0.0
    assert driver.relative_error([1.0], [0.0]) == float("inf")
    assert driver.relative_error([[1, 2], [3, 4]], [[1, 2], [3, 5]]) == pytest.approx(1 / np.sqrt(39))


def test_adaptive_driver_resumes_from_checkpoint(tmp_path):
    """A run stopped after 2 rounds and resumed from its checkpoint with a
    fresh session ends with the same bits as an uninterrupted run."""
    full = driver.adaptive_mlmc(OracleSession(2, 4, 3, 99), 2, 4, 3, eps=1.0, n_pilot=64, max_rounds=5)
    ck = str(tmp_path / "run")
    part = driver.adaptive_mlmc(OracleSession(2, 4, 3, 99), 2, 4, 3, eps=1.0, n_pilot=64, max_rounds=2,
                                checkpoint=ck)
    assert part.rounds == 2 and os.path.exists(ck + ".rank0")
    resumed = driver.adaptive_mlmc(OracleSession(2, 4, 3, 99), 2, 4, 3, eps=1.0, n_pilot=64, max_rounds=5,
                                   checkpoint=ck)
    assert resumed.rounds == full.rounds
    assert resumed.N == full.N and resumed.history == full.history
    assert np.array_equal(resumed.value, full.value)
    assert resumed.rmse_estimate == full.rmse_estimate
