"""Adaptive multilevel driver over the round API, sharded across ranks.

The reference plans N_l a priori only (planner.cpp:65-81, make_plan :94-100;
adaptive allocation is an explicit non-goal).  BASELINE
configs 2, 3 and 5 need the standard MLMC allocation computed from measured
level variances, so this module adds the classic adaptive loop (Giles,
"Multilevel Monte Carlo methods", Acta Numerica 2015, Alg. 1 with fixed L):

  1. pilot round of N_pilot replications per level;
  2. V_l = E||Y_l||_F^2 - ||E Y_l||_F^2 from the per-level sums, C_l = cost of
     one level-l replication (c_l + c_{l-1} sampled indices x cells, the
     reference's cost units, estimators.cpp:34-40);
  3. N_l = ceil( (1/(theta eps^2)) sqrt(V_l / C_l) sum_k sqrt(V_k C_k) ),
     run the missing dN_l = N_l - n_l; repeat until nothing is missing.

Every level's identity-target sketch is unbiased for E[A B],
so the MSE is the variance sum_l V_l / N_l <= theta eps^2 (theta = 1 by
default; 1/2 reserves half of the MSE for a bias term).

Multi-GPU: one process per GPU.  Rank r runs the 64-replication chunks
q = r (mod world) of every round (the library's exec option), then ONE
all-reduce of the packed per-level buffer [(sum Y, sum ||Y||^2, count)] per
round -- NCCL on the device buffer when the process group's backend is NCCL,
gloo on a host copy otherwise.  Every rank then holds the same global
statistics and computes the same next allocation; there is no other
communication.  Matrix sums then differ across world sizes by reassociation
(ulp level); `ShardedSession` (fixed virtual shards, one all-gather and a
vshard-ordered sum per round) makes results bit-identical for any world
size dividing its shard count.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np


@dataclass
class LevelStats:
    """Global (all-rank) per-level accumulators."""

    sums: np.ndarray       # [L+1, cells]
    sumsq: np.ndarray      # [L+1]
    counts: np.ndarray     # [L+1]

    @property
    def estimates(self) -> np.ndarray:
        return self.sums / np.maximum(self.counts, 1)[:, None]

    @property
    def variances(self) -> np.ndarray:
        """V_l = E||Y||^2 - ||E Y||^2 (Frobenius), floored at 0."""
        n = np.maximum(self.counts, 1)
        meansq = self.sumsq / n
        return np.maximum(meansq - np.sum(self.estimates ** 2, axis=1), 0.0)

    @property
    def value(self) -> np.ndarray:
        return self.estimates.sum(axis=0)

    @property
    def mse(self) -> float:
        n = np.maximum(self.counts, 1)
        return float(np.sum(self.variances / n))


@dataclass
class AdaptiveResult:
    value: np.ndarray
    stats: LevelStats
    rounds: int
    N: List[int]
    eps: float
    rmse_estimate: float
    cost_units: int
    history: List[List[int]] = field(default_factory=list)


def pack(sums: np.ndarray, sumsq: np.ndarray, counts: np.ndarray) -> np.ndarray:
    L1, cells = sums.shape
    buf = np.zeros((L1, cells + 2))
    buf[:, :cells] = sums
    buf[:, cells] = sumsq
    buf[:, cells + 1] = counts
    return buf.ravel()


def unpack(buf: np.ndarray, levels: int) -> LevelStats:
    b = np.asarray(buf, dtype=np.float64).reshape(levels, -1)
    cells = b.shape[1] - 2
    return LevelStats(b[:, :cells].copy(), b[:, cells].copy(), np.rint(b[:, cells + 1]).astype(np.int64))


class ShardedSession:
    """Deterministic multi-GPU split: the samples are dealt to `vshards`
    VIRTUAL shards (64-replication chunk q -> virtual shard q mod vshards, the
    library's rank/world sharding with world = vshards), and rank r of `world`
    (world dividing vshards) runs the virtual shards v = r (mod world), each in
    its own session.  Every virtual shard's sums then do not depend on how many
    GPUs run them, and `gather_ordered_stats` adds the vshards' buffers in
    vshard order -- so the statistics, and every decision taken from them, are
    bit-identical for world = 1, 2, 4, 8 (the reference's thread-count
    invariance, README.md:109-119, test_estimators.cpp:162-186, which a plain
    all-reduce of per-rank sums cannot give: its grouping depends on world).

    `make_session(v, vshards)` builds the session of virtual shard v (an
    MlmcSession with EstimatorOptions(rank=v, world=vshards), or any object
    with run_round / packed_stats / cells)."""

    def __init__(self, make_session, rank: int = 0, world: int = 1, vshards: int = 8):
        if world < 1 or vshards % world != 0 or not 0 <= rank < world:
            raise ValueError("ShardedSession: world must divide vshards and 0 <= rank < world")
        self.rank, self.world, self.vshards = rank, world, vshards
        self.owned = list(range(rank, vshards, world))
        self.sessions = [make_session(v, vshards) for v in self.owned]
        self.cells = self.sessions[0].cells

    def run_round(self, dN: Sequence[int]) -> None:
        for s in self.sessions:
            s.run_round(dN)

    def packed_parts(self) -> List[np.ndarray]:
        """This rank's virtual shards' packed buffers, in self.owned order."""
        return [np.asarray(s.packed_stats(), dtype=np.float64) for s in self.sessions]

    def checkpoint(self) -> bytes:
        """The owned virtual shards' images, length-prefixed, in owned order."""
        import struct

        out = b""
        for s in self.sessions:
            img = s.checkpoint()
            out += struct.pack("<q", len(img)) + img
        return out

    def restore(self, image: bytes) -> None:
        import struct

        off = 0
        for s in self.sessions:
            (n,) = struct.unpack_from("<q", image, off)
            off += 8
            s.restore(image[off:off + n])
            off += n
        if off != len(image):
            raise ValueError("ShardedSession.restore: the image holds a different number of shards")

    def close(self) -> None:
        for s in self.sessions:
            if hasattr(s, "close"):
                s.close()


def ordered_sum(parts: Sequence[np.ndarray]) -> np.ndarray:
    """sum of the virtual shards' buffers, strictly in vshard order from 0.0"""
    total = np.zeros_like(parts[0])
    for p in parts:
        total = total + p
    return total


def gather_ordered_stats(session: ShardedSession, levels: int, group=None) -> LevelStats:
    """All ranks' virtual-shard buffers (one all-gather), added in vshard
    order on every rank: the same bits for any world size."""
    import torch.distributed as dist

    mine = session.packed_parts()
    if group is None and not (dist.is_available() and dist.is_initialized()):
        if session.world != 1:
            raise RuntimeError("gather_ordered_stats: world > 1 needs an initialised process group")
        return unpack(ordered_sum(mine), levels)
    import torch

    world = dist.get_world_size(group)
    if world != session.world:
        raise ValueError("gather_ordered_stats: process group size != session world")
    n = mine[0].size
    local = torch.from_numpy(np.concatenate(mine))
    on_dev = dist.get_backend(group) == "nccl"
    if on_dev:
        local = local.cuda()
    bufs = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(bufs, local, group=group)
    per_v = [None] * session.vshards
    for r, b in enumerate(bufs):
        b = b.cpu().numpy()
        for j, v in enumerate(range(r, session.vshards, world)):
            per_v[v] = b[j * n:(j + 1) * n]
    return unpack(ordered_sum(per_v), levels)


def allreduce_stats(session, levels: int, group=None) -> LevelStats:
    """One all-reduce of the packed level buffer across the process group
    (a ShardedSession: the fixed-order all-gather reduction instead)."""
    import torch.distributed as dist

    if isinstance(session, ShardedSession):
        return gather_ordered_stats(session, levels, group)
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return unpack(session.packed_stats(), levels)
    backend = dist.get_backend(group)
    if backend == "nccl" and hasattr(session, "level_buffer"):
        import torch

        ptr, n = session.level_buffer()
        # the pack runs on the session's stream, which need not be torch's
        # current stream: wait for it before NCCL reads the buffer
        session.synchronize()
        t = torch.as_tensor(_DevBuf(ptr, n), device="cuda")
        dist.all_reduce(t, group=group)
        return unpack(t.double().cpu().numpy(), levels)
    import torch

    t = torch.from_numpy(session.packed_stats())
    dist.all_reduce(t, group=group)
    return unpack(t.numpy(), levels)


class _DevBuf:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "stream": None}


def optimal_allocation(V: Sequence[float], C: Sequence[float], eps: float, theta: float = 1.0) -> List[int]:
    """N_l = ceil( sqrt(V_l/C_l) * sum_k sqrt(V_k C_k) / (theta eps^2) )."""
    V = np.asarray(V, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    s = float(np.sum(np.sqrt(V * C)))
    return [int(math.ceil(math.sqrt(v / c) * s / (theta * eps * eps))) if v > 0 else 1 for v, c in zip(V, C)]


def level_costs(M: int, c0: int, L: int, cells: int) -> List[float]:
    """Reference cost units per replication: (c_l + [l>0] c_{l-1}) * cells."""
    out = []
    for l in range(L + 1):
        c = c0 * M ** l
        out.append(float((c + (c // M if l > 0 else 0)) * cells))
    return out


def _rank_of(group) -> int:
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(group)
    except Exception:
        pass
    return 0


def save_checkpoint(path: str, session, n: Sequence[int], history, rounds: int, group=None) -> None:
    """Driver state + this rank's session image, written atomically to
    `path`.rank<r> (checkpoint/resume: the reference has
    none; a long adaptive run -- config 3 at eps = 1e-3 is hours -- survives a
    lost process)."""
    import json
    import os
    import struct

    meta = json.dumps({"version": 1, "n": [int(x) for x in n], "history": history, "rounds": rounds}).encode()
    img = session.checkpoint()
    f = f"{path}.rank{_rank_of(group)}"
    tmp = f + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(b"MLSKDRV1" + struct.pack("<q", len(meta)) + meta + img)
    os.replace(tmp, f)


def load_checkpoint(path: str, session, group=None):
    """(n, history, rounds) after restoring this rank's session image, or None."""
    import json
    import os
    import struct

    f = f"{path}.rank{_rank_of(group)}"
    if not os.path.exists(f):
        return None
    data = open(f, "rb").read()
    if data[:8] != b"MLSKDRV1":
        raise ValueError(f"{f}: not an adaptive-driver checkpoint")
    (k,) = struct.unpack_from("<q", data, 8)
    meta = json.loads(data[16:16 + k].decode())
    session.restore(data[16 + k:])
    return meta["n"], meta["history"], meta["rounds"]


def adaptive_mlmc(session, M: int, c0: int, L: int, eps: float, n_pilot: int = 256, theta: float = 1.0,
                  max_rounds: int = 20, max_total: Optional[int] = None, group=None,
                  checkpoint: Optional[str] = None) -> AdaptiveResult:
    """Run rounds on `session` (an MlmcSession, or any object with run_round /
    packed_stats / cells) until sum_l V_l / N_l <= theta eps^2.

    `session` must be created with rank / world matching the process group:
    each rank then runs its chunk share of every round's dN.  A
    ShardedSession makes the whole run bit-identical across world sizes.

    `checkpoint`: a path prefix; the driver state and the session image are
    saved after every round, and a run started with an existing checkpoint
    resumes from it (the session must be freshly created with the same
    arguments).  A resumed run gives the same bits as one that never stopped.
    """
    levels = L + 1
    cells = session.cells
    C = level_costs(M, c0, L, cells)
    resumed = load_checkpoint(checkpoint, session, group) if checkpoint else None
    if resumed is not None:
        n, history, rounds = resumed
        n = [int(x) for x in n]
    else:
        session.run_round([n_pilot] * levels)
        n = [n_pilot] * levels
        history = [list(n)]
        rounds = 1
    stats = allreduce_stats(session, levels, group)
    if checkpoint and resumed is None:
        save_checkpoint(checkpoint, session, n, history, rounds, group)
    while rounds < max_rounds:
        target = optimal_allocation(stats.variances, C, eps, theta)
        dN = [max(0, t - k) for t, k in zip(target, n)]
        if max_total is not None:
            room = max(0, max_total - sum(n))
            if sum(dN) > room:
                scale = room / max(sum(dN), 1)
                dN = [int(d * scale) for d in dN]
        if sum(dN) == 0:
            break
        session.run_round(dN)
        n = [a + b for a, b in zip(n, dN)]
        history.append(list(dN))
        stats = allreduce_stats(session, levels, group)
        rounds += 1
        if checkpoint:
            save_checkpoint(checkpoint, session, n, history, rounds, group)
    cost = int(sum(k * c for k, c in zip(stats.counts, C)))
    return AdaptiveResult(stats.value, stats, rounds, [int(x) for x in stats.counts], eps,
                          math.sqrt(stats.mse), cost, history)


def relative_error(estimate, reference) -> float:
    """Frobenius relative error, +inf when the reference is 0 (tensor.cpp:152-174)."""
    e = np.asarray(estimate, dtype=np.float64).ravel()
    r = np.asarray(reference, dtype=np.float64).ravel()
    den = float(np.sum(r * r))
    num = float(np.sum((e - r) ** 2))
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return math.sqrt(num / den)
