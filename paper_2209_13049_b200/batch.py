"""Splitting a batch of independent MPC instances across ranks (one GPU per rank).

Config 5 of BASELINE.json: 1024 instances that share H and J and differ in the initial
state (reduction.cpp:270-280 `refresh_initial_state`). Instances are independent, so the
split needs no collective on the data path: each rank solves a contiguous share with
`ipm.BatchSolver`; only the timing (max over ranks) and, optionally, the results are
exchanged (torch.distributed, NCCL on GPUs or gloo on CPU).
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[first, first + count) of `total` instances owned by `rank` (balanced, contiguous)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def instance_affine(base_qp, x_bar):
    """(h, h0, d) of the instance with initial state x_bar (same H and J as base_qp)."""
    from . import problem as P
    q = P.DenseQp(H=base_qp.H, h=base_qp.h, h0=base_qp.h0, J=np.zeros((0, base_qp.n)),
                  d=np.zeros(0), source=base_qp.source.copy(), gk=base_qp.gk, x0=None)
    q.d = base_qp.d.copy()
    P.refresh_initial_state(q, x_bar)
    return q.h, q.h0, q.d


def gather_rows(dist, local: np.ndarray, total: int, world: int, rank: int) -> np.ndarray:
    """All ranks' result rows in instance order (object all-gather; small results only)."""
    if dist is None or world == 1:
        return local
    parts = [None] * world
    dist.all_gather_object(parts, (rank, local))
    parts.sort(key=lambda x: x[0])
    out = np.concatenate([p[1] for p in parts], axis=0)
    assert out.shape[0] == total
    return out
