"""The N > 1 host logic of the batch split (config 5), on CPU with gloo and world_size 2:
the shards partition the batch, and a distributed solve of the shards (oracle as the
per-instance solver on CPU) gathers to exactly the serial results."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_13049_b200 import batch, problem as P


@pytest.mark.parametrize("total,world", [(1024, 8), (1024, 3), (10, 4), (3, 8)])
def test_shards_partition_the_batch(total, world):
    seen = []
    for r in range(world):
        f, c = batch.shard_range(total, world, r)
        seen.extend(range(f, f + c))
    assert seen == list(range(total))
    counts = [batch.shard_range(total, world, r)[1] for r in range(world)]
    assert max(counts) - min(counts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _solve_share(rank, world, port, total, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    data = P.heat2d_problem(6, 5, T=6, splits=([3], [3], [2], [2]))
    base = P.build_dense_qp(data)
    xbs = P.batch_initial_states(data.A.shape[0], total, seed=3)
    first, count = batch.shard_range(total, world, rank)
    rows = []
    for xb in xbs[first:first + count]:
        h, h0, d = batch.instance_affine(base, xb)
        r = O.solve(O.qp_from_arrays(base.H, h, h0, base.J, d))
        rows.append(np.concatenate([[r.iter, r.objective], r.v]))
    res = batch.gather_rows(dist, np.array(rows).reshape(count, -1), total, world, rank)
    if rank == 0:
        np.save(os.path.join(out_dir, "dist.npy"), res)
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_batch_matches_serial(tmp_path):
    total, world = 6, 2
    mp.spawn(_solve_share, args=(world, _free_port(), total, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "dist.npy")
    from oracle import oracle as O
    data = P.heat2d_problem(6, 5, T=6, splits=([3], [3], [2], [2]))
    base = P.build_dense_qp(data)
    for i, xb in enumerate(P.batch_initial_states(data.A.shape[0], total, seed=3)):
        h, h0, d = batch.instance_affine(base, xb)
        r = O.solve(O.qp_from_arrays(base.H, h, h0, base.J, d))
        assert got[i, 0] == r.iter and got[i, 1] == r.objective
        assert np.array_equal(got[i, 2:], r.v)
        fresh = data.copy()
        fresh.x_bar = xb
        q2 = P.build_dense_qp(fresh)
        assert np.allclose(q2.h, h, rtol=1e-13, atol=1e-12) and np.allclose(q2.d, d, rtol=1e-13, atol=1e-12)
