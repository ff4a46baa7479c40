"""The row-sharded iteration's reduction plan (device side: vec.cu
launch_residuals / launch_rhs_partial / launch_recover / launch_trial and ipm_host.cpp
seg_step), on CPU with gloo, world_size 2 and 3.

Each rank holds rows J_g, d_g and the matching s_g, lambda_g, z_g; v, H, h are replicated.
The numpy loop below restates proj/src/ipm.cpp:160-268 with every per-row quantity formed
from the rank's rows and combined with exactly the collective the device issues:
  sum  M partial (H added once), J' lambda, J'(r2 - sigma r3), sum |r3|, sum log s,
       sum ps/s, the trial's sum log s_t and sum |J v_t - d + s_t|
  max  |r3|, |s z - mu|, |lambda|, |s|, |z| (residual packet), trial positivity violation
  min  the fraction-to-boundary ratios
and the kkt scaling uses the total row count. Every rank then takes the same decisions; the
result must be the oracle's unsharded solve (same iteration count, iterates within 1e-8)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_13049_b200 import problem as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ar(x, op):
    t = torch.as_tensor(np.atleast_1d(np.asarray(x, dtype=np.float64)).copy())
    dist.all_reduce(t, op=op)
    return t.numpy()


def sharded_solve(qp, rows, tol=1e-8, mu_init=1e-1, kappa=0.2, tau=0.995, eta=1e-4, max_iter=200):
    """ipm.cpp:160-268 on this rank's rows; returns (status, iter, v, kkt, objective)."""
    H, h, h0 = qp.H, qp.h, qp.h0
    J, d = qp.J[rows], qp.d[rows]
    n, m_all = qp.n, qp.m
    SUM, MAX, MIN = dist.ReduceOp.SUM, dist.ReduceOp.MAX, dist.ReduceOp.MIN
    v = np.zeros(n)
    s = np.maximum(1.0, d)
    mu = mu_init
    z = mu / s
    lam = z.copy()
    hmax = np.abs(h).max(initial=0.0)

    def residuals(v, s, lam, z, mu):
        Jtl = _ar(J.T @ lam, SUM)
        r1 = H @ v + h + Jtl
        r2 = lam - mu / s
        r3 = J @ v - d + s
        sums = _ar([np.log(s).sum(), np.abs(r3).sum()], SUM)
        mx = _ar([np.abs(r3).max(initial=0.0), np.abs(s * z - mu).max(initial=0.0),
                  np.abs(lam).max(initial=0.0), np.abs(s).max(initial=0.0),
                  np.abs(z).max(initial=0.0)], MAX)
        sd = max(1.0, max(hmax, mx[2]) / (n + m_all))
        sc = max(1.0, max(mx[3], mx[4]) / (2 * m_all))
        kkt = max(np.abs(r1).max() / sd, mx[0], mx[1] / sc)
        return r1, r2, r3, kkt, sums, mx

    r1, r2, r3, kkt, sums, mx = residuals(v, s, lam, z, mu)
    it = 0
    while True:
        if kkt <= tol and mu <= tol:
            return "converged", it, v, kkt, 0.5 * v @ H @ v + h @ v + h0
        if it >= max_iter:
            return "max_iter", it, v, kkt, None
        if kkt <= 10.0 * mu:
            mu = max(tol / 10.0, kappa * mu)
            r1, r2, r3, kkt, sums, mx = residuals(v, s, lam, z, mu)
        sig = z / s
        M = _ar(((J * sig[:, None]).T @ J).ravel(), SUM).reshape(n, n) + H
        L = None
        for delta in (0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1.0, 1e2):
            try:
                L = np.linalg.cholesky(M + delta * np.eye(n))
                break
            except np.linalg.LinAlgError:
                continue
        if L is None:
            return "factorization_failure", it, v, kkt, None
        rhs = -r1 + _ar(J.T @ (r2 - sig * r3), SUM)
        pv = np.linalg.solve(L.T, np.linalg.solve(L, rhs))
        Jpv = J @ pv
        ps = -r3 - Jpv
        pl = -r2 + sig * (r3 + Jpv)
        pz = mu / s - z - sig * ps
        neg_s, neg_z = ps < 0, pz < 0
        mins = _ar([np.min(tau * (-s[neg_s] / ps[neg_s]), initial=np.inf),
                    np.min(tau * (-z[neg_z] / pz[neg_z]), initial=np.inf)], MIN)
        a_max, a_z = min(1.0, mins[0]), min(1.0, mins[1])
        rho = 10.0 * mx[2] + 1.0
        phi0 = 0.5 * v @ H @ v + h @ v - mu * sums[0] + rho * sums[1]
        D = (H @ v + h) @ pv - mu * _ar((ps / s).sum(), SUM)[0] - rho * sums[1]
        alpha, acc = a_max, None
        for _ in range(31):
            st = s + alpha * ps
            vt = v + alpha * pv
            bad = _ar(float(np.any(st <= 0)), MAX)[0]
            if bad == 0:
                tsum = _ar([np.log(st).sum(), np.abs(J @ vt - d + st).sum()], SUM)
                phi = 0.5 * vt @ H @ vt + h @ vt - mu * tsum[0] + rho * tsum[1]
                if (D <= 0 and phi <= phi0 + eta * alpha * D) or \
                        abs(phi - phi0) <= 10 * np.finfo(float).eps * (1 + abs(phi0)):
                    acc = alpha
                    break
            alpha *= 0.5
        if acc is None:
            return "line_search_failure", it, v, kkt, None
        v, s, lam, z = v + acc * pv, s + acc * ps, lam + acc * pl, z + a_z * pz
        it += 1
        r1, r2, r3, kkt, sums, mx = residuals(v, s, lam, z, mu)


def _rank_main(rank, world, port, out_dir, which):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    qp = _problem(which)
    rows = P.shard_rows(qp, world)[rank]
    st, it, v, kkt, obj = sharded_solve(qp, rows)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.concatenate([[it, kkt, obj or 0.0], v]))
    with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
        f.write(st)
    dist.barrier()
    dist.destroy_process_group()


def _problem(which):
    if which == "heat":
        return P.build_dense_qp(P.heat2d_problem(6, 5, T=8, splits=([3], [3], [2], [2])))
    rng = np.random.default_rng(5)  # a bare dense QP: contiguous equal-count shards
    n, m = 12, 40
    G = rng.uniform(-1, 1, (n, n))
    return P.DenseQp(H=G.T @ G + np.eye(n), h=rng.uniform(-1, 1, n), h0=0.0,
                     J=rng.uniform(-1, 1, (m, n)), d=rng.uniform(0.5, 2.0, m))


@pytest.mark.parametrize("which,world", [("heat", 2), ("heat", 3), ("dense", 2)])
def test_sharded_reduction_plan_reproduces_the_unsharded_solve(tmp_path, O, which, world):
    mp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path), which), nprocs=world, join=True)
    qp = _problem(which)
    ref = O.solve(O.qp_from_arrays(qp.H, qp.h, qp.h0, qp.J, qp.d))
    outs = [np.load(tmp_path / f"r{r}.npy") for r in range(world)]
    for r in range(world):
        assert (tmp_path / f"r{r}.txt").read_text() == ref.status
        np.testing.assert_array_equal(outs[r], outs[0])  # every rank took the same decisions
    it, kkt, obj, v = outs[0][0], outs[0][1], outs[0][2], outs[0][3:]
    assert int(it) == ref.iter
    assert np.abs(v - ref.v).max() <= 1e-8 * (1 + np.abs(ref.v).max())
    assert abs(obj - ref.objective) <= 1e-8 * (1 + abs(ref.objective))


def test_shard_rows_keep_stages_whole_and_balance_work():
    qp = P.build_dense_qp(P.heat2d_problem(20, 25, T=30))
    w = qp.row_width.astype(float) ** 2 + 1
    for world in (2, 4, 8):
        parts = P.shard_rows(qp, world)
        assert sorted(np.concatenate(parts).tolist()) == list(range(qp.m))
        stages = [set(qp.row_stage[p].tolist()) for p in parts]
        for a in range(world):
            for b in range(a + 1, world):
                assert not stages[a] & stages[b]  # whole stages: the +- row pairs stay together
        share = np.array([w[p].sum() for p in parts]) / w.sum()
        assert share.max() <= 1.0 / world + 0.12  # stage granularity (T = 30)
    bare = P.DenseQp(H=np.eye(3), h=np.zeros(3), h0=0.0, J=np.ones((10, 3)), d=np.ones(10))
    parts = P.shard_rows(bare, 4)
    assert np.array_equal(np.concatenate(parts), np.arange(10))  # contiguous blocks, in order
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
