"""Batch of independent instances sharing H and J (config 5 semantics): each instance of the
batch equals its own single solve and the oracle's."""
import numpy as np
import pytest

from _cmpc_helpers import oracle_qp, rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = pytest.mark.gpu


def instances(data, count, seed=5):
    base = P.build_dense_qp(data)
    xbs = P.batch_initial_states(data.A.shape[0], count, seed=seed)
    out = []
    for xb in xbs:
        d2 = data.copy()
        d2.x_bar = xb
        out.append(P.build_dense_qp(d2))
    return base, out


def test_worker_batch_matches_single_solves_bitwise(O):
    data = P.heat2d_problem(10, 8, T=12, splits=([5], [5], [4], [4]))
    base, insts = instances(data, 12)
    bs = ipm.BatchSolver(base, len(insts), mode="workers")
    for i, q in enumerate(insts):
        bs.set_instance(i, q.h, q.h0, q.d)
    res = bs.solve(threads=4)
    assert all(s == "converged" for s in res.status)
    for i, q in enumerate(insts):
        single = ipm.solve(q)
        assert res.iter[i] == single.iter
        assert np.array_equal(res.v[i], single.v)  # same kernels, same order: bitwise
        o = O.solve(oracle_qp(O, q))
        assert res.iter[i] == o.iter and rel(res.v[i], o.v) <= 1e-8
    bs.close()


def test_lockstep_batch_matches_single_solves_and_oracle(O):
    # the lockstep batch (csrc/batch.cu) takes every decision of ipm.cpp:160-268 per instance:
    # same iterations and barrier sequence as the oracle, iterates within the north-star 1e-8
    data = P.heat2d_problem(10, 8, T=12, splits=([5], [5], [4], [4]))
    base, insts = instances(data, 12)
    bs = ipm.BatchSolver(base, len(insts))
    assert bs.mode == "lockstep"
    for i, q in enumerate(insts):
        bs.set_instance(i, q.h, q.h0, q.d)
    res = bs.solve()
    assert all(s == "converged" for s in res.status)
    for i, q in enumerate(insts):
        single = ipm.solve(q)
        assert res.iter[i] == single.iter and rel(res.v[i], single.v) <= 1e-10
        assert abs(res.objective[i] - single.objective) <= 1e-10 * (1 + abs(single.objective))
        o = O.solve(oracle_qp(O, q))
        assert res.iter[i] == o.iter and rel(res.v[i], o.v) <= 1e-8
        assert abs(res.objective[i] - o.objective) <= 1e-8 * (1 + abs(o.objective))
        assert abs(res.kkt_error[i] - o.kkt_error) <= 1e-9 * (1 + abs(o.kkt_error))
    # a second solve after new instance data reuses the batch context
    for i, q in enumerate(insts[:3]):
        bs.set_instance(i, insts[-1 - i].h, insts[-1 - i].h0, insts[-1 - i].d)
    res2 = bs.solve()
    for i in range(3):
        assert res2.iter[i] == res.iter[len(insts) - 1 - i]
        assert rel(res2.v[i], res.v[len(insts) - 1 - i]) <= 1e-12
    bs.close()


def test_config5_batch_slice():
    data = P.heat2d_problem(20, 25, T=30)
    base, insts = instances(data, 8, seed=11)
    for mode in ("lockstep", "workers"):
        bs = ipm.BatchSolver(base, len(insts), mode=mode)
        for i, q in enumerate(insts):
            bs.set_instance(i, q.h, q.h0, q.d)
        res = bs.solve(threads=2)
        assert all(s == "converged" for s in res.status)
        for i in (0, 3, 7):
            single = ipm.solve(insts[i])
            tol = 1e-14 if mode == "workers" else 1e-10
            assert res.iter[i] == single.iter and rel(res.v[i], single.v) <= tol
            assert abs(res.objective[i] - single.objective) <= 1e-10 * (1 + abs(single.objective))
        bs.close()


def test_batch_solvers_can_be_created_again_on_the_same_base():
    """Closing a batch solver closes its root context; the QP's cached device context is
    re-created for the next one (regression: the second construction dereferenced a closed
    context)."""
    data = P.heat2d_problem(10, 8, T=12, splits=([5], [5], [4], [4]))
    base, insts = instances(data, 6)
    iters = []
    for _ in range(3):
        bs = ipm.BatchSolver(base, len(insts), workers=3, mode="workers")
        for i, q in enumerate(insts):
            bs.set_instance(i, q.h, q.h0, q.d)
        res = bs.solve()
        assert all(s == "converged" for s in res.status)
        iters.append(list(res.iter))
        bs.close()
    assert iters[0] == iters[1] == iters[2]


@pytest.mark.parametrize("shape", ["heat_small", "config5"])
def test_batch_condensation_matches_fp64(shape):
    # the lockstep condensation kernel (csrc/bsyrk.cu) alone: M_b = H + J' diag(sigma_b) J
    # (lower triangle) and tq_b = J' w_b for every instance, against an fp64 numpy product
    # (assemble_condensed, ipm.cpp:72-77; the right-hand side's J'w, ipm.cpp:79-103)
    if shape == "heat_small":
        data = P.heat2d_problem(10, 8, T=12, splits=([5], [5], [4], [4]))
    else:
        import bench
        data = bench.build_problem("c5")
    base = P.build_dense_qp(data)
    cnt = 7
    rng = np.random.default_rng(3)
    m, n = base.m, base.n
    sigma = np.exp(rng.uniform(-6, 6, size=(cnt, m)))
    w = rng.standard_normal((cnt, m))
    bs = ipm.BatchSolver(base, cnt, mode="lockstep")
    M, tq = bs.condense(sigma, w)
    bs.close()
    J, H = base.J, base.H
    for b in range(cnt):
        ref = H + J.T @ (sigma[b][:, None] * J)
        scale = np.abs(H).max() + (np.abs(J).T @ (sigma[b][:, None] * np.abs(J))).max()
        lo = np.tril_indices(n)
        err = np.abs(M[b][lo] - ref[lo]).max() / scale
        assert err <= 1e-13, (b, err)
        tref = J.T @ w[b]
        terr = np.abs(tq[b] - tref).max() / (np.abs(J).T @ np.abs(w[b])).max()
        assert terr <= 1e-13, (b, terr)


def _ragged_qp(n, m, seed):
    """A random strictly convex QP whose constraint rows have ragged nonzero prefixes (widths
    1..n, some repeated up to sign, some all-zero): exercises the batch kernels' region plan and
    chunk widths away from the MPC layout."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n))
    H = G @ G.T + n * np.eye(n)
    J = rng.standard_normal((m, n))
    widths = rng.integers(0, n + 1, size=m)
    for r, w in enumerate(widths):
        J[r, w:] = 0.0
    J[m // 2: m // 2 + 10] = -J[:10]  # exact negations merge into one prototype
    x0 = rng.standard_normal(n) * 0.1
    d = J @ x0 + rng.uniform(0.5, 2.0, size=m)  # strictly feasible at x0
    return P.DenseQp(H=H, h=rng.standard_normal(n), h0=0.0, J=J, d=d)


@pytest.mark.parametrize("n", [2, 17, 37, 100, 160])
def test_batch_kernels_ragged_shapes(n, O):
    # the condensation and the Cholesky of the lockstep batch at n not a multiple of 16 / 32,
    # up to the n = 160 limit: condensation vs fp64, every instance's solve vs its single
    # solve and the oracle
    base = _ragged_qp(n, 3 * n + 20, seed=n)
    cnt = 5
    rng = np.random.default_rng(7)
    m = base.m
    sigma = np.exp(rng.uniform(-4, 4, size=(cnt, m)))
    w = rng.standard_normal((cnt, m))
    bs = ipm.BatchSolver(base, cnt, mode="lockstep")
    M, tq = bs.condense(sigma, w)
    J, H = base.J, base.H
    for b in range(cnt):
        ref = H + J.T @ (sigma[b][:, None] * J)
        lo = np.tril_indices(n)
        scale = np.abs(H).max() + (np.abs(J).T @ (sigma[b][:, None] * np.abs(J))).max()
        assert np.abs(M[b][lo] - ref[lo]).max() <= 1e-13 * scale
        assert np.abs(tq[b] - J.T @ w[b]).max() <= 1e-13 * (np.abs(J).T @ np.abs(w[b])).max()
    qps = []
    for i in range(cnt):
        q = P.DenseQp(H=base.H, h=base.h + 0.1 * rng.standard_normal(n), h0=0.0, J=base.J,
                      d=base.d + 0.05 * rng.uniform(0, 1, size=m))
        qps.append(q)
        bs.set_instance(i, q.h, q.h0, q.d)
    res = bs.solve()
    bs.close()
    for i, q in enumerate(qps):
        single = ipm.solve(q)
        o = O.solve(oracle_qp(O, q))
        assert res.status[i] == single.status.name == o.status
        assert res.iter[i] == single.iter == o.iter
        assert rel(res.v[i], o.v) <= 1e-8
