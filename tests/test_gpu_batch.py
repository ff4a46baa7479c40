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


def test_batch_matches_single_solves_and_oracle(O):
    data = P.heat2d_problem(10, 8, T=12, splits=([5], [5], [4], [4]))
    base, insts = instances(data, 12)
    bs = ipm.BatchSolver(base, len(insts))
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


def test_config5_batch_slice():
    data = P.heat2d_problem(20, 25, T=30)
    base, insts = instances(data, 8, seed=11)
    bs = ipm.BatchSolver(base, len(insts))
    for i, q in enumerate(insts):
        bs.set_instance(i, q.h, q.h0, q.d)
    res = bs.solve(threads=2)  # two workers: each solves several instances in turn
    assert all(s == "converged" for s in res.status)
    for i in (0, 3, 7):
        single = ipm.solve(insts[i])
        assert res.iter[i] == single.iter and rel(res.v[i], single.v) <= 1e-14
        # h0 differs per instance; a worker context replays graphs captured for an earlier one
        assert abs(res.objective[i] - single.objective) <= 1e-12 * (1 + abs(single.objective))


def test_batch_solvers_can_be_created_again_on_the_same_base():
    """Closing a batch solver closes its root context; the QP's cached device context is
    re-created for the next one (regression: the second construction dereferenced a closed
    context)."""
    data = P.heat2d_problem(10, 8, T=12, splits=([5], [5], [4], [4]))
    base, insts = instances(data, 6)
    iters = []
    for _ in range(3):
        bs = ipm.BatchSolver(base, len(insts), workers=3)
        for i, q in enumerate(insts):
            bs.set_instance(i, q.h, q.h0, q.d)
        res = bs.solve()
        assert all(s == "converged" for s in res.status)
        iters.append(list(res.iter))
        bs.close()
    assert iters[0] == iters[1] == iters[2]
