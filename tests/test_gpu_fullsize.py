"""BASELINE.json configurations at full size: size-independent properties (the oracle is
too slow for whole solves here): convergence, the oracle's iteration count, KKT error
recomputed independently on the host from the dense J, first-iteration parity with the
oracle, bitwise determinism, feasibility of the recovered trajectory."""
import os

import numpy as np
import pytest

from _cmpc_helpers import oracle_qp, rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

# iteration counts of the oracle's full solves (recorded in profiles/oracle_fullsize.json)
ORACLE_ITERS = {"c3": 34, "c5": 31}


def host_kkt(qp, r, mu):
    """compute_residuals (ipm.cpp:46-70) in numpy on the final iterate."""
    n, m = qp.n, qp.m
    r1 = qp.H @ r.v + qp.h + qp.J.T @ r.lambda_
    r3 = qp.J @ r.v - qp.d + r.s
    ds = max(1.0, max(np.abs(qp.h).max(), np.abs(r.lambda_).max()) / (n + m))
    cs = max(1.0, max(np.abs(r.s).max(), np.abs(r.z).max()) / (2 * m))
    comp = np.abs(r.s * r.z - mu).max()
    return max(np.abs(r1).max() / ds, np.abs(r3).max(), comp / cs)


@pytest.fixture(scope="module")
def c3():
    return P.build_dense_qp(P.heat2d_problem(50, 50, T=50))


def test_config3_converges_like_the_reference(c3):
    log = []
    r = ipm.solve(c3, ipm.IpmOptions(log=log.append))
    assert r.status == ipm.IpmStatus.converged
    assert r.iter == ORACLE_ITERS["c3"]
    k = host_kkt(c3, r, log[-1].mu)
    assert k <= 1e-8
    assert r.kkt_error <= 1e-8
    x = r.solution.x
    assert x.min() >= -150.0 - 1e-6 and x.max() <= 200.0 + 1e-6
    assert r.solution.u.min() >= -50.0 - 1e-6 and r.solution.u.max() <= 150.0 + 1e-6


def test_config3_first_iteration_matches_oracle(O, c3):
    O.set_threads(os.cpu_count() or 1)
    o = O.solve(oracle_qp(O, c3), max_iter=1)
    r = ipm.solve(c3, ipm.IpmOptions(max_iter=1))
    assert r.iter == o.iter == 1
    assert rel(r.v, o.v) <= 1e-8 and rel(r.s, o.s) <= 1e-8
    assert rel(r.lambda_, o.lam) <= 1e-8 and rel(r.z, o.z) <= 1e-8
    assert abs(r.kkt_error - o.kkt_error) <= 1e-9 * (1 + abs(o.kkt_error))


def test_config3_is_bitwise_deterministic(c3):
    a = ipm.solve(c3)
    b = ipm.solve(c3)
    assert a.iter == b.iter
    assert np.array_equal(a.v, b.v) and np.array_equal(a.s, b.s) and np.array_equal(a.z, b.z)


def test_config5_instance_and_refresh():
    qp = P.build_dense_qp(P.heat2d_problem(20, 25, T=30))
    r = ipm.solve(qp)
    assert r.status == ipm.IpmStatus.converged and r.iter == ORACLE_ITERS["c5"]
    # receding-horizon re-solve: same H and J, refreshed h, h0, d on the device context
    xb = P.batch_initial_states(500, 1, seed=5)[0]
    P.refresh_initial_state(qp, xb)
    r2 = ipm.solve(qp)
    assert r2.status == ipm.IpmStatus.converged
    fresh = P.build_dense_qp(P.heat2d_problem(20, 25, T=30, x_bar=xb))
    r3 = ipm.solve(fresh)
    assert r2.iter == r3.iter and rel(r2.v, r3.v) <= 1e-12


def test_config4_long_horizon():
    qp = P.build_dense_qp(P.heat2d_problem(40, 25, T=200))
    r = ipm.solve(qp)
    assert r.status == ipm.IpmStatus.converged
    assert host_kkt(qp, r, 1e-9) <= 1e-8
