"""BASELINE.json configurations at full size, checked against the oracle (CPU restatement of
the reference solver) decision for decision (north star: same iteration count, objective and
iterates within 1e-8 relative, KKT within 1e-9; the log's barrier values, shifts and accepted
trials exactly):

* config 3 (2-D plate 50x50, T=50): the oracle's whole solve runs live beside the device
  (skip-zeros test mode: bitwise the dense loops' results, ~15 s on the box) and every iterate
  is compared in full; also against the committed fixture.
* config 4 (40x25 plate, T = 50, 100, 150, 200): against the committed fixtures of the
  oracle's whole solves (tests/golden/make_fullsize.py): the full log, v, the objective and
  kkt, and a fixed sample of s, lambda, z rows plus their full-vector sums.
Plus size-independent properties: KKT recomputed on the host from the dense J, bitwise
determinism, feasibility of the recovered trajectory, the receding-horizon refresh."""
import os

import numpy as np
import pytest

from _cmpc_helpers import assert_log_parity, oracle_qp, rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-8


def host_kkt(qp, r, mu):
    """compute_residuals (ipm.cpp:46-70) in numpy on the final iterate."""
    n, m = qp.n, qp.m
    r1 = qp.H @ r.v + qp.h + qp.J.T @ r.lambda_
    r3 = qp.J @ r.v - qp.d + r.s
    ds = max(1.0, max(np.abs(qp.h).max(), np.abs(r.lambda_).max()) / (n + m))
    cs = max(1.0, max(np.abs(r.s).max(), np.abs(r.z).max()) / (2 * m))
    comp = np.abs(r.s * r.z - mu).max()
    return max(np.abs(r1).max() / ds, np.abs(r3).max(), comp / cs)


def fixture(name):
    return np.load(os.path.join(HERE, "golden", f"fullsize_{name}.npz"))


def assert_matches_fixture(r, log, g):
    assert r.status.name == str(g["status"])
    assert r.iter == int(g["iter"])
    obj = float(g["objective"])
    assert abs(r.objective - obj) <= TOL * (1 + abs(obj))
    assert abs(r.kkt_error - float(g["kkt_error"])) <= 1e-9
    assert rel(r.v, g["v"]) <= TOL
    rows = g["rows"]
    for got, key in ((r.s, "s"), (r.lambda_, "lam"), (r.z, "z")):
        want = g[key]
        scale = 1.0 + float(g[key + "_sum"][2])  # the full vector's max |x|
        assert np.abs(got[rows] - want).max() <= TOL * scale, key
        s = g[key + "_sum"]
        assert abs(got.sum() - s[0]) <= TOL * scale * got.size, key
        assert abs((got * got).sum() - s[1]) <= 2 * TOL * scale * scale * got.size, key
        assert abs(np.abs(got).max() - s[2]) <= TOL * scale, key
    assert_log_parity(log, g["log"])


@pytest.fixture(scope="module")
def c3():
    return P.build_dense_qp(P.heat2d_problem(50, 50, T=50))


@pytest.fixture(scope="module")
def c3_solve(c3):
    log = []
    r = ipm.solve(c3, ipm.IpmOptions(log=log.append))
    return r, log


def test_config3_full_solve_matches_the_oracle_live(O, c3, c3_solve):
    r, log = c3_solve
    O.set_threads(os.cpu_count() or 1)
    O.set_skip_zeros(True)
    try:
        o = O.solve(oracle_qp(O, c3))
    finally:
        O.set_skip_zeros(False)
    assert r.status.name == o.status == "converged"
    assert r.iter == o.iter
    assert abs(r.objective - o.objective) <= TOL * (1 + abs(o.objective))
    assert rel(r.v, o.v) <= TOL
    assert rel(r.s, o.s) <= TOL and rel(r.lambda_, o.lam) <= TOL and rel(r.z, o.z) <= TOL
    assert abs(r.kkt_error - o.kkt_error) <= 1e-9
    assert_log_parity(log, o.log)


def test_config3_full_solve_matches_the_committed_fixture(c3_solve):
    assert_matches_fixture(*c3_solve, fixture("c3"))


def test_config3_kkt_and_trajectory_on_the_host(c3, c3_solve):
    r, log = c3_solve
    assert r.status == ipm.IpmStatus.converged
    assert host_kkt(c3, r, log[-1].mu) <= 1e-8
    assert r.kkt_error <= 1e-8
    x = r.solution.x
    assert x.min() >= -150.0 - 1e-6 and x.max() <= 200.0 + 1e-6
    assert r.solution.u.min() >= -50.0 - 1e-6 and r.solution.u.max() <= 150.0 + 1e-6


def test_config3_is_bitwise_deterministic(c3, c3_solve):
    a, _ = c3_solve
    b = ipm.solve(c3)
    assert a.iter == b.iter
    assert np.array_equal(a.v, b.v) and np.array_equal(a.s, b.s) and np.array_equal(a.z, b.z)


@pytest.mark.parametrize("T", [50, 100, 150, 200])
def test_config4_long_horizon_sweep_matches_the_oracle(T):
    qp = P.build_dense_qp(P.heat2d_problem(40, 25, T=T))
    log = []
    r = ipm.solve(qp, ipm.IpmOptions(log=log.append))
    qp.invalidate_device()
    assert_matches_fixture(r, log, fixture(f"c4_T{T}"))
    assert host_kkt(qp, r, log[-1].mu) <= 1e-8


def test_config5_instance_and_refresh():
    qp = P.build_dense_qp(P.heat2d_problem(20, 25, T=30))
    r = ipm.solve(qp)
    assert r.status == ipm.IpmStatus.converged and r.iter == 31
    # receding-horizon re-solve: same H and J, refreshed h, h0, d on the device context
    xb = P.batch_initial_states(500, 1, seed=5)[0]
    P.refresh_initial_state(qp, xb)
    r2 = ipm.solve(qp)
    assert r2.status == ipm.IpmStatus.converged
    fresh = P.build_dense_qp(P.heat2d_problem(20, 25, T=30, x_bar=xb))
    r3 = ipm.solve(fresh)
    assert r2.iter == r3.iter and rel(r2.v, r3.v) <= 1e-12
