"""Device solve vs the oracle (CPU restatement of the reference) on identical QPs:
same iteration count, same barrier/shift/line-search decisions, objective and iterates
within 1e-8 relative, KKT error within 1e-9 (BASELINE.json north star). Also against the
committed golden fixtures."""
import json
import os
import sys

import numpy as np
import pytest

from _cmpc_helpers import lq_from_oracle, oracle_qp, rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
TOL = 1e-8


def solve_both(O, qp):
    log = []
    r = ipm.solve(qp, ipm.IpmOptions(log=log.append))
    o = O.solve(oracle_qp(O, qp))
    return r, o, log


def assert_parity(r, o, log):
    assert r.status.name == o.status
    assert r.iter == o.iter
    assert abs(r.objective - o.objective) <= TOL * (1 + abs(o.objective))
    assert rel(r.v, o.v) <= TOL
    assert rel(r.s, o.s) <= TOL and rel(r.lambda_, o.lam) <= TOL and rel(r.z, o.z) <= TOL
    assert abs(r.kkt_error - o.kkt_error) <= 1e-9
    # decision-for-decision: barrier value, shift and accepted trial of every iteration
    assert [x.mu for x in log] == [row[1] for row in o.log]
    assert [x.delta for x in log] == [row[6] for row in o.log]
    assert [x.trial for x in log] == [int(row[7]) for row in o.log]
    for x, row in zip(log, o.log):
        assert x.alpha == pytest.approx(row[2], rel=1e-6, abs=1e-12)


@pytest.mark.parametrize("i", range(20))
def test_config1_random_ensemble(O, i):
    p = O.random_problem(O.instance_rng(42, i), fixed=(10, 2, 0, 10))
    assert_parity(*solve_both(O, P.build_dense_qp(lq_from_oracle(p))))


@pytest.mark.parametrize("N,T", [(2, 10), (4, 50)])
def test_reference_heat_cube(O, N, T):
    assert_parity(*solve_both(O, P.build_dense_qp(P.build_heat_problem(P.HeatParams(N=N, T=T)))))


def test_config2_heat_rod_full_size(O):
    O.set_threads(os.cpu_count() or 1)
    assert_parity(*solve_both(O, P.build_dense_qp(P.heat1d_problem(200, 50))))


@pytest.mark.parametrize("shape", [(20, 20, 20), (40, 25, 10), (10, 10, 60)])
def test_heat_plates_scaled(O, shape):
    nx, ny, T = shape
    O.set_threads(os.cpu_count() or 1)
    assert_parity(*solve_both(O, P.build_dense_qp(P.heat2d_problem(nx, ny, T=T))))


def test_config5_instance_full_size(O):
    O.set_threads(os.cpu_count() or 1)
    assert_parity(*solve_both(O, P.build_dense_qp(P.heat2d_problem(20, 25, T=30))))


def test_inequality_mix_with_mixed_constraints_and_feedback(O):
    for i in range(10):
        p = O.random_problem(O.instance_rng(99, i), max_n_x=4, max_n_u=3, max_n_c=2, max_T=5)
        assert_parity(*solve_both(O, P.build_dense_qp(lq_from_oracle(p))))


GOLD = json.load(open(os.path.join(HERE, "golden", "oracle_golden.json")))


@pytest.mark.parametrize("name", sorted(GOLD))
def test_device_matches_golden_fixtures(name):
    import make_golden
    qp = make_golden.cases()[name]
    want = GOLD[name]
    log = []
    r = ipm.solve(qp, ipm.IpmOptions(log=log.append))
    assert r.status.name == want["status"] and r.iter == want["iter"]
    assert abs(r.objective - want["objective"]) <= TOL * (1 + abs(want["objective"]))
    assert rel(r.v, want["v"]) <= TOL and rel(r.z, want["z"]) <= TOL
    assert [x.trial for x in log] == [int(row[7]) for row in want["log"]]


def _with_dead_column(qp, h_dead: float):
    """The QP with one extra variable that no constraint touches and H couples to nothing:
    M's extra diagonal entry is exactly h_dead at every iteration, so the reference's shift
    ladder (ipm.cpp:205-221) decides every factorization; the variable's gradient stays 0."""
    n = qp.n
    H = np.zeros((n + 1, n + 1))
    H[:n, :n] = qp.H
    H[n, n] = h_dead
    J = np.zeros((qp.m, n + 1))
    J[:, :n] = qp.J
    return P.DenseQp(H=H, h=np.append(qp.h, 0.0), h0=qp.h0, J=J, d=qp.d)


@pytest.mark.parametrize("h_dead,delta", [(0.0, 1e-8), (-5e-7, 1e-6), (-0.5, 1.0)])
def test_shift_ladder_rescues_every_step_like_the_reference(O, h_dead, delta):
    # proj/src/ipm.cpp:205-221 (the reference's own test covers only total failure,
    # proj/tests/test_ipm.cpp:397-403): the zero pivot fails at delta = 0 and the ladder's
    # first sufficient shift is used and logged, on the device as in the oracle
    p = O.random_problem(O.instance_rng(42, 3), fixed=(10, 2, 0, 10))
    qp = _with_dead_column(P.build_dense_qp(lq_from_oracle(p)), h_dead)
    r, o, log = solve_both(O, qp)
    assert_parity(r, o, log)
    assert r.status == ipm.IpmStatus.converged
    assert {x.delta for x in log} == {delta}


def test_inspected_kkt_matches_the_reference_after_every_barrier_update(O):
    # compute_residuals at the new mu (ipm.cpp:197): the device recomputes only the
    # complementarity part; the kkt seen by inspect must be the reference's at every iteration
    for i in range(3):
        p = O.random_problem(O.instance_rng(42, i), fixed=(10, 2, 0, 10))
        qp = P.build_dense_qp(lq_from_oracle(p))
        dev, ref = [], []
        r = ipm.solve(qp, ipm.IpmOptions(inspect=lambda s: dev.append((s.state.mu, s.residuals.kkt_error))))
        O.solve(oracle_qp(O, qp), inspect=lambda d: ref.append((d["mu"], d["kkt"])))
        assert r.status == ipm.IpmStatus.converged and len(dev) == len(ref) == r.iter
        mus = [m for m, _ in ref]
        assert [m for m, _ in dev] == mus
        assert len(set(mus)) > 3  # the barrier moved several times
        for (_, kd), (_, kr) in zip(dev, ref):
            assert abs(kd - kr) <= 1e-9 * (1 + abs(kr))


def test_failure_exit_reports_the_reference_kkt(O):
    # every shift fails (a dead column with M entry -1e3 < -1e2): factorization_failure after
    # the first barrier decision, returning the residual kkt at the current mu (ipm.cpp:219-226)
    p = O.random_problem(O.instance_rng(42, 0), fixed=(10, 2, 0, 10))
    qp = _with_dead_column(P.build_dense_qp(lq_from_oracle(p)), -1e3)
    r = ipm.solve(qp)
    o = O.solve(oracle_qp(O, qp))
    assert r.status.name == o.status == "factorization_failure"
    assert r.iter == o.iter == 0
    assert abs(r.kkt_error - o.kkt_error) <= 1e-9 * (1 + abs(o.kkt_error))
