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
