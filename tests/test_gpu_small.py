"""The one-CTA solver (csrc/small.cu: the whole ipm::solve loop in one kernel for QPs with
n <= 32 whose J fits in shared memory) and the general host-driven path must both match the
oracle decision for decision: the parity tests of test_gpu_parity.py run through the one-CTA
solver at config 1; these run the same QPs through both paths explicitly."""
import numpy as np
import pytest

from _cmpc_helpers import lq_from_oracle, oracle_qp, rel
from paper_2209_13049_b200 import ipm, problem as P
from test_gpu_parity import _with_dead_column, assert_parity

pytestmark = pytest.mark.gpu


def _solve(qp, small: bool):
    dq = ipm.DeviceQp(qp)
    dq.set_option("small_path", 1 if small else 0)
    log = []
    r = ipm.solve_loaded(dq, qp, ipm.IpmOptions(log=log.append))
    dq.close()
    return r, log


@pytest.mark.parametrize("i", range(8))
def test_both_paths_match_the_oracle_config1(O, i):
    p = O.random_problem(O.instance_rng(42, i), fixed=(10, 2, 0, 10))
    qp = P.build_dense_qp(lq_from_oracle(p))
    o = O.solve(oracle_qp(O, qp))
    rs, ls = _solve(qp, True)
    rg, lg = _solve(qp, False)
    assert rs.launches == 1 and rg.launches > 1  # the one-CTA solver is one kernel
    assert_parity(rs, o, ls)
    assert_parity(rg, o, lg)
    assert rel(rs.v, rg.v) <= 1e-10


@pytest.mark.parametrize("h_dead", [0.0, -0.5])
def test_shift_ladder_through_the_one_cta_solver(O, h_dead):
    p = O.random_problem(O.instance_rng(42, 3), fixed=(10, 2, 0, 10))
    qp = _with_dead_column(P.build_dense_qp(lq_from_oracle(p)), h_dead)
    o = O.solve(oracle_qp(O, qp))
    r, log = _solve(qp, True)
    assert r.launches == 1
    assert_parity(r, o, log)
    assert all(x.delta > 0 for x in log)


def test_failure_exits_through_the_one_cta_solver(O):
    # total factorization failure (the reference's own test_ipm.cpp:397-403 case) and max_iter
    qp = P.DenseQp(H=np.array([[-1e10]]), h=np.zeros(1), h0=0.0, J=np.zeros((0, 1)), d=np.zeros(0))
    r, _ = _solve(qp, True)
    assert r.status == ipm.IpmStatus.factorization_failure and r.launches == 1
    p = O.random_problem(O.instance_rng(42, 1), fixed=(10, 2, 0, 10))
    qp = P.build_dense_qp(lq_from_oracle(p))
    dq = ipm.DeviceQp(qp)
    r = ipm.solve_loaded(dq, qp, ipm.IpmOptions(max_iter=3))
    o = O.solve(oracle_qp(O, qp), max_iter=3)
    dq.close()
    assert r.status == ipm.IpmStatus.max_iter and r.iter == 3 == o.iter
    assert rel(r.v, o.v) <= 1e-8
