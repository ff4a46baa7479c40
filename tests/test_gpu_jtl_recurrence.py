"""J'lambda carried along the iteration: after a step the residual pass takes
J'lambda + alpha J'p_lambda with J'p_lambda = (M - H) pv - J'(r2 - sigma r3) instead of a pass
over J. The reference recomputes J'lambda from lambda (ipm.cpp:46-70); the two must give the
same solve: same iterations, iterates within the parity tolerance, and a final kkt that the
direct residual pass confirms."""
import numpy as np
import pytest

from _cmpc_helpers import rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = pytest.mark.gpu


def _solve(qp, recur: bool):
    dq = ipm.DeviceQp(qp)
    dq.set_option("jtl_recurrence", 1 if recur else 0)  # per context: no process-wide switch
    return dq, dq.solve()


@pytest.mark.parametrize("shape", [(12, 10, 14), (20, 25, 30)])
def test_carried_jtl_matches_the_direct_pass(shape):
    nx, ny, T = shape
    qp = P.build_dense_qp(P.heat2d_problem(nx, ny, T=T))
    dq_a, a = _solve(qp, True)
    dq_b, b = _solve(qp, False)
    try:
        assert a.status == b.status == ipm.IpmStatus.converged
        assert a.iter == b.iter
        assert rel(a.v, b.v) <= 1e-9 and rel(a.lambda_, b.lambda_) <= 1e-9
        assert abs(a.objective - b.objective) <= 1e-10 * (1 + abs(b.objective))
        # the final state's residuals by the direct pass (the reference's compute_residuals)
        res = ipm.compute_residuals(qp, ipm.IpmState(v=a.v, s=a.s, lambda_=a.lambda_, z=a.z,
                                                     mu=1e-9))
        r1_direct = res.r1
        r1_ref = qp.H @ a.v + qp.h + qp.J.T @ a.lambda_
        assert np.abs(r1_direct - r1_ref).max() <= 1e-9 * (1 + np.abs(r1_ref).max())
        assert a.kkt_error <= 1e-8 and np.abs(r1_direct).max() <= 1e-6 * (1 + np.abs(qp.h).max())
    finally:
        dq_a.close()
        dq_b.close()


def test_separate_rhs_pass_matches_the_fused_one():
    """the separate P'q pass (option rhs_pass = 2) against the SYRK-fused right-hand side, on
    two contexts of one process (the options are per context)"""
    qp = P.build_dense_qp(P.heat2d_problem(12, 10, T=14))
    out = {}
    for mode in (1, 2):
        dq = ipm.DeviceQp(qp)
        dq.set_option("rhs_pass", mode)
        out[mode] = dq.solve()
        dq.close()
    a, b = out[1], out[2]
    assert a.status == b.status == ipm.IpmStatus.converged and a.iter == b.iter
    assert rel(a.v, b.v) <= 1e-9
    assert abs(a.objective - b.objective) <= 1e-10 * (1 + abs(b.objective))


def test_options_are_per_context_and_checked():
    qp = P.build_dense_qp(P.heat2d_problem(8, 6, T=8))
    a, b = ipm.DeviceQp(qp), ipm.DeviceQp(qp)
    a.set_option("graphs", 0)  # eager launches on a only
    ra, rb = a.solve(), b.solve()
    assert ra.iter == rb.iter and np.array_equal(ra.v, rb.v)  # same kernels, same order
    for key, val in (("graphs", 2), ("rhs_pass", 3), ("no_such_option", 1)):
        with pytest.raises(Exception):
            a.set_option(key, val)
    a.close()
    b.close()
