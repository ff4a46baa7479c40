"""J'lambda carried along the iteration: after a step the residual pass takes
J'lambda + alpha J'p_lambda with J'p_lambda = (M - H) pv - J'(r2 - sigma r3) instead of a pass
over J. The reference recomputes J'lambda from lambda (ipm.cpp:46-70); the two must give the
same solve: same iterations, iterates within the parity tolerance, and a final kkt that the
direct residual pass confirms."""
import os

import numpy as np
import pytest

from _cmpc_helpers import rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = pytest.mark.gpu


def _solve(qp, recur: bool):
    if recur:
        os.environ.pop("CMPC_NO_RECUR", None)
    else:
        os.environ["CMPC_NO_RECUR"] = "1"
    try:
        dq = ipm.DeviceQp(qp)  # the switch is read when the context loads the QP
        return dq, dq.solve()
    finally:
        os.environ.pop("CMPC_NO_RECUR", None)


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
    """n > 1024 takes a separate P'q pass instead of the SYRK-fused right-hand side;
    run both forms at a small size (one process each: the switch is read once) and compare."""
    import json
    import subprocess
    import sys
    code = (
        "import json, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "from paper_2209_13049_b200 import ipm, problem as P;"
        "qp = P.build_dense_qp(P.heat2d_problem(12, 10, T=14));"
        "r = ipm.solve(qp);"
        "print(json.dumps({'iter': r.iter, 'status': r.status.name, 'v': r.v.tolist(), 'obj': r.objective}))")
    out = {}
    for mode in ("fused", "separate"):
        env = dict(os.environ, CMPC_RHS_PASS=mode)
        res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert res.returncode == 0, res.stderr[-2000:]
        out[mode] = json.loads(res.stdout.strip().splitlines()[-1])
    a, b = out["fused"], out["separate"]
    assert a["status"] == b["status"] == "converged" and a["iter"] == b["iter"]
    assert rel(np.array(a["v"]), np.array(b["v"])) <= 1e-9
    assert abs(a["obj"] - b["obj"]) <= 1e-10 * (1 + abs(b["obj"]))
