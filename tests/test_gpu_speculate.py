"""Speculative step segment (option "speculate", csrc/ipm_host.cpp): the update + residual
segment is enqueued behind the factor/step segment before the host has seen the step, gated
on the device's own evaluation of line-search trial 0 (trial0_decide, csrc/vec.cu). The host
re-evaluates trial 0 from the same packet and runs the rest of the line search / the shift
ladder itself when the device refused it. Speculation must not change one bit of the solve:
same records (iterations, mu, alpha, alpha_z, kkt, objective, shift, trial), same iterates.
The problems cover accepted trial 0, refused trial 0 (j > 0) and the shift ladder."""
import numpy as np
import pytest

from _cmpc_helpers import lq_from_oracle, oracle_qp, rel
from paper_2209_13049_b200 import ipm, problem as P
from test_gpu_parity import _with_dead_column, assert_parity

pytestmark = pytest.mark.gpu


def _solve(qp, spec: bool, opts=None):
    dq = ipm.DeviceQp(qp)
    dq.set_option("small_path", 0)  # the host-driven loop (the one-CTA solver has no segments)
    dq.set_option("speculate", 1 if spec else 0)
    log = []
    o = opts or ipm.IpmOptions()
    o.log = log.append
    r = ipm.solve_loaded(dq, qp, o)
    dq.close()
    return r, log


def _problems(O):
    out = []
    for i in range(6):
        p = O.random_problem(O.instance_rng(42, i), fixed=(10, 2, 0, 10))
        out.append(("c1_%d" % i, P.build_dense_qp(lq_from_oracle(p))))
    p = O.random_problem(O.instance_rng(42, 3), fixed=(10, 2, 0, 10))
    base = P.build_dense_qp(lq_from_oracle(p))
    out.append(("dead0", _with_dead_column(base, 0.0)))
    out.append(("dead-", _with_dead_column(base, -0.5)))
    out.append(("heat", P.build_dense_qp(P.heat2d_problem(12, 10, T=14))))
    for i in range(4):
        p = O.random_problem(O.instance_rng(7, i), max_n_x=6, max_n_u=3, max_n_c=2, max_T=12)
        out.append(("rand_%d" % i, P.build_dense_qp(lq_from_oracle(p))))
    return out


def test_speculation_changes_nothing(O):
    seen_refused = seen_shift = 0
    for name, qp in _problems(O):
        ra, la = _solve(qp, True)
        rb, lb = _solve(qp, False)
        assert ra.status == rb.status and ra.iter == rb.iter, name
        assert la == lb, name  # every record field, bit for bit
        for x, y in ((ra.v, rb.v), (ra.s, rb.s), (ra.lambda_, rb.lambda_), (ra.z, rb.z)):
            assert np.array_equal(x, y), name
        seen_refused += sum(1 for x in la if x.trial > 0)
        seen_shift += sum(1 for x in la if x.delta > 0)
    # both fallbacks of the speculative segment ran somewhere in the set
    assert seen_refused > 0 and seen_shift > 0


def test_speculative_solve_matches_the_oracle(O):
    p = O.random_problem(O.instance_rng(42, 5), fixed=(10, 2, 0, 10))
    qp = _with_dead_column(P.build_dense_qp(lq_from_oracle(p)), -0.5)
    o = O.solve(oracle_qp(O, qp))
    r, log = _solve(qp, True)
    assert_parity(r, o, log)


def test_speculation_with_a_max_iter_exit(O):
    p = O.random_problem(O.instance_rng(42, 1), fixed=(10, 2, 0, 10))
    qp = P.build_dense_qp(lq_from_oracle(p))
    ra, la = _solve(qp, True, ipm.IpmOptions(max_iter=3))
    rb, lb = _solve(qp, False, ipm.IpmOptions(max_iter=3))
    assert ra.status == rb.status == ipm.IpmStatus.max_iter and la == lb
    assert rel(ra.v, rb.v) == 0.0
