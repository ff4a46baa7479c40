"""Shared test helpers (the oracle is test infrastructure only)."""
import numpy as np


def lq_from_oracle(p):
    from paper_2209_13049_b200 import problem as P
    d = p.as_dict()
    T = d.pop("T")
    return P.LqProblemData(T=T, **d)


def oracle_qp(O, qp):
    """Oracle DenseQp holding exactly the arrays of a product DenseQp."""
    return O.qp_from_arrays(qp.H, qp.h, qp.h0, qp.J, qp.d)


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / (1.0 + np.abs(b).max()))


def assert_log_parity(log, ref_rows, tol=1e-8):
    """Decision-for-decision agreement of a device iteration log with the oracle's
    (iter, mu, alpha, alpha_z, kkt, objective, delta, trial) rows: barrier values, shifts and
    accepted trials exactly; step lengths, kkt and objective to the north-star tolerances."""
    ref_rows = [list(r) for r in ref_rows]
    assert len(log) == len(ref_rows)
    for x, row in zip(log, ref_rows):
        assert x.iter == int(row[0])
        assert x.mu == row[1], (x.iter, x.mu, row[1])
        assert x.delta == row[6], (x.iter, x.delta, row[6])
        assert x.trial == int(row[7]), (x.iter, x.trial, row[7])
        assert abs(x.alpha - row[2]) <= 1e-6 * row[2] + 1e-12, (x.iter, x.alpha, row[2])
        assert abs(x.alpha_z - row[3]) <= 1e-6 * row[3] + 1e-12, (x.iter, x.alpha_z, row[3])
        assert abs(x.kkt_error - row[4]) <= 1e-9 * (1 + abs(row[4])), (x.iter, x.kkt_error, row[4])
        assert abs(x.objective - row[5]) <= tol * (1 + abs(row[5])), (x.iter, x.objective, row[5])
