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
