"""The exact structure analysis of J (distinct rows up to sign, prefix widths, singleton and
all-zero rows) must be invisible: every J product equals the dense one."""
import numpy as np
import pytest

from _cmpc_helpers import oracle_qp, rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = pytest.mark.gpu


def planted_J(rng, m_base, n):
    rows = []
    for _ in range(m_base):
        w = int(rng.integers(2, n + 1))
        r = np.zeros(n)
        r[:w] = rng.uniform(-1, 1, w)
        rows.append(r)
    base = list(rows)
    rows += [-r for r in base[: m_base // 2]]             # exact negations (upper/lower bounds)
    rows += [r.copy() for r in base[: m_base // 3]]       # exact duplicates
    rows += [-2.0 * r for r in base[:3]]                  # same pattern, different scale
    rows += [np.zeros(n) for _ in range(5)]               # all-zero rows
    for k in range(6):                                    # singletons, repeated columns
        e = np.zeros(n)
        e[k % 3] = [1.0, -1.0, 2.5][k % 3]
        rows.append(e)
    z = np.zeros(n)
    z[0] = -0.0
    z[1] = 3.0
    rows.append(z)                                        # signed zero inside a singleton
    nearly = base[0].copy()
    nearly[0] = np.nextafter(nearly[0], 2.0)
    rows.append(nearly)                                   # one ulp away: a different row
    J = np.array(rows)
    return J[rng.permutation(J.shape[0])]


@pytest.mark.parametrize("n", [3, 17, 64, 65, 130])
def test_products_match_dense_algebra(n):
    rng = np.random.default_rng(n)
    J = planted_J(rng, 40, n)
    m = J.shape[0]
    G = rng.uniform(-1, 1, (n, n))
    H = G.T @ G + np.eye(n)
    qp = P.DenseQp(H=H, h=rng.uniform(-1, 1, n), h0=0.5, J=J, d=rng.uniform(1, 2, m))
    st = ipm.IpmState(rng.uniform(-1, 1, n), rng.uniform(0.5, 2, m), rng.uniform(-1, 1, m),
                      rng.uniform(0.5, 2, m), 0.1)
    res = ipm.compute_residuals(qp, st)
    assert rel(res.r1, H @ st.v + qp.h + J.T @ st.lambda_) <= 1e-14
    assert rel(res.r3, J @ st.v - qp.d + st.s) <= 1e-14
    sigma = rng.uniform(0.01, 100, m)
    M = ipm.assemble_condensed(qp, sigma)
    ref = H + J.T @ (sigma[:, None] * J)
    assert rel(M, ref) <= 1e-13
    info = ipm.device_qp(qp).info()
    assert info["prototypes"] < m  # duplicates and negations were merged


def test_solve_on_planted_structure_matches_oracle(O):
    rng = np.random.default_rng(7)
    n = 24
    J = planted_J(rng, 30, n)
    m = J.shape[0]
    G = rng.uniform(-1, 1, (n, n))
    v0 = rng.uniform(-0.5, 0.5, n)
    d = J @ v0 + rng.uniform(0.5, 1.5, m)  # strictly feasible at v0
    d[np.all(J == 0, axis=1)] = 1.0
    qp = P.DenseQp(H=G.T @ G + np.eye(n), h=rng.uniform(-3, 3, n), h0=0.0, J=J, d=d)
    r = ipm.solve(qp)
    o = O.solve(oracle_qp(O, qp))
    assert r.status.name == o.status == "converged"
    assert r.iter == o.iter
    assert rel(r.v, o.v) <= 1e-8 and abs(r.objective - o.objective) <= 1e-8 * (1 + abs(o.objective))


def test_dense_unstructured_J_uses_every_row(O):
    rng = np.random.default_rng(3)
    n, m = 70, 300
    J = rng.uniform(-1, 1, (m, n))
    G = rng.uniform(-1, 1, (n, n))
    qp = P.DenseQp(H=G.T @ G + np.eye(n), h=rng.uniform(-1, 1, n), h0=0.0, J=J,
                   d=rng.uniform(1, 2, m))
    info = ipm.device_qp(qp).info()
    assert info["prototypes"] == m and info["syrk_prototypes"] == m
    r = ipm.solve(qp)
    o = O.solve(oracle_qp(O, qp))
    assert r.iter == o.iter and rel(r.v, o.v) <= 1e-8
