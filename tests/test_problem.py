"""Product-side setup (lean reduction + generators) against the oracle's faithful
restatement of proj/src/reduction.cpp and heat3d.cpp. CPU only."""
import numpy as np
import pytest

from paper_2209_13049_b200 import problem as P
from paper_2209_13049_b200._lib import DimensionError
from _cmpc_helpers import lq_from_oracle, rel


def check_same_qp(q1, q2, tol=1e-12):
    assert q1.H.shape == q2.H.shape and q1.J.shape == q2.J.shape
    assert rel(q1.H, q2.H) <= tol
    assert rel(q1.J, q2.J) <= tol
    assert rel(q1.h, q2.h_vec) <= tol
    assert rel(q1.d, q2.d) <= tol
    assert abs(q1.h0 - q2.h0) <= tol * (1 + abs(q2.h0))


@pytest.mark.parametrize("seed", range(8))
def test_lean_reduction_matches_reference_reduction(O, seed):
    p = O.random_problem(O.instance_rng(11, seed), max_n_x=4, max_n_u=3, max_n_c=2, max_T=5,
                         cap_rows_for_oracle=False)
    check_same_qp(P.build_dense_qp(lq_from_oracle(p)), O.build_dense_qp(p))


def test_lean_reduction_with_feedback_and_infinite_bounds(O):
    rng = np.random.default_rng(3)
    nx, nu, T = 3, 2, 6
    A = rng.uniform(-0.5, 0.5, (nx, nx))
    B = rng.uniform(-1, 1, (nx, nu))
    G = rng.uniform(-1, 1, (nx, nx))
    Q = G.T @ G + 0.1 * np.eye(nx)
    K = rng.uniform(-0.3, 0.3, (nu, nx))
    xl = np.array([-5.0, -np.inf, -4.0])
    xu = np.array([5.0, 6.0, np.inf])
    p = O.problem_from_arrays(A=A, B=B, Q=Q, Qf=Q, R=np.eye(nu), S=rng.uniform(-0.1, 0.1, (nx, nu)),
                              E=rng.uniform(-1, 1, (1, nx)), F=rng.uniform(-1, 1, (1, nu)),
                              gl=[-3.0], gu=[np.inf], xl=xl, xu=xu, ul=[-1.0, -np.inf],
                              uu=[1.0, 2.0], w=rng.uniform(-0.1, 0.1, (T, nx)),
                              x_bar=rng.uniform(-1, 1, nx), K=K, T=T)
    check_same_qp(P.build_dense_qp(lq_from_oracle(p)), O.build_dense_qp(p))


def test_heat3d_generator_matches_reference(O):
    for N, T in [(2, 10), (4, 50)]:
        op = O.heat3d_problem(N, T)
        pp = P.build_heat_problem(P.HeatParams(N=N, T=T))
        for f in ("A", "B", "Q", "R", "xl", "xu", "ul", "uu", "x_bar"):
            assert np.array_equal(op.get(f), getattr(pp, f)), f
        assert np.abs(op.get("w") - pp.w).max() <= 1e-12
        check_same_qp(P.build_dense_qp(pp), O.build_dense_qp(op))


def test_baseline_config_shapes():
    # (n_x, n_u, T) -> (n, m) with every bound finite: m = 2T(n_x + n_u)
    d = P.heat1d_problem(200, 50)
    assert (d.A.shape[0], d.B.shape[1], d.T) == (200, 4, 50)
    d = P.heat2d_problem(50, 50, T=50)
    assert (d.A.shape[0], d.B.shape[1]) == (2500, 10)
    d = P.heat2d_problem(40, 25, T=50)
    assert (d.A.shape[0], d.B.shape[1]) == (1000, 10)
    d = P.heat2d_problem(20, 25, T=30)
    assert (d.A.shape[0], d.B.shape[1]) == (500, 5)
    q = P.build_dense_qp(P.heat2d_problem(20, 25, T=4))
    assert q.n == 4 * 5 and q.m == 2 * 4 * (500 + 5)


@pytest.mark.parametrize("gen", [lambda: P.rod_system(200, P.HeatParams()),
                                 lambda: P.plate_system(50, 50, [17, 34], [17, 34], [25], [25], P.HeatParams()),
                                 lambda: P.plate_system(20, 25, [10], [], [], [], P.HeatParams())])
def test_generators_conserve_row_sums(gen):
    A, B = gen()
    assert np.abs(A.sum(1) + B.sum(1) - 1.0).max() <= 1e-14
    assert (A >= 0).all() and (B >= 0).all()


def test_refresh_initial_state_matches_fresh_build(O):
    d = P.heat2d_problem(6, 5, T=8, splits=([3], [3], [2], [2]))
    q = P.build_dense_qp(d)
    xb = np.linspace(-60, -40, d.x_bar.size)
    P.refresh_initial_state(q, xb)
    d2 = d.copy()
    d2.x_bar = xb
    fresh = P.build_dense_qp(d2)
    assert np.array_equal(q.H, fresh.H) and np.array_equal(q.J, fresh.J)
    assert rel(q.h, fresh.h) == 0.0 and rel(q.d, fresh.d) == 0.0 and q.h0 == fresh.h0
    with pytest.raises(DimensionError):
        P.refresh_initial_state(q, np.zeros(d.x_bar.size + 1))
    # and the oracle's refresh (reduction.cpp:270-280) agrees
    op = O.problem_from_arrays(**{k: getattr(d, k) for k in ("A", "B", "Q", "Qf", "R", "S", "E", "F",
                                                            "gl", "gu", "xl", "xu", "ul", "uu",
                                                            "w", "x_bar", "K", "T")})
    oq = O.build_dense_qp(op)
    oq.refresh_initial_state(xb)
    assert rel(q.h, oq.h_vec) <= 1e-12 and rel(q.d, oq.d) <= 1e-12


@pytest.mark.parametrize("seed", range(5))
def test_recover_trajectory_matches_reference(O, seed):
    p = O.random_problem(O.instance_rng(23, seed), max_n_c=2)
    q = P.build_dense_qp(lq_from_oracle(p))
    oq = O.build_dense_qp(p)
    v = np.random.default_rng(seed).uniform(-1, 1, q.n)
    tr = P.recover_trajectory(q, v)
    xs, us, obj = oq.recover_trajectory(v)
    assert rel(tr.x, xs) <= 1e-12 and rel(tr.u, us) <= 1e-12
    assert abs(tr.objective - obj) <= 1e-10 * (1 + abs(obj))
    assert abs(P.dense_objective(q, v) - oq.dense_objective(v)) <= 1e-10 * (1 + abs(obj))
    with pytest.raises(DimensionError):
        P.recover_trajectory(q, np.zeros(q.n + 1))
    with pytest.raises(DimensionError):
        P.dense_objective(q, np.zeros(q.n + 1))


def test_dims_validation():
    d = P.heat1d_problem(10, 3)
    P.dims(d)
    bad = d.copy()
    bad.B = np.zeros((9, 4))
    with pytest.raises(DimensionError):
        P.dims(bad)
    bad = d.copy()
    bad.T = 4
    with pytest.raises(DimensionError):
        P.dims(bad)


def test_device_cache_is_not_copied_and_tracks_reassignment():
    # dataclasses.replace must not carry the cached device context over, and
    # reassigning H/h/h0/J/d must change the fingerprint the cache is checked against
    import dataclasses
    qp = P.DenseQp(H=[[4.0]], h=[2.0], h0=0.0, J=[[-1.0]], d=[0.0])
    qp._device, qp._device_key = object(), qp.device_key()
    other = dataclasses.replace(qp, d=np.array([1.0]))
    assert other._device is None and other._device_key is None
    k0 = qp.device_key()
    qp.d = np.array([0.5])
    assert qp.device_key() != k0
    k1 = qp.device_key()
    qp.h0 = 1.0
    assert qp.device_key() != k1
    assert qp.device_key() == qp.device_key()
