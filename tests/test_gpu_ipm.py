"""Device IPM steps vs the reference's proj/tests/test_ipm.cpp cases (same names, same
tolerances), through the C ABI."""
import numpy as np
import pytest

from paper_2209_13049_b200 import ipm, linalg, problem as P
from paper_2209_13049_b200._lib import DimensionError

pytestmark = pytest.mark.gpu


def plain_qp(H, h, h0, J, d):
    return P.DenseQp(H=H, h=h, h0=h0, J=J, d=d)


def bound_toy():  # min 0.5*4 v^2 + 2 v  s.t.  v >= 0
    return plain_qp([[4.0]], [2.0], 0.0, [[-1.0]], [0.0])


def augmented_matrix(qp, sigma):
    n, m = qp.n, qp.m
    full = np.zeros((n + 2 * m, n + 2 * m))
    full[:n, :n] = qp.H
    if m:
        full[:n, n + m:] = qp.J.T
        full[n:n + m, n:n + m] = np.diag(sigma)
        full[n:n + m, n + m:] = np.eye(m)
        full[n + m:, :n] = qp.J
        full[n + m:, n:n + m] = np.eye(m)
    return full


def augmented_residual(qp, st, res, dirs):
    sigma = st.z / st.s if qp.m else np.zeros(0)
    full = augmented_matrix(qp, sigma)
    p = np.concatenate([dirs.pv, dirs.ps, dirs.plambda])
    r = np.concatenate([res.r1, res.r2, res.r3])
    denom = np.abs(full).sum(1).max() * np.abs(p).max() + np.abs(r).max()
    return np.abs(full @ p + r).max() / max(denom, 1e-300)


def factor_condensed(qp, st):
    sigma = st.z / st.s if qp.m else np.zeros(0)
    return linalg.make_backend("cuda").factorize(ipm.assemble_condensed(qp, sigma))


def state(v, s, lam, z, mu):
    return ipm.IpmState(np.asarray(v, float), np.asarray(s, float), np.asarray(lam, float),
                        np.asarray(z, float), mu)


def test_residuals_evaluate_their_defining_formulas():
    res = ipm.compute_residuals(bound_toy(), state([0.0], [1.0], [0.0], [0.3], 0.3))
    assert res.r1[0] == pytest.approx(2.0, rel=1e-15)
    assert res.r2[0] == pytest.approx(-0.3, rel=1e-15)
    assert res.r3[0] == pytest.approx(1.0, rel=1e-15)
    assert res.kkt_error == pytest.approx(2.0, rel=1e-15)


def test_residuals_vanish_at_unconstrained_stationary_point():
    qp = plain_qp([[4.0]], [2.0], 2.0, np.zeros((0, 1)), np.zeros(0))
    res = ipm.compute_residuals(qp, state([-0.5], [], [], [], 1e-9))
    assert res.r1[0] == 0.0 and res.kkt_error == 0.0


def test_residuals_are_linear_in_the_multipliers(O):
    from _cmpc_helpers import lq_from_oracle
    qp = P.build_dense_qp(lq_from_oracle(O.random_problem(O.Rng(211))))
    m = qp.m
    rng = np.random.default_rng(1)
    st = state(rng.uniform(-1, 1, qp.n), np.full(m, 0.7), rng.uniform(-1, 1, m), np.full(m, 0.4), 0.05)
    base = ipm.compute_residuals(qp, st)
    delta = np.full(m, 0.25)
    st.lambda_ = st.lambda_ + delta
    moved = ipm.compute_residuals(qp, st)
    assert np.abs(moved.r1 - (base.r1 + qp.J.T @ delta)).max() <= 1e-14
    assert np.abs(moved.r2 - (base.r2 + delta)).max() <= 1e-14
    assert np.abs(moved.r3 - base.r3).max() == 0.0


def test_state_shape_mismatch_is_rejected():
    with pytest.raises(DimensionError):
        ipm.compute_residuals(bound_toy(), state([0.0, 1.0], [1.0], [0.0], [1.0], 0.1))
    with pytest.raises(DimensionError):
        ipm.compute_residuals(bound_toy(), state([0.0], [1.0, 2.0], [0.0], [1.0], 0.1))


def test_condensed_matrix_without_rows_is_H_itself():
    qp = plain_qp(np.eye(3), np.zeros(3), 0.0, np.zeros((0, 3)), np.zeros(0))
    assert np.abs(ipm.assemble_condensed(qp, np.zeros(0)) - np.eye(3)).max() == 0.0


def test_identity_rows_with_unit_weights_double_the_identity():
    qp = plain_qp(np.eye(2), np.zeros(2), 0.0, np.eye(2), np.zeros(2))
    assert np.abs(ipm.assemble_condensed(qp, np.ones(2)) - 2 * np.eye(2)).max() == 0.0


def test_weighted_term_never_destroys_positive_definiteness():
    rng = np.random.default_rng(223)
    for _ in range(20):
        n, m = rng.integers(1, 9, size=2)
        G = rng.uniform(-1, 1, (n, n))
        qp = plain_qp(G.T @ G + 0.1 * np.eye(n), np.zeros(n), 0.0, rng.uniform(-1, 1, (m, n)), np.zeros(m))
        sigma = rng.uniform(0.01, 50.0, m)
        M = ipm.assemble_condensed(qp, sigma)
        assert linalg.is_symmetric(M, 1e-12)
        ref = qp.H + qp.J.T @ (sigma[:, None] * qp.J)
        assert np.abs(M - ref).max() <= 1e-12 * (1 + np.abs(ref).max())
        linalg.make_backend("cuda").factorize(M)


def test_step_directions_reproduce_the_hand_worked_toy():
    qp = bound_toy()
    st = state([0.0], [1.0], [1.0], [1.0], 0.1)
    res = ipm.compute_residuals(qp, st)
    assert (res.r1[0], res.r2[0], res.r3[0]) == (pytest.approx(1.0), pytest.approx(0.9), pytest.approx(1.0))
    d = ipm.step_directions(qp, st, res, factor_condensed(qp, st))
    assert d.pv[0] == pytest.approx(-0.18, rel=1e-14)
    assert d.ps[0] == pytest.approx(-1.18, rel=1e-14)
    assert d.plambda[0] == pytest.approx(0.28, rel=1e-14)
    assert d.pz[0] == pytest.approx(0.28, rel=1e-14)
    assert augmented_residual(qp, st, res, d) <= 1e-15


def test_without_inequalities_the_step_is_the_plain_newton_step():
    qp = plain_qp([[4.0]], [2.0], 0.0, np.zeros((0, 1)), np.zeros(0))
    st = state([1.0], [], [], [], 0.1)
    res = ipm.compute_residuals(qp, st)
    d = ipm.step_directions(qp, st, res, factor_condensed(qp, st))
    assert d.pv[0] == pytest.approx(-res.r1[0] / 4.0, rel=1e-15)
    assert d.ps.size == d.plambda.size == d.pz.size == 0


def test_condensed_directions_solve_the_full_block_system():
    rng = np.random.default_rng(227)
    for _ in range(20):
        n, m = int(rng.integers(1, 7)), int(rng.integers(1, 11))
        G = rng.uniform(-1, 1, (n, n))
        qp = plain_qp(G.T @ G + 0.2 * np.eye(n), rng.uniform(-1, 1, n), 0.0,
                      rng.uniform(-1, 1, (m, n)), rng.uniform(-1, 1, m))
        st = state(rng.uniform(-1, 1, n), rng.uniform(0.2, 3.0, m), rng.uniform(-1, 1, m),
                   rng.uniform(0.2, 3.0, m), 0.05)
        res = ipm.compute_residuals(qp, st)
        d = ipm.step_directions(qp, st, res, factor_condensed(qp, st))
        direct = np.linalg.solve(augmented_matrix(qp, st.z / st.s),
                                 -np.concatenate([res.r1, res.r2, res.r3]))
        scale = 1 + np.abs(direct).max()
        assert np.abs(d.pv - direct[:n]).max() <= 1e-9 * scale
        assert np.abs(d.ps - direct[n:n + m]).max() <= 1e-9 * scale
        assert np.abs(d.plambda - direct[n + m:]).max() <= 1e-9 * scale
        assert augmented_residual(qp, st, res, d) <= 1e-8


def test_fraction_to_boundary():
    assert ipm.fraction_to_boundary(np.ones(3), np.ones(3), np.ones(3), np.zeros(3), 0.995) == (1.0, 1.0)
    a, az = ipm.fraction_to_boundary(np.ones(1), -np.ones(1), np.ones(1), np.ones(1), 0.995)
    assert a == pytest.approx(0.995, rel=1e-15) and az == 1.0
    a, _ = ipm.fraction_to_boundary([2.0, 1.0], [-4.0, -1.0], np.ones(2), np.zeros(2), 0.9)
    assert a == pytest.approx(0.45, rel=1e-15)
    rng = np.random.default_rng(229)
    for _ in range(50):
        s = np.abs(rng.uniform(-1, 1, 6)) + 0.01
        ps = rng.uniform(-1, 1, 6) * 3.0
        a, _ = ipm.fraction_to_boundary(s, ps, s, ps, 0.995)
        assert ((s + a * ps) >= (1 - 0.995) * s - 1e-15).all()
    with pytest.raises(DimensionError):
        ipm.fraction_to_boundary(np.ones(1), np.ones(1), np.ones(1), np.ones(1), 1.5)


def test_line_search_accepts_a_clean_descent_step_immediately():
    qp = plain_qp(np.eye(1), np.zeros(1), 0.0, np.zeros((0, 1)), np.zeros(0))
    st = state([10.0], [], [], [], 0.1)
    z = np.zeros(0)
    assert ipm.line_search(qp, st, ipm.StepDirections(np.array([-1.0]), z, z, z), 1.0) == 1.0


def test_line_search_refuses_an_ascent_direction():
    qp = plain_qp(np.eye(1), np.zeros(1), 0.0, np.zeros((0, 1)), np.zeros(0))
    st = state([10.0], [], [], [], 0.1)
    z = np.zeros(0)
    assert ipm.line_search(qp, st, ipm.StepDirections(np.array([5.0]), z, z, z), 1.0) is None


def test_line_search_makes_progress_on_the_toy_problem():
    qp = bound_toy()
    st = state([0.0], [1.0], [1.0], [1.0], 0.1)
    res = ipm.compute_residuals(qp, st)
    d = ipm.step_directions(qp, st, res, factor_condensed(qp, st))
    amax, _ = ipm.fraction_to_boundary(st.s, d.ps, st.z, d.pz, 0.995)
    alpha = ipm.line_search(qp, st, d, amax)
    assert alpha is not None and alpha > 0
    rho = 10 * np.abs(st.lambda_).max() + 1

    def merit(v, s):
        return 0.5 * v @ (qp.H @ v) + qp.h @ v - st.mu * np.log(s[0]) + rho * abs((qp.J @ v - qp.d + s)[0])
    assert merit(st.v + alpha * d.pv, st.s + alpha * d.ps) < merit(st.v, st.s)


def test_solve_finds_the_unconstrained_minimum_through_the_whole_stack():
    data = P.LqProblemData.basic(np.eye(1), np.eye(1), np.eye(1), np.eye(1), np.eye(1), np.ones(1), 1)
    r = ipm.solve(P.build_dense_qp(data))
    assert r.status == ipm.IpmStatus.converged
    assert r.v[0] == pytest.approx(-0.5, rel=1e-8)
    assert r.objective == pytest.approx(1.5, rel=1e-8)
    assert r.solution.u[0, 0] == pytest.approx(-0.5, rel=1e-8)
    assert r.kkt_error <= 1e-8 and r.iter >= 1
    assert r.total_seconds > 0 and r.linalg_seconds <= r.total_seconds


def test_solve_pushes_an_active_bound_to_its_multiplier():
    r = ipm.solve(bound_toy())
    assert r.status == ipm.IpmStatus.converged
    assert abs(r.v[0]) <= 1e-7
    assert r.z[0] == pytest.approx(2.0, rel=1e-5)
    assert r.s[0] > 0 and r.z[0] > 0
    assert np.abs(r.lambda_ - r.z).max() <= 10 * 1e-8


def test_solve_caps_the_iteration_count():
    r = ipm.solve(bound_toy(), ipm.IpmOptions(max_iter=1))
    assert r.status == ipm.IpmStatus.max_iter and r.iter == 1


def test_an_unfactorizable_condensed_matrix_is_reported_not_hidden():
    qp = plain_qp([[-1e10]], [0.0], 0.0, np.zeros((0, 1)), np.zeros(0))
    assert ipm.solve(qp).status == ipm.IpmStatus.factorization_failure


def test_interior_monotone_barrier_and_block_residual_at_every_iteration(O):
    from _cmpc_helpers import lq_from_oracle
    rng = O.Rng(233)
    for _ in range(5):
        qp = P.build_dense_qp(lq_from_oracle(O.random_problem(rng)))
        last_mu = [0.1]
        seen = [0]

        def inspect(snap):
            seen[0] += 1
            assert snap.state.s.min() > 0 and snap.state.z.min() > 0
            assert snap.state.mu <= last_mu[0]
            last_mu[0] = snap.state.mu
            assert snap.delta == 0.0
            assert augmented_residual(qp, snap.state, snap.residuals, snap.dirs) <= 1e-8

        r = ipm.solve(qp, ipm.IpmOptions(inspect=inspect))
        assert r.status == ipm.IpmStatus.converged and seen[0] == r.iter
        assert r.s.min() > 0 and r.z.min() > 0
        assert np.abs(r.lambda_ - r.z).max() <= 10 * 1e-8


def test_two_runs_produce_bitwise_identical_iterates(O):
    from _cmpc_helpers import lq_from_oracle
    qp = P.build_dense_qp(lq_from_oracle(O.random_problem(O.Rng(239))))

    def capture():
        its = []
        ipm.solve(qp, ipm.IpmOptions(inspect=lambda s: its.extend(
            [s.state.v, s.state.s, s.state.lambda_, s.state.z])))
        return its

    a, b = capture(), capture()
    assert len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))


def test_iteration_log_reports_the_advertised_columns():
    log = []
    r = ipm.solve(bound_toy(), ipm.IpmOptions(log=log.append))
    assert r.status == ipm.IpmStatus.converged and len(log) == r.iter
    for i, rec in enumerate(log):
        assert rec.iter == i + 1 and rec.mu > 0 and 0 < rec.alpha <= 1 and rec.alpha_z > 0
        assert rec.kkt_error >= 0
        if i:
            assert rec.mu <= log[i - 1].mu


def test_solver_and_enumeration_oracle_agree_across_the_random_ensemble(O):
    from _cmpc_helpers import lq_from_oracle
    for i in range(100):
        p = O.random_problem(O.instance_rng(7, i))
        qp = P.build_dense_qp(lq_from_oracle(p))
        truth = O.solve_enumeration(O.build_dense_qp(p))
        assert truth["status"] == "optimal"
        r = ipm.solve(qp)
        assert r.status == ipm.IpmStatus.converged, i
        assert abs(r.objective - truth["objective"]) / (1 + abs(truth["objective"])) <= 1e-6
        ref_u = P.recover_trajectory(qp, truth["v"]).u
        assert np.abs(r.solution.u - ref_u).max() <= 1e-5


def test_options_are_validated():
    for bad in (dict(tau=1.5), dict(kappa_mu=0.0), dict(tol=0.0)):
        with pytest.raises(DimensionError):
            ipm.solve(bound_toy(), ipm.IpmOptions(**bad))
