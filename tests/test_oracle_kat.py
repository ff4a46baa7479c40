"""Pin the oracle (CPU restatement of the reference) to the reference's own known-answer
tests: proj/tests/test_ipm.cpp, test_dense_linalg.cpp, test_reduction.cpp,
test_heat3d.cpp and proj/tests/acceptance.cpp. CPU only."""
import math

import numpy as np
import pytest


def toy(O):  # min 0.5*4 v^2 + 2 v s.t. v >= 0  (test_ipm.cpp:27-31)
    return O.qp_from_arrays([[4.0]], [2.0], 0.0, [[-1.0]], [0.0])


def test_residual_kat(O):  # test_ipm.cpp:71-86
    st = O.State(np.zeros(1), np.ones(1), np.zeros(1), np.full(1, 0.3), 0.3)
    r1, r2, r3, kkt = O.compute_residuals(toy(O), st)
    assert r1[0] == pytest.approx(2.0, rel=1e-15)
    assert r2[0] == pytest.approx(-0.3, rel=1e-15)
    assert r3[0] == pytest.approx(1.0, rel=1e-15)
    assert kkt == pytest.approx(2.0, rel=1e-15)


def test_condensed_kats(O):  # test_ipm.cpp:125-136
    q = O.qp_from_arrays(np.eye(3), np.zeros(3), 0.0, np.zeros((0, 3)), np.zeros(0))
    assert np.abs(O.assemble_condensed(q, np.zeros(0)) - np.eye(3)).max() == 0.0
    q = O.qp_from_arrays(np.eye(2), np.zeros(2), 0.0, np.eye(2), np.zeros(2))
    assert np.abs(O.assemble_condensed(q, np.ones(2)) - 2 * np.eye(2)).max() == 0.0


def test_step_direction_kat(O):  # test_ipm.cpp:156-176
    q = toy(O)
    st = O.State(np.zeros(1), np.ones(1), np.ones(1), np.ones(1), 0.1)
    r1, r2, r3, _ = O.compute_residuals(q, st)
    assert (r1[0], r2[0], r3[0]) == (pytest.approx(1.0), pytest.approx(0.9), pytest.approx(1.0))
    L = O.factorize(O.assemble_condensed(q, st.z / st.s))
    pv, ps, pl, pz = O.step_directions(q, st, r1, r2, r3, L)
    assert pv[0] == pytest.approx(-0.18, rel=1e-14)
    assert ps[0] == pytest.approx(-1.18, rel=1e-14)
    assert pl[0] == pytest.approx(0.28, rel=1e-14)
    assert pz[0] == pytest.approx(0.28, rel=1e-14)


def test_fraction_to_boundary_kats(O):  # test_ipm.cpp:227-258
    assert O.fraction_to_boundary(np.ones(3), np.ones(3), np.ones(3), np.zeros(3), 0.995) == (1.0, 1.0)
    a, az = O.fraction_to_boundary(np.ones(1), -np.ones(1), np.ones(1), np.ones(1), 0.995)
    assert a == pytest.approx(0.995, rel=1e-15) and az == 1.0
    a, _ = O.fraction_to_boundary([2.0, 1.0], [-4.0, -1.0], np.ones(2), np.zeros(2), 0.9)
    assert a == pytest.approx(0.45, rel=1e-15)


def test_line_search_kats(O):  # test_ipm.cpp:260-294
    q = O.qp_from_arrays(np.eye(1), np.zeros(1), 0.0, np.zeros((0, 1)), np.zeros(0))
    st = O.State(np.full(1, 10.0), np.zeros(0), np.zeros(0), np.zeros(0), 0.1)
    z0 = np.zeros(0)
    a, j = O.line_search(q, st, (np.full(1, -1.0), z0, z0, z0), 1.0)
    assert a == 1.0 and j == 0
    a, j = O.line_search(q, st, (np.full(1, 5.0), z0, z0, z0), 1.0)
    assert a is None


def test_barrier_and_termination_rules(O):  # test_ipm.cpp:322-361
    assert O.update_barrier(0.1, 1e-3) == pytest.approx(0.02, rel=1e-15)
    assert O.update_barrier(0.1, 10.0) == 0.1
    assert O.update_barrier(1e-9, 0.0) == 1e-9


def test_whole_solve_kats(O):  # test_ipm.cpp:363-403
    p = O.problem_from_arrays(A=[[1.0]], B=[[1.0]], Q=[[1.0]], Qf=[[1.0]], R=[[1.0]], x_bar=[1.0], T=1)
    q = O.build_dense_qp(p)
    r = O.solve(q)
    assert r.status == "converged"
    assert r.v[0] == pytest.approx(-0.5, rel=1e-8)
    assert r.objective == pytest.approx(1.5, rel=1e-8)
    assert r.u[0, 0] == pytest.approx(-0.5, rel=1e-8)
    r = O.solve(toy(O))
    assert r.status == "converged" and abs(r.v[0]) <= 1e-7
    assert r.z[0] == pytest.approx(2.0, rel=1e-5)
    assert np.abs(r.lam - r.z).max() <= 1e-7
    assert O.solve(toy(O), max_iter=1).iter == 1
    bad = O.qp_from_arrays([[-1e10]], [0.0], 0.0, np.zeros((0, 1)), np.zeros(0))
    assert O.solve(bad).status == "factorization_failure"


def test_cholesky_kats(O):  # test_dense_linalg.cpp:33-116
    for be in ("reference", "eigen"):
        L = O.factorize(np.array([[4.0, 2.0], [2.0, 3.0]]), be)
        assert L[0, 0] == pytest.approx(2.0) and L[1, 0] == pytest.approx(1.0)
        assert L[1, 1] == pytest.approx(math.sqrt(2.0)) and L[0, 1] == 0.0
        with pytest.raises(O.NotPositiveDefinite) as e:
            O.factorize(np.array([[1.0, 0.0], [0.0, -1.0]]), be)
        assert e.value.pivot == 1
    with pytest.raises(O.NotPositiveDefinite) as e:
        O.factorize(np.array([[-1.0]]))
    assert e.value.pivot == 0
    rng = np.random.default_rng(31)
    for n in (63, 64, 65, 150):
        G = rng.uniform(-1, 1, (n, n))
        M = G.T @ G + np.eye(n)
        L = O.factorize(M)
        assert np.abs(L @ L.T - M).max() <= 1e-12 * n * np.abs(M).max()
    with pytest.raises(ValueError):
        O.factorize(np.eye(2), "cuda")


def test_gram_kat(O):  # test_dense_linalg.cpp:171-202
    G = O.gram_weighted(np.array([[1.0, 2.0], [3.0, 4.0]]), [2.0, 3.0])
    assert np.allclose(G, [[29.0, 40.0], [40.0, 56.0]], rtol=1e-15)
    rng = np.random.default_rng(53)
    for _ in range(10):
        m, n = rng.integers(1, 30, size=2)
        J = rng.uniform(-1, 1, (m, n))
        s = rng.uniform(0.1, 4.0, m)
        ref = J.T @ (s[:, None] * J)
        G = O.gram_weighted(J, s)
        assert np.abs(G - ref).max() <= 1e-12 * (1 + np.abs(ref).max())
        assert np.array_equal(G, G.T)


def test_reduction_scalar_kat(O):  # test_reduction.cpp:56-74
    p = O.problem_from_arrays(A=[[1.0]], B=[[1.0]], Q=[[1.0]], Qf=[[1.0]], R=[[1.0]], x_bar=[1.0], T=1)
    q = O.build_dense_qp(p)
    assert q.H[0, 0] == pytest.approx(4.0) and q.h_vec[0] == pytest.approx(2.0)
    assert q.h0 == pytest.approx(2.0) and q.m == 0
    assert q.dense_objective([-0.5]) == pytest.approx(1.5)
    xs, us, obj = q.recover_trajectory([-0.5])
    assert xs[1, 0] == pytest.approx(0.5) and us[0, 0] == pytest.approx(-0.5)
    assert obj == pytest.approx(1.5)


def test_row_order_kat(O):  # test_reduction.cpp:221-259
    p = O.problem_from_arrays(A=[[2.0]], B=[[3.0]], Q=[[1.0]], Qf=[[1.0]], R=[[1.0]], x_bar=[1.0],
                              T=2, E=[[5.0]], F=[[7.0]], gl=[-10.0], gu=[10.0], xl=[-20.0],
                              xu=[20.0], ul=[-8.0], uu=[8.0], w=[[0.5], [0.0]])
    q = O.build_dense_qp(p)
    expected = np.array([[7, 0], [15, 7], [-7, 0], [-15, -7], [3, 0], [6, 3], [-3, 0], [-6, -3],
                         [1, 0], [0, 1], [-1, 0], [0, -1]], dtype=float)
    expected_d = np.array([10 - 5, 10 - 12.5, 5 + 10, 12.5 + 10, 20 - 2.5, 20 - 5, 2.5 + 20,
                           5 + 20, 8, 8, 8, 8])
    assert np.abs(q.J - expected).max() <= 1e-14
    assert np.abs(q.d - expected_d).max() <= 1e-14


def test_heat3d_kats(O):  # test_heat3d.cpp:9-105
    c = 400.0 / (8960.0 * 386.0) * 0.1 / 0.0004
    assert c == pytest.approx(0.0289138, rel=1e-5)
    A, B = O.laplacian_system(1)
    assert A[0, 0] == pytest.approx(1 - 6 * c, rel=1e-14)
    assert np.allclose(B[0], c, rtol=1e-14)
    for N in (2, 3, 4):
        A, B = O.laplacian_system(N)
        assert np.abs(A.sum(1) + B.sum(1) - 1).max() <= 1e-14
    p = O.heat3d_problem(4, 50)
    assert (p.n_x, p.n_u, p.n_c, p.T) == (64, 6, 0, 50)
    p = O.heat3d_problem(2, 10)
    assert np.all(p.get("x_bar") == -50.0)
    assert np.abs(p.get("w")).max() <= 1e-10


def test_acceptance_step_equivalence(O):  # acceptance.cpp:88-108 (criterion 2)
    q = O.build_dense_qp(O.heat3d_problem(2, 10))
    H, J = q.H, q.J
    worst = [0.0]

    def inspect(d):
        sig = d["z"] / d["s"]
        n, m = q.n, q.m
        full = np.zeros((n + 2 * m, n + 2 * m))
        full[:n, :n] = H
        full[:n, n + m:] = J.T
        full[n:n + m, n:n + m] = np.diag(sig)
        full[n:n + m, n + m:] = np.eye(m)
        full[n + m:, :n] = J
        full[n + m:, n:n + m] = np.eye(m)
        p = np.concatenate([d["pv"], d["ps"], d["plambda"]])
        r = np.concatenate([d["r1"], d["r2"], d["r3"]])
        denom = np.abs(full).sum(1).max() * np.abs(p).max() + np.abs(r).max()
        worst[0] = max(worst[0], np.abs(full @ p + r).max() / max(denom, 1e-300))

    r = O.solve(q, inspect=inspect)
    assert r.status == "converged" and worst[0] <= 1e-8


def test_acceptance_convergence_envelope(O):  # acceptance.cpp:110-125 (criterion 3)
    r = O.solve(O.build_dense_qp(O.heat3d_problem(4, 50)))
    assert r.status == "converged" and r.iter <= 60


@pytest.mark.parametrize("seed", [7, 42])
def test_oracle_agreement_ensemble(O, seed):  # test_ipm.cpp:477-488, acceptance.cpp:73-86
    for i in range(100):
        p = O.random_problem(O.instance_rng(seed, i))
        q = O.build_dense_qp(p)
        e = O.solve_enumeration(q)
        assert e["status"] == "optimal"
        r = O.solve(q)
        assert r.status == "converged", i
        assert abs(r.objective - e["objective"]) / (1 + abs(e["objective"])) <= 1e-6
        _, us, _ = q.recover_trajectory(e["v"])
        assert np.abs(r.u - us).max() <= 1e-5


def test_acceptance_reduction_correctness(O):  # acceptance.cpp:149-177 (criterion 5, 50 draws)
    rng = np.random.default_rng(5150)
    orng = O.Rng(5150)
    for _ in range(50):
        p = O.random_problem(orng)
        q = O.build_dense_qp(p)
        v = rng.uniform(-1, 1, q.n)
        xs, us, obj = q.recover_trajectory(v)
        A, B, w = p.get("A"), p.get("B"), p.get("w")
        scale = 1 + np.abs(xs).max()
        for t in range(p.T):
            assert np.abs(xs[t + 1] - (A @ xs[t] + B @ us[t] + w[t])).max() / scale <= 1e-10
        dense = q.dense_objective(v)
        assert abs(obj - dense) / (1 + abs(dense)) <= 1e-8


def test_bitwise_determinism(O):  # test_ipm.cpp:432-457
    q = O.build_dense_qp(O.random_problem(O.Rng(239)))
    a = O.solve(q)
    b = O.solve(q)
    assert a.log == b.log and np.array_equal(a.v, b.v) and np.array_equal(a.z, b.z)


def test_thread_count_does_not_change_results(O):
    q = O.build_dense_qp(O.heat3d_problem(2, 10))
    O.set_threads(1)
    a = O.solve(q)
    O.set_threads(4)
    b = O.solve(q)
    O.set_threads(1)
    assert a.log == b.log and np.array_equal(a.v, b.v)
