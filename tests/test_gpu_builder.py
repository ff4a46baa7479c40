"""build_dense_qp, refresh_initial_state and recover_trajectory on
the device, against the oracle's faithful restatement of proj/src/reduction.cpp (with the
reference's bigA / bigAtilde / bigB) and against solves of the host-built QP."""
import numpy as np
import pytest

from _cmpc_helpers import lq_from_oracle, rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = pytest.mark.gpu


def random_arrays(seed, nx, nu, nc, T, K=True, S=True, inf_frac=0.25):
    """A well-posed random LQ problem with every feature of reduction.cpp exercised: feedback K,
    cross weight S, mixed constraints E/F, disturbances w, and some infinite bounds."""
    r = np.random.default_rng(seed)
    A = r.uniform(-1, 1, (nx, nx))
    A *= 0.9 / max(1e-9, np.abs(np.linalg.eigvals(A)).max())
    B = r.uniform(-1, 1, (nx, nu))
    M = r.uniform(-1, 1, (nx, nx))
    Q = M.T @ M + 0.5 * np.eye(nx)
    M = r.uniform(-1, 1, (nx, nx))
    Qf = M.T @ M + 0.5 * np.eye(nx)
    M = r.uniform(-1, 1, (nu, nu))
    R = M.T @ M + 0.5 * np.eye(nu)
    Sx = 0.05 * r.uniform(-1, 1, (nx, nu)) if S else np.zeros((nx, nu))
    Kx = 0.1 * r.uniform(-1, 1, (nu, nx)) if K else np.zeros((nu, nx))
    E = r.uniform(-1, 1, (nc, nx))
    F = r.uniform(-1, 1, (nc, nu))

    def bounds(k, lo, hi):
        l, u = np.full(k, lo), np.full(k, hi)
        l[r.uniform(size=k) < inf_frac] = -np.inf
        u[r.uniform(size=k) < inf_frac] = np.inf
        return l, u

    gl, gu = bounds(nc, -5.0, 5.0)
    xl, xu = bounds(nx, -4.0, 4.0)
    ul, uu = bounds(nu, -3.0, 3.0)
    return dict(A=A, B=B, Q=Q, Qf=Qf, R=R, S=Sx, E=E, F=F, gl=gl, gu=gu, xl=xl, xu=xu, ul=ul,
                uu=uu, w=0.05 * r.uniform(-1, 1, (T, nx)), x_bar=r.uniform(-1, 1, nx), K=Kx, T=T)


CASES = [(11, 4, 2, 0, 5, True, True), (12, 5, 3, 2, 6, True, True), (13, 6, 2, 3, 4, False, True),
         (14, 7, 3, 0, 8, True, False), (15, 3, 1, 1, 10, False, False)]


@pytest.mark.parametrize("case", CASES)
def test_device_build_matches_the_reference_reduction(O, case):
    seed, nx, nu, nc, T, K, S = case
    arrs = random_arrays(seed, nx, nu, nc, T, K, S)
    op = O.problem_from_arrays(**arrs)
    oq = O.build_dense_qp(op)                       # the reference's dense reduction
    data = lq_from_oracle(op)
    dq = ipm.DeviceQp.from_problem(data)
    assert (dq.m, dq.n) == oq.J.shape
    H, h, h0, d = dq.get_qp()
    assert rel(H, oq.H) <= 1e-13 and rel(h, oq.h_vec) <= 1e-13 and rel(d, oq.d) <= 1e-13
    assert abs(h0 - oq.h0) <= 1e-12 * (1.0 + abs(oq.h0))
    # J through the residual r3 = J v - d + s at s = 0 (the analysed device copy of J)
    rng = np.random.default_rng(seed)
    v = rng.uniform(-1, 1, dq.n)
    from paper_2209_13049_b200 import _lib
    L = _lib.lib()
    zm, om = np.zeros(dq.m), np.ones(dq.m)
    _lib.check(L.cmpc_set_state(dq.h, _lib.ptr(v), _lib.ptr(zm), _lib.ptr(zm), _lib.ptr(om), 1.0))
    r1, r2, r3, kkt = np.zeros(dq.n), np.zeros(dq.m), np.zeros(dq.m), np.zeros(1)
    _lib.check(L.cmpc_compute_residuals(dq.h, _lib.ptr(r1), _lib.ptr(r2), _lib.ptr(r3), _lib.ptr(kkt)))
    assert rel(r3 + d, oq.J @ v) <= 1e-13
    qp_host = P.DenseQp(H=oq.H, h=oq.h_vec, h0=oq.h0, J=oq.J, d=oq.d)
    dq.close()
    # the solve: same iterations and iterates as the host-built QP
    a = ipm.solve_problem(data)
    b = ipm.solve(qp_host)
    assert a.status == b.status and a.iter == b.iter
    assert rel(a.v, b.v) <= 1e-8 and abs(a.objective - b.objective) <= 1e-8 * (1 + abs(b.objective))
    # device trajectory recovery == the reference's recover_trajectory
    xs, us, obj = oq.recover_trajectory(a.v)
    assert rel(a.solution.x, xs) <= 1e-12 and rel(a.solution.u, us) <= 1e-12
    assert abs(a.solution.objective - obj) <= 1e-10 * (1 + abs(obj))


def test_refresh_initial_state_matches_a_rebuild(O):
    arrs = random_arrays(21, 5, 2, 2, 6)
    op = O.problem_from_arrays(**arrs)
    data = lq_from_oracle(op)
    dq = ipm.DeviceQp.from_problem(data)
    first = dq.solve()
    xb = np.random.default_rng(5).uniform(-1, 1, 5)
    dq.refresh_initial_state(xb)
    oq = O.build_dense_qp(op)
    oq.refresh_initial_state(xb)                    # reduction.cpp:270-280
    H, h, h0, d = dq.get_qp()
    assert rel(h, oq.h_vec) <= 1e-13 and rel(d, oq.d) <= 1e-13 and rel(H, oq.H) <= 1e-13
    assert abs(h0 - oq.h0) <= 1e-12 * (1 + abs(oq.h0))
    again = dq.solve()
    fresh = ipm.solve(P.DenseQp(H=oq.H, h=oq.h_vec, h0=oq.h0, J=oq.J, d=oq.d))
    assert again.iter == fresh.iter and rel(again.v, fresh.v) <= 1e-8
    xs, us, obj = oq.recover_trajectory(again.v)
    assert rel(again.solution.x, xs) <= 1e-12 and abs(again.solution.objective - obj) <= 1e-10 * (1 + abs(obj))
    assert first.status.name == "converged"
    dq.close()


def test_heat_plate_device_build_equals_host_build():
    """A scaled config-3 plate (the configs' generators): device build == host build, same
    solve, device trajectory == host recover_trajectory."""
    data = P.heat2d_problem(12, 10, T=14)
    qp = P.build_dense_qp(data)
    dq = ipm.DeviceQp.from_problem(data)
    H, h, h0, d = dq.get_qp()
    assert rel(H, qp.H) <= 1e-13 and rel(h, qp.h) <= 1e-13 and rel(d, qp.d) <= 1e-13
    a = dq.solve()
    b = ipm.solve(qp)
    assert a.iter == b.iter and rel(a.v, b.v) <= 1e-8
    host = P.recover_trajectory(qp, a.v)
    assert rel(a.solution.x, host.x) <= 1e-12 and rel(a.solution.u, host.u) <= 1e-12
    assert abs(a.solution.objective - host.objective) <= 1e-10 * (1 + abs(host.objective))
    dq.close()


def test_loading_a_bare_qp_drops_the_problem():
    data = P.heat2d_problem(6, 5, T=6)
    dq = ipm.DeviceQp.from_problem(data)
    qp = P.build_dense_qp(data)
    from paper_2209_13049_b200 import _lib
    _lib.check(_lib.lib().cmpc_load_qp(dq.h, qp.n, qp.m, _lib.ptr(qp.H), _lib.ptr(qp.h), qp.h0,
                                        _lib.ptr(qp.J), _lib.ptr(qp.d), 0))
    with pytest.raises(ipm.DimensionError):
        dq.refresh_initial_state(data.x_bar)
    dq.close()


def test_column_major_and_row_major_inputs_build_the_same_qp(O):
    """cmpc_lq_problem.layout: 0 = Eigen column-major (the reference's storage, the C++ binding
    of INTEGRATION.md), 1 = row-major (numpy C order, transposed on the device)."""
    import ctypes as C
    from paper_2209_13049_b200 import _lib
    arrs = random_arrays(31, 6, 3, 2, 7)
    data = lq_from_oracle(O.problem_from_arrays(**arrs))
    dm = P.dims(data)
    L = _lib.lib()
    got = []
    for layout in (0, 1):
        keep = []

        def arr(a, order):
            a = np.asarray(a, dtype=np.float64)
            a = np.asfortranarray(a) if order == "F" else np.ascontiguousarray(a)
            keep.append(a)
            return a.ctypes.data_as(_lib.D) if a.size else None

        pr = _lib.LqProblem(nx=dm.n_x, nu=dm.n_u, nc=dm.n_c, T=dm.T, layout=layout)
        for f in ("A", "B", "Q", "Qf", "R", "S", "E", "F", "K"):
            setattr(pr, f, arr(getattr(data, f), "F" if layout == 0 else "C"))
        for f in ("gl", "gu", "xl", "xu", "ul", "uu", "x_bar", "w"):
            setattr(pr, f, arr(getattr(data, f), "C"))
        h = C.c_void_p()
        _lib.check(L.cmpc_ctx_create(C.byref(h), 0))
        try:
            _lib.check(L.cmpc_build_qp(h, C.byref(pr)))
            info = (C.c_int64 * 8)()
            L.cmpc_qp_info(h, info)
            n, m = int(info[0]), int(info[1])
            H, hv, d, h0 = np.zeros((n, n), order="F"), np.zeros(n), np.zeros(m), np.zeros(1)
            _lib.check(L.cmpc_get_qp(h, _lib.ptr(H), _lib.ptr(hv), _lib.ptr(h0), _lib.ptr(d)))
            got.append((H, hv, d, h0[0]))
        finally:
            L.cmpc_ctx_destroy(h)
    (H0, h0v, d0, c0), (H1, h1v, d1, c1) = got
    assert np.array_equal(H0, H1) and np.array_equal(h0v, h1v) and np.array_equal(d0, d1) and c0 == c1
