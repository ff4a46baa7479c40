"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of ``liborc.so``, the CPU restatement of the reference
``condmpc`` solver (/root/reference/proj/src/{ipm,dense_linalg,reduction,heat3d,
random_problems,oracle}.cpp). Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs import this module;
the product path (``paper_2209_13049_b200``) never does.

Parity pinning: the reference cannot be compiled here (no Eigen), so this
restatement is pinned against the reference tests' known-answer values
(tests/test_oracle_kat.py). At the BASELINE.json sizes it is unpinned beyond
those KATs and defines the reference CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
LOG_FN = C.CFUNCTYPE(None, C.c_void_p, _D)
INSPECT_FN = C.CFUNCTYPE(None, C.c_void_p, _D, _D, _D, _D, C.c_double, _D, _D, _D, C.c_double,
                         _D, _D, _D, _D, C.c_double)


def build(force: bool = False) -> str:
    so = os.path.join(_HERE, "liborc.so")
    if force or not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        so = build()
        L = C.CDLL(so)
        vp = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        for name in ("orc_rng_new",):
            getattr(L, name).restype = vp
            getattr(L, name).argtypes = [C.c_uint64]
        L.orc_rng_instance.restype = vp
        L.orc_rng_instance.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_rng_free.argtypes = [vp]
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_uniform.argtypes = [vp, C.c_double, C.c_double]
        L.orc_rng_int.restype = C.c_int64
        L.orc_rng_int.argtypes = [vp, C.c_int64, C.c_int64]
        L.orc_problem_random.restype = vp
        L.orc_problem_random.argtypes = [vp, _I64, _D]
        L.orc_problem_heat3d.restype = vp
        L.orc_problem_heat3d.argtypes = [C.c_int64, C.c_int64, _D]
        L.orc_laplacian_system.argtypes = [C.c_int64, _D, _D, _D]
        L.orc_problem_new.restype = vp
        L.orc_problem_new.argtypes = [C.c_int64] * 4 + [_D] * 17
        L.orc_problem_dims.argtypes = [vp, _I64]
        L.orc_problem_get.argtypes = [vp, C.c_char_p, _D]
        L.orc_problem_free.argtypes = [vp]
        L.orc_build_dense_qp.restype = vp
        L.orc_build_dense_qp.argtypes = [vp]
        L.orc_qp_new.restype = vp
        L.orc_qp_new.argtypes = [C.c_int64, C.c_int64, _D, _D, C.c_double, _D, _D]
        L.orc_qp_dims.argtypes = [vp, _I64]
        L.orc_qp_get.argtypes = [vp, C.c_char_p, _D]
        L.orc_qp_refresh.argtypes = [vp, _D]
        L.orc_qp_recover.argtypes = [vp, _D, _D, _D, _D]
        L.orc_dense_objective.restype = C.c_double
        L.orc_dense_objective.argtypes = [vp, _D]
        L.orc_qp_free.argtypes = [vp]
        L.orc_compute_residuals.argtypes = [vp, _D, _D, _D, _D, C.c_double, _D, _D, _D, _D]
        L.orc_assemble_condensed.argtypes = [vp, _D, _D]
        L.orc_gram_weighted.argtypes = [C.c_int64, C.c_int64, _D, _D, C.c_int64, _D]
        L.orc_factorize.argtypes = [C.c_char_p, C.c_int64, _D, _D, _I64]
        L.orc_factor_solve.argtypes = [C.c_int64, _D, _D, C.c_int64, _D]
        L.orc_step_directions.argtypes = [vp, _D, _D, _D, _D, C.c_double, _D, _D, _D, _D, _D, _D,
                                          _D, _D]
        L.orc_fraction_to_boundary.argtypes = [C.c_int64, _D, _D, _D, _D, C.c_double, _D]
        L.orc_line_search.argtypes = [vp, _D, _D, _D, _D, C.c_double, _D, _D, _D, _D, C.c_double,
                                      C.c_double, _D]
        L.orc_merit.restype = C.c_double
        L.orc_merit.argtypes = [vp, _D, _D, C.c_double, C.c_double]
        L.orc_solve.argtypes = [vp, _D, C.c_int64, C.c_char_p, _D, _D, _D, _D, _D, _D, _D, LOG_FN,
                                INSPECT_FN, vp]
        L.orc_solve_enumeration.argtypes = [vp, _D, _D, _I64, _I64, _D]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_set_skip_zeros.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        _LIB = L
    return _LIB


class OracleError(RuntimeError):
    pass


class DimensionError(OracleError):
    pass


class NotPositiveDefinite(OracleError):
    def __init__(self, pivot, msg):
        super().__init__(msg)
        self.pivot = pivot


def _err():
    return lib().orc_last_error().decode()


def _check(rc):
    if rc < 0:
        msg = _err()
        if "must" in msg or "does not match" in msg or "length" in msg or "mismatch" in msg:
            raise DimensionError(msg)
        raise OracleError(msg)
    return rc


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def _f(a, shape=None):
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape, order="F")
    return a


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return lib().orc_get_threads()


def set_skip_zeros(on: bool):
    """Test-speed mode: solve() leaves J's all-zero 512-row column chunks out of every J
    product. Bitwise the same results (only exact-zero products are skipped, sums keep their
    order); the timed CPU baseline never sets it."""
    lib().orc_set_skip_zeros(1 if on else 0)


class Rng:
    """std::mt19937_64 (seeded like the reference tests)."""

    def __init__(self, seed: int | None = None, _h=None):
        self.h = _h if _h is not None else lib().orc_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_rng_free(self.h)
            self.h = None

    def uniform(self, lo, hi):
        return lib().orc_rng_uniform(self.h, lo, hi)


def instance_rng(seed: int, index: int) -> Rng:
    return Rng(_h=lib().orc_rng_instance(seed, index))


class Problem:
    """LqProblemData (proj/include/condmpc/problem.hpp:22-45)."""

    FIELDS = ("A", "B", "Q", "Qf", "R", "S", "E", "F", "gl", "gu", "xl", "xu", "ul", "uu",
              "w", "x_bar", "K")

    def __init__(self, h):
        if not h:
            raise OracleError(_err())
        self.h = h
        d = (C.c_int64 * 4)()
        lib().orc_problem_dims(h, d)
        self.n_x, self.n_u, self.n_c, self.T = (int(x) for x in d)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_problem_free(self.h)
            self.h = None

    def shape(self, f):
        nx, nu, nc, T = self.n_x, self.n_u, self.n_c, self.T
        return {"A": (nx, nx), "B": (nx, nu), "Q": (nx, nx), "Qf": (nx, nx), "R": (nu, nu),
                "S": (nx, nu), "E": (nc, nx), "F": (nc, nu), "gl": (nc,), "gu": (nc,),
                "xl": (nx,), "xu": (nx,), "ul": (nu,), "uu": (nu,), "w": (T, nx),
                "x_bar": (nx,), "K": (nu, nx)}[f]

    def get(self, f):
        shp = self.shape(f)
        if f == "w":
            out = np.zeros(shp, dtype=np.float64)  # row t = w_t (C order)
        else:
            out = np.zeros(shp, dtype=np.float64, order="F")
        _check(lib().orc_problem_get(self.h, f.encode(), _p(out)))
        return out

    def as_dict(self):
        return {f: self.get(f) for f in self.FIELDS} | {"T": self.T}


def problem_from_arrays(A, B, Q, Qf, R, S=None, E=None, F=None, gl=None, gu=None, xl=None,
                        xu=None, ul=None, uu=None, w=None, x_bar=None, K=None, T=None):
    A = _f(A)
    nx = A.shape[0]
    B = _f(B, (nx, -1))
    nu = B.shape[1]
    E = _f(np.zeros((0, nx)) if E is None else E)
    nc = E.shape[0]
    T = int(T)
    inf = np.inf
    args = dict(
        A=A, B=B, Q=_f(Q), Qf=_f(Qf), R=_f(R, (nu, nu)),
        S=_f(np.zeros((nx, nu)) if S is None else S, (nx, nu)), E=E,
        F=_f(np.zeros((nc, nu)) if F is None else F, (nc, nu)),
        gl=_f(np.full(nc, -inf) if gl is None else gl), gu=_f(np.full(nc, inf) if gu is None else gu),
        xl=_f(np.full(nx, -inf) if xl is None else xl), xu=_f(np.full(nx, inf) if xu is None else xu),
        ul=_f(np.full(nu, -inf) if ul is None else ul), uu=_f(np.full(nu, inf) if uu is None else uu),
        w=np.ascontiguousarray(np.zeros((T, nx)) if w is None else np.asarray(w, dtype=np.float64).reshape(T, nx)),
        x_bar=_f(x_bar), K=_f(np.zeros((nu, nx)) if K is None else K, (nu, nx)))
    keep = list(args.values())
    h = lib().orc_problem_new(nx, nu, nc, T, *[_p(args[k]) for k in Problem.FIELDS])
    del keep
    return Problem(h)


def random_problem(rng: Rng, max_n_x=3, max_n_u=2, max_n_c=0, max_T=4, cap_rows_for_oracle=True,
                   bound_margin=0.5, spectral_radius_cap=1.05, fixed=None) -> Problem:
    """random_problems.cpp:39-126; ``fixed=(n_x, n_u, n_c, T)`` replaces the dimension draw."""
    fx = fixed or (0, 0, 0, 0)
    oi = (C.c_int64 * 10)(max_n_x, max_n_u, max_n_c, max_T, int(cap_rows_for_oracle),
                          int(fixed is not None), *fx)
    od = (C.c_double * 2)(bound_margin, spectral_radius_cap)
    return Problem(lib().orc_problem_random(rng.h, oi, od))


HEAT_DEFAULTS = dict(dt=0.1, dw=0.02, rho=8960.0, cp=386.0, conductivity=400.0,
                     q_weight=10.0 * 0.02 * 0.02, r_weight=0.1 * 0.02 * 0.02, x_min=200.0,
                     x_max=550.0, u_min=300.0, u_max=500.0, x_init=300.0, setpoint=350.0)


def _heat_params(kw):
    p = dict(HEAT_DEFAULTS)
    p.update(kw)
    return (C.c_double * 13)(*[p[k] for k in HEAT_DEFAULTS])


def heat3d_problem(N=4, T=50, **kw) -> Problem:
    """heat3d.cpp:39-60."""
    return Problem(lib().orc_problem_heat3d(N, T, _heat_params(kw)))


def laplacian_system(N, **kw):
    nx = N ** 3
    A = np.zeros((nx, nx), order="F")
    B = np.zeros((nx, 6), order="F")
    _check(lib().orc_laplacian_system(N, _heat_params(kw), _p(A), _p(B)))
    return A, B


class Qp:
    """DenseQp (proj/include/condmpc/reduction.hpp:25-33)."""

    def __init__(self, h, problem: Problem | None = None):
        if not h:
            raise OracleError(_err())
        self.h = h
        self.problem = problem
        d = (C.c_int64 * 2)()
        lib().orc_qp_dims(h, d)
        self.n, self.m = int(d[0]), int(d[1])

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_qp_free(self.h)
            self.h = None

    def _get(self, f, shape):
        out = np.zeros(shape, dtype=np.float64, order="F")
        _check(lib().orc_qp_get(self.h, f.encode(), _p(out)))
        return out

    @property
    def H(self):
        return self._get("H", (self.n, self.n))

    @property
    def h_vec(self):
        return self._get("h", (self.n,))

    @property
    def h0(self):
        return float(self._get("h0", (1,))[0])

    @property
    def J(self):
        return self._get("J", (self.m, self.n))

    @property
    def d(self):
        return self._get("d", (self.m,))

    def arrays(self):
        return dict(H=self.H, h=self.h_vec, h0=self.h0, J=self.J, d=self.d)

    def refresh_initial_state(self, x_bar):
        x = _f(x_bar)
        _check(lib().orc_qp_refresh(self.h, _p(x)))

    def recover_trajectory(self, v):
        p = self.problem
        v = _f(v)
        xs = np.zeros((p.T + 1, p.n_x))
        us = np.zeros((p.T, p.n_u))
        obj = C.c_double()
        _check(lib().orc_qp_recover(self.h, _p(v), _p(xs), _p(us), C.byref(obj)))
        return xs, us, obj.value

    def dense_objective(self, v):
        v = _f(v)
        return lib().orc_dense_objective(self.h, _p(v))


def build_dense_qp(problem: Problem) -> Qp:
    return Qp(lib().orc_build_dense_qp(problem.h), problem)


def qp_from_arrays(H, h, h0, J, d) -> Qp:
    H = _f(H)
    n = H.shape[0]
    h = _f(h, (n,))
    J = _f(J)
    if J.size == 0:
        J = np.zeros((0, n), order="F")
    m = J.shape[0]
    d = _f(d, (m,))
    return Qp(lib().orc_qp_new(n, m, _p(H), _p(h), float(h0), _p(J), _p(d)))


# ------------------------------------------------------------ per-step API (ipm.hpp:83-120)
@dataclass
class State:
    v: np.ndarray
    s: np.ndarray
    lam: np.ndarray
    z: np.ndarray
    mu: float
    iter: int = 0


def _st(st: State):
    return [_f(st.v), _f(st.s), _f(st.lam), _f(st.z)]


def compute_residuals(qp: Qp, st: State):
    v, s, l, z = _st(st)
    r1 = np.zeros(qp.n)
    r2 = np.zeros(qp.m)
    r3 = np.zeros(qp.m)
    kkt = C.c_double()
    _check(lib().orc_compute_residuals(qp.h, _p(v), _p(s), _p(l), _p(z), st.mu, _p(r1), _p(r2),
                                       _p(r3), C.byref(kkt)))
    return r1, r2, r3, kkt.value


def assemble_condensed(qp: Qp, sigma):
    sigma = _f(sigma)
    M = np.zeros((qp.n, qp.n), order="F")
    _check(lib().orc_assemble_condensed(qp.h, _p(sigma), _p(M)))
    return M


def gram_weighted(J, sigma):
    J = _f(J)
    sigma = _f(sigma)
    m, n = J.shape
    G = np.zeros((n, n), order="F")
    _check(lib().orc_gram_weighted(m, n, _p(J), _p(sigma), sigma.size, _p(G)))
    return G


def factorize(M, backend="reference"):
    M = _f(M)
    n = M.shape[0]
    L = np.zeros((n, n), order="F")
    piv = C.c_int64(-1)
    rc = lib().orc_factorize(backend.encode(), n, _p(M), _p(L), C.byref(piv))
    if rc == 1:
        raise NotPositiveDefinite(piv.value, _err())
    if rc < 0:
        msg = _err()
        if "unknown factorization backend" in msg:
            raise ValueError(msg)
        raise OracleError(msg)
    return L


def factor_solve(L, b):
    L = _f(L)
    b = _f(b)
    x = np.zeros(b.size)
    _check(lib().orc_factor_solve(L.shape[0], _p(L), _p(b), b.size, _p(x)))
    return x


def step_directions(qp: Qp, st: State, r1, r2, r3, L):
    v, s, l, z = _st(st)
    r1, r2, r3, L = _f(r1), _f(r2), _f(r3), _f(L)
    pv = np.zeros(qp.n)
    ps, pl, pz = np.zeros(qp.m), np.zeros(qp.m), np.zeros(qp.m)
    _check(lib().orc_step_directions(qp.h, _p(v), _p(s), _p(l), _p(z), st.mu, _p(r1), _p(r2),
                                     _p(r3), _p(L), _p(pv), _p(ps), _p(pl), _p(pz)))
    return pv, ps, pl, pz


def fraction_to_boundary(s, ps, z, pz, tau):
    s, ps, z, pz = _f(s), _f(ps), _f(z), _f(pz)
    out = np.zeros(2)
    _check(lib().orc_fraction_to_boundary(s.size, _p(s), _p(ps), _p(z), _p(pz), tau, _p(out)))
    return float(out[0]), float(out[1])


def line_search(qp: Qp, st: State, dirs, alpha_max, eta=1e-4):
    """Returns (alpha, trial) or (None, -1)."""
    v, s, l, z = _st(st)
    pv, ps, pl, pz = (_f(x) for x in dirs)
    a = C.c_double()
    j = lib().orc_line_search(qp.h, _p(v), _p(s), _p(l), _p(z), st.mu, _p(pv), _p(ps), _p(pl),
                              _p(pz), alpha_max, eta, C.byref(a))
    if j == -1:
        _check(-1)
    if j == -2:
        return None, -1
    return a.value, j


def merit(qp: Qp, v, s, mu, rho):
    v, s = _f(v), _f(s)
    return lib().orc_merit(qp.h, _p(v), _p(s), mu, rho)


def update_barrier(mu, kkt, tol=1e-8, kappa_mu=0.2):
    return max(tol / 10.0, kappa_mu * mu) if kkt <= 10.0 * mu else mu


STATUS = ("converged", "max_iter", "factorization_failure", "line_search_failure")


@dataclass
class Result:
    status: str
    v: np.ndarray
    s: np.ndarray
    lam: np.ndarray
    z: np.ndarray
    iter: int
    kkt_error: float
    objective: float
    total_seconds: float
    linalg_seconds: float
    solution_objective: float
    x: np.ndarray | None
    u: np.ndarray | None
    log: list


def solve(qp: Qp, tol=1e-8, mu_init=0.1, kappa_mu=0.2, tau=0.995, max_iter=200, armijo_eta=1e-4,
          backend="reference", log=True, inspect=None) -> Result:
    """ipm::solve (ipm.cpp:160-268). ``log`` collects (iter, mu, alpha, alpha_z, kkt,
    objective, delta, trial) rows; ``inspect(dict)`` is called per iteration."""
    n, m = qp.n, qp.m
    v, s, l, z = np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(m)
    scal = np.zeros(8)
    rows = []
    has_prob = qp.problem is not None
    xs = np.zeros((qp.problem.T + 1, qp.problem.n_x)) if has_prob else None
    us = np.zeros((qp.problem.T, qp.problem.n_u)) if has_prob else None

    def _log(user, rec):
        rows.append(tuple(rec[i] for i in range(8)))

    def _insp(user, v_, s_, l_, z_, mu, r1, r2, r3, kkt, pv, ps, pl, pz, delta):
        vec = lambda p, k: np.ctypeslib.as_array(p, shape=(k,)).copy() if k else np.zeros(0)
        inspect(dict(v=vec(v_, n), s=vec(s_, m), lam=vec(l_, m), z=vec(z_, m), mu=mu,
                     r1=vec(r1, n), r2=vec(r2, m), r3=vec(r3, m), kkt=kkt, pv=vec(pv, n),
                     ps=vec(ps, m), plambda=vec(pl, m), pz=vec(pz, m), delta=delta))

    lf = LOG_FN(_log) if log else LOG_FN()
    inf_ = INSPECT_FN(_insp) if inspect else INSPECT_FN()
    od = (C.c_double * 5)(tol, mu_init, kappa_mu, tau, armijo_eta)
    rc = lib().orc_solve(qp.h, od, max_iter, backend.encode(), _p(v), _p(s), _p(l), _p(z),
                         _p(scal), _p(xs), _p(us), lf, inf_, None)
    if rc < 0:
        msg = _err()
        if "unknown factorization backend" in msg:
            raise ValueError(msg)
        raise DimensionError(msg)
    has_sol = scal[7] > 0
    return Result(STATUS[int(scal[0])], v, s, l, z, int(scal[1]), scal[2], scal[3], scal[4],
                  scal[5], scal[6], xs if has_sol else None, us if has_sol else None, rows)


def solve_enumeration(qp: Qp):
    v = np.zeros(qp.n)
    obj = C.c_double()
    act = np.zeros(max(qp.m, 1), dtype=np.int64)
    na = C.c_int64()
    mult = np.zeros(max(qp.m, 1))
    st = lib().orc_solve_enumeration(qp.h, _p(v), C.byref(obj), act.ctypes.data_as(_I64),
                                     C.byref(na), _p(mult))
    _check(st)
    k = na.value
    return dict(status=("optimal", "infeasible", "unbounded_guard")[st], v=v,
                objective=obj.value, active_set=act[:k].copy(), multipliers=mult[:k].copy())
