"""Problem data, dense reduction and workload generators (setup; not the hot path).

Mirrors proj/include/condmpc/problem.hpp (LqProblemData, dims), reduction.hpp
(DenseQp, Trajectory, build_dense_qp, refresh_initial_state, recover_trajectory,
dense_objective) and heat3d.hpp. The reduction here is *lean*: it never forms the
(T+1)n_x x T n_x bigAtilde of proj/src/reduction.cpp:32 (127 GB at the 2-D heat config)
nor the powers bigA; the free response uses the recursion x0_{t+1} = A_K x0_t + w_t and
bigB's first block column the reference's own recursion (reduction.cpp:43-51). Row order
of J and d follows reduction.cpp:191-251 exactly. tests/test_problem.py checks it
against the oracle's faithful restatement.

New workload generators for the BASELINE.json configurations (the reference ships only
the 3-D cube): 1-D rod (config 2) and 2-D plates (configs 3-5), built with the cube's
conventions.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np

from ._lib import DimensionError

INF = np.inf


@dataclass
class LqProblemData:
    """proj/include/condmpc/problem.hpp:22-45 (w stored as a T x n_x array)."""

    A: np.ndarray
    B: np.ndarray
    Q: np.ndarray
    Qf: np.ndarray
    R: np.ndarray
    S: np.ndarray
    E: np.ndarray
    F: np.ndarray
    gl: np.ndarray
    gu: np.ndarray
    xl: np.ndarray
    xu: np.ndarray
    ul: np.ndarray
    uu: np.ndarray
    w: np.ndarray
    x_bar: np.ndarray
    K: np.ndarray
    T: int

    @staticmethod
    def basic(A, B, Q, R, Qf, x_bar, T) -> "LqProblemData":
        """problem.cpp:10-34."""
        A = np.asarray(A, dtype=np.float64)
        B = np.asarray(B, dtype=np.float64)
        nx, nu = A.shape[0], B.shape[1]
        return LqProblemData(
            A=A, B=B, Q=np.asarray(Q, float), Qf=np.asarray(Qf, float), R=np.asarray(R, float),
            S=np.zeros((nx, nu)), E=np.zeros((0, nx)), F=np.zeros((0, nu)), gl=np.zeros(0),
            gu=np.zeros(0), xl=np.full(nx, -INF), xu=np.full(nx, INF), ul=np.full(nu, -INF),
            uu=np.full(nu, INF), w=np.zeros((int(T), nx)), x_bar=np.asarray(x_bar, float).copy(),
            K=np.zeros((nu, nx)), T=int(T))

    def copy(self) -> "LqProblemData":
        return dataclasses.replace(self, **{f.name: (np.array(getattr(self, f.name), copy=True)
                                                     if isinstance(getattr(self, f.name), np.ndarray)
                                                     else getattr(self, f.name))
                                            for f in dataclasses.fields(self)})


@dataclass
class Dims:
    n_x: int
    n_u: int
    n_c: int
    T: int


def dims(d: LqProblemData) -> Dims:
    """problem.cpp:42-69."""
    nx, nu, nc, T = d.A.shape[0], d.B.shape[1], d.E.shape[0], d.w.shape[0]

    def bad(msg):
        raise DimensionError("dimension mismatch: " + msg)

    if d.A.shape != (nx, nx):
        bad("A is not square")
    if d.B.shape[0] != nx:
        bad("B rows do not match A")
    if d.Q.shape != (nx, nx) or d.Qf.shape != (nx, nx):
        bad("Q/Qf do not match A")
    if d.R.shape != (nu, nu):
        bad("R does not match B")
    if d.S.shape != (nx, nu):
        bad("S does not match A and B")
    if nc > 0 and d.E.shape[1] != nx:
        bad("E cols do not match A")
    if d.F.shape[0] != nc or (nc > 0 and d.F.shape[1] != nu):
        bad("F does not match E and B")
    if d.gl.size != nc or d.gu.size != nc:
        bad("gl/gu do not match E")
    if d.xl.size != nx or d.xu.size != nx:
        bad("xl/xu do not match A")
    if d.ul.size != nu or d.uu.size != nu:
        bad("ul/uu do not match B")
    if d.x_bar.size != nx:
        bad("x_bar does not match A")
    if d.K.shape != (nu, nx):
        bad("K does not match B and A")
    if d.T != T:
        bad("T field does not match w")
    if T < 1:
        bad("horizon T must be positive")
    return Dims(nx, nu, nc, T)


@dataclass
class Trajectory:
    """reduction.hpp:35-40 (x: (T+1) x n_x, u, v: T x n_u)."""

    x: np.ndarray | None = None
    u: np.ndarray | None = None
    v: np.ndarray | None = None
    objective: float = 0.0


@dataclass
class DenseQp:
    """reduction.hpp:25-33: min 1/2 v'Hv + h'v + h0  s.t.  J v <= d (column-major arrays).

    ``source`` is the structured problem (None for a bare QP); the lean reduction keeps
    the first block column of bigB (``gk``) and the free response ``x0`` instead of the
    reference's BlockMatrices."""

    H: np.ndarray
    h: np.ndarray
    h0: float
    J: np.ndarray
    d: np.ndarray
    source: LqProblemData | None = None
    gk: np.ndarray | None = None     # T x n_x x n_u: A_K^k B
    x0: np.ndarray | None = None     # (T+1) x n_x free response
    # per row of J: (stage t, nonzero prefix width) from the builder (None for a bare QP);
    # used to shard rows across GPUs by whole stages
    row_stage: np.ndarray | None = None
    row_width: np.ndarray | None = None
    # the cached device context (ipm.device_qp) and the fingerprint of the arrays it was loaded
    # from: never copied by dataclasses.replace, re-checked on every solve
    _device: object = field(init=False, default=None, repr=False, compare=False)
    _device_key: object = field(init=False, default=None, repr=False, compare=False)
    _version: int = field(init=False, default=0, repr=False, compare=False)

    _QP_FIELDS = ("H", "h", "h0", "J", "d")

    def __setattr__(self, name, value):
        if name in DenseQp._QP_FIELDS:  # reassigning an array or h0 invalidates the upload
            object.__setattr__(self, "_version", getattr(self, "_version", 0) + 1)
        object.__setattr__(self, name, value)

    def device_key(self):
        """Cheap fingerprint of the arrays a device upload holds: the array objects, their
        data pointers, shapes and strides, h0, and a counter bumped on reassignment. In-place
        edits of the arrays' contents are not seen: call invalidate_device() after them."""
        def arr(a):
            return (id(a), a.__array_interface__["data"][0], a.shape, a.strides)
        return (self._version, arr(self.H), arr(self.h), arr(self.J), arr(self.d), self.h0)

    def __post_init__(self):
        self.H = np.asfortranarray(np.asarray(self.H, dtype=np.float64))
        n = self.H.shape[0] if self.H.ndim == 2 else 0
        self.h = np.asarray(self.h, dtype=np.float64).reshape(n)
        J = np.asarray(self.J, dtype=np.float64)
        if J.size == 0:
            J = np.zeros((0, n))
        self.J = np.asfortranarray(J)
        self.d = np.asarray(self.d, dtype=np.float64).reshape(self.J.shape[0])
        self.h0 = float(self.h0)

    @property
    def n(self) -> int:
        return self.H.shape[0]

    @property
    def m(self) -> int:
        return self.J.shape[0]

    def invalidate_device(self):
        """Call after mutating H/h/h0/J/d in place so the next solve re-uploads."""
        if self._device is not None:
            self._device.close()
        self._device = None
        self._device_key = None


def _apply_Q(Qt, X, diag):
    return (diag[:, None] * X) if diag is not None else Qt @ X


def _diag_or_none(Mx):
    d = np.diag(Mx).copy()
    return d if np.count_nonzero(Mx) == np.count_nonzero(d) else None


def free_response(A_K, x_bar, w):
    """x0_0 = x_bar, x0_{t+1} = A_K x0_t + w_t (equals bigA x_bar + bigAtilde w)."""
    T = w.shape[0]
    x0 = np.zeros((T + 1, A_K.shape[0]))
    x0[0] = x_bar
    for t in range(T):
        x0[t + 1] = A_K @ x0[t] + w[t]
    return x0


def _affine(data: LqProblemData, gk, x0, Q_K, S_K):
    """h, h0, d (reduction.cpp:119-180)."""
    dm = dims(data)
    nx, nu, nc, T = dm.n_x, dm.n_u, dm.n_c, dm.T
    h = np.zeros(T * nu)
    h0 = 0.0
    for t in range(T + 1):
        Qt = data.Qf if t == T else Q_K
        Qx = Qt @ x0[t]
        h0 += float(x0[t] @ Qx)
        if t > 0:
            # bigB block row t = [G_{t-1} ... G_0]: column block j is G_{t-1-j}
            for j in range(t):
                h[j * nu:(j + 1) * nu] += 2.0 * (gk[t - 1 - j].T @ Qx)
        if t < T:
            h[t * nu:(t + 1) * nu] += 2.0 * (S_K.T @ x0[t])
    EFK = data.E + data.F @ data.K if nc > 0 else np.zeros((0, nx))
    parts = []

    def emit(bound, off, upper):
        fin = np.isfinite(bound)
        parts.append((bound - off)[fin] if upper else (off - bound)[fin])

    for upper in (1, 0):
        if nc > 0:
            for t in range(T):
                emit(data.gu if upper else data.gl, EFK @ x0[t], upper)
    for upper in (1, 0):
        for t in range(1, T + 1):
            emit(data.xu if upper else data.xl, x0[t], upper)
    for upper in (1, 0):
        for t in range(T):
            emit(data.uu if upper else data.ul, data.K @ x0[t], upper)
    d = np.concatenate(parts) if parts else np.zeros(0)
    return h, h0, d


def build_dense_qp(data: LqProblemData) -> DenseQp:
    """Lean restatement of build_dense_qp (reduction.cpp:255-268)."""
    dm = dims(data)
    nx, nu, nc, T = dm.n_x, dm.n_u, dm.n_c, dm.T
    n = T * nu
    A_K = data.A + data.B @ data.K
    gk = np.zeros((T, nx, nu))
    gk[0] = data.B
    for k in range(1, T):
        gk[k] = A_K @ gk[k - 1]
    SK = data.S @ data.K
    Q_K = data.Q + SK + SK.T + data.K.T @ data.R @ data.K
    S_K = data.S + data.K.T @ data.R

    # Hessian (reduction.cpp:88-117): H = 2 (R_bar + sum_t Bt' Q_t Bt + cross), symmetrised
    H = np.zeros((n, n), order="F")
    for t in range(T):
        H[t * nu:(t + 1) * nu, t * nu:(t + 1) * nu] = data.R
    qd, qfd = _diag_or_none(Q_K), _diag_or_none(data.Qf)
    for t in range(1, T + 1):
        w = t * nu
        Bt = np.concatenate([gk[t - 1 - j] for j in range(t)], axis=1)  # nx x w
        if t == T:
            QB = _apply_Q(data.Qf, Bt, qfd)
        else:
            QB = _apply_Q(Q_K, Bt, qd)
        H[:w, :w] += Bt.T @ QB
    for t in range(1, T):
        w = t * nu
        Bt = np.concatenate([gk[t - 1 - j] for j in range(t)], axis=1)
        cross = Bt.T @ S_K
        H[:w, t * nu:(t + 1) * nu] += cross
        H[t * nu:(t + 1) * nu, :w] += cross.T
    H *= 2.0
    H = np.asfortranarray(0.5 * (H + H.T))

    x0 = free_response(A_K, data.x_bar, data.w)
    h, h0, d = _affine(data, gk, x0, Q_K, S_K)

    # inequality rows (reduction.cpp:182-251)
    EFK = data.E + data.F @ data.K if nc > 0 else np.zeros((0, nx))
    cnt = lambda lo, hi: int(np.isfinite(lo).sum() + np.isfinite(hi).sum()) * T
    m = cnt(data.gl, data.gu) + cnt(data.xl, data.xu) + cnt(data.ul, data.uu)
    J = np.zeros((m, n), order="F")
    row_stage = np.zeros(m, dtype=np.int64)
    row_width = np.zeros(m, dtype=np.int64)
    r = 0

    def brow(t):  # bigB block row t (nx x t*nu)
        return np.concatenate([gk[t - 1 - j] for j in range(t)], axis=1) if t > 0 else np.zeros((nx, 0))

    for upper in (1, 0):
        sign = 1.0 if upper else -1.0
        bound = data.gu if upper else data.gl
        for t in range(T if nc > 0 else 0):
            Bt = brow(t)
            for i in range(nc):
                if not np.isfinite(bound[i]):
                    continue
                if t > 0:
                    J[r, :t * nu] = sign * (EFK[i] @ Bt)
                J[r, t * nu:(t + 1) * nu] += sign * data.F[i]
                row_stage[r], row_width[r] = t, (t + 1) * nu
                r += 1
    for upper in (1, 0):
        sign = 1.0 if upper else -1.0
        bound = data.xu if upper else data.xl
        fin = np.flatnonzero(np.isfinite(bound))
        for t in range(1, T + 1):
            Bt = brow(t)
            k = fin.size
            J[r:r + k, :t * nu] = sign * Bt[fin]
            row_stage[r:r + k], row_width[r:r + k] = t, t * nu
            r += k
    for upper in (1, 0):
        sign = 1.0 if upper else -1.0
        bound = data.uu if upper else data.ul
        for t in range(T):
            Bt = brow(t)
            for i in range(nu):
                if not np.isfinite(bound[i]):
                    continue
                if t > 0:
                    J[r, :t * nu] = sign * (data.K[i] @ Bt)
                J[r, t * nu + i] += sign
                row_stage[r] = t
                row_width[r] = t * nu + i + 1 if np.any(data.K) else 1
                r += 1
    assert r == m, "inequality assembly row count mismatch"
    return DenseQp(H=H, h=h, h0=h0, J=J, d=d, source=data, gk=gk, x0=x0, row_stage=row_stage,
                   row_width=row_width)


# ------------------------------------------------------------------ row sharding (§8(e))
def shard_rows(qp: DenseQp, nranks: int) -> list:
    """Partition the rows of J for the row-sharded solve (one GPU per part).

    J' Sigma J = sum_g J_g' Sigma_g J_g holds for any partition; this one cuts at whole
    stages (every row of a stage — upper and lower bound of the same quantity, the mirror
    rows of the plate — lands in one shard, so each shard's exact-duplicate analysis finds
    the same merges as the whole) and balances the condensation work, which grows with the
    square of a row's nonzero prefix width. A bare QP (no builder metadata) is cut into
    contiguous blocks of equal row count. Returns ascending row-index arrays."""
    m = qp.m
    if nranks < 1:
        raise DimensionError("nranks must be positive")
    if qp.row_stage is None or qp.row_width is None or m == 0:
        edges = np.linspace(0, m, nranks + 1).round().astype(np.int64)
        return [np.arange(edges[g], edges[g + 1], dtype=np.int64) for g in range(nranks)]
    stage = np.asarray(qp.row_stage)
    work = np.asarray(qp.row_width, dtype=np.float64) ** 2 + 1.0
    nst = int(stage.max()) + 1
    per_stage = np.bincount(stage, weights=work, minlength=nst)
    cum = np.cumsum(per_stage)
    total = cum[-1]
    # stage boundaries: the first stage whose cumulative work reaches g / nranks of the total
    bounds = [0]
    for g in range(1, nranks):
        b = int(np.searchsorted(cum, total * g / nranks, side="left")) + 1
        bounds.append(min(max(b, bounds[-1]), nst))
    bounds.append(nst)
    return [np.flatnonzero((stage >= bounds[g]) & (stage < bounds[g + 1])) for g in range(nranks)]


def shard_qp(qp: DenseQp, rows) -> DenseQp:
    """The QP restricted to `rows` of J and d (H, h, h0 are replicated on every shard)."""
    rows = np.asarray(rows, dtype=np.int64)
    return DenseQp(H=qp.H, h=qp.h, h0=qp.h0, J=qp.J[rows], d=qp.d[rows],
                   row_stage=None if qp.row_stage is None else qp.row_stage[rows],
                   row_width=None if qp.row_width is None else qp.row_width[rows])


def refresh_initial_state(qp: DenseQp, x_bar) -> None:
    """reduction.cpp:270-280: new x_bar, same H and J; refreshes h, h0, d."""
    data = qp.source
    x_bar = np.asarray(x_bar, dtype=np.float64)
    if x_bar.size != data.x_bar.size:
        raise DimensionError("refresh_initial_state: x_bar length mismatch")
    data.x_bar = x_bar.copy()
    A_K = data.A + data.B @ data.K
    SK = data.S @ data.K
    Q_K = data.Q + SK + SK.T + data.K.T @ data.R @ data.K
    S_K = data.S + data.K.T @ data.R
    qp.x0 = free_response(A_K, data.x_bar, data.w)
    fresh = qp._device is not None and qp._device_key == qp.device_key()
    qp.h, qp.h0, qp.d = _affine(data, qp.gk, qp.x0, Q_K, S_K)
    if fresh:  # same H and J on the device: only h, h0, d travel
        qp._device.update_affine(qp.h, qp.h0, qp.d)
        qp._device_key = qp.device_key()


def recover_trajectory(qp: DenseQp, v) -> Trajectory:
    """reduction.cpp:282-314: x = (bigA x_bar + bigAtilde w) + bigB v, u_t = K x_t + v_t, and
    the Eq. (1a) objective. Uses the cached free response x0 and bigB's first block column
    (x_t = x0_t + sum_{j<t} A_K^{t-1-j} B v_j), never the stacked matrices."""
    data = qp.source
    dm = dims(data)
    v = np.asarray(v, dtype=np.float64)
    if v.size != dm.T * dm.n_u:
        raise DimensionError(f"recover_trajectory: v has length {v.size}, expected {dm.T * dm.n_u}")
    vt = v.reshape(dm.T, dm.n_u)
    if qp.gk is None or qp.x0 is None:
        A_K = data.A + data.B @ data.K
        qp.gk = np.zeros((dm.T, dm.n_x, dm.n_u))
        qp.gk[0] = data.B
        for k in range(1, dm.T):
            qp.gk[k] = A_K @ qp.gk[k - 1]
        qp.x0 = free_response(A_K, data.x_bar, data.w)
    x = qp.x0.copy()
    # x_t = x0_t + sum_{k<t} G_k v_{t-1-k}: one GEMM of the block-Toeplitz arrangement of v
    # (row t-1 holds v_{t-1}, .., v_0) with [G_0' ; .. ; G_{T-1}'] (a GEMM per lag costs ~3x
    # more at config 3)
    T, nu = dm.T, dm.n_u
    gc = data.__dict__.setdefault("_gcat_cache", {})  # shared by every DenseQp of this data
    if gc.get("key") is not qp.gk:
        gc.clear()
        gc["key"] = qp.gk
        gc["gcat"] = np.ascontiguousarray(qp.gk.transpose(0, 2, 1).reshape(T * nu, dm.n_x))
    gcat = gc["gcat"]
    W = np.zeros((T, T * nu))
    for r in range(T):
        W[r, :(r + 1) * nu] = vt[r::-1].reshape(-1)
    x[1:] += W @ gcat
    u = x[:-1] @ data.K.T + vt
    # the diagonal-weight check scans n_x^2 entries: cache it on the problem data, which
    # every DenseQp built from it (e.g. a fresh upload per solve) shares
    cache = data.__dict__.setdefault("_quad_cache", {})
    key = (id(data.Q), id(data.Qf), id(data.R), id(data.S))
    if cache.get("key") != key:
        cache.clear()
        cache["key"] = key
        cache.update(Q=_diag_or_none(data.Q), Qf=_diag_or_none(data.Qf),
                     R=_diag_or_none(data.R), S0=not np.any(data.S))

    def quad(X, Mx, d):
        return (X * X) @ d if d is not None else np.einsum("ti,ti->t", X @ Mx, X)

    obj = float(quad(x[-1:], data.Qf, cache["Qf"])[0])
    cross = 0.0 if cache["S0"] else 2.0 * np.einsum("ti,ti->t", x[:-1] @ data.S, u)
    per_t = quad(x[:-1], data.Q, cache["Q"]) + cross + quad(u, data.R, cache["R"])
    obj += float(per_t.sum())
    return Trajectory(x=x, u=u, v=vt.copy(), objective=obj)


def dense_objective(qp: DenseQp, v) -> float:
    """reduction.cpp:316-321 (host helper; the solve computes it on the device)."""
    v = np.asarray(v, dtype=np.float64)
    if v.size != qp.n:
        raise DimensionError(f"dense_objective: v has length {v.size}, expected {qp.n}")
    return float(0.5 * v @ (qp.H @ v) + qp.h @ v + qp.h0)


# ---------------------------------------------------------------------- generators
@dataclass
class HeatParams:
    """heat3d.hpp:20-42 (Table I copper constants)."""

    N: int = 4
    T: int = 50
    dt: float = 0.1
    dw: float = 0.02
    rho: float = 8960.0
    cp: float = 386.0
    conductivity: float = 400.0
    q_weight: float = 10.0 * 0.02 * 0.02
    r_weight: float = 0.1 * 0.02 * 0.02
    x_min: float = 200.0
    x_max: float = 550.0
    u_min: float = 300.0
    u_max: float = 500.0
    x_init: float = 300.0
    setpoint: float = 350.0

    def diffusivity(self):
        return self.conductivity / (self.rho * self.cp)

    def stability_factor(self):
        return self.diffusivity() * self.dt / (self.dw * self.dw)


class StabilityError(RuntimeError):
    pass


def laplacian_system(N: int, params: HeatParams):
    """heat3d.cpp:7-37: 3-D cube, x-fastest cells, faces x0, xL, y0, yL, z0, zL as inputs."""
    if N < 1:
        raise DimensionError("grid must have at least one interior point per dimension")
    c = params.stability_factor()
    if not c < 1.0 / 6.0:
        raise StabilityError(f"explicit Euler unstable: diffusivity*dt/dw^2 = {c} must be below 1/6")
    nx = N ** 3
    A = np.zeros((nx, nx))
    B = np.zeros((nx, 6))
    cell = lambda i, j, k: i + N * j + N * N * k
    for k in range(N):
        for j in range(N):
            for i in range(N):
                r = cell(i, j, k)
                A[r, r] = 1.0 - 6.0 * c
                for cond, nb, face in ((i > 0, (i - 1, j, k), 0), (i < N - 1, (i + 1, j, k), 1),
                                       (j > 0, (i, j - 1, k), 2), (j < N - 1, (i, j + 1, k), 3),
                                       (k > 0, (i, j, k - 1), 4), (k < N - 1, (i, j, k + 1), 5)):
                    if cond:
                        A[r, cell(*nb)] = c
                    else:
                        B[r, face] += c
    return A, B


def _heat_problem(A, B, params: HeatParams, T: int, x_bar=None) -> LqProblemData:
    """heat3d.cpp:39-60 conventions: deviation variables about the set point."""
    nx, nu = A.shape[0], B.shape[1]
    q, r = params.q_weight, params.r_weight
    xb = np.full(nx, params.x_init - params.setpoint) if x_bar is None else np.asarray(x_bar, float)
    data = LqProblemData.basic(A, B, q * np.eye(nx), r * np.eye(nu), q * np.eye(nx), xb, T)
    defect = (A.sum(axis=1) + B.sum(axis=1) - 1.0) * params.setpoint
    data.w = np.tile(defect, (T, 1))
    data.xl = np.full(nx, params.x_min - params.setpoint)
    data.xu = np.full(nx, params.x_max - params.setpoint)
    data.ul = np.full(nu, params.u_min - params.setpoint)
    data.uu = np.full(nu, params.u_max - params.setpoint)
    return data


def build_heat_problem(params: HeatParams) -> LqProblemData:
    """heat3d.cpp:39-60 (the reference's 3-D cube, n_u = 6)."""
    if params.T < 1:
        raise DimensionError("horizon must be at least 1")
    A, B = laplacian_system(params.N, params)
    return _heat_problem(A, B, params, params.T)


def to_physical(traj: Trajectory, params: HeatParams) -> Trajectory:
    """heat3d.cpp:62-66."""
    return Trajectory(x=traj.x + params.setpoint, u=traj.u + params.setpoint, v=traj.v,
                      objective=traj.objective)


def rod_system(ncells: int, params: HeatParams):
    """1-D rod (config 2): inputs 0/1 = left/right end (Dirichlet), 2/3 = lateral heater
    zones over the two halves with coupling c. Rows of [A B] sum to 1."""
    c = params.stability_factor()
    if not 3.0 * c < 1.0:
        raise StabilityError("explicit Euler unstable for the rod")
    A = np.zeros((ncells, ncells))
    B = np.zeros((ncells, 4))
    half = ncells // 2
    for i in range(ncells):
        A[i, i] = 1.0 - 3.0 * c
        if i > 0:
            A[i, i - 1] = c
        else:
            B[i, 0] += c
        if i < ncells - 1:
            A[i, i + 1] = c
        else:
            B[i, 1] += c
        B[i, 2 if i < half else 3] += c
    return A, B


def _segments(length, splits):
    """index -> segment id for boundaries [0, s1, s2, ..., length)."""
    seg = np.zeros(length, dtype=int)
    for k, b in enumerate(splits):
        seg[b:] = k + 1
    return seg


def plate_system(nx: int, ny: int, bottom, top, left, right, params: HeatParams):
    """2-D plate nx x ny (x-fastest). Edge cells whose stencil neighbour is missing couple
    to the input of the edge segment they lie on; ``bottom``/``top`` are split points
    along x, ``left``/``right`` along y. Inputs are numbered bottom, top, left, right."""
    c = params.stability_factor()
    if not c < 0.25:
        raise StabilityError("explicit Euler unstable for the plate")
    sb, st = _segments(nx, bottom), _segments(nx, top)
    sl, sr = _segments(ny, left), _segments(ny, right)
    nb, nt, nl = len(bottom) + 1, len(top) + 1, len(left) + 1
    nu = nb + nt + nl + len(right) + 1
    n = nx * ny
    A = np.zeros((n, n))
    B = np.zeros((n, nu))
    cell = lambda i, j: i + nx * j
    for j in range(ny):
        for i in range(nx):
            r = cell(i, j)
            A[r, r] = 1.0 - 4.0 * c
            if i > 0:
                A[r, cell(i - 1, j)] = c
            else:
                B[r, nb + nt + sl[j]] += c
            if i < nx - 1:
                A[r, cell(i + 1, j)] = c
            else:
                B[r, nb + nt + nl + sr[j]] += c
            if j > 0:
                A[r, cell(i, j - 1)] = c
            else:
                B[r, sb[i]] += c
            if j < ny - 1:
                A[r, cell(i, j + 1)] = c
            else:
                B[r, nb + st[i]] += c
    return A, B


# BASELINE.json configurations
def heat1d_problem(ncells=200, T=50, params: HeatParams | None = None) -> LqProblemData:
    """config 2: 1-D rod, n_x = 200, n_u = 4, T = 50."""
    p = params or HeatParams()
    A, B = rod_system(ncells, p)
    return _heat_problem(A, B, p, T)


def heat2d_problem(nx=50, ny=50, T=50, splits=None, params: HeatParams | None = None,
                   x_bar=None) -> LqProblemData:
    """config 3 (50 x 50, n_u = 10), config 4 (40 x 25, n_u = 10), config 5 (20 x 25, n_u = 5)."""
    p = params or HeatParams()
    if splits is None:
        splits = default_splits(nx, ny)
    A, B = plate_system(nx, ny, *splits, p)
    return _heat_problem(A, B, p, T, x_bar)


def default_splits(nx, ny):
    if (nx, ny) == (50, 50):
        return ([17, 34], [17, 34], [25], [25])
    if (nx, ny) == (40, 25):
        return ([14, 27], [14, 27], [13], [13])
    if (nx, ny) == (20, 25):
        return ([10], [], [], [])
    # generic: two segments per edge
    return ([nx // 2], [nx // 2], [ny // 2], [ny // 2])


def batch_initial_states(n_x: int, count: int, seed: int = 42, spread: float = 20.0,
                         params: HeatParams | None = None) -> np.ndarray:
    """config 5: per-instance x_bar = 300 K + U[-spread, spread] per cell, in deviation units."""
    p = params or HeatParams()
    rng = np.random.default_rng(seed)
    return (p.x_init - p.setpoint) + rng.uniform(-spread, spread, size=(count, n_x))
