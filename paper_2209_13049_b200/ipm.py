"""condmpc::ipm on the B200 (proj/include/condmpc/ipm.hpp, proj/src/ipm.cpp).

Same names, argument meaning and error behaviour as the reference: ``solve(qp, opts)``
runs the C++ host loop of csrc/ipm_host.cpp over the device kernels; the per-step
functions (``compute_residuals``, ``assemble_condensed``, ``step_directions``,
``line_search`` ...) run the same kernels on the QP's device context so they can be
unit-tested like proj/tests/test_ipm.cpp. ``update_barrier`` and ``check_termination``
are the host-side scalar rules (identical to the C++ loop's).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import DimensionError, check, f64, ptr
from . import linalg as _linalg
from .linalg import Factor, NotPositiveDefinite
from .problem import DenseQp, Trajectory, recover_trajectory


class IpmStatus(enum.Enum):
    converged = 0
    max_iter = 1
    factorization_failure = 2
    line_search_failure = 3


def to_string(status: IpmStatus) -> str:
    return status.name


class Termination(enum.Enum):
    converged = 0
    max_iter = 1
    keep_going = 2


@dataclass
class IpmState:
    v: np.ndarray
    s: np.ndarray
    lambda_: np.ndarray
    z: np.ndarray
    mu: float = 0.0
    iter: int = 0


@dataclass
class Residuals:
    r1: np.ndarray
    r2: np.ndarray
    r3: np.ndarray
    kkt_error: float = 0.0


@dataclass
class StepDirections:
    pv: np.ndarray
    ps: np.ndarray
    plambda: np.ndarray
    pz: np.ndarray


@dataclass
class IterationRecord:
    iter: int
    mu: float
    alpha: float
    alpha_z: float
    kkt_error: float
    objective: float
    delta: float = 0.0  # extension: shift used by the factorization
    trial: int = 0      # extension: accepted line-search trial j


@dataclass
class IterationInspection:
    state: IpmState
    residuals: Residuals
    dirs: StepDirections
    delta: float


@dataclass
class IpmOptions:
    tol: float = 1e-8
    mu_init: float = 1e-1
    kappa_mu: float = 0.2
    tau: float = 0.995
    max_iter: int = 200
    armijo_eta: float = 1e-4
    backend: str = "cuda"
    log: Optional[Callable[[IterationRecord], None]] = None
    inspect: Optional[Callable[[IterationInspection], None]] = None


@dataclass
class IpmResult:
    status: IpmStatus = IpmStatus.max_iter
    solution: Trajectory = field(default_factory=Trajectory)
    v: np.ndarray = None
    s: np.ndarray = None
    lambda_: np.ndarray = None
    z: np.ndarray = None
    iter: int = 0
    kkt_error: float = 0.0
    objective: float = 0.0
    total_seconds: float = 0.0
    linalg_seconds: float = 0.0
    device_seconds: float = 0.0
    launches: int = 0
    syncs: int = 0
    trials: int = 0
    syrk_seconds: float = 0.0     # device time of the condensation (SYRK + reduce)
    chol_seconds: float = 0.0     # device time of the first factorization attempts
    condensations: int = 0
    syrk_kernel_seconds: float = 0.0  # device time of the SYRK kernel alone (k_syrk)


class DeviceQp:
    """One device context (stream + HBM buffers) holding a loaded DenseQp."""

    def __init__(self, qp: DenseQp, device: int | None = None, on_device_ptrs=None):
        L = _lib.lib()
        device = _linalg.DEVICE if device is None else device
        h = C.c_void_p()
        check(L.cmpc_ctx_create(C.byref(h), device))
        self.h = h
        self.n, self.m = qp.n, qp.m
        if on_device_ptrs is not None:
            H, hv, J, d = on_device_ptrs
            check(L.cmpc_load_qp(self.h, qp.n, qp.m, C.cast(H, _lib.D), C.cast(hv, _lib.D),
                                 qp.h0, C.cast(J, _lib.D), C.cast(d, _lib.D), 1))
        else:
            check(L.cmpc_load_qp(self.h, qp.n, qp.m, ptr(qp.H), ptr(qp.h), qp.h0, ptr(qp.J),
                                 ptr(qp.d), 0))

    @classmethod
    def from_problem(cls, data, device: int | None = None, options: dict | None = None) -> "DeviceQp":
        """build_dense_qp (reduction.cpp:255-268) on the device: only the
        structured data crosses PCIe; J is never stored (the analysis generates its rows) and,
        when every SYRK prototype is a state row, neither is P: the SYRK and the P products
        read the Markov table of B-responses (option "markov": 1, the
        default, when P would exceed 64 MB; 2 always; 0 never). ``options``: per-context
        options applied before the build (set_option)."""
        from . import problem as P
        dm = P.dims(data)
        L = _lib.lib()
        device = _linalg.DEVICE if device is None else device
        out = cls.__new__(cls)
        h = C.c_void_p()
        check(L.cmpc_ctx_create(C.byref(h), device))
        out.h = h
        for k, v in (options or {}).items():
            out.set_option(k, v)
        keep = {}

        def arr(name, a):
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))  # no copy for C-ordered input
            keep[name] = a
            return a.ctypes.data_as(_lib.D) if a.size else None

        # matrices go across row-major (layout 1) and are transposed on the device
        pr = _lib.LqProblem(nx=dm.n_x, nu=dm.n_u, nc=dm.n_c, T=dm.T, layout=1)
        for f in ("A", "B", "Q", "Qf", "R", "S", "E", "F", "K", "gl", "gu", "xl", "xu", "ul", "uu", "x_bar"):
            setattr(pr, f, arr(f, getattr(data, f)))
        pr.w = arr("w", data.w)
        check(L.cmpc_build_qp(out.h, C.byref(pr)))
        info = (C.c_int64 * 8)()
        L.cmpc_qp_info(out.h, info)
        out.n, out.m = int(info[0]), int(info[1])
        out.source = data
        return out

    def get_qp(self):
        """(H, h, h0, d) of the loaded QP, read back from the device."""
        H = np.zeros((self.n, self.n), order="F")
        h, d, h0 = np.zeros(self.n), np.zeros(self.m), np.zeros(1)
        check(_lib.lib().cmpc_get_qp(self.h, ptr(H), ptr(h), ptr(h0), ptr(d)))
        return H, h, float(h0[0]), d

    def refresh_initial_state(self, x_bar):
        """refresh_initial_state (reduction.cpp:270-280) on the device."""
        xb = np.ascontiguousarray(np.asarray(x_bar, dtype=np.float64))
        check(_lib.lib().cmpc_refresh_initial_state(self.h, ptr(xb)))
        self.source = dataclasses.replace(self.source, x_bar=xb.copy())

    def recover_trajectory(self, v=None) -> "Trajectory":
        """recover_trajectory (reduction.cpp:282-314) on the device (v None: the last solve's)."""
        from . import problem as P
        dm = P.dims(self.source)
        x = np.zeros((dm.T + 1, dm.n_x))
        u = np.zeros((dm.T, dm.n_u))
        obj = np.zeros(1)
        vv = None if v is None else np.ascontiguousarray(np.asarray(v, dtype=np.float64))
        check(_lib.lib().cmpc_recover_trajectory(self.h, ptr(vv), ptr(x), ptr(u), ptr(obj)))
        return P.Trajectory(x=x, u=u, v=None if v is None else vv.reshape(dm.T, dm.n_u).copy(),
                            objective=float(obj[0]))

    def solve(self, opts: "IpmOptions" = None) -> "IpmResult":
        """ipm::solve on the loaded QP; the trajectory is recovered on the device when the
        QP was built there."""
        opts = opts or IpmOptions()
        _check_options(opts)
        return solve_loaded(self, None, opts)

    def close(self):
        if getattr(self, "h", None):
            try:
                _lib.lib().cmpc_ctx_destroy(self.h)
            except (AttributeError, TypeError):  # interpreter shutdown: the module is gone
                pass
            self.h = None

    __del__ = close

    def info(self):
        out = (C.c_int64 * 8)()
        _lib.lib().cmpc_qp_info(self.h, out)
        lay = (C.c_int64 * 4)()
        _lib.lib().cmpc_qp_layout(self.h, lay)
        return dict(n=out[0], m=out[1], prototypes=out[2], syrk_prototypes=out[3],
                    singletons=out[4], syrk_units=out[5], syrk_flops=out[6], p_bytes=out[7],
                    markov=bool(lay[0]), markov_rows=lay[1], markov_cols=lay[2],
                    stored_bytes=lay[3])

    PHASES = dict(condense_all=0, condense=1, cholesky=2, chol_solve=3, residuals=4, recover=5,
                  trial=6, Jx=7, Jty=8, prepare=9, chol_fused=10, condense_rhs=11)

    def time_phase(self, name: str, reps: int = 10) -> float:
        """Device milliseconds of one phase (CUDA events, back-to-back launches)."""
        ms = C.c_double()
        check(_lib.lib().cmpc_time_phase(self.h, self.PHASES[name], int(reps), C.byref(ms)))
        return ms.value

    def clone(self) -> "DeviceQp":
        """A new context with a device copy of this QP and its J structure."""
        out = DeviceQp.__new__(DeviceQp)
        h = C.c_void_p()
        check(_lib.lib().cmpc_ctx_clone(self.h, C.byref(h)))
        out.h, out.n, out.m = h, self.n, self.m
        return out

    def update_affine(self, h, h0, d):
        h, d = f64(h), f64(d)
        check(_lib.lib().cmpc_update_qp_affine(self.h, ptr(h), float(h0), ptr(d), 0))

    def set_option(self, key: str, value: int):
        """Per-context switches (no process-wide environment): "jtl_recurrence" (1: carry
        J'lambda across a step, 0: recompute it by a pass over J as compute_residuals does),
        "rhs_pass" (0/1: fused into the condensation, 2: its own pass over P), "graphs" (1:
        CUDA-graph replay of the per-iteration segments, 0: eager launches), "small_path" (1:
        the whole solve in one CTA when n <= 32 and J fits in shared memory, 0: never),
        "speculate" (1: the step update and next residual pass are enqueued before the host
        has seen the step, gated on the device's evaluation of line-search trial 0; 0: off)."""
        check(_lib.lib().cmpc_ctx_set_option(self.h, key.encode(), int(value)))

    def set_state(self, st: IpmState):
        v, s, l, z = _state_arrays(st, self.n, self.m)
        check(_lib.lib().cmpc_set_state(self.h, ptr(v), ptr(s), ptr(l), ptr(z), float(st.mu)))


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for a row-sharded solve; create it on rank 0 and
    broadcast it to the other ranks (any host channel: torch.distributed, MPI, a file)."""
    buf = C.create_string_buffer(128)
    check(_lib.lib().cmpc_comm_unique_id(buf))
    return buf.raw


NCCL_DETERMINISM = {"NCCL_ALGO": "Ring", "NCCL_PROTO": "Simple"}


class ShardedQp:
    """This rank's part of a row-sharded QP: rows `rows` of J and d (from
    problem.shard_rows) on this process's GPU, attached to an NCCL communicator over all
    ranks. solve() runs ipm::solve cooperatively — every rank must call it with the same
    options — and returns the same v, kkt, objective, iteration count and status on every
    rank, with s, lambda, z for this rank's rows."""

    def __init__(self, qp: DenseQp, rows, uid: bytes, nranks: int, rank: int):
        import os
        from .problem import shard_qp
        # a fixed reduction algorithm and protocol: NCCL's choice may change with the message
        # size or topology, and with it the summation order (bitwise reproducible solves,
        # proj/tests/test_ipm.cpp:432-457); must be set before the communicator exists
        for k, v in NCCL_DETERMINISM.items():
            os.environ.setdefault(k, v)
        self.rows = np.asarray(rows, dtype=np.int64)
        self.m_total = qp.m
        self.local = shard_qp(qp, self.rows)
        self.dq = DeviceQp(self.local)
        if len(uid) != 128:
            raise DimensionError("the NCCL unique id is 128 bytes")
        check(_lib.lib().cmpc_ctx_attach_comm(self.dq.h, uid, int(nranks), int(rank),
                                              int(self.m_total)))
        self.nranks, self.rank = nranks, rank

    def solve(self, opts: IpmOptions = None) -> IpmResult:
        opts = opts or IpmOptions()
        _check_options(opts)
        return solve_loaded(self.dq, self.local, opts)

    def reload(self, local: DenseQp):
        """Upload a new copy of this rank's rows (same shape) into the same context: the
        communicator and the total row count stay attached (end-to-end timing)."""
        if local.m != self.local.m or local.n != self.local.n:
            raise DimensionError("reload: the shard's shape changed")
        check(_lib.lib().cmpc_load_qp(self.dq.h, local.n, local.m, ptr(local.H), ptr(local.h),
                                      local.h0, ptr(local.J), ptr(local.d), 0))
        self.local = local

    def close(self):
        if getattr(self, "dq", None) is not None:
            self.dq.close()
            self.dq = None


class LoopbackShards:
    """The row-sharded solve (ShardedQp's C++ loop and kernels) with `nranks` ranks inside one
    process on one GPU: the shards (problem.shard_rows) are attached to an in-process loopback
    communicator instead of NCCL, and solve() drives every rank from its own host thread, as
    torchrun would drive one process per GPU. Tests of the multi-rank path without a multi-GPU
    node; the results of every rank are returned."""

    def __init__(self, qp: DenseQp, nranks: int, device: int | None = None):
        from .problem import shard_qp, shard_rows
        device = _linalg.DEVICE if device is None else device
        L = _lib.lib()
        g = C.c_void_p()
        check(L.cmpc_loop_create(int(nranks), int(device), C.byref(g)))
        self.group = g
        self.rows = shard_rows(qp, nranks)
        self.locals = [shard_qp(qp, r) for r in self.rows]
        self.dqs = [DeviceQp(loc, device=device) for loc in self.locals]
        for r, dq in enumerate(self.dqs):
            check(L.cmpc_ctx_attach_loop(dq.h, self.group, r, int(qp.m)))
        self.nranks = nranks

    def solve(self, opts: IpmOptions = None) -> list:
        import threading
        opts = opts or IpmOptions()
        _check_options(opts)
        out = [None] * self.nranks
        errs = []

        def run(r):
            try:
                out[r] = solve_loaded(self.dqs[r], self.locals[r], opts)
            except Exception as e:  # re-raised in the caller
                errs.append(e)

        th = [threading.Thread(target=run, args=(r,)) for r in range(self.nranks)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        return out

    def close(self):
        for dq in getattr(self, "dqs", []):
            dq.close()
        self.dqs = []
        if getattr(self, "group", None) is not None:
            _lib.lib().cmpc_loop_destroy(self.group)
            self.group = None


def device_qp(qp: DenseQp) -> DeviceQp:
    """The QP's cached device context: re-created when it was closed or when the QP's arrays
    are no longer the ones it was loaded from (DenseQp.device_key). The reference takes the QP
    by const reference on every call, so a solve always sees the current arrays."""
    key = qp.device_key()
    if qp._device is not None and getattr(qp._device, "h", None) is not None and qp._device_key == key:
        return qp._device
    if qp._device is not None and qp._device_key is not None and qp._device_key != key:
        qp._device.close()  # the arrays changed under the cached context
    qp._device = DeviceQp(qp)
    qp._device_key = key
    return qp._device


def _state_arrays(st: IpmState, n, m):
    v, s, l, z = (f64(x).reshape(-1) for x in (st.v, st.s, st.lambda_, st.z))
    if v.size != n:
        raise DimensionError("state.v does not match the QP")
    if s.size != m or l.size != m or z.size != m:
        raise DimensionError("state slack/dual lengths do not match the QP row count")
    return v, s, l, z


def _check_options(opts: IpmOptions):
    """ipm.cpp:17-23."""
    if not opts.tol > 0.0:
        raise DimensionError("tol must be positive")
    if not (0.0 < opts.kappa_mu < 1.0):
        raise DimensionError("kappa_mu must lie in (0,1)")
    if not (0.0 < opts.tau < 1.0):
        raise DimensionError("tau must lie in (0,1)")
    if not opts.mu_init > 0.0:
        raise DimensionError("mu_init must be positive")
    if not opts.max_iter >= 1:
        raise DimensionError("max_iter must be at least 1")


# ------------------------------------------------------------------ per-step API
def compute_residuals(qp: DenseQp, state: IpmState) -> Residuals:
    """ipm.cpp:46-70."""
    dq = device_qp(qp)
    dq.set_state(state)
    r1, r2, r3 = np.zeros(qp.n), np.zeros(qp.m), np.zeros(qp.m)
    kkt = C.c_double()
    check(_lib.lib().cmpc_compute_residuals(dq.h, ptr(r1), ptr(r2), ptr(r3), C.byref(kkt)))
    return Residuals(r1, r2, r3, kkt.value)


def assemble_condensed(qp: DenseQp, sigma) -> np.ndarray:
    """ipm.cpp:72-77: H + J' diag(sigma) J (full symmetric)."""
    sigma = f64(sigma).reshape(-1)
    if sigma.size != qp.m:
        raise DimensionError("sigma length does not match the QP row count")
    dq = device_qp(qp)
    M = np.zeros((qp.n, qp.n), order="F")
    check(_lib.lib().cmpc_assemble_condensed(dq.h, ptr(sigma) if qp.m > 0 else None, ptr(M)))
    return M


def step_directions(qp: DenseQp, state: IpmState, res: Residuals, factor: Factor) -> StepDirections:
    """ipm.cpp:79-103 with the given factor of the condensed matrix."""
    dq = device_qp(qp)
    dq.set_state(state)
    L = _lib.lib()
    r1, r2, r3 = (f64(x).reshape(-1) for x in (res.r1, res.r2, res.r3))
    check(L.cmpc_set_residuals(dq.h, ptr(r1), ptr(r2), ptr(r3)))
    Lf = f64(factor.lower())
    if Lf.shape != (qp.n, qp.n):
        raise DimensionError("factor dimension does not match the QP")
    check(L.cmpc_set_factor(dq.h, ptr(Lf)))
    pv, ps, pl, pz = np.zeros(qp.n), np.zeros(qp.m), np.zeros(qp.m), np.zeros(qp.m)
    alpha = np.zeros(2)
    check(L.cmpc_step_directions(dq.h, 0.5, ptr(pv), ptr(ps), ptr(pl), ptr(pz), ptr(alpha)))
    return StepDirections(pv, ps, pl, pz)


def fraction_to_boundary(s, ps, z, pz, tau):
    """ipm.cpp:105-116: (alpha_max, alpha_z)."""
    if not (0.0 < tau < 1.0):
        raise DimensionError("tau must lie in (0,1)")
    s, ps, z, pz = (f64(x).reshape(-1) for x in (s, ps, z, pz))
    out = np.zeros(2)
    check(_lib.lib().cmpc_fraction_to_boundary(_linalg.DEVICE, s.size, ptr(s), ptr(ps), ptr(z), ptr(pz),
                                                float(tau), ptr(out)))
    return float(out[0]), float(out[1])


def line_search(qp: DenseQp, state: IpmState, dirs: StepDirections, alpha_max: float,
                opts: IpmOptions = IpmOptions()) -> Optional[float]:
    """ipm.cpp:118-144: first accepted alpha_max * 2^-j, or None."""
    if not (0.0 < alpha_max <= 1.0):
        raise DimensionError("alpha_max must lie in (0,1]")
    dq = device_qp(qp)
    dq.set_state(state)
    L = _lib.lib()
    pv, ps, pl, pz = (f64(x).reshape(-1) for x in (dirs.pv, dirs.ps, dirs.plambda, dirs.pz))
    check(L.cmpc_set_directions(dq.h, ptr(pv), ptr(ps) if qp.m else None, ptr(pl) if qp.m else None,
                                ptr(pz) if qp.m else None))
    a = C.c_double()
    j = C.c_int()
    check(L.cmpc_line_search(dq.h, float(alpha_max), float(opts.armijo_eta), C.byref(a), C.byref(j)))
    return a.value if j.value >= 0 else None


def update_barrier(state: IpmState, res: Residuals, opts: IpmOptions) -> float:
    """ipm.cpp:146-151."""
    if res.kkt_error <= 10.0 * state.mu:
        return max(opts.tol / 10.0, opts.kappa_mu * state.mu)
    return state.mu


def check_termination(res: Residuals, state: IpmState, opts: IpmOptions) -> Termination:
    """ipm.cpp:153-158."""
    if res.kkt_error <= opts.tol and state.mu <= opts.tol:
        return Termination.converged
    if state.iter >= opts.max_iter:
        return Termination.max_iter
    return Termination.keep_going


# ------------------------------------------------------------------ solve
def solve_problem(data, opts: IpmOptions = None) -> IpmResult:
    """build_dense_qp + ipm::solve + recover_trajectory, all on the device (SURVEY §8(f)
    rows 1 and 3): the structured problem in, the trajectory out."""
    dq = DeviceQp.from_problem(data)
    try:
        return dq.solve(opts)
    finally:
        dq.close()


def solve(qp: DenseQp, opts: IpmOptions = None) -> IpmResult:
    """ipm.cpp:160-268: the whole solve on the device, host loop in C++."""
    opts = opts or IpmOptions()
    _check_options(opts)
    if qp.h.size != qp.n:
        raise DimensionError("qp.h length does not match qp.H")
    if qp.d.size != qp.m:
        raise DimensionError("qp.d length does not match qp.J")
    if opts.backend not in _linalg.BACKEND_NAMES:
        raise ValueError(f"unknown factorization backend: {opts.backend}")
    t0 = time.perf_counter()
    dq = device_qp(qp)
    return solve_loaded(dq, qp, opts, t0)


def solve_loaded(dq: DeviceQp, qp: DenseQp | None, opts: IpmOptions, t0=None) -> IpmResult:
    t0 = time.perf_counter() if t0 is None else t0
    n, m = (qp.n, qp.m) if qp is not None else (dq.n, dq.m)
    v, s, l, z = np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(m)
    out = np.zeros(14)
    L = _lib.lib()

    def _log(user, rec):
        opts.log(IterationRecord(int(rec[0]), rec[1], rec[2], rec[3], rec[4], rec[5], rec[6],
                                 int(rec[7])))

    def _insp(user, v_, s_, l_, z_, mu, r1, r2, r3, kkt, pv, ps, pl, pz, delta):
        vec = lambda p, k: np.ctypeslib.as_array(p, shape=(k,)).copy() if k else np.zeros(0)
        st = IpmState(vec(v_, n), vec(s_, m), vec(l_, m), vec(z_, m), mu)
        opts.inspect(IterationInspection(st, Residuals(vec(r1, n), vec(r2, m), vec(r3, m), kkt),
                                         StepDirections(vec(pv, n), vec(ps, m), vec(pl, m),
                                                        vec(pz, m)), delta))

    lf = _lib.LOG_FN(_log) if opts.log else _lib.LOG_FN()
    inf_ = _lib.INSPECT_FN(_insp) if opts.inspect else _lib.INSPECT_FN()
    od = (C.c_double * 5)(opts.tol, opts.mu_init, opts.kappa_mu, opts.tau, opts.armijo_eta)
    check(L.cmpc_solve(dq.h, od, int(opts.max_iter), ptr(v), ptr(s), ptr(l), ptr(z), ptr(out), lf,
                       inf_, None))
    res = IpmResult(status=IpmStatus(int(out[0])), v=v, s=s, lambda_=l, z=z, iter=int(out[1]),
                    kkt_error=float(out[2]), objective=float(out[3]), linalg_seconds=float(out[5]),
                    device_seconds=float(out[6]), launches=int(out[7]), syncs=int(out[8]),
                    trials=int(out[9]), syrk_seconds=float(out[10]), chol_seconds=float(out[11]),
                    condensations=int(out[12]), syrk_kernel_seconds=float(out[13]))
    if qp is None and getattr(dq, "source", None) is not None:
        res.solution = dq.recover_trajectory()
        res.solution.v = v.reshape(res.solution.u.shape).copy()
    elif qp is not None and qp.source is not None:
        res.solution = recover_trajectory(qp, v)
    else:
        res.solution = Trajectory(objective=res.objective)
    res.total_seconds = time.perf_counter() - t0
    return res


@dataclass
class BatchResult:
    status: list
    iter: np.ndarray
    objective: np.ndarray
    kkt_error: np.ndarray
    v: np.ndarray            # count x n
    device_seconds: np.ndarray
    launches: int
    wall_seconds: float


LOCKSTEP_MAX_N = 160  # csrc/batch.cu keeps each instance's condensed matrix in shared memory


class BatchSolver:
    """Independent instances that share H and J and differ in (h, h0, d) — the
    receding-horizon / config-5 case (refresh_initial_state, reduction.cpp:270-280).

    mode "lockstep" (the default when n <= 160 and J has rows): ONE host loop drives every
    instance, each kernel covering all active instances in one launch (csrc/batch.cu,
    csrc/bsyrk.cu: one CTA per instance for the condensation over the shared P and for the
    Cholesky, DGEMMs for the products with P and H); every instance still takes the
    reference's decisions (ipm.cpp:160-268) on its own scalars.
    mode "workers": a few worker device contexts (cloned from the base QP's analysed
    structure, one host thread and one CUDA stream each) take the instances in turn, each
    running the single-instance loop."""

    def __init__(self, base: DenseQp, count: int, workers: int | None = None, mode: str = "auto"):
        import os
        self.base = base
        self.count = count
        if mode == "auto":
            mode = "lockstep" if (0 < base.m and base.n <= LOCKSTEP_MAX_N) else "workers"
        if mode not in ("lockstep", "workers"):
            raise ValueError(f"unknown batch mode: {mode}")
        self.mode = mode
        self.h_all = np.repeat(f64(base.h).reshape(1, -1), count, axis=0)
        self.h0_all = np.full(count, float(base.h0))
        self.d_all = np.repeat(f64(base.d).reshape(1, -1), count, axis=0)
        self._pinned = []
        self.ctxs = []
        self._batch = None
        self._root = None
        if mode == "lockstep":
            self.workers = 1
            self._root = DeviceQp(base)
            h = C.c_void_p()
            check(_lib.lib().cmpc_batch_create(self._root.h, int(count), C.byref(h)))
            self._batch = h
            self._dirty = True
        else:
            # workers per process: the cores this process may use (under torchrun every rank
            # gets its share of the host, not all of it), one left for the interpreter
            try:
                cores = len(os.sched_getaffinity(0))
            except AttributeError:
                cores = os.cpu_count() or 2
            local = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
            cores = max(1, cores // max(1, local))
            self.workers = max(1, min(count, workers or max(1, cores - 1)))
            root = device_qp(base)
            self.ctxs = [root.clone() for _ in range(self.workers)]
            root.close()
        for a in (self.h_all, self.d_all):  # page-locked: the per-instance uploads are plain DMA
            if a.nbytes and _lib.lib().cmpc_host_register(a.ctypes.data, a.nbytes) == 0:
                self._pinned.append(a)

    def set_instance(self, i: int, h, h0: float, d):
        self.h_all[i] = np.asarray(h, dtype=np.float64)
        self.h0_all[i] = float(h0)
        self.d_all[i] = np.asarray(d, dtype=np.float64)
        self._dirty = True

    def condense(self, sigma, w):
        """Lockstep mode: the condensation step alone for every instance (assemble_condensed +
        the right-hand side's J'w, ipm.cpp:72-103): sigma, w count x m -> (M count x n x n with
        the lower triangle of H + J' diag(sigma_b) J, tq count x n = J' w_b)."""
        if self.mode != "lockstep":
            raise ValueError("condense needs the lockstep batch")
        n, m, cnt = self.base.n, self.base.m, self.count
        sg = np.ascontiguousarray(sigma, dtype=np.float64).reshape(cnt, m)
        ww = np.ascontiguousarray(w, dtype=np.float64).reshape(cnt, m)
        M = np.zeros((cnt, n, n))
        tq = np.zeros((cnt, n))
        check(_lib.lib().cmpc_batch_condense(self._batch, ptr(sg), ptr(ww), ptr(M), ptr(tq)))
        return M.transpose(0, 2, 1), tq  # column-major per instance

    def solve(self, opts: IpmOptions = None, threads: int | None = None) -> BatchResult:
        opts = opts or IpmOptions()
        _check_options(opts)
        n, cnt = self.base.n, self.count
        if self.mode == "lockstep":
            L = _lib.lib()
            if self._dirty:
                check(L.cmpc_batch_set_affine(self._batch, ptr(self.h_all), ptr(self.h0_all), ptr(self.d_all)))
                self._dirty = False
            v = np.zeros((cnt, n))
            scal = np.zeros((cnt, 14))
            stats = np.zeros(10)
            od = (C.c_double * 5)(opts.tol, opts.mu_init, opts.kappa_mu, opts.tau, opts.armijo_eta)
            t0 = time.perf_counter()
            check(L.cmpc_batch_solve(self._batch, od, int(opts.max_iter), ptr(v), ptr(scal), ptr(stats)))
            wall = time.perf_counter() - t0
            self.last_stats = dict(batch_iterations=int(stats[0]), device_seconds=float(stats[1]),
                                   wall_seconds=float(stats[2]), launches=int(stats[3]),
                                   syncs=int(stats[4]), rounds=int(stats[5]),
                                   condense_seconds=float(stats[6]), condense_launches=int(stats[7]),
                                   condense_instances=float(stats[8]),
                                   condense_flops_per_instance=float(stats[9]))
            return BatchResult(status=[IpmStatus(int(x)).name for x in scal[:, 0]], iter=scal[:, 1].astype(int),
                               objective=scal[:, 3].copy(), kkt_error=scal[:, 2].copy(), v=v,
                               device_seconds=np.full(cnt, float(stats[1]) / cnt), launches=int(stats[3]),
                               wall_seconds=wall)
        nw = max(1, min(self.workers, threads or self.workers))
        v = np.zeros((cnt, n))
        scal = np.zeros((cnt, 14))
        arr = (C.c_void_p * nw)(*[c.h.value if isinstance(c.h, C.c_void_p) else c.h for c in self.ctxs[:nw]])
        od = (C.c_double * 5)(opts.tol, opts.mu_init, opts.kappa_mu, opts.tau, opts.armijo_eta)
        t0 = time.perf_counter()
        check(_lib.lib().cmpc_solve_batch_affine(arr, nw, cnt, ptr(self.h_all), ptr(self.h0_all),
                                                 ptr(self.d_all), od, int(opts.max_iter), ptr(v), ptr(scal)))
        wall = time.perf_counter() - t0
        return BatchResult(status=[IpmStatus(int(x)).name for x in scal[:, 0]], iter=scal[:, 1].astype(int),
                           objective=scal[:, 3].copy(), kkt_error=scal[:, 2].copy(), v=v,
                           device_seconds=scal[:, 6].copy(), launches=int(scal[:, 7].sum()),
                           wall_seconds=wall)

    def close(self):
        if getattr(self, "_batch", None) is not None:
            try:
                _lib.lib().cmpc_batch_destroy(self._batch)
            except (AttributeError, TypeError):  # interpreter shutdown
                pass
            self._batch = None
        if getattr(self, "_root", None) is not None:
            self._root.close()
            self._root = None
        for c in getattr(self, "ctxs", []):
            c.close()
        self.ctxs = []
        for a in getattr(self, "_pinned", []):
            try:
                _lib.lib().cmpc_host_unregister(a.ctypes.data)
            except (AttributeError, TypeError):  # interpreter shutdown
                pass
        self._pinned = []

    __del__ = close
