"""condmpc::linalg on the GPU (proj/include/condmpc/dense_linalg.hpp:12-59).

The reference's plug point is ``Backend::factorize``; here the registry knows
``"cuda"`` (the only backend this package ships — the reference's "reference" and
"eigen" CPU backends are not part of the product). Every call runs on the device
through ``libcondmpc_cuda.so``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import DimensionError, check, f64, ptr

DEVICE = 0


class NotPositiveDefinite(RuntimeError):
    """dense_linalg.hpp:12-16: carries the failing pivot index."""

    def __init__(self, pivot: int, msg: str):
        super().__init__(msg)
        self.pivot = pivot


class Factor:
    """Lower Cholesky factor (dense_linalg.hpp:18-35); immutable."""

    def __init__(self, lower: np.ndarray, seconds: float = 0.0):
        self._lower = np.asfortranarray(lower)
        self._lower.setflags(write=False)
        self._seconds = seconds

    def lower(self) -> np.ndarray:
        return self._lower

    def dim(self) -> int:
        return self._lower.shape[0]

    def factorize_seconds(self) -> float:
        return self._seconds

    def solve(self, rhs) -> np.ndarray:
        """Two triangular solves against L L' on the device (dense_linalg.cpp:102-110)."""
        rhs = f64(rhs).reshape(-1)
        n = self.dim()
        if rhs.size != n:
            raise DimensionError(f"cholesky_solve: rhs length {rhs.size} does not match factor "
                                 f"dimension {n}")
        x = np.zeros(n)
        check(_lib.lib().cmpc_cholesky_solve(DEVICE, n, ptr(self._lower), ptr(rhs), ptr(x)))
        return x


class Backend:
    def name(self) -> str:
        raise NotImplementedError

    def in_place(self) -> bool:
        raise NotImplementedError

    def parallel(self) -> bool:
        raise NotImplementedError

    def factorize(self, sym) -> Factor:
        raise NotImplementedError


class CudaBackend(Backend):
    """Blocked FP64 Cholesky on the B200 (csrc/chol.cu)."""

    def name(self):
        return "cuda"

    def in_place(self):
        return False

    def parallel(self):
        return True

    def factorize(self, sym) -> Factor:
        import time
        sym = f64(sym)
        n = sym.shape[0]
        if sym.ndim != 2 or sym.shape[1] != n:
            raise DimensionError("cholesky_factorize: matrix must be square")
        L = np.zeros((n, n), order="F")
        piv = C.c_int64(-1)
        t0 = time.perf_counter()
        rc = _lib.lib().cmpc_cholesky(DEVICE, n, ptr(sym), ptr(L), C.byref(piv))
        dt = time.perf_counter() - t0
        if rc == _lib.CMPC_NOT_PD:
            raise NotPositiveDefinite(piv.value, _lib.last_error())
        check(rc)
        return Factor(L, dt)


# The reference's names (dense_linalg.cpp:112-116: "reference" = blocked right-looking
# Cholesky, "eigen" = Eigen::LLT) select the same device factorization here: both compute
# the lower Cholesky factor of the same matrix, so code written against the reference keeps
# working; "cuda" names it explicitly. Anything else throws like the reference.
BACKEND_NAMES = ("cuda", "reference", "eigen")


def make_backend(name: str) -> Backend:
    """dense_linalg.cpp:112-116 with the B200 registry."""
    if name in BACKEND_NAMES:
        return CudaBackend()
    raise ValueError(f"unknown factorization backend: {name}")


def is_symmetric(m: np.ndarray, rel_tol: float) -> bool:
    """types.hpp:25-29."""
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        return False
    if m.size == 0:
        return True
    return float(np.abs(m - m.T).max()) <= rel_tol * (1.0 + float(np.abs(m).max()))


def cholesky_factorize(backend: Backend, sym) -> Factor:
    """dense_linalg.cpp:118-124."""
    sym = np.asarray(sym, dtype=np.float64)
    if sym.ndim != 2 or sym.shape[0] != sym.shape[1]:
        raise DimensionError("cholesky_factorize: matrix must be square")
    if not is_symmetric(sym, 1e-10):
        raise ValueError("cholesky_factorize: matrix not symmetric within 1e-10 relative")
    return backend.factorize(sym)


def cholesky_solve(factor: Factor, rhs) -> np.ndarray:
    return factor.solve(rhs)


def gram_weighted(J, sigma) -> np.ndarray:
    """J' diag(sigma) J on DMMA tensor cores (dense_linalg.cpp:128-137), full symmetric."""
    J = f64(J)
    if J.ndim != 2:
        raise DimensionError("gram_weighted: J must be a matrix")
    m, n = J.shape
    sigma = f64(sigma).reshape(-1)
    if sigma.size != m:
        raise DimensionError("gram_weighted: sigma length must equal row count of J")
    G = np.zeros((n, n), order="F")
    if m == 0 or n == 0:
        return G
    check(_lib.lib().cmpc_gram_weighted(DEVICE, m, n, ptr(J), ptr(sigma), ptr(G)))
    return G
