"""ctypes binding of ``libcondmpc_cuda.so`` (C ABI: include/condmpc_cuda.h).

No CPU fallback: if the library or a CUDA device is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcondmpc_cuda.so")

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
LOG_FN = C.CFUNCTYPE(None, C.c_void_p, D)


class LqProblem(C.Structure):
    """cmpc_lq_problem (include/condmpc_cuda.h): LqProblemData for the device builder."""
    _fields_ = [("nx", C.c_int64), ("nu", C.c_int64), ("nc", C.c_int64), ("T", C.c_int64)] + [
        (f, D) for f in ("A", "B", "Q", "Qf", "R", "S", "E", "F", "gl", "gu", "xl", "xu", "ul", "uu",
                         "w", "x_bar", "K")] + [("layout", C.c_int64)]


INSPECT_FN = C.CFUNCTYPE(None, C.c_void_p, D, D, D, D, C.c_double, D, D, D, C.c_double, D, D, D,
                         D, C.c_double)

CMPC_OK, CMPC_NOT_PD, CMPC_ERR_DIM, CMPC_ERR_ARG, CMPC_ERR_CUDA = 0, 1, -1, -2, -3

_lib = None

# every exported entry point and its signature (the .so must export all of them)
SIGNATURES = {
    "cmpc_abi_version": (C.c_int, []),
    "cmpc_last_error": (C.c_char_p, []),
    "cmpc_launch_count": (C.c_longlong, []),
    "cmpc_ctx_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "cmpc_ctx_destroy": (None, [C.c_void_p]),
    "cmpc_load_qp": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, D, D, C.c_double, D, D, C.c_int]),
    "cmpc_qp_info": (C.c_int, [C.c_void_p, I64]),
    "cmpc_qp_layout": (C.c_int, [C.c_void_p, I64]),
    "cmpc_build_qp": (C.c_int, [C.c_void_p, C.POINTER(LqProblem)]),
    "cmpc_refresh_initial_state": (C.c_int, [C.c_void_p, D]),
    "cmpc_get_qp": (C.c_int, [C.c_void_p, D, D, D, D]),
    "cmpc_recover_trajectory": (C.c_int, [C.c_void_p, D, D, D, D]),
    "cmpc_debug_syrk_timeline": (C.c_int, [C.c_void_p, D, C.c_int64, I64]),
    "cmpc_update_qp_affine": (C.c_int, [C.c_void_p, D, C.c_double, D, C.c_int]),
    "cmpc_set_state": (C.c_int, [C.c_void_p, D, D, D, D, C.c_double]),
    "cmpc_get_state": (C.c_int, [C.c_void_p, D, D, D, D]),
    "cmpc_compute_residuals": (C.c_int, [C.c_void_p, D, D, D, D]),
    "cmpc_set_residuals": (C.c_int, [C.c_void_p, D, D, D]),
    "cmpc_assemble_condensed": (C.c_int, [C.c_void_p, D, D]),
    "cmpc_factorize_condensed": (C.c_int, [C.c_void_p, C.c_double, I64]),
    "cmpc_get_factor": (C.c_int, [C.c_void_p, D]),
    "cmpc_set_factor": (C.c_int, [C.c_void_p, D]),
    "cmpc_step_directions": (C.c_int, [C.c_void_p, C.c_double, D, D, D, D, D]),
    "cmpc_set_directions": (C.c_int, [C.c_void_p, D, D, D, D]),
    "cmpc_line_search": (C.c_int, [C.c_void_p, C.c_double, C.c_double, D, C.POINTER(C.c_int)]),
    "cmpc_merit": (C.c_int, [C.c_void_p, C.c_double, C.c_double, D]),
    "cmpc_apply_step": (C.c_int, [C.c_void_p, C.c_double, C.c_double]),
    "cmpc_dense_objective": (C.c_int, [C.c_void_p, D]),
    "cmpc_solve": (C.c_int, [C.c_void_p, D, C.c_int64, D, D, D, D, D, LOG_FN, INSPECT_FN,
                             C.c_void_p]),
    "cmpc_gram_weighted": (C.c_int, [C.c_int, C.c_int64, C.c_int64, D, D, D]),
    "cmpc_cholesky": (C.c_int, [C.c_int, C.c_int64, D, D, I64]),
    "cmpc_cholesky_solve": (C.c_int, [C.c_int, C.c_int64, D, D, D]),
    "cmpc_fraction_to_boundary": (C.c_int, [C.c_int, C.c_int64, D, D, D, D, C.c_double, D]),
    "cmpc_time_phase": (C.c_int, [C.c_void_p, C.c_int, C.c_int, D]),
    "cmpc_ctx_clone": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "cmpc_solve_batch": (C.c_int, [C.POINTER(C.c_void_p), C.c_int64, D, C.c_int64, D, D, C.c_int]),
    "cmpc_host_register": (C.c_int, [C.c_void_p, C.c_int64]),
    "cmpc_host_unregister": (C.c_int, [C.c_void_p]),
    "cmpc_solve_batch_affine": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int64, D, D, D, D,
                                          C.c_int64, D, D]),
    "cmpc_batch_create": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    "cmpc_batch_set_affine": (C.c_int, [C.c_void_p, D, D, D]),
    "cmpc_batch_solve": (C.c_int, [C.c_void_p, D, C.c_int64, D, D, D]),
    "cmpc_ctx_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "cmpc_batch_condense": (C.c_int, [C.c_void_p, D, D, D, D]),
    "cmpc_batch_destroy": (None, [C.c_void_p]),
    "cmpc_loop_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "cmpc_loop_destroy": (None, [C.c_void_p]),
    "cmpc_ctx_attach_loop": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int64]),
    "cmpc_comm_unique_id": (C.c_int, [C.c_void_p]),
    "cmpc_ctx_attach_comm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int64]),
    "cmpc_ctx_detach_comm": (C.c_int, [C.c_void_p]),
}


class DimensionError(RuntimeError):
    """The reference's condmpc::DimensionError (types.hpp:17-19)."""


class CudaError(RuntimeError):
    pass


def lib(build_if_missing: bool = True):
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            if not build_if_missing:
                raise CudaError(f"{LIB_PATH} is not built")
            from . import build as _b
            _b.build()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().cmpc_last_error().decode()


def check(rc: int) -> int:
    if rc >= 0:
        return rc
    msg = last_error()
    if rc == CMPC_ERR_DIM:
        raise DimensionError(msg)
    if rc == CMPC_ERR_CUDA:
        raise CudaError(msg)
    raise ValueError(msg)


def ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(D)


def f64(a, shape=None):
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape, order="F")
    return a


def launch_count() -> int:
    return int(lib().cmpc_launch_count())
