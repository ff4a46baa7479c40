"""The C-ABI library builds, loads and exports every entry point include/condmpc_cuda.h
declares; the product never routes through the oracle; no silent CPU fallback. CPU only."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "condmpc_cuda.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cmpc_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2209_13049_b200 import _lib
    L = _lib.lib()
    names = declared()
    assert len(names) >= 25
    for name in names:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (cmpc_\w+)", out))
    assert set(names) <= exported
    assert L.cmpc_abi_version() == 1


def test_library_is_sm100a_only():
    from paper_2209_13049_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass          # FP64 tensor-core MMA in the SYRK / Cholesky updates
    assert "UTMALDG" in sass       # TMA tile loads in the SYRK pipeline


def test_product_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_2209_13049_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liborc" not in txt, f


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2209_13049_b200 import ipm, problem as P
    from paper_2209_13049_b200._lib import CudaError
    qp = P.DenseQp(H=[[4.0]], h=[2.0], h0=0.0, J=[[-1.0]], d=[0.0])
    with pytest.raises(CudaError):
        ipm.solve(qp)


def test_error_codes_surface_as_exceptions():
    from paper_2209_13049_b200 import ipm, problem as P
    from paper_2209_13049_b200._lib import DimensionError
    qp = P.DenseQp(H=[[4.0]], h=[2.0], h0=0.0, J=[[-1.0]], d=[0.0])
    for bad in (dict(tau=1.5), dict(kappa_mu=0.0), dict(tol=0.0), dict(mu_init=-1.0), dict(max_iter=0)):
        with pytest.raises(DimensionError):
            ipm.solve(qp, ipm.IpmOptions(**bad))
    with pytest.raises(ValueError):
        ipm.solve(qp, ipm.IpmOptions(backend="lapack"))


def test_host_side_rules():  # test_ipm.cpp:322-361 on the host mirror
    from paper_2209_13049_b200 import ipm
    st = ipm.IpmState(np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0), mu=0.1)
    o = ipm.IpmOptions(tol=1e-8, max_iter=10)
    res = ipm.Residuals(np.zeros(0), np.zeros(0), np.zeros(0), 1e-3)
    assert ipm.update_barrier(st, res, o) == pytest.approx(0.02, rel=1e-15)
    res.kkt_error = 10.0
    assert ipm.update_barrier(st, res, o) == 0.1
    st.mu, res.kkt_error = 1e-9, 0.0
    assert ipm.update_barrier(st, res, o) == 1e-9
    st.iter, res.kkt_error = 3, 1e-9
    assert ipm.check_termination(res, st, o) == ipm.Termination.converged
    res.kkt_error = 1e-3
    assert ipm.check_termination(res, st, o) == ipm.Termination.keep_going
    res.kkt_error, st.mu = 1e-9, 1e-4
    assert ipm.check_termination(res, st, o) == ipm.Termination.keep_going
    st.iter = 10
    assert ipm.check_termination(res, st, o) == ipm.Termination.max_iter


def test_backend_registry():  # test_dense_linalg.cpp:162-169 with the B200 registry
    from paper_2209_13049_b200 import linalg
    assert linalg.make_backend("cuda").name() == "cuda"
    assert linalg.make_backend("cuda").parallel()
    # the reference's names select the device factorization (same factor)
    for alias in ("reference", "eigen"):
        assert linalg.make_backend(alias).name() == "cuda"
    for unknown in ("reference-cpu", "Eigen", "nonexistent", ""):
        with pytest.raises(ValueError):
            linalg.make_backend(unknown)


def test_null_context_is_an_error_not_a_crash():
    """A closed (null) context handle is rejected with an error code (no dereference)."""
    from paper_2209_13049_b200 import _lib
    L = _lib.lib()
    h = ctypes.c_void_p()
    assert L.cmpc_ctx_clone(None, ctypes.byref(h)) == _lib.CMPC_ERR_ARG
    assert "null context" in _lib.last_error()
    out = (ctypes.c_int64 * 8)()
    assert L.cmpc_update_qp_affine(None, None, 0.0, None, 0) == _lib.CMPC_ERR_DIM
