"""B200-native condensed-space interior-point hot path for linear-quadratic MPC
(arXiv 2209.13049; reference API: /root/reference/proj/include/condmpc).

    from paper_2209_13049_b200 import problem, ipm, linalg
    qp = problem.build_dense_qp(problem.heat2d_problem(50, 50, T=50))
    result = ipm.solve(qp, ipm.IpmOptions())        # backend "cuda"

The device path lives in ``libcondmpc_cuda.so`` (csrc/, C ABI include/condmpc_cuda.h);
there is no CPU fallback.
"""
from . import _lib, ipm, linalg, problem  # noqa: F401
from ._lib import CudaError, DimensionError  # noqa: F401

__all__ = ["ipm", "linalg", "problem", "DimensionError", "CudaError"]
