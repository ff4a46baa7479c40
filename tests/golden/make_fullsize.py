"""Generate tests/golden/fullsize_<case>.npz: the oracle's (CPU restatement of the reference
solver, pinned by tests/test_oracle_kat.py) whole solves at the BASELINE.json full-size heat
configurations, so the GPU tests can check the device solve decision for decision without
re-running minutes of CPU work on the box.

    python tests/golden/make_fullsize.py [case ...]     (all cases: ~30 min on 8 cores)

Each fixture holds the status, iteration count, objective, kkt, the per-iteration log (iter,
mu, alpha, alpha_z, kkt, objective, delta, trial), the full v (n), and for s, lambda, z (m
each, up to 3.2 MB apiece) a fixed sample of rows (every k-th row plus each vector's
largest entries) together with the full vectors' sum, sum of squares and max, so the
fixtures stay small. The oracle runs in its skip-zeros test mode (bitwise the dense loops'
results: oracle/oracle_core.cpp ZeroMap) on all host cores.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2209_13049_b200 import problem as P  # noqa: E402

NSAMPLE = 4096
NTOP = 64


def cases():
    """name -> structured problem (BASELINE.json configs 3 and 4; SURVEY Appendix B shapes)."""
    out = {"c3": lambda: P.heat2d_problem(50, 50, T=50)}
    for T in (50, 100, 150, 200):
        out[f"c4_T{T}"] = (lambda T=T: P.heat2d_problem(40, 25, T=T))
    return out


def sample_rows(m: int, extra: np.ndarray) -> np.ndarray:
    base = np.unique(np.linspace(0, m - 1, min(NSAMPLE, m)).astype(np.int64))
    return np.unique(np.concatenate([base, extra.astype(np.int64)]))


def summarize(x: np.ndarray) -> np.ndarray:
    return np.array([x.sum(), (x * x).sum(), np.abs(x).max() if x.size else 0.0])


def make(name: str) -> str:
    qp = P.build_dense_qp(cases()[name]())
    O.set_threads(os.cpu_count() or 1)
    O.set_skip_zeros(True)
    t = time.time()
    r = O.solve(O.qp_from_arrays(qp.H, qp.h, qp.h0, qp.J, qp.d))
    secs = time.time() - t
    O.set_skip_zeros(False)
    top = np.concatenate([np.argsort(-np.abs(a))[:NTOP] for a in (r.s, r.lam, r.z)])
    rows = sample_rows(qp.m, top)
    path = os.path.join(HERE, f"fullsize_{name}.npz")
    np.savez_compressed(
        path, status=np.array(r.status), iter=np.array(r.iter), objective=np.array(r.objective),
        kkt_error=np.array(r.kkt_error), log=np.array(r.log, dtype=np.float64), v=r.v,
        rows=rows, s=r.s[rows], lam=r.lam[rows], z=r.z[rows], s_sum=summarize(r.s),
        lam_sum=summarize(r.lam), z_sum=summarize(r.z), n=np.array(qp.n), m=np.array(qp.m),
        oracle_seconds=np.array(secs), oracle_threads=np.array(O.get_threads()))
    print(f"{name}: {r.status} in {r.iter} iterations, objective {r.objective!r}, "
          f"{secs:.1f} s on {O.get_threads()} threads -> {path}", flush=True)
    return path


if __name__ == "__main__":
    O.build()
    for name in (sys.argv[1:] or list(cases())):
        make(name)
