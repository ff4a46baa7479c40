import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2209_13049_b200 import _lib, ipm, problem as P
from test_gpu_builder import random_arrays
from _cmpc_helpers import lq_from_oracle
from oracle import oracle as O
seed, nx, nu, T = 54, 40, 2, 5
arrs = random_arrays(seed, nx, nu, 0, T, K=False, S=False, inf_frac=0.3)
data = lq_from_oracle(O.problem_from_arrays(**arrs))
qp = P.build_dense_qp(data)
L = _lib.lib()
print("xl finite", np.isfinite(arrs["xl"]).sum(), "xu finite", np.isfinite(arrs["xu"]).sum())
for mk in (2, 0):
    dq = ipm.DeviceQp.from_problem(data, options={"markov": mk})
    print("markov", mk, dq.info())
    rng = np.random.default_rng(1)
    n, m = dq.n, dq.m
    v, lam = rng.uniform(-1, 1, n), rng.uniform(-1, 1, m)
    s, z = rng.uniform(0.5, 2, m), rng.uniform(0.5, 2, m)
    _lib.check(L.cmpc_set_state(dq.h, _lib.ptr(v), _lib.ptr(s), _lib.ptr(lam), _lib.ptr(z), 0.1))
    r1, r2, r3, kkt = np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(1)
    _lib.check(L.cmpc_compute_residuals(dq.h, _lib.ptr(r1), _lib.ptr(r2), _lib.ptr(r3), _lib.ptr(kkt)))
    e1 = r1 - (qp.H @ v + qp.h + qp.J.T @ lam)
    e3 = r3 - (qp.J @ v - qp.d + s)
    print(" r1 err", np.abs(e1).max(), np.round(e1, 4))
    bad = np.flatnonzero(np.abs(e3) > 1e-10)
    print(" r3 err", np.abs(e3).max(), "bad rows", bad[:20], len(bad))
    sigma = rng.uniform(0.01, 100, m)
    M = np.zeros((n, n), order="F")
    _lib.check(L.cmpc_assemble_condensed(dq.h, _lib.ptr(sigma), _lib.ptr(M)))
    eM = M - (qp.H + qp.J.T @ (sigma[:, None] * qp.J))
    print(" M err", np.abs(eM).max())
    dq.close()
