"""Solve config-5 instances one at a time (single context), printing progress: finds an
instance that hangs or fails. python tools/batch_find.py first last"""
import sys
import time

sys.path.insert(0, ".")
from paper_2209_13049_b200 import batch, ipm, problem as P  # noqa: E402

first, last = int(sys.argv[1]), int(sys.argv[2])
data = P.heat2d_problem(20, 25, T=30)
base = P.build_dense_qp(data)
xbs = P.batch_initial_states(500, 1024, seed=42)
dq = ipm.device_qp(base)
for i in range(first, last):
    h, h0, d = batch.instance_affine(base, xbs[i])
    dq.update_affine(h, h0, d)
    print(f"instance {i} ...", end=" ", flush=True)
    t0 = time.perf_counter()
    q = P.DenseQp(H=base.H, h=h, h0=h0, J=base.J, d=d)
    r = ipm.solve_loaded(dq, q, ipm.IpmOptions())
    print(f"{r.status.name} iter {r.iter} {time.perf_counter() - t0:.3f}s", flush=True)
