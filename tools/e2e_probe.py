import os, sys, time
sys.path.insert(0, ".")
os.environ["CMPC_VERBOSE"] = "1"
import numpy as np, torch
from paper_2209_13049_b200 import ipm, problem as P
import bench
qp = P.build_dense_qp(P.heat2d_problem(50, 50, T=50))
pin = dict(H=bench.pinned_like(qp.H), h=bench.pinned_like(qp.h), J=bench.pinned_like(qp.J), d=bench.pinned_like(qp.d))
for k in range(8):
    fresh = P.DenseQp(H=pin["H"], h=pin["h"], h0=qp.h0, J=pin["J"], d=pin["d"], source=qp.source, gk=qp.gk, x0=qp.x0)
    t0 = time.perf_counter()
    dq = ipm.device_qp(fresh)
    t1 = time.perf_counter()
    r = ipm.solve(fresh)
    t2 = time.perf_counter()
    fresh.invalidate_device()
    t3 = time.perf_counter()
    print(f"e2e {k}: load {1e3*(t1-t0):.1f} ms solve(+recover) {1e3*(t2-t1):.1f} ms (device {1e3*r.device_seconds:.1f}) free {1e3*(t3-t2):.1f} ms", file=sys.stderr)
