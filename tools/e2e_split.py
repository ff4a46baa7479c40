"""Where the e2e time of config 3 goes: context + load (H2D, analysis, plan), solve, D2H and
the host trajectory recovery. python tools/e2e_split.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

data = bench.build_problem("c3")
qp = P.build_dense_qp(data)
pin = {k: bench.pinned_like(getattr(qp, k)) for k in ("H", "h", "J", "d")}
for rep in range(4):
    fresh = P.DenseQp(H=pin["H"], h=pin["h"], h0=qp.h0, J=pin["J"], d=pin["d"], source=qp.source,
                      gk=qp.gk, x0=qp.x0)
    t0 = time.perf_counter()
    dq = ipm.device_qp(fresh)
    t1 = time.perf_counter()
    r = ipm.solve_loaded(dq, fresh, ipm.IpmOptions())
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms, solve_loaded {1e3*(t2-t1):.2f} ms (device {1e3*r.device_seconds:.2f}, "
          f"host loop {1e3*r.total_seconds:.2f}), sync {1e3*(t3-t2):.2f}", flush=True)
    t4 = time.perf_counter()
    tr = P.recover_trajectory(fresh, r.v)
    print(f"   host recover_trajectory alone {1e3*(time.perf_counter()-t4):.2f} ms", flush=True)
    fresh.invalidate_device()
