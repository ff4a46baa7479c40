"""Where the config-3 end-to-end time goes besides the solve (tools only): CMPC_VERBOSE load
phases and CMPC_SOLVE_TIMES for ipm.solve on a fresh DenseQp from pinned host arrays."""
import os
import sys
import time

os.environ["CMPC_VERBOSE"] = "1"
os.environ["CMPC_SOLVE_TIMES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

data = bench.build_problem("c3")
qp = P.build_dense_qp(data)
pin = dict(H=bench.pinned_like(qp.H), h=bench.pinned_like(qp.h), J=bench.pinned_like(qp.J), d=bench.pinned_like(qp.d))
for k in range(4):
    fresh = P.DenseQp(H=pin["H"], h=pin["h"], h0=qp.h0, J=pin["J"], d=pin["d"], source=qp.source, gk=qp.gk, x0=qp.x0)
    t0 = time.perf_counter()
    r = ipm.solve(fresh, ipm.IpmOptions())
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    print(f"e2e {dt:.2f} ms, device solve {r.device_seconds * 1e3:.2f} ms, total_seconds {r.total_seconds * 1e3:.2f}",
          file=sys.stderr, flush=True)
    fresh.invalidate_device()
