"""Host-loop vs device time of solves with fresh (untouched) output arrays, as ipm.solve makes."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

qp = P.build_dense_qp(bench.build_problem("c3"))
dq = ipm.DeviceQp(qp)
for rep in range(4):
    t0 = time.perf_counter()
    r = ipm.solve_loaded(dq, qp, ipm.IpmOptions())
    print(f"wall {1e3*(time.perf_counter()-t0):.2f} host {1e3*r.total_seconds:.2f} device "
          f"{1e3*r.device_seconds:.2f} iter {r.iter}", flush=True)
