"""Host-loop time vs device time of a solve: fresh context (graphs captured during the solve),
second solve on the same context (graphs replayed), eager (option graphs = 0)."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

qp = P.build_dense_qp(bench.build_problem("c3"))
for rep in range(3):
    dq = ipm.DeviceQp(qp)
    if rep == 2:
        dq.set_option("graphs", 0)
    for k in range(2):
        t0 = time.perf_counter()
        r = ipm.solve_loaded(dq, qp, ipm.IpmOptions())
        print(f"context {rep} solve {k}: wall {1e3*(time.perf_counter()-t0):.2f} ms, host loop "
              f"{1e3*r.total_seconds:.2f}, device {1e3*r.device_seconds:.2f}", flush=True)
    dq.close()
