"""Device dense-QP build at a config: build time, solve, recovery, parity with the host build.
python tools/builder_probe.py c3"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
data = bench.build_problem(cfg)
t0 = time.perf_counter()
qp = P.build_dense_qp(data)
t1 = time.perf_counter()
print(f"host build {1e3 * (t1 - t0):.0f} ms  n={qp.n} m={qp.m}", flush=True)
for rep in range(3):
    t0 = time.perf_counter()
    dq = ipm.DeviceQp.from_problem(data)
    t1 = time.perf_counter()
    r = dq.solve()
    t2 = time.perf_counter()
    print(f"device build+load {1e3 * (t1 - t0):.1f} ms, solve+recover {1e3 * (t2 - t1):.1f} ms "
          f"(device {1e3 * r.device_seconds:.1f} ms) iter {r.iter} {r.status.name}", flush=True)
    if rep < 2:
        dq.close()
H, h, h0, d = dq.get_qp()
rel = lambda a, b: float(np.abs(a - b).max() / (1 + np.abs(b).max()))
print(f"rel diff vs host build: H {rel(H, qp.H):.2e} h {rel(h, qp.h):.2e} d {rel(d, qp.d):.2e} "
      f"h0 {abs(h0 - qp.h0) / (1 + abs(qp.h0)):.2e}")
b = ipm.solve(qp)
print(f"host-built solve: iter {b.iter} obj {b.objective:.15e}; device-built obj {r.objective:.15e}; "
      f"v rel {rel(r.v, b.v):.2e}; traj obj {r.solution.objective:.12e} vs {b.solution.objective:.12e}")
