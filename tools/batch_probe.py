"""Time ipm.BatchSolver on config-5 instances: python tools/batch_probe.py [count ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2209_13049_b200 import batch, ipm, problem as P  # noqa: E402

data = P.heat2d_problem(20, 25, T=30)
base = P.build_dense_qp(data)
for count in [int(x) for x in sys.argv[1:]] or [16, 64, 256]:
    xbs = P.batch_initial_states(500, count, seed=42)
    t0 = time.perf_counter()
    bs = ipm.BatchSolver(base, count, workers=int(os.environ.get('WORKERS', '0')) or None)
    for i, xb in enumerate(xbs):
        bs.set_instance(i, *batch.instance_affine(base, xb))
    t1 = time.perf_counter()
    res = bs.solve(ipm.IpmOptions())
    t2 = time.perf_counter()
    res = bs.solve(ipm.IpmOptions())
    t3 = time.perf_counter()
    print(f"count {count} workers {bs.workers}: setup {t1 - t0:.2f} s, first solve {t2 - t1:.3f} s, second {t3 - t2:.3f} s "
          f"= {(t3 - t2) / count * 1e3:.3f} ms/instance, iters {np.mean(res.iter):.1f}", flush=True)
    bs.close()
