"""Clone timing growth (config 5 contexts): python tools/clone_probe.py N"""
import sys
import time

sys.path.insert(0, ".")
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
base = P.build_dense_qp(P.heat2d_problem(20, 25, T=30))
root = ipm.device_qp(base)
ctxs = []
t0 = time.perf_counter()
for i in range(N):
    ctxs.append(root.clone())
    if (i + 1) % 64 == 0:
        t1 = time.perf_counter()
        print(f"{i + 1} clones, last 64 in {t1 - t0:.2f} s", flush=True)
        t0 = t1
