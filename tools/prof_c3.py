"""C3 solve for profiling: one warm solve, then one profiled solve."""
import sys, time
sys.path.insert(0, ".")
from paper_2209_13049_b200 import ipm, problem as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
if cfg == "c3":
    qp = P.build_dense_qp(P.heat2d_problem(50, 50, T=50))
elif cfg == "c2":
    qp = P.build_dense_qp(P.heat1d_problem())
elif cfg == "c4":
    qp = P.build_dense_qp(P.heat2d_problem(40, 25, T=int(sys.argv[2]) if len(sys.argv) > 2 else 200))
dq = ipm.device_qp(qp)
print(dq.info(), flush=True)
for k in range(2):
    r = ipm.solve(qp)
    print(r.status.name, r.iter, r.total_seconds, r.device_seconds, r.linalg_seconds, r.launches, flush=True)
