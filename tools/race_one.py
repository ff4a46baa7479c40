"""One small solve (config-5 instance) for compute-sanitizer racecheck / synccheck."""
import sys
sys.path.insert(0, ".")
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402
qp = P.build_dense_qp(P.heat2d_problem(8, 6, T=8))
r = ipm.solve(qp, ipm.IpmOptions(max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 3))
print(r.status.name, r.iter)
