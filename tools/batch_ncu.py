# one lockstep batch solve of 1024 config-5 instances, capped at a few iterations (ncu target)
import sys
sys.path.insert(0, ".")
from paper_2209_13049_b200 import ipm, problem as P, batch
cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
data = P.heat2d_problem(20, 25, T=30)
base = P.build_dense_qp(data)
xbs = P.batch_initial_states(500, cnt, seed=42)
bs = ipm.BatchSolver(base, cnt)
for i, xb in enumerate(xbs):
    bs.set_instance(i, *batch.instance_affine(base, xb))
res = bs.solve(ipm.IpmOptions(max_iter=3))
print(bs.last_stats)
