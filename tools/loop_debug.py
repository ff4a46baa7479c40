import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P
qp = P.build_dense_qp(P.heat2d_problem(12, 10, T=14, splits=([6], [6], [5], [5])))
n = int(sys.argv[1])
sh = ipm.LoopbackShards(qp, n)
print("rows per rank", [len(r) for r in sh.rows], "m", [d.m for d in sh.dqs], flush=True)
print([dq.info() for dq in sh.dqs], flush=True)
out = sh.solve()
print([r.iter for r in out], flush=True)
