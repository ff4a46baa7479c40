import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P
data = P.heat2d_problem(20, 25, T=30)
base = P.build_dense_qp(data)
cnt = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(3)
sigma = np.exp(rng.uniform(-6, 6, size=(cnt, base.m))); w = rng.standard_normal((cnt, base.m))
bs = ipm.BatchSolver(base, cnt, mode="lockstep")
for r in range(reps):
    M, tq = bs.condense(sigma, w)
bs.close()
print("condense ok", cnt, reps, flush=True)
