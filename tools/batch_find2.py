import sys, subprocess
sys.path.insert(0, ".")
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P, batch
cnt, seed, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
data = P.heat2d_problem(20, 25, T=30)
base = P.build_dense_qp(data)
bs = ipm.BatchSolver(base, cnt)
for i, xb in enumerate(P.batch_initial_states(500, cnt, seed=seed)):
    bs.set_instance(i, *batch.instance_affine(base, xb))
for r in range(reps):
    res = bs.solve()
    print(cnt, seed, r, sum(s == "converged" for s in res.status), res.iter.max(), flush=True)
'''
for cnt, seed, reps in [(int(a), 9, 1) for a in sys.argv[1:]]:
    p = subprocess.run([sys.executable, "-c", code, str(cnt), str(seed), str(reps)], capture_output=True, text=True,
                       env={**__import__("os").environ, "CUDA_LAUNCH_BLOCKING": "1"})
    print("case", cnt, seed, reps, "rc", p.returncode, p.stdout.strip().replace("\n", " | "), p.stderr.strip().splitlines()[-12:] if p.returncode else "")
