"""Create / destroy cycles of cloned contexts (config 5), with and without solves."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_2209_13049_b200 import batch, ipm, problem as P  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
base = P.build_dense_qp(P.heat2d_problem(20, 25, T=30))
for cyc in range(4):
    if mode == "plain":
        root = ipm.device_qp(base)
        cl = [root.clone() for _ in range(k)]
        root.close()
        for c in cl:
            c.close()
    else:
        bs = ipm.BatchSolver(base, k, workers=min(k, 15))
        if mode == "solve":
            res = bs.solve()
            print("  iters", np.mean(res.iter), flush=True)
        bs.close()
        del bs
    print("cycle", cyc, "ok", flush=True)
