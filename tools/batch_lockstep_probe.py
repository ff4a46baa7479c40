import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P, batch
cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
data = P.heat2d_problem(20, 25, T=30)
base = P.build_dense_qp(data)
xbs = P.batch_initial_states(500, cnt, seed=42)
bs = ipm.BatchSolver(base, cnt)
for i, xb in enumerate(xbs):
    bs.set_instance(i, *batch.instance_affine(base, xb))
for rep in range(3):
    res = bs.solve()
    st = bs.last_stats
    print(f"count {cnt} mode {bs.mode}: conv {sum(s == 'converged' for s in res.status)} iters mean {res.iter.mean():.1f} max {res.iter.max()} "
          f"wall {res.wall_seconds*1e3:.1f} ms device {st['device_seconds']*1e3:.1f} ms batch-iters {st['batch_iterations']} "
          f"-> {st['device_seconds']*1e3/st['batch_iterations']:.2f} ms/batch-iter, {res.wall_seconds*1e3/cnt:.3f} ms/solve; launches {st['launches']} syncs {st['syncs']} rounds {st['rounds']}", flush=True)
single = ipm.solve(P.build_dense_qp(data.copy() if False else data))
