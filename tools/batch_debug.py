import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P
from test_gpu_batch import instances
data = P.heat2d_problem(10, 8, T=12, splits=([5], [5], [4], [4]))
base, insts = instances(data, 12)
dq = ipm.device_qp(base)
print("info", dq.info())
bs = ipm.BatchSolver(base, len(insts))
for i, q in enumerate(insts):
    bs.set_instance(i, q.h, q.h0, q.d)
res = bs.solve()
print(res.status, res.iter, bs.last_stats)
for i, q in enumerate(insts[:4]):
    log = []
    single = ipm.solve(q, ipm.IpmOptions(log=log.append))
    print(i, single.status.name, single.iter, res.iter[i], np.abs(res.v[i] - single.v).max(), res.objective[i], single.objective)
    print("   mu:", [round(x.mu, 12) for x in log][:12])
    print("   j:", [x.trial for x in log])
log = []
single = ipm.solve(insts[0], ipm.IpmOptions(log=log.append))
for x in log[:8]:
    print(f"[single] iter {x.iter} mu {x.mu:.6g} alpha {x.alpha:.10g} alpha_z {x.alpha_z:.10g} kkt {x.kkt_error:.10g} obj {x.objective:.12g} j {x.trial}")
