import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P
data = P.heat2d_problem(20, 25, T=30)
base = P.build_dense_qp(data)
xbs = P.batch_initial_states(data.A.shape[0], 8, seed=11)
insts = []
for xb in xbs:
    d2 = data.copy(); d2.x_bar = xb; insts.append(P.build_dense_qp(d2))
a = ipm.solve(insts[0]); b = ipm.solve(insts[0])
print("single twice equal:", np.array_equal(a.v, b.v))
q = insts[0]; q2 = P.DenseQp(H=q.H, h=q.h, h0=q.h0, J=q.J, d=q.d)
c = ipm.solve(q2)
print("fresh ctx equal:", np.array_equal(a.v, c.v), np.abs(a.v - c.v).max())
for w in (15,) * 16:
    bs = ipm.BatchSolver(base, len(insts), workers=w)
    for i, qq in enumerate(insts): bs.set_instance(i, qq.h, qq.h0, qq.d)
    res = bs.solve()
    print("workers", w, [float(np.abs(res.v[i] - ipm.solve(insts[i]).v).max()) for i in (0, 1, 7)])
    bs.close()
