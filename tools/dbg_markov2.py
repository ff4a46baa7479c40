import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2209_13049_b200 import _lib, ipm, problem as P
from test_gpu_builder import random_arrays
from _cmpc_helpers import lq_from_oracle, oracle_qp, rel
from oracle import oracle as O
seed, nx, nu, T = 55, 2, 4, 33
arrs = random_arrays(seed, nx, nu, 0, T, K=False, S=False, inf_frac=0.3)
data = lq_from_oracle(O.problem_from_arrays(**arrs))
qp = P.build_dense_qp(data)
o = O.solve(oracle_qp(O, qp))
print("oracle", o.status, o.iter, [int(r[7]) for r in o.log], [r[6] for r in o.log])
for mk in (2, 0):
    dq = ipm.DeviceQp.from_problem(data, options={"markov": mk})
    log = []
    r = ipm.solve_loaded(dq, None, ipm.IpmOptions(log=log.append))
    print("markov", mk, dq.info()["markov"], r.status.name, r.iter, [x.trial for x in log], [x.delta for x in log], rel(r.v, o.v))
    dq.close()
    log = []
    r = ipm.solve_loaded(ipm.DeviceQp(qp), qp, ipm.IpmOptions(log=log.append))
    print("dense ", r.status.name, r.iter, [x.trial for x in log], rel(r.v, o.v))
for opt in ({"jtl_recurrence": 0}, {"small_path": 0}, {"speculate": 0}):
    dq = ipm.DeviceQp(qp)
    for k, v in opt.items():
        dq.set_option(k, v)
    log = []
    r = ipm.solve_loaded(dq, qp, ipm.IpmOptions(log=log.append))
    print(opt, r.iter, [x.trial for x in log][-3:], [f"{x.alpha:.17g}" for x in log][-2:])
    dq.close()
print("oracle alphas", [f"{r_[2]:.17g}" for r_ in o.log][-2:])
