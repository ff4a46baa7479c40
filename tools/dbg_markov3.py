import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2209_13049_b200 import ipm, problem as P
from test_gpu_builder import random_arrays
from _cmpc_helpers import lq_from_oracle, oracle_qp, rel
from oracle import oracle as O
for case in [(42, 6, 2, 3, 7, False, True), (43, 4, 3, 2, 9, True, True), (44, 9, 2, 4, 12, True, False)]:
    seed, nx, nu, nc, T, K, S = case
    arrs = random_arrays(seed, nx, nu, nc, T, K=K, S=S)
    data = lq_from_oracle(O.problem_from_arrays(**arrs))
    qp = P.build_dense_qp(data)
    o = O.solve(oracle_qp(O, qp))
    print(case, "oracle", o.iter, [int(r[7]) for r in o.log])
    for mk in (2, 0):
        dq = ipm.DeviceQp.from_problem(data, options={"markov": mk})
        log = []
        r = ipm.solve_loaded(dq, None, ipm.IpmOptions(log=log.append))
        print("  markov", mk, dq.info()["markov"], r.iter, [x.trial for x in log], "rel v", rel(r.v, o.v))
        dq.close()
    log = []
    r = ipm.solve_loaded(ipm.DeviceQp(qp), qp, ipm.IpmOptions(log=log.append))
    print("  dense", r.iter, [x.trial for x in log], "rel v", rel(r.v, o.v))
