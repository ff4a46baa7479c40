"""A few iterations of a device-built QP on the Markov-table path (tools only: the ncu target
for k_syrk / k_mk_gemv with P never stored).  python tools/markov_solve.py [c3|c4] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
data = P.heat2d_problem(50, 50, T=50) if cfg == "c3" else P.heat2d_problem(40, 25, T=200)
dq = ipm.DeviceQp.from_problem(data, options={"markov": 2})
assert dq.info()["markov"]
r = dq.solve(ipm.IpmOptions(max_iter=iters))
print(cfg, "markov", r.iter, r.status.name, dq.info()["stored_bytes"])
dq.close()
