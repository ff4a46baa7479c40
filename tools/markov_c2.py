"""Markov table vs materialised P at config 2 (tools only): device ms per solve, P x, P' q."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

d = P.heat1d_problem(200, 50)
for mk in (1, 0):
    dq = ipm.DeviceQp.from_problem(d, options={"markov": 2 * mk})
    ts = [dq.solve().device_seconds * 1e3 for _ in range(8)][2:]
    print("c2 markov", mk, round(statistics.median(ts), 3), "Jx", round(dq.time_phase("Jx", 20) * 1e3, 1),
          "Jty", round(dq.time_phase("Jty", 20) * 1e3, 1), flush=True)
    dq.close()
