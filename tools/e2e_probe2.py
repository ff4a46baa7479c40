"""e2e outlier hunt: the bench's e2e loop with (a) another loaded context alive, (b) the clock
sampler running; per-step ms."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

qp = P.build_dense_qp(P.heat2d_problem(50, 50, T=50))
pin = dict(H=bench.pinned_like(qp.H), h=bench.pinned_like(qp.h), J=bench.pinned_like(qp.J), d=bench.pinned_like(qp.d))
mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
keep = None
if mode in ("ctx", "both", "ctxreuse"):
    keep = ipm.DeviceQp(qp)
    qp._device = keep
    for _ in range(3):
        ipm.solve_loaded(keep, qp, ipm.IpmOptions())
samp = bench.ClockSampler(0) if mode in ("clock", "both") else None
if samp:
    samp.__enter__()
out = []
from paper_2209_13049_b200 import _lib  # noqa: E402
reuse = ipm.DeviceQp(qp) if "reuse" in mode else None
for k in range(14):
    if reuse is not None:
        fresh = P.DenseQp(H=pin["H"], h=pin["h"], h0=qp.h0, J=pin["J"], d=pin["d"], source=qp.source, gk=qp.gk, x0=qp.x0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(_lib.lib().cmpc_load_qp(reuse.h, fresh.n, fresh.m, _lib.ptr(fresh.H), _lib.ptr(fresh.h), fresh.h0,
                                            _lib.ptr(fresh.J), _lib.ptr(fresh.d), 0))
        t1 = time.perf_counter()
        r = ipm.solve_loaded(reuse, fresh, ipm.IpmOptions())
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out.append((round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1), round(r.device_seconds * 1e3, 1)))
        continue
    fresh = P.DenseQp(H=pin["H"], h=pin["h"], h0=qp.h0, J=pin["J"], d=pin["d"], source=qp.source, gk=qp.gk, x0=qp.x0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ipm.solve(fresh)
    torch.cuda.synchronize()
    out.append(round((time.perf_counter() - t0) * 1e3, 1))
    fresh.invalidate_device()
if samp:
    samp.__exit__(None, None, None)
print(mode, out)
