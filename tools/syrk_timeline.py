"""Per-CTA timeline of one condensation (cmpc_debug_syrk_timeline) after a solve: imbalance,
per-mode step cost fit, SM occupancy over time. Usage: python tools/syrk_timeline.py c3"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import _lib, ipm, problem as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
qp = P.build_dense_qp(bench.build_problem(cfg))
dq = ipm.device_qp(qp)
print(dq.info())
for name in ("condense", "condense"):
    print(name, f"{dq.time_phase(name, 10) * 1e3:.1f} us")
cap = 1 << 16
out = np.zeros(cap * 8)
nb = C.c_int64()
for rep in range(3):
    _lib.check(_lib.lib().cmpc_debug_syrk_timeline(dq.h, _lib.ptr(out), cap, C.byref(nb)))
t = out[: nb.value * 8].reshape(-1, 8)
st, en, sm = t[:, 0], t[:, 1], t[:, 2].astype(int)
nseg, steps = t[:, 3], t[:, 4:8]  # full off, thin off, full diag, thin diag
W = np.array([1.0, 0.6, 0.8, 0.35])
cost = steps @ W
dur = en - st
X = np.column_stack([steps, nseg])
coef, *_ = np.linalg.lstsq(X, dur, rcond=None)
print("  regression us per step: full-off %.3f thin-off %.3f full-diag %.3f thin-diag %.3f per-seg %.2f" % tuple(coef))
print("  relative to full-off:", np.round(coef[:4] / coef[0], 3))
for name, mask in (("sm even", sm % 2 == 0), ("sm odd", sm % 2 == 1), ("sm < 74", sm < 74), ("sm >= 74", sm >= 74)):
    print(f"  {name:9s} mean dur {dur[mask].mean():.1f}  mean resid {(dur - X @ coef)[mask].mean():+.2f}")
print(f"pieces {len(t)}  makespan {en.max():.1f} us  mean dur {dur.mean():.1f}  min {dur.min():.1f}  max {dur.max():.1f}")
print(f"  sum(dur)/(296) = {dur.sum() / 296:.1f} us (ideal makespan at 2 CTAs/SM)")
ok = cost > 0
k = np.polyfit(cost[ok], dur[ok], 1)
print(f"  fit dur = {k[0]:.3f} us/weighted-step * cost + {k[1]:.2f} us")
resid = dur - np.polyval(k, cost)
print(f"  residual sd {resid.std():.2f} us; worst +{resid.max():.1f}")
# end-time distribution (tail)
q = np.percentile(en, [50, 90, 99, 100])
print("  end-time pct 50/90/99/100:", np.round(q, 1))
print("  start-time pct 50/90/99/100:", np.round(np.percentile(st, [50, 90, 99, 100]), 1))
# busy SM count over time
grid = np.linspace(0, en.max(), 21)
for g0, g1 in zip(grid[:-1], grid[1:]):
    busy = ((st < g1) & (en > g0)).sum()
    print(f"   {g0:7.1f}-{g1:7.1f} us  running CTAs {busy}")
