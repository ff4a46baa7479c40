"""Executed / algorithmic SYRK work of a 64 x 64-tile plan vs the row granularity of its segment
shapes, over a QP's prototype prefix widths:
    python tools/syrk_waste_model.py c3
A tile (I, J) executes ceil((hi - 64 I) / g) * g of its 64 rows per prototype row reaching it;
diagonal tiles their lower part (rows x (rows + 8))."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import problem as P  # noqa: E402


def prefix_widths(cfg):
    qp = P.build_dense_qp(bench.build_problem(cfg))
    J = qp.J
    m, n = J.shape
    nz = J != 0
    hi = np.where(nz.any(1), n - np.argmax(nz[:, ::-1], axis=1), 0)
    first = np.argmax(nz, 1)
    sgn = np.sign(J[np.arange(m), first])
    sgn[sgn == 0] = 1
    Jn = np.ascontiguousarray(J * sgn[:, None] + 0.0)  # + 0.0: no negative zeros
    _, idx = np.unique(Jn.view(np.void(Jn.dtype.itemsize * n)), return_index=True)
    cnt = nz[idx].sum(1)
    return np.sort(hi[idx][cnt > 1]), n


h, n = prefix_widths(sys.argv[1] if len(sys.argv) > 1 else "c3")
alg = (h * (h + 1.0)).sum()
T = 64
nt = (n + T - 1) // T
print(f"{len(h)} SYRK prototype rows, {alg / 1e9:.3f} GFLOP algorithmic")
for g in (64, 32, 16, 8):
    ex = 0.0
    for I in range(nt):
        r = np.minimum(np.ceil((h[h > T * I] - T * I) / g) * g, T)
        ex += (r * (r + 8)).sum() + I * (2 * r * T).sum()  # diagonal tile + I off-diagonal ones
    print(f"granularity {g:2d}: executed / algorithmic {ex / alg:.3f}")
