"""Condensation determinism under concurrency: K threads call cmpc_assemble_condensed with the
same sigma on cloned contexts; report differing entries of M vs a single-threaded reference
(which tile rows/cols, and whether they lie in thin / diagonal regions)."""
import sys
import threading

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import _lib, ipm, problem as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 15
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
qp = P.build_dense_qp(bench.build_problem(cfg))
root = ipm.device_qp(qp)
ctxs = [root.clone() for _ in range(K)]
sigma = np.random.default_rng(0).uniform(0.1, 10.0, qp.m)
L = _lib.lib()


def cond(ctx, out):
    _lib.check(L.cmpc_assemble_condensed(ctx.h, _lib.ptr(sigma), _lib.ptr(out)))


ref = np.zeros((qp.n, qp.n), order="F")
cond(ctxs[0], ref)
bad = 0
for rep in range(reps):
    outs = [np.zeros((qp.n, qp.n), order="F") for _ in range(K)]

    def run(i):
        for _ in range(5):
            cond(ctxs[i], outs[i])

    ths = [threading.Thread(target=run, args=(i,)) for i in range(K)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for i, o in enumerate(outs):
        d = np.argwhere(o != ref)
        if len(d):
            bad += 1
            rows, cols = d[:, 0], d[:, 1]
            low = rows >= cols
            print(f"rep {rep} ctx {i}: {len(d)} entries differ (lower {low.sum()}), max rel "
                  f"{np.abs((o - ref)[o != ref]).max() / np.abs(ref).max():.2e}; tiles "
                  f"{sorted(set(zip((rows[low] // 64).tolist(), (cols[low] // 64).tolist())))[:8]} "
                  f"row%64 {sorted(set((rows[low] % 64).tolist()))[:12]} col%64 {sorted(set((cols[low] % 64).tolist()))[:12]}", flush=True)
print("differing outputs:", bad, "of", reps * K)
