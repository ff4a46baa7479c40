"""Concurrency determinism probe: K host threads solve the same QP on K cloned contexts at the
same time, recording per-iteration hashes of every inspected vector; prints the first quantity
and iteration at which any thread differs from thread 0."""
import hashlib
import sys
import threading

import numpy as np

sys.path.insert(0, ".")
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 15
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
data = P.heat2d_problem(20, 25, T=30)
qp = P.build_dense_qp(data)
root = ipm.device_qp(qp)
ctxs = [root.clone() for _ in range(K)]


def h(a):
    return hashlib.md5(np.ascontiguousarray(a).tobytes()).hexdigest()[:10]


for rep in range(reps):
    recs = [[] for _ in range(K)]

    def run(i):
        def insp(it):
            recs[i].append(dict(v=h(it.state.v), s=h(it.state.s), lam=h(it.state.lambda_), z=h(it.state.z),
                                r1=h(it.residuals.r1), r2=h(it.residuals.r2), r3=h(it.residuals.r3),
                                pv=h(it.dirs.pv), ps=h(it.dirs.ps), pl=h(it.dirs.plambda), pz=h(it.dirs.pz),
                                delta=it.delta))
        if len(sys.argv) > 3 and sys.argv[3] == "log":
            def lg(rec):
                recs[i].append(dict(kkt=rec.kkt_error if hasattr(rec, "kkt_error") else rec[4], full=repr(rec)))
            r = ipm.solve_loaded(ctxs[i], qp, ipm.IpmOptions(log=lg))
            recs[i].append(dict(v=h(r.v)))
        elif len(sys.argv) > 3 and sys.argv[3] == "final":
            r = ipm.solve_loaded(ctxs[i], qp, ipm.IpmOptions())
            recs[i].append(dict(v=h(r.v), s=h(r.s), lam=h(r.lambda_), z=h(r.z), it=r.iter))
        else:
            ipm.solve_loaded(ctxs[i], qp, ipm.IpmOptions(inspect=insp))

    ths = [threading.Thread(target=run, args=(i,)) for i in range(K)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    bad = None
    for i in range(1, K):
        for it, (a, b) in enumerate(zip(recs[0], recs[i])):
            diff = [k for k in a if a[k] != b[k]]
            if diff:
                if bad is None or it < bad[1]:
                    bad = (i, it, diff)
                break
    print(f"rep {rep}: iters {[len(r) for r in recs][:4]}...", "clean" if bad is None else f"thread {bad[0]} differs at iteration {bad[1]} in {bad[2]}", flush=True)
    if bad is not None and "full" in recs[0][0]:
        print("   t0:", recs[0][bad[1]]["full"])
        print("   t%d:" % bad[0], recs[bad[0]][bad[1]]["full"])
