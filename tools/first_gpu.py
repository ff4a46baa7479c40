"""Ad-hoc GPU bring-up check: device path vs the oracle on small cases, C3 timing."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2209_13049_b200 import ipm, linalg, problem as P  # noqa: E402


def lq_from_oracle(p):
    d = p.as_dict()
    T = d.pop("T")
    return P.LqProblemData(T=T, **d)


def cmp_solve(name, qp, oq=None):
    t = time.perf_counter()
    r = ipm.solve(qp, ipm.IpmOptions(log=lambda rec: logs.append(rec)))
    tg = time.perf_counter() - t
    if oq is None:
        oq = O.qp_from_arrays(qp.H, qp.h, qp.h0, qp.J, qp.d)
    t = time.perf_counter()
    o = O.solve(oq)
    to = time.perf_counter() - t
    dv = np.abs(r.v - o.v).max() / (1 + np.abs(o.v).max())
    ds = np.abs(r.s - o.s).max() / (1 + np.abs(o.s).max()) if qp.m else 0
    dz = np.abs(r.z - o.z).max() / (1 + np.abs(o.z).max()) if qp.m else 0
    print(f"{name}: gpu {r.status.name} it={r.iter} obj={r.objective:.12g} kkt={r.kkt_error:.3g} "
          f"t={tg*1e3:.1f}ms | oracle {o.status} it={o.iter} obj={o.objective:.12g} t={to*1e3:.1f}ms "
          f"| dv={dv:.2e} ds={ds:.2e} dz={dz:.2e} launches={r.launches} syncs={r.syncs}")
    if r.iter != o.iter:
        for a, b in zip(logs, o.log):
            print("   gpu", a.iter, a.mu, a.alpha, a.alpha_z, a.kkt_error, a.trial, "| ora", b)
    logs.clear()
    return r, o


logs = []
print("gram:", end=" ")
rng = np.random.default_rng(0)
for (m, n) in [(2, 2), (30, 17), (300, 130), (1000, 65)]:
    J = rng.uniform(-1, 1, (m, n))
    sig = rng.uniform(0.1, 4, m)
    G = linalg.gram_weighted(J, sig)
    ref = J.T @ (sig[:, None] * J)
    print(f"({m},{n}) {np.abs(G - ref).max() / (1 + np.abs(ref).max()):.2e}", end=" ")
print()
J = np.array([[1.0, 2.0], [3.0, 4.0]])
print("gram KAT", linalg.gram_weighted(J, [2.0, 3.0]))
for n in [1, 2, 5, 63, 64, 65, 150, 500]:
    G = rng.uniform(-1, 1, (n, n))
    M = G.T @ G + np.eye(n)
    L = linalg.make_backend("cuda").factorize(M).lower()
    b = rng.uniform(-1, 1, n)
    x = linalg.make_backend("cuda").factorize(M).solve(b)
    print(f"chol n={n} recon {np.abs(L @ L.T - M).max() / np.abs(M).max():.2e} solve {np.abs(M @ x - b).max():.2e}")
try:
    linalg.make_backend("cuda").factorize(np.array([[1.0, 0.0], [0.0, -1.0]]))
except linalg.NotPositiveDefinite as e:
    print("NPD pivot", e.pivot)

# toy
toy = P.DenseQp(H=[[4.0]], h=[2.0], h0=0.0, J=[[-1.0]], d=[0.0])
st = ipm.IpmState(np.zeros(1), np.ones(1), np.zeros(1), np.full(1, 0.3), 0.3)
print("toy residuals", ipm.compute_residuals(toy, st))
cmp_solve("toy", toy)
unc = P.build_dense_qp(P.LqProblemData.basic(np.eye(1), np.eye(1), np.eye(1), np.eye(1), np.eye(1), np.ones(1), 1))
cmp_solve("unconstrained", unc)
for N, T in [(2, 10), (4, 50)]:
    p = O.heat3d_problem(N, T)
    qp = P.build_dense_qp(lq_from_oracle(p))
    cmp_solve(f"heat3d N={N} T={T}", qp)
for i in range(10):
    p = O.random_problem(O.instance_rng(7, i))
    qp = P.build_dense_qp(lq_from_oracle(p))
    cmp_solve(f"rand{i}", qp)
for i in range(3):
    p = O.random_problem(O.instance_rng(42, i), fixed=(10, 2, 0, 10))
    qp = P.build_dense_qp(lq_from_oracle(p))
    cmp_solve(f"C1 rand{i}", qp)
qp = P.build_dense_qp(P.heat1d_problem())
O.set_threads(16)
cmp_solve("C2 heat1d", qp)
qp = P.build_dense_qp(P.heat2d_problem(10, 10, T=20))
cmp_solve("heat2d 10x10 T20", qp)
t = time.perf_counter()
qp = P.build_dense_qp(P.heat2d_problem(50, 50, T=50))
print("C3 build", time.perf_counter() - t)
t = time.perf_counter()
dq = ipm.device_qp(qp)
print("C3 upload+analyze", time.perf_counter() - t, dq.info())
for k in range(3):
    r = ipm.solve(qp, ipm.IpmOptions(log=lambda rec: logs.append(rec)))
    print(f"C3 gpu {r.status.name} it={r.iter} obj={r.objective:.12g} kkt={r.kkt_error:.3g} total={r.total_seconds*1e3:.1f}ms "
          f"device={r.device_seconds*1e3:.1f}ms linalg={r.linalg_seconds*1e3:.1f}ms launches={r.launches} syncs={r.syncs} trials={r.trials}")
    if k == 0:
        for a in logs:
            print("   ", a)
    logs.clear()
