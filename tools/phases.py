"""Per-phase device times (CUDA events) on a converged state, for C2/C3/C4/C5-shaped QPs."""
import sys, time
sys.path.insert(0, ".")
from paper_2209_13049_b200 import ipm, problem as P

cfgs = sys.argv[1:] or ["c2", "c3"]
for cfg in cfgs:
    if cfg == "c2":
        qp = P.build_dense_qp(P.heat1d_problem())
    elif cfg == "c3":
        qp = P.build_dense_qp(P.heat2d_problem(50, 50, T=50))
    elif cfg.startswith("c4"):
        T = int(cfg[2:] or 200)
        qp = P.build_dense_qp(P.heat2d_problem(40, 25, T=T))
    elif cfg == "c5":
        qp = P.build_dense_qp(P.heat2d_problem(20, 25, T=30))
    t = time.perf_counter()
    dq = ipm.device_qp(qp)
    t_load = time.perf_counter() - t
    info = dq.info()
    r = ipm.solve(qp)
    r = ipm.solve(qp)
    print(f"== {cfg}: n={qp.n} m={qp.m} load={t_load*1e3:.1f}ms {info}")
    print(f"   solve: {r.status.name} iter={r.iter} total={r.total_seconds*1e3:.2f}ms device={r.device_seconds*1e3:.2f}ms "
          f"syrk={r.syrk_seconds*1e3:.2f}ms chol={r.chol_seconds*1e3:.2f}ms launches={r.launches} syncs={r.syncs}")
    per = {}
    for ph in ["prepare", "condense", "condense_rhs", "cholesky", "chol_solve", "chol_fused", "residuals", "recover", "trial", "Jx", "Jty"]:
        per[ph] = dq.time_phase(ph, 20)
    for k, v in per.items():
        extra = ""
        if k in ("condense", "condense_rhs"):
            extra = f"  {info['syrk_flops'] / (v * 1e-3) / 1e12:.2f} TF/s ({100 * info['syrk_flops'] / (v * 1e-3) / 37.1e12:.1f}% of 37.1)"
        if k in ("Jx", "Jty"):
            extra = f"  {info['p_bytes'] / (v * 1e-3) / 1e9:.0f} GB/s of P"
        print(f"   {k:11s} {v * 1e3:9.1f} us{extra}")
    print(f"   per-iter estimate {1e3 * (per['prepare'] + per['condense'] + per['cholesky'] + per['chol_solve'] + per['residuals'] + per['recover'] + per['trial']):.1f} us; measured {r.device_seconds / max(r.iter, 1) * 1e6:.1f} us")
