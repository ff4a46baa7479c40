"""Markov table vs materialised P on a device-built QP (tools only): per-solve device time,
the SYRK kernel's share and DMMA fraction, the P x pass, stored bytes.
  python tools/markov_ab.py [c3|c4|c5] [T for c4] [solves]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402

PEAK_FP64 = 37.1e12  # profiles/r01_fp64_peak_probe.txt


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    T4 = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    data = {"c3": lambda: P.heat2d_problem(50, 50, T=50), "c4": lambda: P.heat2d_problem(40, 25, T=T4),
            "c5": lambda: P.heat2d_problem(20, 25, T=30)}[cfg]()
    res = {}
    order = (0, 1) if len(sys.argv) > 4 and sys.argv[4] == "rev" else (1, 0)
    for mk in order:
        dq = ipm.DeviceQp.from_problem(data, options={"markov": 2 * mk})
        info = dq.info()
        ts, syrk, cond, it = [], [], 0, 0
        for i in range(k + 2):
            r = dq.solve()
            if i >= 2:
                ts.append(r.device_seconds * 1e3)
                syrk.append(r.syrk_kernel_seconds / max(1, r.condensations))
            it = r.iter
        jx = dq.time_phase("Jx", 20)
        cd = dq.time_phase("condense", 10)
        ph = {name: dq.time_phase(name, 10) * 1e3 for name in ("condense_rhs", "chol_fused", "residuals",
                                                               "recover", "trial", "Jty", "prepare")}
        print("   phases (us): " + ", ".join(f"{k} {v:.1f}" for k, v in ph.items()), flush=True)
        syrk_us = statistics.median(syrk) * 1e6
        frac = info["syrk_flops"] / (syrk_us * 1e-6) / PEAK_FP64
        print(f"{cfg} markov={mk}: {statistics.median(ts):.3f} ms/solve ({it} it), syrk {syrk_us:.1f} us "
              f"(frac {frac:.3f}), condense phase {cd * 1e3:.1f} us, Jx {jx * 1e3:.1f} us, "
              f"stored {info['stored_bytes'] / 1e6:.1f} MB (table rows {info['markov_rows']})", flush=True)
        res[mk] = r
        dq.close()
    import numpy as np
    a, b = res[1], res[0]
    print(f"  same iterations: {a.iter == b.iter}, max |dv|/|v| {np.abs(a.v - b.v).max() / np.abs(b.v).max():.2e}")


if __name__ == "__main__":
    main()
