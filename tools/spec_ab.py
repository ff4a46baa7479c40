"""A/B of the per-context option "speculate" (tools only): the same QP in two contexts, solves
alternating between them, device time per solve from the solve's own CUDA events.
  python tools/spec_ab.py [c2|c3] [solves]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2209_13049_b200 import ipm, problem as P  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    qp = P.build_dense_qp(bench.build_problem(cfg))
    ctx = {}
    for spec in (1, 0):
        dq = ipm.DeviceQp(qp)
        dq.set_option("speculate", spec)
        ctx[spec] = dq
    t = {1: [], 0: []}
    for i in range(k + 3):
        for spec in (1, 0):
            r = ipm.solve_loaded(ctx[spec], qp, ipm.IpmOptions())
            if i >= 3:
                t[spec].append(r.device_seconds * 1e3)
    for spec in (1, 0):
        print(f"{cfg} speculate={spec}: median {statistics.median(t[spec]):.3f} ms, "
              f"min {min(t[spec]):.3f} ms, iterations {r.iter}")
    for dq in ctx.values():
        dq.close()


if __name__ == "__main__":
    main()
