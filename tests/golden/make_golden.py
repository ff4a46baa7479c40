"""Generate tests/golden/oracle_golden.json: per-case iteration logs and solutions of the
oracle (the CPU restatement of the reference solver, pinned by tests/test_oracle_kat.py).

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from _cmpc_helpers import lq_from_oracle  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2209_13049_b200 import problem as P  # noqa: E402


def cases():
    """name -> product DenseQp (identical arrays go to the oracle and to the device)."""
    out = {}
    out["toy"] = P.DenseQp(H=[[4.0]], h=[2.0], h0=0.0, J=[[-1.0]], d=[0.0])
    out["unconstrained"] = P.build_dense_qp(P.LqProblemData.basic(
        np.eye(1), np.eye(1), np.eye(1), np.eye(1), np.eye(1), np.ones(1), 1))
    out["heat3d_N2_T10"] = P.build_dense_qp(P.build_heat_problem(P.HeatParams(N=2, T=10)))
    for i in range(5):
        out[f"c1_random_{i}"] = P.build_dense_qp(lq_from_oracle(
            O.random_problem(O.instance_rng(42, i), fixed=(10, 2, 0, 10))))
    out["heat1d_20_T10"] = P.build_dense_qp(P.heat1d_problem(20, 10))
    out["heat2d_6x5_T8"] = P.build_dense_qp(P.heat2d_problem(6, 5, T=8, splits=([3], [3], [2], [2])))
    return out


def solve_case(qp):
    r = O.solve(O.qp_from_arrays(qp.H, qp.h, qp.h0, qp.J, qp.d))
    return {"status": r.status, "iter": r.iter, "objective": r.objective, "kkt_error": r.kkt_error,
            "v": r.v.tolist(), "s": r.s.tolist(), "lambda": r.lam.tolist(), "z": r.z.tolist(),
            "log": [list(x) for x in r.log]}


if __name__ == "__main__":
    gold = {name: solve_case(qp) for name, qp in cases().items()}
    with open(os.path.join(HERE, "oracle_golden.json"), "w") as f:
        json.dump(gold, f, indent=0)
    print({k: (v["status"], v["iter"]) for k, v in gold.items()})
