import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P
for n in [32, 64, 96, 128, 160, 256, 512]:
    rng = np.random.default_rng(0)
    G = rng.uniform(-1, 1, (n, n))
    qp = P.DenseQp(H=G.T @ G + n * np.eye(n), h=np.zeros(n), h0=0.0, J=np.zeros((0, n)), d=np.zeros(0))
    dq = ipm.device_qp(qp)
    ipm.assemble_condensed(qp, np.zeros(0))
    print(n, " ".join(f"{ph} {dq.time_phase(ph, 50) * 1e3:7.1f}" for ph in ["cholesky", "chol_fused"]), flush=True)
