import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2209_13049_b200 import ipm, problem as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(0)
G = rng.uniform(-1, 1, (n, n))
qp = P.DenseQp(H=G.T @ G + n * np.eye(n), h=np.zeros(n), h0=0.0, J=np.zeros((0, n)), d=np.zeros(0))
dq = ipm.device_qp(qp)
ipm.assemble_condensed(qp, np.zeros(0))
for ph in ["cholesky", "chol_solve", "chol_fused"]:
    print(n, ph, dq.time_phase(ph, 20) * 1e3, "us")
