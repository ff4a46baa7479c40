"""Staged host->device upload (csrc/upload.cpp): pageable sources above 4 MB go through pinned
slots copied by several host threads. A load of a random QP whose J spans several 8 MB slots
(and ends in a partial one) must arrive bit-exact: H, h, d read back, J through r3 = J v - d + s."""
import numpy as np
import pytest

from _cmpc_helpers import rel
from paper_2209_13049_b200 import _lib, ipm, problem as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m", [(120, 9001), (300, 13_337), (64, 65_537)])
def test_staged_upload_is_exact(n, m):
    r = np.random.default_rng(n + m)
    J = np.asfortranarray(r.standard_normal((m, n)))          # 8.6 / 32 / 33.5 MB, pageable
    M = r.standard_normal((n, n))
    H = np.asfortranarray(M @ M.T + n * np.eye(n))
    qp = P.DenseQp(H=H, h=r.standard_normal(n), h0=0.5, J=J, d=r.uniform(1, 2, m))
    dq = ipm.DeviceQp(qp)
    try:
        H2, h2, h02, d2 = dq.get_qp()
        assert np.array_equal(H2, H) and np.array_equal(h2, qp.h) and np.array_equal(d2, qp.d)
        assert h02 == 0.5
        L = _lib.lib()
        v = r.standard_normal(n)
        zm, om = np.zeros(m), np.ones(m)
        _lib.check(L.cmpc_set_state(dq.h, _lib.ptr(v), _lib.ptr(zm), _lib.ptr(zm), _lib.ptr(om), 1.0))
        r1, r2, r3, kkt = np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(1)
        _lib.check(L.cmpc_compute_residuals(dq.h, _lib.ptr(r1), _lib.ptr(r2), _lib.ptr(r3), _lib.ptr(kkt)))
        assert rel(r3 + qp.d, J @ v) <= 1e-13
    finally:
        dq.close()
