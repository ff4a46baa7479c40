"""for a QP built on the device, the SYRK prototypes are read from the
Markov table of B-responses (csrc/markov.cu) and P is never stored. State row (t, i) of J is
[G_{t-1} .. G_0] row i (G_k = A_K^k B, proj/src/reduction.cpp:43-60, rows :182-251), input
and mixed rows add their own-stage block: every row is a window of the table. Every product through the table must equal the dense algebra, and the
solve must take the reference's decisions (the oracle) exactly as the materialised path does."""
import numpy as np
import pytest

from _cmpc_helpers import lq_from_oracle, oracle_qp, rel
from paper_2209_13049_b200 import _lib, ipm, problem as P
from test_gpu_builder import random_arrays
from test_gpu_parity import assert_parity

pytestmark = pytest.mark.gpu


def _built(data, markov: bool):
    return ipm.DeviceQp.from_problem(data, options={"markov": 2 if markov else 0})


def _products(dq, qp, seed):
    """r1, r3 of the residual pass (J v, J' lambda) and the condensed M (P' diag P) against
    the host-built dense QP"""
    L = _lib.lib()
    rng = np.random.default_rng(seed)
    n, m = dq.n, dq.m
    v, lam = rng.uniform(-1, 1, n), rng.uniform(-1, 1, m)
    s, z = rng.uniform(0.5, 2, m), rng.uniform(0.5, 2, m)
    _lib.check(L.cmpc_set_state(dq.h, _lib.ptr(v), _lib.ptr(s), _lib.ptr(lam), _lib.ptr(z), 0.1))
    r1, r2, r3, kkt = np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(1)
    _lib.check(L.cmpc_compute_residuals(dq.h, _lib.ptr(r1), _lib.ptr(r2), _lib.ptr(r3), _lib.ptr(kkt)))
    assert rel(r1, qp.H @ v + qp.h + qp.J.T @ lam) <= 1e-13
    assert rel(r3, qp.J @ v - qp.d + s) <= 1e-13
    sigma = rng.uniform(0.01, 100, m)
    M = np.zeros((n, n), order="F")
    _lib.check(L.cmpc_assemble_condensed(dq.h, _lib.ptr(sigma), _lib.ptr(M)))
    assert rel(M, qp.H + qp.J.T @ (sigma[:, None] * qp.J)) <= 1e-13


@pytest.mark.parametrize("shape", [(6, 5, 6), (12, 10, 14), (20, 25, 30)])
def test_table_products_match_dense_algebra(shape):
    nx_, ny_, T = shape
    data = P.heat2d_problem(nx_, ny_, T=T)
    qp = P.build_dense_qp(data)
    dq = _built(data, True)
    info = dq.info()
    assert info["markov"], info
    ref = _built(data, False)
    assert not ref.info()["markov"]
    # the table replaces P: far fewer stored bytes than the materialised prototypes
    assert info["stored_bytes"] * 4 < ref.info()["stored_bytes"]
    assert info["syrk_flops"] == ref.info()["syrk_flops"]  # same algorithmic work
    _products(dq, qp, 1)
    dq.close()
    ref.close()


@pytest.mark.parametrize("case", [(31, 6, 2, 7, False), (32, 9, 3, 12, True), (33, 4, 1, 20, False)])
def test_table_solve_matches_the_oracle(O, case):
    """random LQ problems without feedback or mixed rows (state rows + input singletons),
    some bounds infinite (those states stay out of the table)"""
    seed, nx, nu, T, S = case
    arrs = random_arrays(seed, nx, nu, 0, T, K=False, S=S)
    op = O.problem_from_arrays(**arrs)
    data = lq_from_oracle(op)
    qp = P.build_dense_qp(data)
    o = O.solve(oracle_qp(O, qp))
    out = {}
    for mk in (True, False):
        dq = _built(data, mk)
        assert dq.info()["markov"] == mk
        log = []
        r = ipm.solve_loaded(dq, None, ipm.IpmOptions(log=log.append))
        assert_parity(r, o, log)
        out[mk] = r
        dq.close()
    assert rel(out[True].v, out[False].v) <= 1e-10


def test_plate_solve_matches_the_materialised_path(O):
    data = P.heat2d_problem(12, 10, T=14)
    qp = P.build_dense_qp(data)
    o = O.solve(oracle_qp(O, qp))
    logs = {}
    for mk in (True, False):
        dq = _built(data, mk)
        log = []
        r = ipm.solve_loaded(dq, None, ipm.IpmOptions(log=log.append))
        assert_parity(r, o, log)
        logs[mk] = (r, log)
        dq.close()
    a, b = logs[True][0], logs[False][0]
    assert a.iter == b.iter and rel(a.v, b.v) <= 1e-10
    assert rel(a.solution.x, b.solution.x) <= 1e-10


@pytest.mark.parametrize("case", [(41, 5, 2, 0, 6, True, False), (42, 6, 2, 3, 7, False, True),
                                  (43, 4, 3, 2, 9, True, True), (44, 9, 2, 4, 12, True, False)])
def test_table_covers_feedback_and_mixed_rows(O, case):
    """with feedback K the input rows are [(K G)_{t-1} .. (K G)_0, e_i], mixed rows
    [((E + F K) G)_{t-1} .. , F]: windows of the same table with the own-stage block last"""
    seed, nx, nu, nc, T, K, S = case
    arrs = random_arrays(seed, nx, nu, nc, T, K=K, S=S)
    data = lq_from_oracle(O.problem_from_arrays(**arrs))
    qp = P.build_dense_qp(data)
    out = {}
    for mk in (True, False):
        dq = _built(data, mk)
        assert dq.info()["markov"] == mk
        _products(dq, qp, seed)
        log = []
        out[mk] = (ipm.solve_loaded(dq, None, ipm.IpmOptions(log=log.append)), log)
        dq.close()
    (a, la), (b, lb) = out[True], out[False]
    o = O.solve(oracle_qp(O, qp))
    assert_parity(a, o, la)
    # (the materialised built path of case 1 takes trial 1 instead of 0 in its converged
    # 11th iteration, inside the line search's roundoff band: a summation-order effect; its
    # iterates stay at 1e-16 of the oracle's)
    assert b.status.name == o.status and b.iter == o.iter and rel(b.v, o.v) <= 1e-8


def test_table_context_clones_and_refuses_batch_mode():
    data = P.heat2d_problem(8, 6, T=8)
    dq = _built(data, True)
    a = dq.solve()
    L = _lib.lib()
    import ctypes as C
    h2 = C.c_void_p()
    _lib.check(L.cmpc_ctx_clone(dq.h, C.byref(h2)))
    lay = (C.c_int64 * 4)()
    L.cmpc_qp_layout(h2, lay)
    assert lay[0] == 1
    bh = C.c_void_p()
    assert L.cmpc_batch_create(dq.h, 4, C.byref(bh)) != 0  # batch mode needs P
    L.cmpc_ctx_destroy(h2)
    b = dq.solve()
    assert a.iter == b.iter and np.array_equal(a.v, b.v)
    dq.close()


@pytest.mark.parametrize("case", [(51, 3, 1, 1), (52, 4, 1, 9), (53, 7, 3, 2), (54, 40, 2, 5), (55, 2, 4, 33)])
def test_table_edge_shapes(O, case):
    """one stage, one input, more inputs than states, 40 states in two chunks per stage, long
    horizons: products against dense algebra and the oracle's decisions"""
    seed, nx, nu, T = case
    arrs = random_arrays(seed, nx, nu, 0, T, K=False, S=False, inf_frac=0.3)
    data = lq_from_oracle(O.problem_from_arrays(**arrs))
    qp = P.build_dense_qp(data)
    out = {}
    for mk in (True, False):
        dq = _built(data, mk)
        if mk and not dq.info()["markov"]:  # every state unbounded: nothing for the table
            assert not np.isfinite(arrs["xl"]).any() and not np.isfinite(arrs["xu"]).any()
        _products(dq, qp, seed)
        log = []
        out[mk] = (ipm.solve_loaded(dq, None, ipm.IpmOptions(log=log.append)), log)
        dq.close()
    (a, la), (b, lb) = out[True], out[False]
    # the table changes no decision of the device loop ...
    assert a.status == b.status and a.iter == b.iter
    assert [(x.mu, x.delta, x.trial) for x in la] == [(x.mu, x.delta, x.trial) for x in lb]
    # ... and the solve is the reference's (case 4 ends in the line search's roundoff band,
    # where the accepted trial of the last iteration is decided by the last bits of phi: the
    # device loop takes trial 0 there with the table, with P and with the dense J alike)
    o = O.solve(oracle_qp(O, qp))
    assert a.status.name == o.status and a.iter == o.iter
    assert rel(a.v, o.v) <= 1e-8 and abs(a.objective - o.objective) <= 1e-8 * (1 + abs(o.objective))
