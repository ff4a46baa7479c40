"""Concurrent solves on cloned contexts (the batch mode's situation: kernels of many contexts
share the SMs) give bitwise the single-context result. Regression for a shared-memory race in
the SYRK pipeline: the consumers' reads of a stage were not ordered before the producer's next
TMA write into it (missing fence.proxy.async), which showed up only under SM contention."""
import threading

import numpy as np
import pytest

from paper_2209_13049_b200 import _lib, ipm, problem as P

pytestmark = pytest.mark.gpu


def test_concurrent_solves_are_bitwise_identical():
    qp = P.build_dense_qp(P.heat2d_problem(20, 25, T=30))
    ref = ipm.solve(qp)
    root = ipm.device_qp(qp)
    K = 12
    ctxs = [root.clone() for _ in range(K)]
    for _ in range(3):
        outs = [None] * K

        def run(i):
            outs[i] = ipm.solve_loaded(ctxs[i], qp, ipm.IpmOptions())

        ths = [threading.Thread(target=run, args=(i,)) for i in range(K)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        for r in outs:
            assert r.iter == ref.iter
            assert np.array_equal(r.v, ref.v) and np.array_equal(r.z, ref.z)
    for c in ctxs:
        c.close()


def test_concurrent_condensations_are_bitwise_identical():
    qp = P.build_dense_qp(P.heat2d_problem(30, 30, T=40))
    sigma = np.random.default_rng(3).uniform(0.1, 10.0, qp.m)
    root = ipm.device_qp(qp)
    L = _lib.lib()
    ref = np.zeros((qp.n, qp.n), order="F")
    _lib.check(L.cmpc_assemble_condensed(root.h, _lib.ptr(sigma), _lib.ptr(ref)))
    K = 12
    ctxs = [root.clone() for _ in range(K)]
    outs = [np.zeros((qp.n, qp.n), order="F") for _ in range(K)]

    def run(i):
        for _ in range(4):
            _lib.check(L.cmpc_assemble_condensed(ctxs[i].h, _lib.ptr(sigma), _lib.ptr(outs[i])))

    ths = [threading.Thread(target=run, args=(i,)) for i in range(K)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for o in outs:
        assert np.array_equal(o, ref)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("shape", [(20, 25, 30), (12, 10, 40)])
def test_concurrent_cholesky_paths_are_bitwise_identical(shape):
    # the dataflow Cholesky (chol.cu) under SM contention: the spine's named barriers and
    # mbarrier signals, the pre-diagonal / panel tasks' flags, the spine backward solve
    # (n = 150) and the per-block backward tasks (n = 320) must give bitwise the same factor
    # and solve whatever the interleaving (compute-sanitizer is not available on this pool;
    # this is the race check)
    nx, ny, T = shape
    qp = P.build_dense_qp(P.heat2d_problem(nx, ny, T=T))
    ref = ipm.solve(qp)
    root = ipm.device_qp(qp)
    K = 10
    ctxs = [root.clone() for _ in range(K)]
    for _ in range(2):
        outs = [None] * K

        def run(i):
            outs[i] = ipm.solve_loaded(ctxs[i], qp, ipm.IpmOptions())

        ths = [threading.Thread(target=run, args=(i,)) for i in range(K)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        for r in outs:
            assert r.iter == ref.iter
            assert np.array_equal(r.v, ref.v) and np.array_equal(r.s, ref.s) and np.array_equal(r.z, ref.z)
    for c in ctxs:
        c.close()


def test_lockstep_batch_is_bitwise_reproducible():
    from paper_2209_13049_b200 import batch
    data = P.heat2d_problem(20, 25, T=30)
    base = P.build_dense_qp(data)
    xbs = P.batch_initial_states(500, 64, seed=9)
    bs = ipm.BatchSolver(base, 64)
    for i, xb in enumerate(xbs):
        bs.set_instance(i, *batch.instance_affine(base, xb))
    a = bs.solve()
    b = bs.solve()
    bs.close()
    assert np.array_equal(a.iter, b.iter) and np.array_equal(a.v, b.v)
    assert all(s == "converged" for s in a.status)
