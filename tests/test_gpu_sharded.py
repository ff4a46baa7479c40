"""Row-sharded solve on the device.

Only one GPU is available to the tests, so the NCCL path runs with a communicator of one
rank: every collective of the sharded iteration (condensed-matrix and right-hand-side sums,
residual maxima and sums, step-length minima, merit sums) is issued and must leave the
solve unchanged. The partition algebra is checked on the device without NCCL: the shards'
condensed matrices and J' y products add up to the whole QP's. The multi-rank reduction
plan is exercised on CPU with gloo in tests/test_shard_protocol.py."""
import numpy as np
import pytest

from _cmpc_helpers import rel
from paper_2209_13049_b200 import ipm, problem as P

pytestmark = pytest.mark.gpu


def heat_qp(nx=12, ny=10, T=14):
    return P.build_dense_qp(P.heat2d_problem(nx, ny, T=T, splits=([6], [6], [5], [5])))


@pytest.mark.parametrize("T", [8, 14])
def test_one_rank_communicator_leaves_the_solve_unchanged(T):
    qp = heat_qp(T=T)
    ref = ipm.solve(qp)
    sh = ipm.ShardedQp(qp, np.arange(qp.m), ipm.nccl_unique_id(), 1, 0)
    try:
        log = []
        r = sh.solve(ipm.IpmOptions(log=log.append))
    finally:
        sh.close()
    assert r.status.name == ref.status.name == "converged"
    assert r.iter == ref.iter
    assert abs(r.objective - ref.objective) <= 1e-12 * (1 + abs(ref.objective))
    assert rel(r.v, ref.v) <= 1e-12
    assert rel(r.s, ref.s) <= 1e-12 and rel(r.z, ref.z) <= 1e-12
    assert len(log) == r.iter


def test_one_rank_communicator_on_config2_shape():
    qp = P.build_dense_qp(P.heat1d_problem(200, 50))
    ref = ipm.solve(qp)
    sh = ipm.ShardedQp(qp, np.arange(qp.m), ipm.nccl_unique_id(), 1, 0)
    try:
        r = sh.solve()
    finally:
        sh.close()
    assert r.iter == ref.iter and r.status.name == ref.status.name
    assert rel(r.v, ref.v) <= 1e-12


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_shard_condensed_matrices_sum_to_the_whole(nranks):
    qp = heat_qp()
    rng = np.random.default_rng(nranks)
    sigma = rng.uniform(0.1, 3.0, qp.m)
    whole = ipm.assemble_condensed(qp, sigma)
    parts = P.shard_rows(qp, nranks)
    assert sorted(np.concatenate(parts).tolist()) == list(range(qp.m))
    acc = np.zeros_like(whole)
    for rows in parts:
        sq = P.shard_qp(qp, rows)
        acc += ipm.assemble_condensed(sq, sigma[rows]) - qp.H  # each shard adds H once
    acc += qp.H
    assert np.abs(acc - whole).max() <= 1e-11 * (1 + np.abs(whole).max())


def test_shard_residuals_partition_the_rows():
    qp = heat_qp()
    rng = np.random.default_rng(3)
    st = ipm.IpmState(rng.uniform(-1, 1, qp.n), rng.uniform(0.5, 2, qp.m), rng.uniform(0.1, 1, qp.m),
                      rng.uniform(0.1, 1, qp.m), 0.3)
    whole = ipm.compute_residuals(qp, st)
    r1_jtl = np.zeros(qp.n)
    for rows in P.shard_rows(qp, 3):
        sq = P.shard_qp(qp, rows)
        part = ipm.compute_residuals(sq, ipm.IpmState(st.v, st.s[rows], st.lambda_[rows], st.z[rows], st.mu))
        np.testing.assert_array_equal(part.r2, whole.r2[rows])
        np.testing.assert_array_equal(part.r3, whole.r3[rows])
        r1_jtl += part.r1 - (qp.H @ st.v + qp.h)  # J_g' lambda_g
    assert np.abs(qp.H @ st.v + qp.h + r1_jtl - whole.r1).max() <= 1e-10 * (1 + np.abs(whole.r1).max())


@pytest.mark.timeout(300)
@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_sharded_loop_at_several_ranks_matches_the_unsharded_solve_and_oracle(O, nranks):
    # the real sharded C++ loop (ipm_host.cpp) and kernels with N ranks: an in-process
    # loopback communicator stands in for NCCL over N contexts on the one GPU, one host
    # thread per rank (ipm.cpp:183-251 on every rank, the row sums combined in rank order)
    from _cmpc_helpers import oracle_qp
    qp = heat_qp(T=14)
    ref_log = []
    ref = ipm.solve(qp, ipm.IpmOptions(log=ref_log.append))
    sh = ipm.LoopbackShards(qp, nranks)
    try:
        assert sum(len(r) for r in sh.rows) == qp.m and len(sh.rows) == nranks
        outs = sh.solve()
    finally:
        sh.close()
    o = O.solve(oracle_qp(O, qp))
    for r in outs:  # identical decisions on every rank: same iterations, same iterate v
        assert r.status.name == ref.status.name == o.status == "converged"
        assert r.iter == ref.iter == o.iter
        assert np.array_equal(r.v, outs[0].v)
        assert r.objective == outs[0].objective and r.kkt_error == outs[0].kkt_error
        assert rel(r.v, ref.v) <= 1e-10 and rel(r.v, o.v) <= 1e-8
        assert abs(r.objective - o.objective) <= 1e-8 * (1 + abs(o.objective))
        assert abs(r.kkt_error - o.kkt_error) <= 1e-9 * (1 + abs(o.kkt_error))
    # each rank holds its rows' slacks and duals: together the unsharded ones
    s_all = np.zeros(qp.m)
    for rows, r in zip(sh.rows, outs):
        s_all[rows] = r.s
    assert rel(s_all, o.s) <= 1e-8


@pytest.mark.timeout(600)
def test_sharded_loop_on_config2_shape_at_two_ranks():
    qp = P.build_dense_qp(P.heat1d_problem(200, 50))
    ref = ipm.solve(qp)
    sh = ipm.LoopbackShards(qp, 2)
    try:
        outs = sh.solve()
    finally:
        sh.close()
    for r in outs:
        assert r.iter == ref.iter and r.status.name == ref.status.name
        assert rel(r.v, ref.v) <= 1e-10
