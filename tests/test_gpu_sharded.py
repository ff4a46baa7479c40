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
