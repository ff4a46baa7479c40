"""Device linear algebra vs the reference's test_dense_linalg.cpp cases and numpy fp64."""
import numpy as np
import pytest

from paper_2209_13049_b200 import linalg
from paper_2209_13049_b200._lib import DimensionError

pytestmark = pytest.mark.gpu


def spd(rng, n, shift=0.5):
    m = rng.uniform(-1, 1, (n, n))
    return m.T @ m + shift * np.eye(n)


def test_two_by_two_factor_kat():  # test_dense_linalg.cpp:33-44
    L = linalg.make_backend("cuda").factorize(np.array([[4.0, 2.0], [2.0, 3.0]])).lower()
    assert L[0, 0] == pytest.approx(2.0, rel=1e-15)
    assert L[1, 0] == pytest.approx(1.0, rel=1e-15)
    assert L[1, 1] == pytest.approx(np.sqrt(2.0), rel=1e-15)
    assert L[0, 1] == 0.0


def test_one_by_one_is_the_square_root():  # :46-50
    f = linalg.make_backend("cuda").factorize(np.array([[4.0]]))
    assert f.lower()[0, 0] == 2.0 and f.dim() == 1


def test_failure_reports_first_nonpositive_pivot():  # :52-70
    be = linalg.make_backend("cuda")
    with pytest.raises(linalg.NotPositiveDefinite) as e:
        be.factorize(np.array([[1.0, 0.0], [0.0, -1.0]]))
    assert e.value.pivot == 1
    with pytest.raises(linalg.NotPositiveDefinite) as e:
        be.factorize(np.array([[-1.0]]))
    assert e.value.pivot == 0
    # failure deep inside a later panel, and a NaN pivot
    rng = np.random.default_rng(5)
    M = spd(rng, 150)
    M[137, 137] = -50.0
    with pytest.raises(linalg.NotPositiveDefinite) as e:
        be.factorize(M)
    assert e.value.pivot == 137
    M = spd(rng, 70)
    M[3, 3] = np.nan
    with pytest.raises(linalg.NotPositiveDefinite) as e:
        be.factorize(M)
    assert e.value.pivot == 3


def test_cholesky_factorize_rejects_asymmetric_input():  # :72-78
    be = linalg.make_backend("cuda")
    with pytest.raises(ValueError):
        linalg.cholesky_factorize(be, np.array([[1.0, 0.5], [0.0, 1.0]]))
    with pytest.raises(DimensionError):
        linalg.cholesky_factorize(be, np.zeros((2, 3)))


@pytest.mark.parametrize("n", [1, 2, 5, 17, 40, 63, 64, 65, 127, 150, 200, 333, 500, 1000, 2000])
def test_factor_reconstructs_and_solves(n):  # :80-116, :118-132
    rng = np.random.default_rng(n)
    M = spd(rng, n, 1.0)
    f = linalg.make_backend("cuda").factorize(M)
    L = f.lower()
    assert np.abs(np.triu(L, 1)).max(initial=0.0) == 0.0
    assert np.abs(L @ L.T - M).max() <= 1e-12 * n * np.abs(M).max()
    b = rng.uniform(-1, 1, n)
    x = f.solve(b)
    assert np.abs(M @ x - b).max() <= 1e-10 * (1 + np.abs(b).max()) * max(1, n / 100)
    # numpy's LAPACK factor agrees
    Lref = np.linalg.cholesky(M)
    assert np.abs(L - Lref).max() <= 1e-9 * (1 + np.abs(Lref).max())


def test_solve_checks_rhs_length_and_is_bitwise_repeatable():  # :103-106, :146-154
    rng = np.random.default_rng(43)
    f = linalg.make_backend("cuda").factorize(spd(rng, 12))
    with pytest.raises(DimensionError):
        f.solve(np.zeros(11))
    b = rng.uniform(-1, 1, 12)
    assert np.array_equal(f.solve(b), f.solve(b))


def test_gram_weighted_kat():  # :171-182
    G = linalg.gram_weighted(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([2.0, 3.0]))
    assert G[0, 0] == pytest.approx(29.0, rel=1e-15)
    assert G[0, 1] == pytest.approx(40.0, rel=1e-15)
    assert G[1, 0] == G[0, 1]
    assert G[1, 1] == pytest.approx(56.0, rel=1e-15)


@pytest.mark.parametrize("seed", range(20))
def test_gram_weighted_matches_naive_triple_product(seed):  # :184-202
    rng = np.random.default_rng(53 + seed)
    m, n = rng.integers(1, 31, size=2)
    J = rng.uniform(-1, 1, (m, n))
    s = rng.uniform(0.1, 4.0, m)
    ref = J.T @ (s[:, None] * J)
    G = linalg.gram_weighted(J, s)
    assert np.abs(G - ref).max() <= 1e-12 * (1 + np.abs(ref).max())
    assert np.array_equal(G, G.T)


@pytest.mark.parametrize("m,n", [(4000, 65), (3000, 200), (20000, 129), (5000, 500)])
def test_gram_weighted_large_tall(m, n):
    rng = np.random.default_rng(m + n)
    J = rng.uniform(-1, 1, (m, n))
    s = rng.uniform(0.01, 10.0, m)
    ref = J.T @ (s[:, None] * J)
    G = linalg.gram_weighted(J, s)
    assert np.abs(G - ref).max() <= 1e-12 * (1 + np.abs(ref).max())


def test_gram_weighted_checks_sigma_length():  # :204-206
    with pytest.raises(DimensionError):
        linalg.gram_weighted(np.eye(2), np.zeros(3))


def test_backend_conformance_acceptance():  # acceptance.cpp:255-296 (criterion 8)
    rng = np.random.default_rng(8080)
    worst_recon = worst_solve = worst_gram = 0.0
    for _ in range(50):
        n = int(rng.integers(1, 101))
        G = rng.uniform(-1, 1, (n, n))
        M = G.T @ G + 0.1 * np.eye(n)
        b = rng.uniform(-1, 1, n)
        f = linalg.make_backend("cuda").factorize(M)
        L = f.lower()
        worst_recon = max(worst_recon, np.abs(L @ L.T - M).max() / (1e-12 * n * np.abs(M).max()))
        x = f.solve(b)
        worst_solve = max(worst_solve, np.abs(M @ x - b).max() / (1e-9 * n * (1 + np.abs(b).max())))
        m = min(n, 12)
        J = G[:m]
        s = 0.01 + np.abs(rng.uniform(-1, 1, m))
        naive = J.T @ np.diag(s) @ J
        gram = linalg.gram_weighted(J, s)
        worst_gram = max(worst_gram, np.abs(gram - naive).max() / (1 + np.abs(naive).max()))
    assert worst_recon <= 1.0 and worst_solve <= 1.0 and worst_gram <= 1e-13
