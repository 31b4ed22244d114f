"""Pins of oracle/krylov.py (the paper's Krylov workload) against
dense algebra built independently with numpy.kron and a dense SVD."""
import numpy as np
import pytest

from oracle import krylov, rounding, tt


def _kron_laplacian(d, n):
    """sum_k I (x) .. (x) L (x) .. (x) I, built with numpy.kron (independent of the TT form)."""
    L = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    I = np.eye(n)
    tot = np.zeros((n ** d, n ** d))
    for k in range(d):
        M = np.ones((1, 1))
        for j in range(d):
            M = np.kron(M, L if j == k else I)
        tot += M
    return tot


@pytest.mark.parametrize("d,n", [(2, 4), (3, 3), (4, 3)])
def test_laplacian_ttm_dense(d, n):
    A = krylov.laplacian_ttm(d, n)
    assert [c.shape[0] for c in A] == [1] + [2] * (d - 1)
    np.testing.assert_allclose(krylov.dense_operator(A), _kron_laplacian(d, n), atol=1e-13)


@pytest.mark.parametrize("d,n", [(2, 5), (3, 4)])
def test_matvec_dense(d, n):
    rng = np.random.Generator(np.random.PCG64(3))
    r = [1] + [3] * (d - 1) + [1]
    x = [rng.standard_normal((r[k], n, r[k + 1])) for k in range(d)]
    y = krylov.matvec(krylov.laplacian_ttm(d, n), x)
    assert tt.ranks(y) == [1] + [6] * (d - 1) + [1]
    np.testing.assert_allclose(tt.densify(y), _kron_laplacian(d, n) @ tt.densify(x), atol=1e-11)


def test_krylov_set_rank_one_normalised_and_first_vectors():
    d, n, m = 2, 6, 5
    S = krylov.krylov_set(d, n, m)
    for a in S:
        assert tt.ranks(a) == [1, 1, 1]
        assert abs(tt.tt_norm(a) - 1.0) <= 1e-14
    np.testing.assert_allclose(np.abs(tt.densify(S[0])), np.full(n * n, 1.0 / n), atol=1e-15)
    # d = 2: TT rounding to rank 1 is the truncated SVD of the n x n unfolding (Eckart-Young)
    y = _kron_laplacian(d, n) @ tt.densify(S[0])
    Y = y.reshape(n, n).T  # psi order: i_1 fastest -> Y[i_1, i_2]
    U, s, Vt = np.linalg.svd(Y)
    best = s[0] * np.outer(U[:, 0], Vt[0])
    best = best / np.linalg.norm(best)
    a2 = tt.densify(S[1]).reshape(n, n).T
    assert min(np.linalg.norm(a2 - best), np.linalg.norm(a2 + best)) <= 1e-13


def test_krylov_conditioning_grows():
    """By construction the Krylov set's condition number grows with k."""
    S = krylov.krylov_set(3, 5, 8)
    A = np.stack([tt.densify(a) for a in S], axis=1)
    kap = [np.linalg.cond(A[:, :k]) for k in range(2, 9)]
    assert all(b >= a * 0.999 for a, b in zip(kap, kap[1:])) and kap[-1] > 1e3
