"""Small dense fp64 algebra used by the drivers (§2.2 Alg. 5, §2.4 Eq. (9)).

Plain loops for the m x m kernels (m <= 100), so that breakdown indices are exact.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

U_ROUND = 2.0 ** -53  # unit round-off u of IEEE fp64 ("u_64 ~ 1e-16")


class SingularGram(Exception):
    """Cholesky met a non-positive pivot: the Gram matrix is numerically singular
    (Remark 1).  ``index`` is the 0-based failing pivot."""

    def __init__(self, index: int):
        super().__init__(f"numerically singular Gram matrix at pivot {index}")
        self.index = index


class SingularTriangular(Exception):
    def __init__(self, index: int):
        super().__init__(f"zero diagonal entry at {index}")
        self.index = index


def cholesky(G: np.ndarray) -> np.ndarray:
    """G = L L^T, L lower triangular (Alg. 5 line "L = cholesky(G)").
    Input symmetrised as (G + G^T)/2; a pivot <= 0 raises SingularGram."""
    G = 0.5 * (np.asarray(G, dtype=np.float64) + np.asarray(G, dtype=np.float64).T)
    m = G.shape[0]
    L = np.zeros_like(G)
    for j in range(m):
        s = G[j, j] - np.dot(L[j, :j], L[j, :j])
        if not (s > 0.0):
            raise SingularGram(j)
        L[j, j] = np.sqrt(s)
        for i in range(j + 1, m):
            L[i, j] = (G[i, j] - np.dot(L[i, :j], L[j, :j])) / L[j, j]
    return L


def invert_upper(R: np.ndarray) -> np.ndarray:
    """Explicit R^{-1} for upper-triangular R (Alg. 5 "R^{-1} = invert(R)", PAPER.md:249,
    Remark 3 PAPER.md:232-234).  Column-by-column back substitution."""
    m = R.shape[0]
    X = np.zeros_like(R, dtype=np.float64)
    for j in range(m):
        if R[j, j] == 0.0:
            raise SingularTriangular(j)
    for j in range(m):
        X[j, j] = 1.0 / R[j, j]
        for i in range(j - 1, -1, -1):
            X[i, j] = -np.dot(R[i, i + 1:j + 1], X[i + 1:j + 1, j]) / R[i, i]
    return X


def loo(G_q: np.ndarray) -> float:
    """Loss of orthogonality ||I_m - Q^T Q||_2, Eq. (9), with
    (Q^T Q)(i,j) = <q_i, q_j> given as ``G_q``.  The 2-norm of the
    symmetric defect is its largest |eigenvalue| (symmetrised per SPEC.md:550)."""
    G_q = np.asarray(G_q, dtype=np.float64)
    D = np.eye(G_q.shape[0]) - 0.5 * (G_q + G_q.T)
    if D.size == 0:
        return 0.0
    return float(np.max(np.abs(np.linalg.eigvalsh(D))))


def truncation_rank(sigma: np.ndarray, tau: float, keep_all: bool = False) -> int:
    """Smallest rho >= 1 with sqrt(sum_{j>rho} sigma_j^2) <= tau (ties: <= drops),
    SPEC.md:59-62.  ``keep_all`` (delta = 0) keeps every value."""
    sigma = np.asarray(sigma, dtype=np.float64)
    p = sigma.shape[0]
    if keep_all or p == 0:
        return max(p, 1)
    # tail[rho] = sqrt(sum_{j >= rho} sigma_j^2) for 0-based j, i.e. the tail after keeping rho
    for rho in range(1, p + 1):
        tail = np.sqrt(np.sum(sigma[rho:] ** 2))
        if tail <= tau:
            return rho
    return p
