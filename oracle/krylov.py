"""The paper's own workload: Krylov sets of TT-vectors built with the
TT-Laplacian.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:475 (Section 3): "Let x_1 be the TT-vector of ones, iteratively we compute
x_{j+1} = -Delta_d a_j where Delta_d is the TT-matrix representing the discretization of the
Laplacian operator of order d with Dirichlet boundary conditions [Kazeev 2012], and a_j is the
normalized output of the TT-round algorithm applied to x_j with the accuracy replaced by a maximum
TT-rank equal to 1."

Readings (A24-A26):
* -Delta_d = sum_k I (x) ... (x) L (x) ... (x) I with L = tridiag(-1, 2, -1) (n x n, Dirichlet, unit
  mesh width): the 1/h^2 factor is dropped because every a_j is normalised (the set is invariant).
* A TT-matrix core is (R_{k-1}, n, n, R_k): A(i_1..i_d, j_1..j_d) = A_1(i_1, j_1) ... A_d(i_d, j_d)
  with A_k(i, j) the R_{k-1} x R_k slice; -Delta_d has the rank-2 form
  [L I], [[I 0], [L I]], ..., [I; L].
* The matrix-vector product has cores Y_k((a, alpha), i, (b, beta)) = sum_j A_k(a, i, j, b)
  X_k(alpha, j, beta) (ranks multiply; (a, alpha) with alpha fastest).
* "maximum TT-rank equal to 1": tt_round with delta = 0 and max_rank = 1, floor off.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .rounding import tt_round
from .tt import TT, ones_tt, tt_norm, tt_scale

TTM = List[np.ndarray]  # operator cores (R_{k-1}, n_k, n_k, R_k)


def laplacian_1d(n: int) -> np.ndarray:
    """L = tridiag(-1, 2, -1): -d^2/dx^2 with Dirichlet boundary conditions, unit mesh width."""
    return 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)


def laplacian_ttm(d: int, n: int) -> TTM:
    """-Delta_d in TT-matrix form, ranks (1, 2, ..., 2, 1) (d >= 2): first core [L I], interior
    [[I 0], [L I]], last [I; L] -- the product telescopes to sum_k I..L..I."""
    L, I = laplacian_1d(n), np.eye(n)
    if d == 1:
        return [L.reshape(1, n, n, 1)]
    first = np.zeros((1, n, n, 2))
    first[0, :, :, 0] = L
    first[0, :, :, 1] = I
    mid = np.zeros((2, n, n, 2))
    mid[0, :, :, 0] = I
    mid[1, :, :, 0] = L
    mid[1, :, :, 1] = I
    last = np.zeros((2, n, n, 1))
    last[0, :, :, 0] = I
    last[1, :, :, 0] = L
    return [first] + [mid.copy() for _ in range(d - 2)] + [last]


def matvec(A: TTM, x: TT) -> TT:
    """y = A x, cores Y_k((a, alpha), i, (b, beta)) = sum_j A_k(a, i, j, b) X_k(alpha, j, beta)."""
    out = []
    for Ak, Xk in zip(A, x):
        ra0, n, _, ra1 = Ak.shape
        rx0, _, rx1 = Xk.shape
        Y = np.einsum("aijb,xjy->axiby", Ak, Xk)
        out.append(Y.reshape(ra0 * rx0, n, ra1 * rx1))
    return out


def krylov_set(d: int, n: int, m: int) -> List[TT]:
    """a_1 = ones / ||ones||; a_{j+1} = round_{rank 1}(-Delta_d a_j) / ||.||."""
    A = laplacian_ttm(d, n)
    x = ones_tt(d, n)
    out: List[TT] = []
    for _ in range(m):
        r, _info = tt_round(x, 0.0, floor_c=0.0, max_rank=1)
        a = tt_scale(r, 1.0 / tt_norm(r))
        out.append(a)
        x = matvec(A, a)
    return out


def dense_operator(A: TTM) -> np.ndarray:
    """Dense matrix of a TT-matrix in psi order (mode 1 fastest): entry
    (psi(i), psi(j)) = A_1(i_1, j_1) ... A_d(i_d, j_d).  For pins on tiny cases."""
    d = len(A)
    n = [c.shape[1] for c in A]
    N = int(np.prod(n))
    M = np.zeros((N, N))
    for p in range(N):
        ip, t = [], p
        for k in range(d):
            ip.append(t % n[k]); t //= n[k]
        for q in range(N):
            jq, t = [], q
            for k in range(d):
                jq.append(t % n[k]); t //= n[k]
            v = A[0][:, ip[0], jq[0], :]
            for k in range(1, d):
                v = v @ A[k][:, ip[k], jq[k], :]
            M[p, q] = v[0, 0]
    return M


def storage_counts(xs: Sequence[TT]) -> List[int]:
    """Numerator of Eq. (1) for each vector (memory per step, Figs. 3-4)."""
    return [int(sum(c.size for c in x)) for x in xs]
