"""TT-rounding ("a rounding algorithm ... proposed in [Oseledets2011]";
contract ||x - x~|| <= delta ||x||; cost O(d n r^3)).  The paper does not restate the
algorithm; the oracle runs Oseledets' TT-SVD rounding step by step (SURVEY.md §8(c) C2,
readings A1-A3, A11, A12):

1. right-to-left orthogonalisation: for k = d..2, Householder QR (numpy.linalg.qr) of the
   transposed unfolding C_k^T ((n_k R'_k) x R_{k-1}); core k <- Q^T, core k-1 <- core k-1 x_3 R^T;
2. ||x|| = ||C_1||_F and the per-split threshold tau = max(delta ||x|| / sqrt(d-1),
   floor_c u s(x)) with s(x) = sum_l |c_l| ||y_l|| the pre-cancellation scale (A2, A12);
3. left-to-right truncation: for k = 1..d-1, SVD (numpy.linalg.svd) of the unfolding
   Y_k ((rho_{k-1} n_k) x R'_k), rho_k = smallest rho >= 1 with tail <= tau, core k <- U_rho,
   core k+1 <- (S_rho V_rho^T) x_1 core k+1;
4. edge cases: ||x|| = 0 -> rank-1 zero tensor; d = 1 -> unchanged; delta = 0 -> no
   truncation and no floor (keep min(rows, cols) values, A11).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .dense import U_ROUND, truncation_rank
from .tt import TT, check_tt, tt_norm, tt_sum

DEFAULT_FLOOR_C = 2048.0  # SURVEY A12; calibrated on the oracle


@dataclass
class RoundInfo:
    ranks: List[int]
    norm: float          # ||x|| = ||C_1||_F after the right-to-left sweep
    tau: float           # per-split truncation threshold
    scale: float         # s(x)
    formal_ranks: List[int] = field(default_factory=list)
    sweep_ranks: List[int] = field(default_factory=list)   # R'_k after right-to-left
    sigmas: List[np.ndarray] = field(default_factory=list)  # singular values per split


def threshold(delta: float, norm: float, d: int, floor_c: float, scale: float) -> float:
    """tau = max(delta ||x|| / sqrt(d-1), floor_c u s(x)) (SURVEY A2 + A12)."""
    if d <= 1:
        return 0.0
    return max(delta * norm / np.sqrt(d - 1.0), floor_c * U_ROUND * scale)


def tt_round(x: TT, delta: float, floor_c: float = 0.0, scale: Optional[float] = None,
             max_rank: Optional[int] = None,
             force_ranks: Optional[Sequence[int]] = None, _owned: bool = False) -> tuple[TT, RoundInfo]:
    """force_ranks (test use only): force rho_k = min(ranks[k], #singular values) at every split
    instead of the threshold rule -- the same truncation as another implementation that chose
    those ranks, for comparing reconstructions where a decision sits inside the window of tau
    (SURVEY.md §8(c) C6 item 1)."""
    check_tt(x)
    d = len(x)
    formal = [1] + [c.shape[2] for c in x]
    # _owned: x is a fresh array list nobody else holds (tt_round_sum's materialised sum), so the
    # sweep may overwrite it instead of copying (memory only: at C5 size the sum is ~60 GB)
    cores = x if _owned else [np.array(c, dtype=np.float64, copy=True) for c in x]
    if d == 1:
        nrm = float(np.linalg.norm(cores[0]))
        return cores, RoundInfo([1, 1], nrm, 0.0, nrm if scale is None else scale, formal, [1, 1])

    # 1. right-to-left orthogonalisation
    for k in range(d - 1, 0, -1):
        r0, n, r1 = cores[k].shape
        A = cores[k].reshape(r0, n * r1).T           # (n_k R'_k) x R_{k-1}
        Q, R = np.linalg.qr(A, mode="reduced")       # Householder QR (LAPACK dgeqrf/dorgqr)
        rn = Q.shape[1]                              # R'_{k-1} = min(n_k R'_k, R_{k-1})
        cores[k] = np.ascontiguousarray(Q.T.reshape(rn, n, r1))
        cores[k - 1] = np.tensordot(cores[k - 1], R.T, axes=([2], [0]))
    sweep = [1] + [c.shape[2] for c in cores]

    # 2. norm and threshold
    nrm = float(np.linalg.norm(cores[0]))
    s = nrm if scale is None else float(scale)
    keep_all = (delta == 0.0)
    tau = 0.0 if keep_all else threshold(delta, nrm, d, floor_c, s)
    if nrm == 0.0:
        z = [np.zeros((1, c.shape[1], 1)) for c in cores]
        return z, RoundInfo([1] * (d + 1), 0.0, tau, s, formal, sweep)

    # 3. left-to-right truncated SVDs
    sigmas = []
    for k in range(d - 1):
        r0, n, r1 = cores[k].shape
        Y = cores[k].reshape(r0 * n, r1)
        U, S, Vt = np.linalg.svd(Y, full_matrices=False)
        rho = truncation_rank(S, tau, keep_all=keep_all)
        if force_ranks is not None:
            rho = max(1, min(int(force_ranks[k + 1]), len(S)))
        if max_rank is not None:
            rho = max(1, min(rho, int(max_rank)))
        sigmas.append(S)
        cores[k] = np.ascontiguousarray(U[:, :rho].reshape(r0, n, rho))
        SV = S[:rho, None] * Vt[:rho, :]
        cores[k + 1] = np.tensordot(SV, cores[k + 1], axes=([1], [0]))
    ranks = [1] + [c.shape[2] for c in cores]
    return cores, RoundInfo(ranks, nrm, tau, s, formal, sweep, sigmas)


def sum_scale(terms: Sequence[TT], coeffs: Sequence[float],
              term_norms: Optional[Sequence[float]] = None) -> float:
    """s(x) = sum_l |c_l| ||y_l|| (SURVEY §8 notation)."""
    if term_norms is None:
        term_norms = [tt_norm(t) for t in terms]
    return float(sum(abs(c) * nr for c, nr in zip(coeffs, term_norms)))


def tt_round_sum(terms: Sequence[TT], coeffs: Sequence[float], delta: float,
                 floor_c: float = 0.0, term_norms: Optional[Sequence[float]] = None,
                 max_rank: Optional[int] = None,
                 force_ranks: Optional[Sequence[int]] = None) -> tuple[TT, RoundInfo]:
    """Round the TT-sum sum_l c_l y_l, materialised literally."""
    s = sum_scale(terms, coeffs, term_norms) if (floor_c > 0.0) else None
    x = tt_sum(terms, coeffs)
    out, info = tt_round(x, delta, floor_c=floor_c, scale=s, max_rank=max_rank, force_ranks=force_ranks, _owned=True)
    return out, info
