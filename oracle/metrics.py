"""Metrics of PAPER.md §1 and §2.4: compression ratio Eq. (1), compression gain Eq. (2),
loss of orthogonality Eq. (9).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .dense import loo
from .tt import TT, compression_gain, compression_ratio, storage_count, tt_dot  # noqa: F401


def q_gram(Q: Sequence[TT]) -> np.ndarray:
    """(Q^T Q)(i,j) = <q_i, q_j>."""
    m = len(Q)
    G = np.zeros((m, m))
    for i in range(m):
        for j in range(i + 1):
            G[i, j] = G[j, i] = tt_dot(Q[i], Q[j])
    return G


def loss_of_orthogonality(Q: Sequence[TT]) -> float:
    """Eq. (9): ||I_m - Q_m^T Q_m||_2."""
    return loo(q_gram(Q))
