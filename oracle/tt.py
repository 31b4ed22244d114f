"""TT-format basics (§1 "Notation and TT-format", lines 17-69).

A TT-vector is a Python list of d numpy fp64 arrays; core k has shape (r_{k-1}, n_k, r_k)
with r_0 = r_d = 1, stored C-order (r_k fastest).
Multi-indices are 1-based in the paper's psi/phi maps; the array
helpers here take 0-based indices unless the name says otherwise.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

TT = List[np.ndarray]


def modes(x: TT) -> List[int]:
    return [c.shape[1] for c in x]


def ranks(x: TT) -> List[int]:
    """TT-ranks (r_0, ..., r_d) ("k-th TT-rank")."""
    return [x[0].shape[0]] + [c.shape[2] for c in x]


def check_tt(x: TT) -> None:
    if len(x) < 1:
        raise ValueError("TT-vector needs d >= 1 cores")
    if x[0].shape[0] != 1 or x[-1].shape[2] != 1:
        raise ValueError("boundary ranks must be r_0 = r_d = 1 (PAPER.md:45)")
    for k in range(len(x) - 1):
        if x[k].shape[2] != x[k + 1].shape[0]:
            raise ValueError(f"rank mismatch between cores {k + 1} and {k + 2}")


# ----------------------------------------------------------------------------------------
# psi / phi and the canonical basis (§2.3)
# ----------------------------------------------------------------------------------------
def psi(idx1: Sequence[int], n: Sequence[int]) -> int:
    """psi(i_1..i_d) = i_1 + sum_{a>=2} (i_a - 1) m_a, m_a = prod_{b<a} n_b.
    1-based in and out."""
    lin = int(idx1[0])
    m_a = 1
    for a in range(1, len(n)):
        m_a *= int(n[a - 1])
        lin += (int(idx1[a]) - 1) * m_a
    return lin


def phi(i1: int, n: Sequence[int]) -> List[int]:
    """Inverse of psi.  1-based in and out."""
    rem = int(i1) - 1
    out = []
    for nk in n:
        out.append(rem % int(nk) + 1)
        rem //= int(nk)
    if rem != 0:
        raise IndexError("linear index out of range")
    return out


def canonical_tt(i1: int, n: Sequence[int]) -> TT:
    """e_i = e_{i_1} (x) ... (x) e_{i_d} with (i_1..i_d) = phi(i)."""
    idx = phi(i1, n)
    cores = []
    for k, nk in enumerate(n):
        c = np.zeros((1, int(nk), 1))
        c[0, idx[k] - 1, 0] = 1.0
        cores.append(c)
    return cores


def ones_tt(d: int, n: int) -> TT:
    """The TT-vector of ones."""
    return [np.ones((1, n, 1)) for _ in range(d)]


# ----------------------------------------------------------------------------------------
# element, densify
# ----------------------------------------------------------------------------------------
def element(x: TT, idx0: Sequence[int]) -> float:
    """x(i_1..i_d) = X_1(i_1) X_2(i_2) ... X_d(i_d), product of slices.
    0-based multi-index."""
    v = x[0][:, idx0[0], :]
    for k in range(1, len(x)):
        v = v @ x[k][:, idx0[k], :]
    return float(v[0, 0])


def densify(x: TT) -> np.ndarray:
    """Dense vector of length prod(n) in psi order (mode 1 fastest), entry
    psi(i) = element(x, i).  Built by contracting cores left to right."""
    d = len(x)
    # full tensor F[i_1, ..., i_k, r_k], then vectorise with i_1 fastest
    F = x[0][0]  # (n_1, r_1)
    for k in range(1, d):
        F = np.tensordot(F, x[k], axes=([F.ndim - 1], [0]))  # (..., n_k, r_k)
    F = F[..., 0]  # (n_1, ..., n_d)
    return np.asarray(F).transpose(list(range(d))[::-1]).reshape(-1)  # i_1 fastest


def storage_count(x: TT) -> int:
    """Numerator of Eq. (1): sum_i r_{i-1} n_i r_i."""
    return int(sum(c.shape[0] * c.shape[1] * c.shape[2] for c in x))


# ----------------------------------------------------------------------------------------
# sum, scale, dot, norm
# ----------------------------------------------------------------------------------------
def tt_scale(x: TT, alpha: float) -> TT:
    """alpha x by multiplying the first core only; ranks unchanged."""
    out = [c.copy() for c in x]
    out[0] = out[0] * alpha
    return out


def tt_sum(terms: Sequence[TT], coeffs: Sequence[float] | None = None) -> TT:
    """x = sum_l c_l y_l with ranks r_k = sum_l r_k^(l): first cores concatenated
    horizontally (c_l applied to term l's first core), interior cores block-diagonal, last
    cores concatenated vertically.  Materialised literally."""
    K = len(terms)
    if coeffs is None:
        coeffs = [1.0] * K
    d = len(terms[0])
    for t in terms:
        if len(t) != d or modes(t) != modes(terms[0]):
            raise ValueError("shape mismatch in TT-sum (SPEC.md:154)")
    if d == 1:
        return [sum(c * t[0] for c, t in zip(coeffs, terms))]
    out = []
    for k in range(d):
        nk = terms[0][k].shape[1]
        r0s = [t[k].shape[0] for t in terms]
        r1s = [t[k].shape[2] for t in terms]
        R0 = 1 if k == 0 else sum(r0s)
        R1 = 1 if k == d - 1 else sum(r1s)
        core = np.zeros((R0, nk, R1))
        o0 = o1 = 0
        for l, t in enumerate(terms):
            blk = t[k] * (coeffs[l] if k == 0 else 1.0)
            a0 = 0 if k == 0 else o0
            a1 = 0 if k == d - 1 else o1
            core[a0:a0 + r0s[l], :, a1:a1 + r1s[l]] = blk
            o0 += r0s[l]
            o1 += r1s[l]
        out.append(core)
    return out


def tt_dot(x: TT, y: TT) -> float:
    """<x, y> = sum_i x(i) y(i) (the Euclidean dot product generalised through
    the tensor contraction), evaluated by the left-to-right contraction
    W_k = sum_{i_k} X_k(i_k)^T W_{k-1} Y_k(i_k), W_0 = 1."""
    if modes(x) != modes(y):
        raise ValueError("shape mismatch in TT-dot (SPEC.md:172)")
    W = np.ones((1, 1))
    for k in range(len(x)):
        Wn = np.zeros((x[k].shape[2], y[k].shape[2]))
        for i in range(x[k].shape[1]):
            Wn += x[k][:, i, :].T @ W @ y[k][:, i, :]
        W = Wn
    return float(W[0, 0])


def tt_norm(x: TT) -> float:
    """||x|| = sqrt(max(<x,x>, 0))."""
    return float(np.sqrt(max(tt_dot(x, x), 0.0)))


def compression_ratio(x: TT) -> float:
    """Eq. (1): sum r_{i-1} n_i r_i / prod n_j."""
    return storage_count(x) / float(np.prod([float(v) for v in modes(x)]))


def compression_gain(before: TT, after: TT) -> float:
    """Eq. (2): ratio of the storage counts before / after rounding."""
    if modes(before) != modes(after):
        raise ValueError("shape mismatch")
    return storage_count(before) / float(storage_count(after))


def tt_hadamard(x: TT, y: TT) -> TT:
    """Elementwise product z(i) = x(i) y(i): core k is the Kronecker product of the slices,
    Z_k(i) = X_k(i) (x) Y_k(i), ranks multiply (SPEC.md:177-185 Hadamard; used only by the
    TTH-vec masking variant)."""
    if modes(x) != modes(y):
        raise ValueError("shape mismatch in TT-Hadamard")
    out = []
    for X, Y in zip(x, y):
        a0, n, a1 = X.shape
        b0, _, b1 = Y.shape
        Z = np.einsum("aib,cid->acibd", X, Y).reshape(a0 * b0, n, a1 * b1)
        out.append(np.ascontiguousarray(Z))
    return out


def mask_geq(n: Sequence[int], L: int) -> TT:
    """Indicator of the canonical indices j >= L + 1, i.e. of the multi-indices whose psi-order
    linear index (mode 1 fastest) is >= L, as a TT of ranks <= 2: a comparison of the
    mixed-radix digits from the most significant (mode d) down, state 0 = equal so far, 1 =
    already greater; core k maps the state before digit k (right index) to the state after it
    (left index); core 1 accepts states 'equal' (digit >= l_1) and 'greater'.  L = 0 gives ones."""
    d = len(n)
    digits, rem = [], int(L)
    for k in range(d):
        digits.append(rem % n[k])
        rem //= n[k]
    if rem:
        raise ValueError("L beyond prod(n)")
    cores = []
    for k in range(d):
        lk = digits[k]
        left = 1 if k == 0 else 2
        right = 1 if k == d - 1 else 2
        C = np.zeros((left, n[k], right))
        for s_in in range(right):          # state from the digits above k (mode d: start 'equal')
            state_in = 0 if k == d - 1 else s_in
            for x in range(n[k]):
                if state_in == 1:
                    s_out = 1
                elif x > lk:
                    s_out = 1
                elif x == lk:
                    s_out = 0
                else:
                    continue               # smaller at the first differing digit: rejected
                if k == 0:
                    C[0, x, s_in] = 1.0    # accept 'equal' (lin == L) and 'greater'
                else:
                    C[s_out, x, s_in] = 1.0
        cores.append(C)
    return cores
