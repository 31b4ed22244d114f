"""The six TT orthogonalization kernels of PAPER.md §2 (Algorithms 1-8), each in two forms:

* ``*_literal``: the listing executed as written, every TT-sum materialised by block
  concatenation and every inner product taken on the materialised train;
* ``*_lazy``: the same arithmetic with the running TT-sums kept as coefficients over the
  stored tensors (SURVEY.md §8(c) C3 "lazy equivalence": <sum_l c_l y_l, q> on the
  concatenated train equals sum_l c_l <y_l, q> up to the order of the final reduction),
  materialised only at the paper's rounding points.  This is the form the CUDA drivers
  implement; tests assert literal == lazy on small inputs.

Readings: R stored at R(j, i) (A4), Gram uses q_i = sum_k R^{-1}(k,i) a_k
(A5), u = w/||w|| (A7), Householder sign per Alg. 6 with sign(0) = +1 (A8), beta from the
first rounding's norm unless hh_beta="literal" (A9), 4m-1 roundings (A10), the redundant
H_i a_i is skipped (A18), the noise floor s(x) uses ||q_j|| = ||u_j|| = ||e_j|| = 1 (unit by
construction) and ||a_i|| from one TT-dot.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .dense import cholesky, invert_upper, loo
from .rounding import DEFAULT_FLOOR_C, RoundInfo, tt_round_sum
from .tt import TT, canonical_tt, element, mask_geq, modes, phi, tt_dot, tt_hadamard, tt_norm, tt_scale, tt_sum


class NumericalDefect(Exception):
    """TTH-vec with the literal beta (Alg. 6 line 10): ||a||^2 - s below
    -1e-12 ||a||^2 (clamped to 0 when within that tolerance).  ``index`` is the
    0-based step."""

    def __init__(self, index: int):
        super().__init__(f"||a||^2 - s < 0 in TTH-vec at step {index}")
        self.index = index


def _literal_beta(a_norm: float, s: float, i: int) -> float:
    """beta = sqrt(||a||^2 - s) as Alg. 6 line 10 prints it, with SPEC.md:436's
    defect rule; i is 1-based."""
    d2 = a_norm * a_norm - s
    if d2 < -1e-12 * a_norm * a_norm:
        raise NumericalDefect(i - 1)
    return float(np.sqrt(max(d2, 0.0)))


class LinearDependence(Exception):
    def __init__(self, index: int):
        super().__init__(f"linear dependence at step {index}")
        self.index = index


@dataclass
class OrthResult:
    Q: List[TT]
    R: np.ndarray
    rounding_calls: int = 0
    infos: List[RoundInfo] = field(default_factory=list)
    U: List[Optional[TT]] = field(default_factory=list)   # Householder vectors
    coeffs: List[np.ndarray] = field(default_factory=list)  # per rounding: the sum's coefficients
    terms: List[list] = field(default_factory=list)         # per rounding (lazy form): the sum's terms
    outputs: List[TT] = field(default_factory=list)         # per rounding (lazy form): its output
    term_norms: List[list] = field(default_factory=list)    # per rounding (lazy form): ||y_l|| used in s(x)

    def loo_per_step(self) -> np.ndarray:
        """LOO_k = ||I_k - Q_k^T Q_k||_2 over prefixes."""
        m = len(self.Q)
        G = np.zeros((m, m))
        for i in range(m):
            for j in range(i + 1):
                G[i, j] = G[j, i] = tt_dot(self.Q[i], self.Q[j])
        return np.array([loo(G[:k, :k]) for k in range(1, m + 1)])


def _record(res: "OrthResult", terms, coefs, norms, out, info) -> None:
    res.rounding_calls += 1
    res.infos.append(info)
    res.coeffs.append(np.array(coefs))
    res.terms.append(list(terms))
    res.term_norms.append(list(norms))
    res.outputs.append(out)


def _last_core_norm(p: TT) -> float:
    """||p|| of a rounding output: cores 1..d-1 are left-orthonormal after the left-to-right
    sweep, so ||p|| = ||X_d||_F."""
    return float(np.linalg.norm(p[-1]))


def _normalise(p: TT, nrm: float) -> TT:
    return tt_scale(p, 1.0 / nrm)  # q = (1/R(i,i)) p, first core


def _ldep_check(nrm: float, a_norm: float, i: int) -> None:
    # SURVEY A22 / SPEC.md:473: ||p|| <= 1e3 u ||a_i|| -> linear dependence
    if nrm <= 1e3 * 2.0 ** -53 * a_norm:
        raise LinearDependence(i)


# ========================================================================================
# Gram-Schmidt family, literal (Algs. 1-4)
# ========================================================================================
def gs_literal(A: Sequence[TT], delta: float, kind: str, floor_c: float = DEFAULT_FLOOR_C) -> OrthResult:
    """kind in {cgs, mgs, cgs2, mgs2}.  Alg. 1 (CGS) PAPER.md:87-109, Alg. 2 (MGS) :111-133,
    Alg. 3 (CGS2) :144-171, Alg. 4 (MGS2) :173-200."""
    m = len(A)
    passes = 2 if kind in ("cgs2", "mgs2") else 1
    modified = kind in ("mgs", "mgs2")
    Rk = [np.zeros((m, m)) for _ in range(passes)]
    Q: List[TT] = []
    res = OrthResult(Q, np.zeros((m, m)))
    a_norms = [tt_norm(a) for a in A]
    for i in range(m):
        p_prev = A[i]
        prev_norm = a_norms[i]
        for k in range(passes):
            p = p_prev
            scale = prev_norm
            terms, coefs = [p_prev], [1.0]
            for j in range(i):
                src = p if modified else p_prev          # line 6/7 of Algs 1-4
                c = tt_dot(src, Q[j])
                Rk[k][j, i] = c
                p = tt_sum([p, Q[j]], [1.0, -c])
                scale += abs(c)
                terms.append(Q[j]); coefs.append(-c)
            # TT-round(p, delta) (Alg. 1 l.9, Alg. 2 l.10, Algs. 3-4 l.10); s(x) = scale
            out, info = _round_materialised(p, delta, floor_c, scale)
            res.rounding_calls += 1
            res.infos.append(info)
            res.coeffs.append(np.array(coefs))
            p_prev = out
            prev_norm = _last_core_norm(out)
        nrm = prev_norm
        _ldep_check(nrm, a_norms[i], i)
        Rk[passes - 1][i, i] = nrm
        Q.append(_normalise(p_prev, nrm))
    res.R = Rk[0] + (Rk[1] if passes == 2 else 0.0)  # R = R1 + R2 (Alg. 3/4 last lines)
    return res


def _round_materialised(p: TT, delta: float, floor_c: float, scale: float):
    from .rounding import tt_round
    return tt_round(p, delta, floor_c=floor_c, scale=scale)


# ========================================================================================
# Gram-Schmidt family, lazy
# ========================================================================================
def gs_lazy(A: Sequence[TT], delta: float, kind: str, floor_c: float = DEFAULT_FLOOR_C) -> OrthResult:
    """Same as gs_literal with coefficients instead of materialised sums.
    CGS:  R(j,i) = <a_i, q_j>.
    MGS:  R(j,i) = <a_i, q_j> - sum_{l<j} R(l,i) <q_l, q_j>  (= <p^(j-1), q_j>).
    Second passes use the rounded p_1 in place of a_i."""
    m = len(A)
    passes = 2 if kind in ("cgs2", "mgs2") else 1
    modified = kind in ("mgs", "mgs2")
    Rk = [np.zeros((m, m)) for _ in range(passes)]
    Q: List[TT] = []
    GQ = np.zeros((m, m))  # <q_l, q_j>
    res = OrthResult(Q, np.zeros((m, m)))
    a_norms = [tt_norm(a) for a in A]
    for i in range(m):
        base = A[i]
        base_norm = a_norms[i]
        for k in range(passes):
            d_bq = np.array([tt_dot(base, Q[j]) for j in range(i)])
            c = np.zeros(i)
            for j in range(i):
                if modified:
                    c[j] = d_bq[j] - np.dot(c[:j], GQ[:j, j])
                else:
                    c[j] = d_bq[j]
                Rk[k][j, i] = c[j]
            terms = [base] + Q[:i]
            coefs = [1.0] + list(-c)
            scale = base_norm + float(np.sum(np.abs(c)))
            tn = [base_norm] + [1.0] * i
            out, info = tt_round_sum(terms, coefs, delta, floor_c=floor_c, term_norms=tn)
            _record(res, terms, coefs, tn, out, info)
            base = out
            base_norm = _last_core_norm(out)
        nrm = base_norm
        _ldep_check(nrm, a_norms[i], i)
        Rk[passes - 1][i, i] = nrm
        qi = _normalise(base, nrm)
        Q.append(qi)
        for j in range(i + 1):
            GQ[j, i] = GQ[i, j] = tt_dot(Q[j], qi)
    res.R = Rk[0] + (Rk[1] if passes == 2 else 0.0)
    return res


# ========================================================================================
# Gram (Alg. 5)
# ========================================================================================
def gram_matrix(A: Sequence[TT]) -> np.ndarray:
    """G(i,j) = G(j,i) = <a_i, a_j> (Alg. 5 lines 2-6; Eq. (3))."""
    m = len(A)
    G = np.zeros((m, m))
    for i in range(m):
        for j in range(i + 1):
            G[i, j] = G[j, i] = tt_dot(A[i], A[j])
    return G


def gram_orth(A: Sequence[TT], delta: float, floor_c: float = DEFAULT_FLOOR_C,
              literal: bool = False) -> OrthResult:
    """TT-Gram: L = chol(G), R = L^T, R^{-1} explicit (Remark 3), q_i = round(sum_{k<=i}
    R^{-1}(k,i) a_k) (PAPER.md:230 equation; A5)."""
    m = len(A)
    G = gram_matrix(A)
    L = cholesky(G)
    R = L.T.copy()
    Rinv = invert_upper(R)
    a_norms = [tt_norm(a) for a in A]
    res = OrthResult([], R)
    for i in range(m):
        coefs = [Rinv[k, i] for k in range(i + 1)]
        if literal:
            p = tt_scale(A[0], coefs[0])                   # Alg. 5 line 8
            for k in range(1, i + 1):                        # Alg. 5 lines 9-11
                p = tt_sum([p, A[k]], [1.0, coefs[k]])
            scale = float(sum(abs(c) * a_norms[k] for k, c in enumerate(coefs)))
            out, info = _round_materialised(p, delta, floor_c, scale)
        else:
            out, info = tt_round_sum(list(A[:i + 1]), coefs, delta, floor_c=floor_c,
                                     term_norms=a_norms[:i + 1])
            _record(res, list(A[:i + 1]), coefs, a_norms[:i + 1], out, info)
        if literal:
            res.rounding_calls += 1
            res.infos.append(info)
            res.coeffs.append(np.array(coefs))
        res.Q.append(out)                                    # Alg. 5 line 12
    return res


# ========================================================================================
# Householder (Algs. 6-8)
# ========================================================================================
def _sign(v: float) -> float:
    return 1.0 if v >= 0.0 else -1.0  # sign(0) = +1


def tth_vec_literal(a: TT, i: int, delta: float, floor_c: float, hh_beta: str = "round_norm",
                    a_norm: Optional[float] = None):
    """Alg. 6 TTH-vec(a, F = {e_1..e_i}, delta); i is 1-based.
    Returns (u or None for the identity reflector, r[0:i], infos, coeffs)."""
    n = modes(a)
    an = tt_norm(a) if a_norm is None else a_norm
    r = np.zeros(i)
    s = 0.0
    w = a
    scale = an
    coefs1 = [1.0]
    for j in range(1, i):                                    # lines 4-8
        e = canonical_tt(j, n)
        r[j - 1] = tt_dot(a, e)
        s += r[j - 1] ** 2
        w = tt_sum([w, e], [1.0, -r[j - 1]])
        scale += abs(r[j - 1])
        coefs1.append(-r[j - 1])
    w1, info1 = _round_materialised(w, delta, floor_c, scale)   # line 9
    ei = canonical_tt(i, n)
    sg = _sign(tt_dot(a, ei))
    if hh_beta == "literal":                                 # line 10 as printed
        beta = _literal_beta(an, s, i)
    else:                                                    # A9: beta = ||round(a - sum r_j e_j)||
        beta = _last_core_norm(w1)
    r[i - 1] = sg * beta
    w2 = tt_sum([w1, ei], [1.0, -r[i - 1]])                  # line 11
    w2r, info2 = _round_materialised(w2, delta, floor_c, _last_core_norm(w1) + abs(r[i - 1]))  # line 12
    nw = _last_core_norm(w2r)
    u = None if nw == 0.0 else _normalise(w2r, nw)           # line 13 (A7: u = w/||w||)
    return u, r, [info1, info2], [np.array(coefs1), np.array([1.0, -r[i - 1]])]


def apply_h_vec(a: TT, u: Optional[TT]):
    """Alg. 7: b = a - 2<a,u>u.  Identity for a degenerate u."""
    if u is None:
        return a, 0.0
    c = 2.0 * tt_dot(a, u)
    if c == 0.0:
        return a, 0.0
    return tt_sum([a, u], [1.0, -c]), c


def householder_literal(A: Sequence[TT], delta: float, floor_c: float = DEFAULT_FLOOR_C,
                        hh_beta: str = "round_norm") -> OrthResult:
    """Alg. 8 TT-Householder executed as listed."""
    m = len(A)
    n = modes(A[0])
    A = list(A)
    scales = [tt_norm(a) for a in A]                       # running s(a_j)
    res = OrthResult([], np.zeros((m, m)))
    w = A[0]                                               # line 3 (not rounded)
    w_norm = scales[0]
    for i in range(1, m + 1):
        u, r, infos, cfs = tth_vec_literal(w, i, delta, floor_c, hh_beta, a_norm=w_norm)
        res.rounding_calls += 2
        res.infos += infos
        res.coeffs += cfs
        res.U.append(u)
        res.R[:i, i - 1] = r
        for j in range(i + 1, m + 1):                      # line 6-8 (j = i skipped, A18)
            A[j - 1], c = apply_h_vec(A[j - 1], u)
            scales[j - 1] += abs(c)
        if i < m:                                          # lines 9-11
            w, info = _round_materialised(A[i], delta, floor_c, scales[i])
            res.rounding_calls += 1
            res.infos.append(info)
            res.coeffs.append(np.array([]))
            w_norm = _last_core_norm(w)
    for i in range(1, m + 1):                              # lines 13-19
        q = canonical_tt(i, n)
        scale = 1.0
        for j in range(i, 0, -1):
            q, c = apply_h_vec(q, res.U[j - 1])
            scale += abs(c)
        q, info = _round_materialised(q, delta, floor_c, scale)
        res.rounding_calls += 1
        res.infos.append(info)
        res.coeffs.append(np.array([]))
        res.Q.append(q)
    return res


def householder_lazy(A: Sequence[TT], delta: float, floor_c: float = DEFAULT_FLOOR_C,
                     hh_beta: str = "round_norm", hh_mask: bool = False) -> OrthResult:
    """Alg. 8 with a~_j = a_j - sum_l gamma_{jl} u_l kept as coefficients:
    gamma_{jl} = 2(<a_j,u_l> - sum_{p<l} gamma_{jp} <u_p,u_l>), and
    q_i = e_i - sum_{j<=i} beta_{ij} u_j with beta_{ij} = 2(<e_i,u_j> - sum_{j<l<=i} beta_{il}<u_l,u_j>)
    (SURVEY.md §8(c) C3).  <x, e_j> is the element x(phi(j)).
    hh_mask (a DEPARTURE from Alg. 6's listing): the first TTH-vec rounding
    takes w with its entries at phi(1..i-1) set to zero exactly -- the Hadamard product with
    the rank-2 mask of the canonical indices >= i (mask_geq) -- instead of the TT-sum
    w - sum_{j<i} r(j) e_j, which equals it in exact arithmetic but cancels in floating point."""
    m = len(A)
    n = modes(A[0])
    a_norms = [tt_norm(a) for a in A]
    res = OrthResult([], np.zeros((m, m)))
    U: List[Optional[TT]] = []
    GU = np.zeros((m, m))                 # <u_p, u_l>
    gamma = np.zeros((m, m))              # gamma[j, l]
    w = A[0]
    w_norm = a_norms[0]
    for i in range(1, m + 1):
        # --- TTH-vec(w, F_i) with element reads ---
        idx = [phi(j, n) for j in range(1, i + 1)]
        ew = np.array([element(w, [t - 1 for t in ix]) for ix in idx])   # <w, e_j>
        r = np.zeros(i)
        r[:i - 1] = ew[:i - 1]
        s = float(np.sum(r[:i - 1] ** 2))
        if hh_mask and i > 1:
            terms = [tt_hadamard(w, mask_geq(n, i - 1))]
            coefs = [1.0]
            tn1 = [tt_norm(terms[0])]
        else:
            terms = [w] + [canonical_tt(j, n) for j in range(1, i)]
            coefs = [1.0] + list(-r[:i - 1])
            tn1 = [w_norm] + [1.0] * (i - 1)
        w1, info1 = tt_round_sum(terms, coefs, delta, floor_c=floor_c, term_norms=tn1)
        _record(res, terms, coefs, tn1, w1, info1)
        sg = _sign(ew[i - 1])
        beta = _literal_beta(w_norm, s, i) if hh_beta == "literal" else _last_core_norm(w1)
        r[i - 1] = sg * beta
        w1n = _last_core_norm(w1)
        t2, c2 = [w1, canonical_tt(i, n)], [1.0, -r[i - 1]]
        w2, info2 = tt_round_sum(t2, c2, delta, floor_c=floor_c, term_norms=[w1n, 1.0])
        _record(res, t2, c2, [w1n, 1.0], w2, info2)
        nw = _last_core_norm(w2)
        u = None if nw == 0.0 else _normalise(w2, nw)
        U.append(u)
        res.R[:i, i - 1] = r
        if u is not None:
            for p in range(i):
                GU[p, i - 1] = GU[i - 1, p] = (tt_dot(U[p], u) if U[p] is not None else 0.0)
        # --- reflections of a_j, j > i, as coefficients ---
        for j in range(i + 1, m + 1):
            if u is None:
                gamma[j - 1, i - 1] = 0.0
                continue
            v = tt_dot(A[j - 1], u) - float(np.dot(gamma[j - 1, :i - 1], GU[:i - 1, i - 1]))
            gamma[j - 1, i - 1] = 2.0 * v
        if i < m:
            live = [l for l in range(i) if U[l] is not None]
            terms = [A[i]] + [U[l] for l in live]
            coefs = [1.0] + [-gamma[i, l] for l in live]
            tn = [a_norms[i]] + [1.0] * len(live)
            w, info = tt_round_sum(terms, coefs, delta, floor_c=floor_c, term_norms=tn)
            _record(res, terms, coefs, tn, w, info)
            w_norm = _last_core_norm(w)
    res.U = U
    for i in range(1, m + 1):
        beta = np.zeros(m)
        for j in range(i, 0, -1):                       # H_i first, then H_{i-1}, ..., H_1
            if U[j - 1] is None:
                continue
            ix = phi(i, n)
            v = element(U[j - 1], [t - 1 for t in ix]) - sum(
                beta[l - 1] * GU[l - 1, j - 1] for l in range(j + 1, i + 1))
            beta[j - 1] = 2.0 * v
        live = [j for j in range(i, 0, -1) if U[j - 1] is not None]
        terms = [canonical_tt(i, n)] + [U[j - 1] for j in live]
        coefs = [1.0] + [-beta[j - 1] for j in live]
        q, info = tt_round_sum(terms, coefs, delta, floor_c=floor_c, term_norms=[1.0] * len(terms))
        _record(res, terms, coefs, [1.0] * len(terms), q, info)
        res.Q.append(q)
    return res


# ========================================================================================
# dispatcher
# ========================================================================================
def orth(kind: str, A: Sequence[TT], delta: float, floor_c: float = DEFAULT_FLOOR_C,
         literal: bool = False, hh_beta: str = "round_norm", hh_mask: bool = False) -> OrthResult:
    kind = kind.lower()
    if kind in ("cgs", "mgs", "cgs2", "mgs2"):
        return (gs_literal if literal else gs_lazy)(A, delta, kind, floor_c)
    if kind == "gram":
        return gram_orth(A, delta, floor_c, literal=literal)
    if kind in ("householder", "hh"):
        if hh_mask:
            return householder_lazy(A, delta, floor_c, hh_beta, hh_mask=True)
        return (householder_literal if literal else householder_lazy)(A, delta, floor_c, hh_beta)
    raise ValueError(kind)
