"""Seeded synthetic inputs for the five BASELINE.json configurations.

Recipe (with the change noted below):

* All draws come from ``numpy.random.Generator(PCG64(seed))`` via ``standard_normal``
  (fp64), in the fixed order documented per function.  seed_c = 221108770 + c.
* TT layout: core k has shape (r_{k-1}, n_k, r_k), C order (r_k fastest).
* Shared-tail sets (C1, C2, C3, C5): a_i = (first core X @ M[:, i]) followed by one common
  right-orthonormal tail T.  With X having orthonormal columns and T orthonormal rows at
  split 1, vec(a_i) = B M[:, i] with B = X (x) T orthonormal, hence EXACTLY
  Gram(A) = M^T M, sigma(A) = sigma(M), R = R_M and q_i = B Q_M[:, i].  Ranks stay r.
  Literal "mixing" of independent tensors would multiply the ranks by m.
* Orthonormal factors are Q-factors of Gaussian draws with diag(R) >= 0 (a random
  orthonormal matrix).  Each tail core is made right-orthonormal on its own (its own
  QR; nothing is propagated between cores), so this module never runs the TT-rounding
  sweep or any other step of the paper's method.

The module holds none of the method's arithmetic: no TT-dot, TT-sum, rounding, Gram-Schmidt
or Householder step.  Norms used here are Frobenius norms of single cores.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

SEED_BASE = 221108770


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _qfactor(g: np.ndarray) -> np.ndarray:
    """Q-factor of a Gaussian draw with diag(R) >= 0 (a random orthonormal basis)."""
    q, r = np.linalg.qr(g, mode="reduced")
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s[None, :]


def tt_ranks_capped(d: int, n: Sequence[int], r: int) -> List[int]:
    """r_k = min(r, n_1..n_k, n_{k+1}..n_d) with r_0 = r_d = 1."""
    ranks = [1]
    for k in range(1, d):
        left = int(np.prod(n[:k], dtype=object))
        right = int(np.prod(n[k:], dtype=object))
        ranks.append(int(min(r, left, right)))
    ranks.append(1)
    return ranks


def _right_orthonormal_core(rng: np.random.Generator, r0: int, n: int, r1: int) -> np.ndarray:
    """Random core with orthonormal rows of its (r0) x (n r1) unfolding (needs r0 <= n r1)."""
    g = rng.standard_normal((r0, n, r1))
    q = _qfactor(g.reshape(r0, n * r1).T)  # (n r1) x r0, orthonormal columns
    return np.ascontiguousarray(q.T.reshape(r0, n, r1))


@dataclass
class SharedTailSet:
    """m TT-vectors a_i = [X M[:, i]] x T with closed-form answers."""

    d: int
    n: List[int]
    ranks: List[int]
    m: int
    kappa: float
    seed: int
    X: np.ndarray               # (n_1 r_1) x m, orthonormal columns
    M: np.ndarray               # m x m mixing matrix, singular values kappa^{-(j-1)/(m-1)}
    tail: List[np.ndarray]      # cores 2..d, right-orthonormal
    tensors: List[List[np.ndarray]] = field(default_factory=list)

    # ---- closed forms of the construction (not computed by the method) ----
    def gram_exact(self) -> np.ndarray:
        return self.M.T @ self.M

    def qr_exact(self) -> Tuple[np.ndarray, np.ndarray]:
        """M = Q_M R_M with diag(R_M) > 0."""
        q, r = np.linalg.qr(self.M)
        s = np.sign(np.diag(r))
        s[s == 0] = 1.0
        return q * s[None, :], r * s[:, None]

    def q_exact(self, i: int) -> List[np.ndarray]:
        """Exact i-th orthonormal vector q_i = B Q_M[:, i] (0-based i)."""
        qm, _ = self.qr_exact()
        return self.first_core_tensor(self.X @ qm[:, i])

    def first_core_tensor(self, v: np.ndarray) -> List[np.ndarray]:
        c1 = np.ascontiguousarray(v.reshape(1, self.n[0], self.ranks[1]))
        return [c1] + [t.copy() for t in self.tail]


def make_shared_tail_set(d: int, n: int | Sequence[int], r: int, m: int, kappa: float,
                         seed: int) -> SharedTailSet:
    """Draw order: tail cores k = 2..d, then X, then U, then V (all standard_normal)."""
    nn = [int(n)] * d if np.isscalar(n) else [int(v) for v in n]
    ranks = tt_ranks_capped(d, nn, r)
    rng = _rng(seed)
    tail = [_right_orthonormal_core(rng, ranks[k - 1], nn[k - 1], ranks[k]) for k in range(2, d + 1)]
    rows = nn[0] * ranks[1]
    if rows < m:
        raise ValueError(f"shared-tail construction needs n_1 r_1 >= m ({rows} < {m})")
    X = _qfactor(rng.standard_normal((rows, m)))
    U = _qfactor(rng.standard_normal((m, m)))
    V = _qfactor(rng.standard_normal((m, m)))
    if m > 1:
        sig = kappa ** (-np.arange(m) / (m - 1.0))
    else:
        sig = np.ones(1)
    M = (U * sig[None, :]) @ V.T
    st = SharedTailSet(d=d, n=nn, ranks=ranks, m=m, kappa=kappa, seed=seed, X=X, M=M, tail=tail)
    st.tensors = [st.first_core_tensor(X @ M[:, i]) for i in range(m)]
    return st


def make_random_tt(d: int, n: int | Sequence[int], ranks: Sequence[int],
                   rng: np.random.Generator, unit_right_orth: bool = False) -> List[np.ndarray]:
    """Gaussian TT cores (r_{k-1}, n_k, r_k).  With unit_right_orth, cores 2..d are random
    right-orthonormal cores and core 1 is scaled to unit Frobenius norm, so the tensor has
    norm exactly 1 by construction (no TT contraction involved)."""
    nn = [int(n)] * d if np.isscalar(n) else [int(v) for v in n]
    if unit_right_orth:
        cores = [rng.standard_normal((ranks[0], nn[0], ranks[1]))]
        for k in range(1, d):
            cores.append(_right_orthonormal_core(rng, ranks[k], nn[k], ranks[k + 1]))
        cores[0] = cores[0] / np.linalg.norm(cores[0])
        return cores
    return [rng.standard_normal((ranks[k], nn[k], ranks[k + 1])) for k in range(d)]


def make_batch_sums(B: int, d: int = 10, n: int = 32, r: int = 16, seed: int = SEED_BASE + 4,
                    eps3: float = 1e-9, eps4: float = 1e-10, omega_odd: float = 1e-9,
                    start: int = 0):
    """C4: x_b = y_1 + w_b y_2 + eps3 y_3 + eps4 y_4 with unit-norm y.

    w_b = 1 for even b, omega_odd for odd b.  Each y has random right-orthonormal cores 2..d
    and a Gaussian first core scaled to unit Frobenius norm (norm exactly 1 by construction).
    Draw order: b-major, then s = 1..4, then the cores of y_{b,s} (core 1 first); items
    [start, start+B) of the full stream are returned.  Same bytes as make_batch_sums_stacked
    (this is its per-item view).  Returns a list of (terms, coeffs), terms a list of 4 core-lists.
    """
    cores, coeffs = make_batch_sums_stacked(B, d, n, r, seed, eps3, eps4, omega_odd, start)
    return [([[cores[s][k][b] for k in range(d)] for s in range(4)], [float(v) for v in coeffs[b]])
            for b in range(B)]


def _qfactor_batched(g: np.ndarray) -> np.ndarray:
    """_qfactor over a stack (..., M, N): LAPACK per matrix, same result as one at a time."""
    q, r = np.linalg.qr(g, mode="reduced")
    s = np.sign(np.diagonal(r, axis1=-2, axis2=-1)).copy()
    s[s == 0] = 1.0
    return q * s[..., None, :]


def make_batch_sums_stacked(B: int, d: int = 10, n: int = 32, r: int = 16, seed: int = SEED_BASE + 4,
                            eps3: float = 1e-9, eps4: float = 1e-10, omega_odd: float = 1e-9,
                            start: int = 0):
    """Same bytes as make_batch_sums(B, ..., start), stacked for the batched API: returns
    (cores, coeffs) with cores[s][k] of shape (B, r_{k-1}, n, r_k) = core k of y_{b,s} for
    b in [start, start+B), coeffs (B, 4).  One standard_normal draw in the documented order
    (b-major, then s, then the cores of y_{b,s}), then the per-core QRs batched."""
    ranks = tt_ranks_capped(d, [n] * d, r)
    sizes = [ranks[k] * n * ranks[k + 1] for k in range(d)]
    per = sum(sizes)
    rng = _rng(seed)
    skip = start * 4 * per
    while skip > 0:  # advance the stream past items [0, start) without holding them
        c = min(skip, 1 << 26)
        rng.standard_normal(c)
        skip -= c
    g = rng.standard_normal(B * 4 * per).reshape(B, 4, per)
    cores = [[None] * d for _ in range(4)]
    off = 0
    for k in range(d):
        blk = g[:, :, off:off + sizes[k]].reshape(B, 4, ranks[k], n, ranks[k + 1])
        off += sizes[k]
        if k == 0:
            c = blk / np.linalg.norm(blk.reshape(B, 4, -1), axis=2)[:, :, None, None, None]
        else:
            r0, r1 = ranks[k], ranks[k + 1]
            q = _qfactor_batched(np.swapaxes(blk.reshape(B, 4, r0, n * r1), -1, -2))  # (B,4,n r1,r0)
            c = np.swapaxes(q, -1, -2).reshape(B, 4, r0, n, r1)
        for s in range(4):
            cores[s][k] = np.ascontiguousarray(c[:, s])
    w = np.where((np.arange(start, start + B) % 2) == 0, 1.0, omega_odd)
    coeffs = np.stack([np.ones(B), w, np.full(B, eps3), np.full(B, eps4)], axis=1)
    return cores, coeffs


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    drivers: Tuple[str, ...]
    m: int
    d: int
    n: int
    r: int
    kappa: float
    delta: float
    seed: int
    batch: int = 0
    note: str = ""


CONFIGS = {
    "C1": ConfigSpec("C1", ("cgs",), 10, 4, 8, 3, 1e8, 1e-8, SEED_BASE + 1,
                     note="BASELINE.json configs[0]"),
    "C2": ConfigSpec("C2", ("mgs", "mgs2"), 30, 8, 32, 10, 1e10, 1e-10, SEED_BASE + 2,
                     note="BASELINE.json configs[1]; the bench workload"),
    "C3": ConfigSpec("C3", ("cgs2", "gram"), 50, 16, 64, 20, 1e6, 1e-5, SEED_BASE + 3,
                     note="delta not given by BASELINE.json; 1e-5 is a paper value (SURVEY A13)"),
    "C4": ConfigSpec("C4", ("batch",), 0, 10, 32, 16, 0.0, 1e-6, SEED_BASE + 4, batch=4096),
    "C5": ConfigSpec("C5", ("householder",), 100, 50, 16, 30, 1e12, 1e-12, SEED_BASE + 5),
}


def config_spec(name: str) -> ConfigSpec:
    return CONFIGS[name]


def make_fuzz_batch(seed: int):
    """Randomised batch for the batched engine's parity sweep (tools/fuzz_batch.py,
    tests/test_gpu_batch.py): random order, mode sizes, term count and ranks (formal rank <= 64),
    optionally graded rank slices (unfolding spectra over many decades), mixed term scales and --
    only with the noise floor on -- near cancellation of the first and last term.  Returns
    (items, delta, floor_c, description); items = [(terms, coeffs), ...].  floor_c is 0.0 (off) or
    None (the caller's default constant)."""
    rng = np.random.Generator(np.random.PCG64(50000 + seed))
    d = int(rng.integers(2, 8))
    n = [int(v) for v in rng.integers(1, 33, size=d)]
    K = int(rng.integers(1, 6))
    rmax = max(1, 64 // K)
    ranks = [[1] + [int(v) for v in rng.integers(1, rmax + 1, size=d - 1)] + [1] for _ in range(K)]
    delta = float(rng.choice([0.0, 1e-1, 1e-3, 1e-6, 1e-10, 1e-14]))
    floor_off = delta == 0.0 or rng.random() < 0.3
    graded = rng.random() < 0.5
    mixed = rng.random() < 0.3
    B = int(rng.integers(1, 4))
    items = []
    for _ in range(B):
        terms = []
        for r in ranks:
            t = make_random_tt(d, n, r, rng)
            if graded:
                for k in range(d - 1):
                    g = 10.0 ** (-rng.uniform(0, 16.0 / max(1, d - 1)) * np.arange(r[k + 1]) / max(1, r[k + 1] - 1))
                    t[k] = t[k] * g[None, None, :]
            if mixed:
                t[0] = t[0] * 10.0 ** float(rng.integers(-40, 41))
            terms.append(t)
        coeffs = [float(v) for v in rng.standard_normal(K)]
        cancel = K >= 2 and rng.random() < 0.3
        if cancel and not floor_off:  # with the floor off the ranks of a cancelling sum are noise (A12)
            terms[-1] = terms[0]
            coeffs[-1] = -coeffs[0] * (1.0 + float(rng.choice([0.0, 1e-12, 1e-7])))
        items.append((terms, coeffs))
    desc = (f"seed {seed} d={d} n={n} K={K} ranks={ranks} delta={delta} floor={'off' if floor_off else 'on'} "
            f"graded={graded} mixed={mixed}")
    return items, delta, (0.0 if floor_off else None), desc
