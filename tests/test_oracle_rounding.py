"""Pins for oracle/rounding.py (TT-rounding).

Pins: dense reconstruction (delta = 0 reproduces x; the contract ||x - x~|| <= delta ||x||
checked on densified tensors), the d = 2 case reduces to the truncated SVD of a matrix
(Eckart-Young, checked against scipy's gesvd driver), exact rank collapse of x + x,
idempotence, monotone ranks, degenerate inputs, and the C4 closed form.
"""
import numpy as np
import pytest
import scipy.linalg

from oracle import rounding, tt
from oracle.dense import U_ROUND
from ttinputs import make_batch_sums, make_random_tt


def _rng(s):
    return np.random.Generator(np.random.PCG64(s))


def _dense_err(x, y):
    return float(np.linalg.norm(tt.densify(x) - tt.densify(y)))


@pytest.mark.parametrize("seed", range(8))
def test_delta_zero_reproduces(seed):
    rng = _rng(100 + seed)
    d = 2 + seed % 4
    n = [int(v) for v in rng.integers(2, 5, size=d)]
    a = make_random_tt(d, n, [1] + [int(v) for v in rng.integers(1, 4, size=d - 1)] + [1], rng)
    b = make_random_tt(d, n, [1] + [int(v) for v in rng.integers(1, 4, size=d - 1)] + [1], rng)
    x = tt.tt_sum([a, b, a], [1.0, -0.5, 2.0])          # rank-deficient on purpose
    y, info = rounding.tt_round(x, 0.0)
    nx = np.linalg.norm(tt.densify(x))
    assert _dense_err(x, y) <= 1e-13 * nx
    assert abs(info.norm - nx) <= 1e-13 * nx
    # delta = 0 keeps the structural caps: rank_k = min(prod n_<=k, prod n_>k, R'_k)
    for k in range(1, d):
        assert info.ranks[k] <= info.formal_ranks[k]


def test_contract_200_cases():
    """SPEC.md:631 acceptance 1: ||x - round(x, delta)|| <= delta ||x|| via densify."""
    rng = _rng(7)
    count = 0
    for case in range(200):
        d = int(rng.integers(2, 5))
        n = [int(v) for v in rng.integers(2, 7, size=d)]
        r = [1] + [int(v) for v in rng.integers(1, 5, size=d - 1)] + [1]
        x = make_random_tt(d, n, r, rng)
        y0 = make_random_tt(d, n, r, rng)
        x = tt.tt_sum([x, y0], [1.0, 10.0 ** -rng.integers(0, 5)])
        delta = [1e-2, 1e-4, 1e-8][case % 3]
        y, info = rounding.tt_round(x, delta)
        nx = np.linalg.norm(tt.densify(x))
        assert _dense_err(x, y) <= delta * nx * (1 + 1e-10) + 1e-14 * nx
        assert all(a <= b for a, b in zip(info.ranks, info.formal_ranks))
        count += int(any(a < b for a, b in zip(info.ranks, info.formal_ranks)))
    assert count > 50  # truncation actually happened in many cases


@pytest.mark.parametrize("seed", range(5))
def test_d2_is_truncated_matrix_svd(seed):
    """d = 2: x is the n1 x n2 matrix X_1 X_2; rounding keeps the top-rho singular triplets
    with rho the smallest rank whose tail <= delta ||X||_F (sqrt(d-1) = 1), so the error is
    exactly the tail (Eckart-Young).  Reference singular values from scipy gesvd."""
    rng = _rng(200 + seed)
    n1, n2, r = 9, 7, 6
    x = make_random_tt(2, [n1, n2], [1, r, 1], rng)
    Xd = tt.densify(x).reshape(n2, n1).T  # psi order: i_1 fastest
    s = scipy.linalg.svd(Xd, compute_uv=False, lapack_driver="gesvd")
    delta = float(s[3] / np.linalg.norm(Xd)) * 1.0001   # threshold between sigma_3.. tails
    y, info = rounding.tt_round(x, delta)
    tau = delta * np.linalg.norm(Xd)
    tails = [np.sqrt(np.sum(s[k:] ** 2)) for k in range(len(s) + 1)]
    rho = next(k for k in range(1, len(s) + 1) if tails[k] <= tau)
    assert info.ranks == [1, rho, 1]
    assert _dense_err(x, y) == pytest.approx(tails[rho], rel=1e-9, abs=1e-13)
    np.testing.assert_allclose(info.sigmas[0][:r], s[:r], rtol=1e-12, atol=1e-14 * s[0])


def test_rank_collapse_x_plus_x():
    """round(x + x) has the ranks of x."""
    rng = _rng(9)
    x = make_random_tt(4, [4, 5, 4, 3], [1, 2, 3, 2, 1], rng)
    y, info = rounding.tt_round(tt.tt_sum([x, x]), 1e-10, floor_c=rounding.DEFAULT_FLOOR_C,
                                scale=2 * tt.tt_norm(x))
    assert info.ranks == tt.ranks(x)
    assert _dense_err(y, tt.tt_scale(x, 2.0)) <= 1e-10 * 2 * tt.tt_norm(x)


def test_idempotent_and_monotone():
    rng = _rng(11)
    a = make_random_tt(4, 4, [1, 3, 4, 3, 1], rng)
    b = make_random_tt(4, 4, [1, 2, 2, 2, 1], rng)
    x = tt.tt_sum([a, b], [1.0, 1e-3])
    y, i1 = rounding.tt_round(x, 1e-2)
    z, i2 = rounding.tt_round(y, 1e-2)
    assert i2.ranks == i1.ranks
    assert _dense_err(y, z) <= 1e-2 * tt.tt_norm(y)
    assert all(p <= q for p, q in zip(i1.ranks, i1.formal_ranks))


def test_degenerate_inputs():
    n = [3, 4, 2]
    z = [np.zeros((1, 3, 2)), np.zeros((2, 4, 2)), np.zeros((2, 2, 1))]
    y, info = rounding.tt_round(z, 1e-6)
    assert info.ranks == [1, 1, 1, 1] and info.norm == 0.0
    assert np.all(tt.densify(y) == 0.0)
    x1 = [np.arange(5.0).reshape(1, 5, 1)]
    y1, _ = rounding.tt_round(x1, 1e-3)
    assert np.array_equal(y1[0], x1[0])                      # d = 1 unchanged
    e = tt.canonical_tt(7, n)
    y, info = rounding.tt_round(e, 1e-3)
    assert info.ranks == [1, 1, 1, 1]
    assert _dense_err(y, e) <= 1e-15
    rng = _rng(12)
    x = make_random_tt(3, n, [1, 3, 2, 1], rng)
    y, info = rounding.tt_round(x, 0.0, max_rank=1)
    assert info.ranks == [1, 1, 1, 1]


def test_cancelled_sum_is_zero_with_floor():
    rng = _rng(13)
    x = make_random_tt(4, 5, [1, 3, 3, 3, 1], rng)
    nx = tt.tt_norm(x)
    y, info = rounding.tt_round(tt.tt_sum([x, x], [1.0, -1.0]), 1e-8,
                                floor_c=rounding.DEFAULT_FLOOR_C, scale=2 * nx)
    assert info.norm <= 64 * U_ROUND * 2 * nx
    assert max(info.ranks) == 1


def test_c4_closed_form():
    """x_b = y1 + w_b y2 + 1e-9 y3 + 1e-10 y4 (unit-norm y) at delta = 1e-6
    rounds to ranks 32 (even b) / 16 (odd b) and to y1 + [w_b = 1] y2 within ~2e-9."""
    items = make_batch_sums(4)
    for b, (terms, coeffs) in enumerate(items):
        y, info = rounding.tt_round(tt.tt_sum(terms, coeffs), 1e-6)
        want = 32 if b % 2 == 0 else 16
        assert info.ranks == [1] + [want] * 9 + [1]
        ref = tt.tt_sum(terms[:2], [1.0, 1.0]) if b % 2 == 0 else terms[0]
        _, dinfo = rounding.tt_round(tt.tt_sum([y, ref], [1.0, -1.0]), 0.0)  # sweep norm
        assert dinfo.norm <= 5e-9 * info.norm
