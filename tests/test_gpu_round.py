"""GPU parity of TT-rounding (tt_round / tt_round_batch) against the oracle.

Bar (north star): ranks identical except where the oracle's tail lies within
the documented window around tau; reconstructions agree to 1e-10 s(x) (TT-difference norm
by an exact oracle rounding); the error contract holds on the GPU output.
"""
import numpy as np
import pytest

from oracle import rounding, tt
from ttinputs import make_batch_sums, make_random_tt, make_shared_tail_set

from gpu_util import assert_round_parity, ctx, cuda_ok, dev, diff_norm

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _rng(s):
    return np.random.Generator(np.random.PCG64(s))


def _case(seed):
    rng = _rng(seed)
    d = int(rng.integers(2, 7))
    n = [int(v) for v in rng.integers(2, 9, size=d)]
    K = int(rng.integers(1, 5))
    terms = []
    for _ in range(K):
        r = [1] + [int(v) for v in rng.integers(1, 6, size=d - 1)] + [1]
        terms.append(make_random_tt(d, n, r, rng))
    coeffs = [float(v) for v in rng.standard_normal(K)]
    if K >= 2:
        terms.append(terms[0])           # exact rank deficiency / cancellation
        coeffs.append(-0.5 * coeffs[0])
    return terms, coeffs


@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("delta", [0.0, 1e-2, 1e-8])
def test_round_random_sums(seed, delta):
    import paper_2211_08770_b200 as P
    terms, coeffs = _case(seed)
    floor_c = 0.0 if delta == 0.0 else rounding.DEFAULT_FLOOR_C
    norms = [tt.tt_norm(t) for t in terms]
    ref, info = rounding.tt_round_sum(terms, coeffs, delta, floor_c=floor_c, term_norms=norms)
    out, ginfo = P.tt_round(ctx(), [dev(t, nr) for t, nr in zip(terms, norms)], coeffs, delta, floor_c=floor_c)
    g = out.to_numpy()
    assert abs(ginfo["norm"] - info.norm) <= 1e-13 * info.scale
    assert_round_parity(g, out.ranks, terms, coeffs, delta, floor_c, norms, info=info, ref=ref, tag=f"round{seed}")
    x = tt.tt_sum(terms, coeffs)
    s = info.scale
    # the contract ||x - x~|| <= delta ||x|| (+ floor) on the GPU output itself
    d = len(terms[0])
    tol = max(delta * info.norm, np.sqrt(d - 1) * info.tau) * (1 + 1e-8) + 1e-13 * s
    assert diff_norm(x, g) <= tol
    # left-orthonormal cores 1..d-1
    for k in range(d - 1):
        U = g[k].reshape(-1, g[k].shape[2])
        assert np.linalg.norm(U.T @ U - np.eye(U.shape[1])) <= 1e-12


def test_round_zero_and_d1():
    import paper_2211_08770_b200 as P
    rng = _rng(50)
    x = make_random_tt(4, 5, [1, 3, 3, 3, 1], rng)
    out, info = P.tt_round(ctx(), [dev(x), dev(x)], [1.0, -1.0], 1e-8)
    assert max(out.ranks) == 1
    assert info["norm"] <= 1e-12 * tt.tt_norm(x)
    x1 = [rng.standard_normal((1, 7, 1))]
    out, _ = P.tt_round(ctx(), [dev(x1), dev(x1)], [2.0, 1.0], 1e-3)
    np.testing.assert_allclose(out.to_numpy()[0], 3.0 * x1[0], rtol=1e-15)


def test_round_c2_shape_mgs_like_sum():
    """One MGS-like sum at the C2 shape (d=8, n=32, r=10, 12 terms), against the oracle."""
    import paper_2211_08770_b200 as P
    st = make_shared_tail_set(8, 32, 10, 12, 1e4, seed=77)
    rng = _rng(51)
    coeffs = [1.0] + [float(v) for v in rng.standard_normal(11) * 0.3]
    terms = st.tensors
    norms = [tt.tt_norm(t) for t in terms]
    ref, info = rounding.tt_round_sum(terms, coeffs, 1e-10, floor_c=rounding.DEFAULT_FLOOR_C, term_norms=norms)
    out, ginfo = P.tt_round(ctx(), [dev(t, nr) for t, nr in zip(terms, norms)], coeffs, 1e-10)
    assert out.ranks == info.ranks == [1] + [10] * 7 + [1]
    assert diff_norm(out.to_numpy(), ref) <= 1e-10 * info.scale


def test_round_c4_closed_form_batch():
    """C4 items: ranks 32 (even b) / 16 (odd b); distance to y1 + [b even] y2 <= 5e-9 ||x||."""
    import paper_2211_08770_b200 as P
    items = make_batch_sums(6)
    batch = [([dev(t, 1.0) for t in terms], coeffs) for terms, coeffs in items]
    outs = P.tt_round_batch(ctx(), batch, 1e-6)
    for b, ((terms, coeffs), o) in enumerate(zip(items, outs)):
        want = 32 if b % 2 == 0 else 16
        assert o.ranks == [1] + [want] * 9 + [1]
        refx = tt.tt_sum(terms[:2], [1.0, 1.0]) if b % 2 == 0 else terms[0]
        g = o.to_numpy()
        assert diff_norm(g, refx) <= 5e-9 * np.sqrt(2.0)
        cpu, info = rounding.tt_round_sum(terms, coeffs, 1e-6, floor_c=rounding.DEFAULT_FLOOR_C,
                                          term_norms=[1.0] * 4)
        assert info.ranks == o.ranks
        assert diff_norm(g, cpu) <= 1e-10 * info.scale


def test_round_theta_small_equals_exact_decision():
    """A tiny QRCP stopping fraction must give the same result as the default (the rank
    decision is the exact-SVD decision either way)."""
    import paper_2211_08770_b200 as P
    terms, coeffs = _case(99)
    o1, _ = P.tt_round(ctx(), [dev(t) for t in terms], coeffs, 1e-3, theta=0.5)
    o2, _ = P.tt_round(ctx(), [dev(t) for t in terms], coeffs, 1e-3, theta=1e-6)
    assert o1.ranks == o2.ranks
    assert diff_norm(o1.to_numpy(), o2.to_numpy()) <= 1e-12 * max(tt.tt_norm(t) for t in terms) * len(terms)


@pytest.mark.parametrize("distinct", [5, 30])
def test_round_tall_panels_qr_then_qrcp(distinct):
    """Right-to-left panels taller than 2c and beyond one cluster (4096 x 480, 5120 x 480) take
    the blocked-QR-then-pivoted-QR-of-R path; with 5 distinct tensors repeated (structural rank
    480, numerical rank 80) the pivoted QR drops rank, with 30 distinct ones it keeps it."""
    import paper_2211_08770_b200 as P
    rng = _rng(60 + distinct)
    d, n, r = 4, 64, 16
    base = [make_random_tt(d, [n] * d, [1, r, r, r, 1], rng) for _ in range(distinct)]
    terms = [base[i % distinct] for i in range(30)]
    coeffs = [float(v) for v in rng.standard_normal(30)]
    norms = [tt.tt_norm(t) for t in terms]
    ref, info = rounding.tt_round_sum(terms, coeffs, 1e-8, floor_c=rounding.DEFAULT_FLOOR_C, term_norms=norms)
    out, ginfo = P.tt_round(ctx(), [dev(t, nr) for t, nr in zip(terms, norms)], coeffs, 1e-8)
    assert abs(ginfo["norm"] - info.norm) <= 1e-13 * info.scale
    if distinct == 5:
        assert out.ranks == [1, 64, 80, 64, 1]
    g = out.to_numpy()
    assert_round_parity(g, out.ranks, terms, coeffs, 1e-8, rounding.DEFAULT_FLOOR_C, norms, info=info, ref=ref,
                        tag="tall")
    x = tt.tt_sum(terms, coeffs)
    assert diff_norm(x, g) <= 1e-8 * info.norm * (1 + 1e-8) + np.sqrt(d - 1) * info.tau


def test_round_wide_panel_grid_qrcp():
    """A 1024 x 1000 right-to-left panel (beyond one cluster, not tall) goes through the
    grid-cooperative pivoted QR; 10 distinct tensors repeated 5 times, the left part has rank
    <= n_1 = 32, so the pivoted QR drops 1000 columns to 32."""
    import paper_2211_08770_b200 as P
    rng = _rng(70)
    d, n, r = 3, 32, 20
    base = [make_random_tt(d, [n] * d, [1, r, r, 1], rng) for _ in range(10)]
    terms = [base[i % 10] for i in range(50)]
    coeffs = [float(v) for v in rng.standard_normal(50)]
    norms = [tt.tt_norm(t) for t in terms]
    ref, info = rounding.tt_round_sum(terms, coeffs, 1e-10, floor_c=rounding.DEFAULT_FLOOR_C, term_norms=norms)
    out, ginfo = P.tt_round(ctx(), [dev(t, nr) for t, nr in zip(terms, norms)], coeffs, 1e-10)
    assert abs(ginfo["norm"] - info.norm) <= 1e-13 * info.scale
    g = out.to_numpy()
    assert_round_parity(g, out.ranks, terms, coeffs, 1e-10, rounding.DEFAULT_FLOOR_C, norms, info=info, ref=ref,
                        tag="grid_qrcp")
    x = tt.tt_sum(terms, coeffs)
    assert diff_norm(x, g) <= 1e-10 * info.norm * (1 + 1e-8) + np.sqrt(d - 1) * info.tau


def test_round_large_rank_grid_jacobi():
    """Kept ranks >= 128 take the whole-GPU Jacobi (same rotations as the one-CTA kernel):
    10 random rank-14 terms with n = (160, 8, 160) keep rank 140 on both bonds."""
    import paper_2211_08770_b200 as P
    rng = _rng(80)
    n = [160, 8, 160]
    terms = [make_random_tt(3, n, [1, 14, 14, 1], rng) for _ in range(10)]
    coeffs = [float(v) for v in rng.standard_normal(10)]
    norms = [tt.tt_norm(t) for t in terms]
    ref, info = rounding.tt_round_sum(terms, coeffs, 1e-10, floor_c=rounding.DEFAULT_FLOOR_C, term_norms=norms)
    out, ginfo = P.tt_round(ctx(), [dev(t, nr) for t, nr in zip(terms, norms)], coeffs, 1e-10)
    assert min(out.ranks[1:-1]) >= 128
    g = out.to_numpy()
    assert_round_parity(g, out.ranks, terms, coeffs, 1e-10, rounding.DEFAULT_FLOOR_C, norms, info=info, ref=ref,
                        tag="grid_jacobi")
    for k in range(2):
        U = g[k].reshape(-1, g[k].shape[2])
        assert np.linalg.norm(U.T @ U - np.eye(U.shape[1])) <= 1e-12
