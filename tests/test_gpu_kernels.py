"""GPU parity of the TT kernels against the oracle (through the C ABI)."""
import numpy as np
import pytest

from oracle import orth, rounding, tt
from ttinputs import CONFIGS, make_random_tt, make_shared_tail_set

from gpu_util import ctx, cuda_ok, dev

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _rng(s):
    return np.random.Generator(np.random.PCG64(s))


def _rand(rng, d, n, rmax):
    r = [1] + [int(v) for v in rng.integers(1, rmax + 1, size=d - 1)] + [1]
    return make_random_tt(d, n, r, rng)


def test_dot_batch_ragged():
    """Relative to ||x|| ||y|| (the dot itself can cancel): <= 1e-12 (north star)."""
    import paper_2211_08770_b200 as P
    c = ctx()
    rng = _rng(1)
    xs, ys, ref, sc = [], [], [], []
    for p in range(40):
        d = int(rng.integers(1, 7))
        n = [int(v) for v in rng.integers(1, 9, size=d)]
        x = _rand(rng, d, n, 9)
        y = _rand(rng, d, n, 13)
        xs.append(dev(x)); ys.append(dev(y))
        ref.append(tt.tt_dot(x, y)); sc.append(tt.tt_norm(x) * tt.tt_norm(y))
    # the kernel groups pairs of different shapes only when d and n agree; test per pair
    for p in range(40):
        got = P.tt_dot_batch(c, [xs[p]], [ys[p]]).cpu().numpy()[0]
        assert abs(got - ref[p]) <= 1e-12 * sc[p], p


def test_dot_batch_many_pairs_same_shape():
    import paper_2211_08770_b200 as P
    c = ctx()
    rng = _rng(2)
    d, n = 6, [7, 5, 8, 3, 9, 4]
    xs = [_rand(rng, d, n, 24) for _ in range(17)]
    ys = [_rand(rng, d, n, 31) for _ in range(17)]
    got = P.tt_dot_batch(c, [dev(x) for x in xs], [dev(y) for y in ys]).cpu().numpy()
    for p in range(17):
        assert abs(got[p] - tt.tt_dot(xs[p], ys[p])) <= 1e-12 * tt.tt_norm(xs[p]) * tt.tt_norm(ys[p])


def test_dot_batch_uniform_blocks_gram_route():
    """Equally shaped operands take the pair-tiled Gram route: a row block (one x against a
    set), a column block, a repeated pair and isolated pairs, output in pair order."""
    import paper_2211_08770_b200 as P
    c = ctx()
    rng = _rng(4)
    d, n, r = 5, [6, 4, 7, 5, 3], [1, 5, 7, 6, 4, 1]
    ts = [make_random_tt(d, n, r, rng) for _ in range(9)]
    dv = [dev(t) for t in ts]
    pairs = [(0, j) for j in range(1, 9)] + [(i, 8) for i in range(2, 6)] + [(3, 3), (3, 3), (7, 1), (2, 6)]
    got = P.tt_dot_batch(c, [dv[i] for i, _ in pairs], [dv[j] for _, j in pairs]).cpu().numpy()
    for q, (i, j) in enumerate(pairs):
        assert abs(got[q] - tt.tt_dot(ts[i], ts[j])) <= 1e-12 * tt.tt_norm(ts[i]) * tt.tt_norm(ts[j]), q


def test_dot_batch_two_rank_profiles_gram_route():
    """First operands share one rank profile, second operands another (a projection of x on a
    set Q): row and column blocks with I-side and J-side shapes that differ per core."""
    import paper_2211_08770_b200 as P
    c = ctx()
    rng = _rng(5)
    d, n = 5, [6, 4, 7, 5, 3]
    qs = [make_random_tt(d, n, [1, 5, 7, 6, 4, 1], rng) for _ in range(7)]
    xs = [make_random_tt(d, n, [1, 3, 9, 2, 5, 1], rng) for _ in range(3)]
    pairs = [(qs[i], xs[0]) for i in range(7)] + [(qs[2], xs[j]) for j in range(3)] + [(qs[5], xs[1])]
    got = P.tt_dot_batch(c, [dev(a) for a, _ in pairs], [dev(b) for _, b in pairs]).cpu().numpy()
    for q, (a, b) in enumerate(pairs):
        assert abs(got[q] - tt.tt_dot(a, b)) <= 1e-12 * tt.tt_norm(a) * tt.tt_norm(b), q


def test_dot_batch_large_ranks_gemm_route():
    """Ranks above 32 (unequal profiles) take the per-core grouped DMMA GEMM route: several pairs with different
    rank profiles (and a pair of small x against large y)."""
    import paper_2211_08770_b200 as P
    c = ctx()
    rng = _rng(6)
    d, n = 4, [5, 3, 4, 6]
    xs = [make_random_tt(d, n, [1, 5, 15, 60, 1], rng), make_random_tt(d, n, [1, 3, 9, 6, 1], rng),
          make_random_tt(d, n, [1, 5, 14, 49, 1], rng)]
    ys = [make_random_tt(d, n, [1, 5, 15, 55, 1], rng), make_random_tt(d, n, [1, 5, 15, 70, 1], rng),
          make_random_tt(d, n, [1, 4, 12, 20, 1], rng)]
    got = P.tt_dot_batch(c, [dev(x) for x in xs], [dev(y) for y in ys]).cpu().numpy()
    for q in range(3):
        assert abs(got[q] - tt.tt_dot(xs[q], ys[q])) <= 1e-12 * tt.tt_norm(xs[q]) * tt.tt_norm(ys[q]), q


def test_dot_large_rank_global_path():
    """Ranks large enough that the per-pair workspace leaves shared memory."""
    import paper_2211_08770_b200 as P
    c = ctx()
    rng = _rng(3)
    x = make_random_tt(3, 4, [1, 4, 130, 1], rng)
    y = make_random_tt(3, 4, [1, 4, 150, 1], rng)
    got = P.tt_dot_batch(c, [dev(x)], [dev(y)]).cpu().numpy()[0]
    assert abs(got - tt.tt_dot(x, y)) <= 1e-12 * tt.tt_norm(x) * tt.tt_norm(y)


@pytest.mark.parametrize("cfg", ["C1", "C3"])
def test_gram_closed_form_and_oracle(cfg):
    """G = M^T M exactly for the shared-tail inputs (C1 full; C3 full shape, m reduced)."""
    import paper_2211_08770_b200 as P
    c = CONFIGS[cfg]
    m = c.m if cfg == "C1" else 12
    st = make_shared_tail_set(c.d, c.n, c.r, m, c.kappa, c.seed)
    G = P.tt_gram(ctx(), [dev(a) for a in st.tensors]).cpu().numpy()
    Gx = st.gram_exact()
    assert np.linalg.norm(G - Gx) <= 1e-10 * np.linalg.norm(Gx)
    Go = orth.gram_matrix(st.tensors)
    assert np.linalg.norm(G - Go) <= 1e-12 * np.linalg.norm(Go)
    assert np.array_equal(G, G.T)


def test_gram_blocks_pack():
    import paper_2211_08770_b200 as P
    rng = _rng(4)
    A = [_rand(rng, 4, 5, 4) for _ in range(7)]
    blocks = [(0, 0, 3, 3), (3, 0, 4, 3), (3, 3, 4, 4)]
    packed = P.tt_gram_blocks(ctx(), [dev(a) for a in A], blocks).cpu().numpy()
    G = orth.gram_matrix(A)
    o = 0
    for i0, j0, bi, bj in blocks:
        blk = packed[o:o + bi * bj].reshape(bi, bj)
        o += bi * bj
        np.testing.assert_allclose(blk, G[i0:i0 + bi, j0:j0 + bj], rtol=1e-12, atol=1e-12 * np.abs(G).max())


def test_element_matches_oracle():
    import paper_2211_08770_b200 as P
    rng = _rng(5)
    n = [4, 3, 5, 2]
    x = make_random_tt(4, n, [1, 3, 7, 2, 1], rng)
    lins = [1, 2, 17, 60, 120, 33]
    got = P.tt_element(ctx(), dev(x), lins).cpu().numpy()
    for t, l in enumerate(lins):
        ref = tt.element(x, [i - 1 for i in tt.phi(l, n)])
        assert abs(got[t] - ref) <= 1e-14 * (1 + abs(ref))
    with pytest.raises(Exception):
        P.tt_element(ctx(), dev(x), [121])


def test_tt_sum_bitexact():
    import paper_2211_08770_b200 as P
    rng = _rng(6)
    n = [3, 4, 2, 5]
    a = make_random_tt(4, n, [1, 2, 3, 2, 1], rng)
    b = make_random_tt(4, n, [1, 1, 4, 3, 1], rng)
    s = P.tt_sum(ctx(), [dev(a), dev(b)], [0.5, -2.0]).to_numpy()
    ref = tt.tt_sum([a, b], [0.5, -2.0])
    assert [c.shape for c in s] == [c.shape for c in ref]
    for x, y in zip(s, ref):
        assert np.array_equal(x, y)


def test_norm_sweep():
    import paper_2211_08770_b200 as P
    rng = _rng(7)
    x = make_random_tt(5, 6, [1, 4, 9, 9, 4, 1], rng)
    assert P.tt_norm(ctx(), dev(x)) == pytest.approx(tt.tt_norm(x), rel=1e-13)


@pytest.mark.parametrize("seed", range(8))
def test_gram_tiled_matches_oracle_and_pairwise(seed):
    """Pair-tiled Gram kernel (equal shapes; odd m, ragged ranks up to 32, d from 1) against the
    oracle (1e-12 ||a_i|| ||a_j||) and the per-pair kernel (TT_B200_GRAM_PAIRWISE)."""
    import os
    import paper_2211_08770_b200 as P
    from oracle import tt
    from ttinputs import make_random_tt
    rng = np.random.Generator(np.random.PCG64(500 + seed))
    d = int(rng.integers(1, 6))
    n = [int(v) for v in rng.integers(1, 12, size=d)]
    r = [1] + [int(v) for v in rng.integers(1, 33, size=d - 1)] + [1]
    m = int(rng.integers(1, 12))
    A = [make_random_tt(d, n, r, rng) for _ in range(m)]
    G = P.tt_gram(ctx(), [dev(a) for a in A]).cpu().numpy()
    nr = np.array([tt.tt_norm(a) for a in A])
    Go = np.array([[tt.tt_dot(a, b) for b in A] for a in A])
    assert np.all(np.abs(G - Go) <= 1e-12 * np.outer(nr, nr))
    assert np.array_equal(G, G.T)
    os.environ["TT_B200_GRAM_PAIRWISE"] = "1"
    try:
        Gp = P.tt_gram(ctx(), [dev(a) for a in A]).cpu().numpy()
    finally:
        del os.environ["TT_B200_GRAM_PAIRWISE"]
    assert np.all(np.abs(G - Gp) <= 1e-13 * np.outer(nr, nr))
