"""GPU parity of the batched TT-rounding engine (tt_round_batch on uniform batches,
csrc/batch_round.cu) against the oracle (BASELINE.json configs[3], "C4").

Every item is compared with oracle.rounding.tt_round_sum on the same bytes: ranks identical
(or inside the documented window around tau), reconstruction within 1e-10 s(x) (TT-difference
norm through an exact oracle rounding), the rounding contract on the GPU output, and
left-orthonormal cores 1..d-1.  Shapes span one stack (<= 192 panel rows), several stacks with
a ragged tail, d = 2, single-term sums, exact cancellation, delta = 0, max_rank and unknown
term norms (computed on the device).
"""
import os

import numpy as np
import pytest

from oracle import rounding, tt
from ttinputs import make_batch_sums, make_random_tt

from gpu_util import assert_round_parity, ctx, cuda_ok, dev, diff_norm

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _rng(s):
    return np.random.Generator(np.random.PCG64(s))


def _batch(seed):
    """B items sharing d, n, K and term ranks (formal ranks <= 64)."""
    rng = _rng(1000 + seed)
    d = int(rng.integers(2, 7))
    n = [int(v) for v in rng.integers(2, 41, size=d)]
    K = int(rng.integers(1, 5))
    rmax = max(1, 60 // (K + 1))
    ranks = []
    for _ in range(K):
        ranks.append([1] + [int(v) for v in rng.integers(1, rmax + 1, size=d - 1)] + [1])
    dup = K >= 2 and seed % 2 == 0      # last term repeats the first: exact cancellation
    B = int(rng.integers(1, 6))
    items = []
    for _ in range(B):
        terms = [make_random_tt(d, n, r, rng) for r in ranks]
        coeffs = [float(v) for v in rng.standard_normal(K)]
        if dup:
            terms.append(terms[0])
            coeffs.append(-0.5 * coeffs[0])
        items.append((terms, coeffs))
    return items


def _check_item(g, ranks, terms, coeffs, delta, floor_c, norms=None, max_rank=None):
    if norms is None:
        norms = [tt.tt_norm(t) for t in terms]
    info = assert_round_parity(g, ranks, terms, coeffs, delta, floor_c, norms, max_rank=max_rank, tag="batch")
    s = info.scale
    d = len(terms[0])
    if max_rank is None:
        x = tt.tt_sum(terms, coeffs)
        tol = max(delta * info.norm, np.sqrt(d - 1) * info.tau) * (1 + 1e-8) + 1e-13 * s
        assert diff_norm(x, g) <= tol
    if delta > 0.0:
        for k in range(d - 1):
            U = g[k].reshape(-1, g[k].shape[2])
            assert np.linalg.norm(U.T @ U - np.eye(U.shape[1])) <= 1e-12
    return info


@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("delta", [0.0, 1e-2, 1e-8])
def test_batch_random_uniform(seed, delta):
    import paper_2211_08770_b200 as P
    items = _batch(seed)
    floor_c = 0.0 if delta == 0.0 else rounding.DEFAULT_FLOOR_C
    norms = [[tt.tt_norm(t) for t in terms] for terms, _ in items]
    batch = [([dev(t, nr) for t, nr in zip(terms, nb)], coeffs) for (terms, coeffs), nb in zip(items, norms)]
    outs = P.tt_round_batch(ctx(), batch, delta, floor_c=floor_c)
    for (terms, coeffs), nb, o in zip(items, norms, outs):
        _check_item(o.to_numpy(), o.ranks, terms, coeffs, delta, floor_c, norms=nb)


def test_batch_matches_serial_path():
    """The batched engine and the per-item rounding (TT_B200_BATCH_SERIAL=1) agree."""
    import paper_2211_08770_b200 as P
    items = _batch(3) + _batch(3)
    batch = [([dev(t) for t in terms], coeffs) for terms, coeffs in items]
    outs = P.tt_round_batch(ctx(), batch, 1e-6)
    os.environ["TT_B200_BATCH_SERIAL"] = "1"
    try:
        ser = P.tt_round_batch(ctx(), batch, 1e-6)
    finally:
        del os.environ["TT_B200_BATCH_SERIAL"]
    for (terms, coeffs), a, b in zip(items, outs, ser):
        s = sum(abs(c) * tt.tt_norm(t) for t, c in zip(terms, coeffs))
        assert a.ranks == b.ranks
        assert diff_norm(a.to_numpy(), b.to_numpy()) <= 1e-10 * s


def test_batch_unknown_norms_and_max_rank():
    import paper_2211_08770_b200 as P
    items = _batch(5)
    batch = [([dev(t) for t in terms], coeffs) for terms, coeffs in items]   # norms NaN
    outs = P.tt_round_batch(ctx(), batch, 1e-8)
    for (terms, coeffs), o in zip(items, outs):
        _check_item(o.to_numpy(), o.ranks, terms, coeffs, 1e-8, rounding.DEFAULT_FLOOR_C)
    outs = P.tt_round_batch(ctx(), batch, 1e-8, max_rank=3)
    for (terms, coeffs), o in zip(items, outs):
        assert max(o.ranks) <= 3
        _check_item(o.to_numpy(), o.ranks, terms, coeffs, 1e-8, rounding.DEFAULT_FLOOR_C, max_rank=3)


def test_batch_zero_items():
    """||x|| = 0 (all coefficients zero) gives the rank-1 zero tensor, next to normal items."""
    import paper_2211_08770_b200 as P
    rng = _rng(77)
    d, n = 5, [6, 9, 4, 7, 5]
    rk = [1, 4, 6, 5, 3, 1]
    items = []
    for b in range(4):
        terms = [make_random_tt(d, n, rk, rng) for _ in range(2)]
        coeffs = [0.0, 0.0] if b % 2 else [1.0, 0.5]
        items.append((terms, coeffs))
    outs = P.tt_round_batch(ctx(), [([dev(t) for t in ts], cs) for ts, cs in items], 1e-8)
    for b, ((terms, coeffs), o) in enumerate(zip(items, outs)):
        if b % 2:
            assert o.ranks == [1] * (d + 1)
            assert all(np.all(c == 0.0) for c in o.to_numpy())
        else:
            _check_item(o.to_numpy(), o.ranks, terms, coeffs, 1e-8, rounding.DEFAULT_FLOOR_C)


def test_batch_c4_shape():
    """C4 items at full shape (d = 10, n = 32, 4 x rank 16): closed form and oracle parity."""
    import paper_2211_08770_b200 as P
    items = make_batch_sums(8)
    outs = P.tt_round_batch(ctx(), [([dev(t, 1.0) for t in terms], coeffs) for terms, coeffs in items], 1e-6)
    for b, ((terms, coeffs), o) in enumerate(zip(items, outs)):
        want = 32 if b % 2 == 0 else 16
        assert o.ranks == [1] + [want] * 9 + [1]
        g = o.to_numpy()
        refx = tt.tt_sum(terms[:2], [1.0, 1.0]) if b % 2 == 0 else terms[0]
        assert diff_norm(g, refx) <= 5e-9 * np.sqrt(2.0)
        if b < 4:
            _check_item(g, o.ranks, terms, coeffs, 1e-6, rounding.DEFAULT_FLOOR_C, norms=[1.0] * 4)


def _stack(items):
    """Per-item (terms, coeffs) -> stacked (B, r0, n, r1) CUDA tensors per (term, core)."""
    import torch
    K, d = len(items[0][0]), len(items[0][0][0])
    cores = [[torch.from_numpy(np.ascontiguousarray(np.stack([it[0][l][k] for it in items]))).cuda()
              for k in range(d)] for l in range(K)]
    coeffs = np.array([it[1] for it in items], dtype=np.float64)
    return cores, coeffs


@pytest.mark.parametrize("seed", [0, 1, 2, 6, 9, 12])
def test_batch_strided_api(seed):
    """tt_round_batch_strided (base pointer + item stride per term core, one result handle)
    equals the oracle item by item; norms given and unknown."""
    import paper_2211_08770_b200 as P
    items = _batch(seed)
    cores, coeffs = _stack(items)
    norms = np.array([[tt.tt_norm(t) for t in terms] for terms, _ in items])
    for nr in (norms, None):
        res = P.tt_round_batch_strided(ctx(), cores, coeffs, 1e-8, norms=nr)
        assert len(res) == len(items)
        for b, (terms, cf) in enumerate(items):
            g = res.item_numpy(b)
            assert [1] + [c.shape[2] for c in g] == list(res.ranks[b])
            _check_item(g, list(res.ranks[b]), terms, cf, 1e-8, rounding.DEFAULT_FLOOR_C, norms=list(norms[b]))


def test_batch_strided_c4_stacked_generator():
    """C4 through the stacked generator and the strided API: closed-form ranks 32/16, distance
    to y1 + [b even] y2, and oracle parity on a sample."""
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked
    B = 40
    cores, coeffs = make_batch_sums_stacked(B)
    dc = [[torch.from_numpy(c).cuda() for c in term] for term in cores]
    res = P.tt_round_batch_strided(ctx(), dc, coeffs, 1e-6, norms=np.ones((B, 4)))
    for b in range(B):
        want = 32 if b % 2 == 0 else 16
        assert list(res.ranks[b]) == [1] + [want] * 9 + [1]
    for b in (0, 1, 17, 38, 39):
        terms = [[cores[s][k][b] for k in range(10)] for s in range(4)]
        g = res.item_numpy(b)
        refx = tt.tt_sum(terms[:2], [1.0, 1.0]) if b % 2 == 0 else terms[0]
        assert diff_norm(g, refx) <= 5e-9 * np.sqrt(2.0)
        _check_item(g, list(res.ranks[b]), terms, list(coeffs[b]), 1e-6, rounding.DEFAULT_FLOOR_C, norms=[1.0] * 4)


def test_batch_host_pipeline_matches_device_call():
    """tt_round_batch_host (host inputs -> host results, 3 pipelined slices) returns the same
    bytes as tt_round_batch_strided on the device copies, items and cores in order."""
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked
    B = 10
    cores, coeffs = make_batch_sums_stacked(B, d=6, n=9, r=5)
    host = [[torch.from_numpy(c).pin_memory() for c in term] for term in cores]
    out, ranks, norms, cnt = P.tt_round_batch_host(ctx(), host, coeffs, 1e-6, norms=np.ones((B, 4)), slices=3)
    res = P.tt_round_batch_strided(ctx(), [[c.cuda() for c in term] for term in host], coeffs, 1e-6,
                                   norms=np.ones((B, 4)))
    assert np.array_equal(ranks, res.ranks)
    flat = np.concatenate([np.concatenate([c.ravel() for c in res.item_numpy(b)]) for b in range(B)])
    assert cnt == flat.size
    assert np.array_equal(out[:cnt].numpy(), flat)
    np.testing.assert_array_equal(norms, res.norms)


def test_batch_host_pipeline_back_to_back_c4_shape():
    """Two back-to-back host-to-host calls at the C4 item shape with 4 slices: the slices'
    device inputs (allocated on the copy stream, read on the context stream) are not recycled
    while still being read; both calls return the device call's bytes."""
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked
    B = 600
    cores, coeffs = make_batch_sums_stacked(B, start=1000)
    host = [[torch.from_numpy(c).pin_memory() for c in term] for term in cores]
    res = P.tt_round_batch_strided(ctx(), [[c.cuda() for c in term] for term in host], coeffs, 1e-6,
                                   norms=np.ones((B, 4)))
    flat = np.concatenate([np.concatenate([c.ravel() for c in res.item_numpy(b)]) for b in range(B)])
    outs = []
    for _ in range(2):
        out, ranks, _, cnt = P.tt_round_batch_host(ctx(), host, coeffs, 1e-6, norms=np.ones((B, 4)), slices=4)
        outs.append((out[:cnt].numpy().copy(), ranks))
    for o, rk in outs:
        assert np.array_equal(rk, res.ranks)
        assert np.array_equal(o, flat)


def test_batch_host_small_buffer_and_strided_items():
    """The C-ABI host call with (a) an output buffer too small for the results: TT_EINVAL with the
    needed count, nothing written past the buffer, and the retry returns the device call's bytes;
    (b) items that are not adjacent in host memory (every other item of a larger pinned tensor:
    item_stride = 2 x the core size, copied with strided host->device copies); (c) one slice per
    item, so slice 0 (an odd-rank item) has a smaller output than later slices."""
    import ctypes as C
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked
    B = 7
    cores, coeffs = make_batch_sums_stacked(2 * B, d=5, n=6, r=4, start=31)
    big = [[torch.from_numpy(c).pin_memory() for c in term] for term in cores]
    host = [[c[1::2] for c in term] for term in big]   # items 1, 3, 5, ... (odd: rank-16-like first)
    cf = np.ascontiguousarray(coeffs[1::2])
    res = P.tt_round_batch_strided(ctx(), [[c.contiguous().cuda() for c in term] for term in host], cf, 1e-6,
                                   norms=np.ones((B, 4)))
    flat = np.concatenate([np.concatenate([c.ravel() for c in res.item_numpy(b)]) for b in range(B)])
    guard = torch.full((flat.size,), -7.0, dtype=torch.float64).pin_memory()
    small = guard[:flat.size // 3]
    # direct C call with the small buffer: TT_EINVAL and the needed count
    K, d = 4, 5
    n = (C.c_int64 * d)(*[6] * d)
    r = (C.c_int64 * (K * (d + 1)))(*[v for _ in range(K) for v in [1, 4, 4, 4, 4, 1]])
    base = (C.c_void_p * (K * d))(*[host[l][k].data_ptr() for l in range(K) for k in range(d)])
    stride = (C.c_int64 * (K * d))(*[int(host[l][k].stride(0)) for l in range(K) for k in range(d)])
    nr = np.ones((B, K))
    o = P.api._opts(1e-6, P.DEFAULT_FLOOR_C, 0, 0.5, False)
    cnt = C.c_int64()
    st = ctx().lib.tt_round_batch_host(ctx().handle, B, K, d, n, r, base, stride,
                                       cf.ctypes.data_as(C.POINTER(C.c_double)),
                                       nr.ctypes.data_as(C.POINTER(C.c_double)), C.byref(o), B,
                                       C.c_void_p(small.data_ptr()), small.numel(), C.byref(cnt), None, None)
    assert st == 1 and cnt.value == flat.size
    assert np.all(guard[flat.size // 3:].numpy() == -7.0)  # nothing written past the capacity
    out, ranks, _, cnt2 = P.tt_round_batch_host(ctx(), host, cf, 1e-6, norms=nr, slices=B, out_host=small.clone())
    assert cnt2 == flat.size and np.array_equal(ranks, res.ranks)
    assert np.array_equal(out[:cnt2].numpy(), flat)


def test_batch_strided_unsupported_shape_and_serial_fallback():
    """Formal rank > 64 is outside the batched engine: tt_round_batch_strided reports
    TT_ENOTSUP, tt_round_batch falls back to the per-item rounding (still oracle-exact)."""
    import paper_2211_08770_b200 as P
    from paper_2211_08770_b200._native import TTError
    rng = _rng(404)
    d, n = 3, [5, 6, 4]
    ranks = [[1, 20, 20, 1], [1, 25, 25, 1], [1, 22, 22, 1]]  # formal interior rank 67
    items = []
    for _ in range(2):
        terms = [make_random_tt(d, n, r, rng) for r in ranks]
        items.append((terms, [1.0, -0.5, 0.25]))
    cores, coeffs = _stack(items)
    with pytest.raises(TTError) as e:
        P.tt_round_batch_strided(ctx(), cores, coeffs, 1e-8)
    assert e.value.name == "TT_ENOTSUP"
    outs = P.tt_round_batch(ctx(), [([dev(t) for t in ts], cs) for ts, cs in items], 1e-8)
    for (terms, cf), o in zip(items, outs):
        _check_item(o.to_numpy(), o.ranks, terms, cf, 1e-8, rounding.DEFAULT_FLOOR_C)


def test_batch_exactly_rank_64_and_single_item():
    """Formal ranks exactly 64 (the engine's limit), one item, one mode size of 1."""
    import paper_2211_08770_b200 as P
    rng = _rng(405)
    d, n = 4, [7, 1, 30, 9]
    ranks = [[1, 7, 1, 9, 1], [1, 40, 1, 30, 1], [1, 17, 1, 25, 1]]  # R_1 = 64, R_3 = 64
    terms = [make_random_tt(d, n, r, rng) for r in ranks]
    items = [(terms, [1.0, 2.0, -1.0])]
    cores, coeffs = _stack(items)
    res = P.tt_round_batch_strided(ctx(), cores, coeffs, 1e-10)
    _check_item(res.item_numpy(0), list(res.ranks[0]), terms, [1.0, 2.0, -1.0], 1e-10, rounding.DEFAULT_FLOOR_C)


def test_batch_c4_full_size_bench_config():
    """BASELINE configs[3] at full size in the launch configuration bench.py times (4096 items,
    tt_round_batch_strided, one call): closed-form ranks for every item, the distance to
    y1 + [b even] y2 on a sample across waves, and oracle parity item by item on that sample."""
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked
    B = 4096
    cores, coeffs = make_batch_sums_stacked(B)
    dc = [[torch.from_numpy(c).cuda() for c in term] for term in cores]
    res = P.tt_round_batch_strided(ctx(), dc, coeffs, 1e-6, norms=np.ones((B, 4)))
    want = np.where(np.arange(B) % 2 == 0, 32, 16)
    assert np.all(res.ranks[:, 1:-1] == want[:, None]) and np.all(res.ranks[:, [0, -1]] == 1)
    for b in (0, 1, 1333, 2048, 2049, 4095):
        terms = [[cores[s][k][b] for k in range(10)] for s in range(4)]
        g = res.item_numpy(b)
        refx = tt.tt_sum(terms[:2], [1.0, 1.0]) if b % 2 == 0 else terms[0]
        assert diff_norm(g, refx) <= 5e-9 * np.sqrt(2.0)
        _check_item(g, list(res.ranks[b]), terms, list(coeffs[b]), 1e-6, rounding.DEFAULT_FLOOR_C, norms=[1.0] * 4)


@pytest.mark.parametrize("case", ["wide_terms", "five_blocks", "one_block", "odd_ranks"])
def test_batch_panel_engine_paths(case):
    """Shapes that steer the compact-WY panel engine (csrc/batch_wy.cuh) through each of its paths,
    all with several 128-row stacks and a ragged last one: term ranks above 16 (the loader's general
    beta-slab loop), 5 and 1 column blocks (cell order with fewer blocks than warps / a single
    chain), column blocks that straddle two terms and ranks that are no multiples of 8."""
    import paper_2211_08770_b200 as P
    rng = _rng({"wide_terms": 71, "five_blocks": 72, "one_block": 73, "odd_ranks": 74}[case])
    if case == "wide_terms":      # R = 60: two terms of rank 30, panels 37 * 60 = 2220 rows
        d, n, ranks = 4, [9, 37, 37, 6], [[1, 9, 30, 6, 1], [1, 9, 30, 6, 1]]
    elif case == "five_blocks":   # R_2 = 38: 5 column blocks, the last one partial
        d, n, ranks = 4, [12, 33, 29, 12], [[1, 12, 19, 12, 1], [1, 12, 19, 12, 1]]
    elif case == "one_block":     # R <= 8: one column block, one warp chain per stack
        d, n, ranks = 4, [5, 40, 40, 5], [[1, 3, 4, 3, 1], [1, 3, 4, 3, 1]]
    else:                         # three terms, blocks straddling terms, R'_k % 8 != 0
        d, n, ranks = 5, [6, 23, 31, 17, 5], [[1, 5, 11, 7, 4, 1], [1, 3, 13, 9, 5, 1], [1, 6, 7, 10, 3, 1]]
    K = len(ranks)
    items = []
    for b in range(3):
        terms = [make_random_tt(d, n, r, rng) for r in ranks]
        coeffs = [float(v) for v in rng.standard_normal(K)]
        if b == 2 and ranks[0] == ranks[1]:  # near cancellation of the first two terms
            terms[1] = terms[0]
            coeffs[1] = -coeffs[0] * (1.0 - 2.0 ** -20)
        items.append((terms, coeffs))
    cores, coeffs = _stack(items)
    for delta in (1e-9, 1e-3):
        res = P.tt_round_batch_strided(ctx(), cores, coeffs, delta)
        for b, (terms, cf) in enumerate(items):
            _check_item(res.item_numpy(b), list(res.ranks[b]), terms, cf, delta, rounding.DEFAULT_FLOOR_C)


def test_batch_two_stream_wave_small_items():
    """A wave large enough to run as two halves on two streams (>= 16 x SMs items), with small
    ragged items: a sample from both halves and the seam against the oracle, and every item's
    ranks against a second call (bitwise reproducible: the cell scheduler orders work only)."""
    import paper_2211_08770_b200 as P
    rng = _rng(75)
    B, d, n = 2600, 3, [6, 21, 5]
    ranks = [[1, 5, 4, 1], [1, 4, 5, 1]]
    items = []
    for b in range(B):
        terms = [make_random_tt(d, n, r, rng) for r in ranks]
        items.append((terms, [1.0, float(rng.standard_normal())]))
    cores, coeffs = _stack(items)
    res = P.tt_round_batch_strided(ctx(), cores, coeffs, 1e-8)
    res2 = P.tt_round_batch_strided(ctx(), cores, coeffs, 1e-8)
    assert np.array_equal(res.ranks, res2.ranks)
    for b in (0, 1, 1299, 1300, 1301, 2599):
        g = res.item_numpy(b)
        assert all(np.array_equal(x, y) for x, y in zip(g, res2.item_numpy(b)))
        _check_item(g, list(res.ranks[b]), items[b][0], items[b][1], 1e-8, rounding.DEFAULT_FLOOR_C)


def _diag_term(d, n, r, off, Q):
    """sum_{j < r} (Q_1 e_{off+j}) x ... x (Q_d e_{off+j}): every unfolding has r singular values
    equal to 1 (up to rounding)."""
    cores = []
    for k in range(d):
        r0, r1 = (1 if k == 0 else r), (1 if k == d - 1 else r)
        G = np.zeros((r0, n, r1))
        for a in range(r):
            G[0 if k == 0 else a, :, 0 if k == d - 1 else a] = Q[k][:, off + a]
        cores.append(G)
    return cores


@pytest.mark.parametrize("r", [4, 8, 16])
def test_batch_repeated_singular_values(r):
    """Sums whose unfoldings carry r-fold repeated singular values (|c_l| each): Jacobi pairs with
    equal column norms rotate by large angles however small their inner product is -- the case
    the tiny-rotation stopping rule of the batched Jacobi (A23) has to count as not tiny.
    Terms 1, 2 are kept (rank 2 r), terms 3, 4 (1e-9) fall below delta = 1e-6."""
    import paper_2211_08770_b200 as P
    d, n, K = 4, 64, 4
    items = []
    for seed in range(3):
        rng = _rng(7700 + 10 * r + seed)
        Q = [np.linalg.qr(rng.standard_normal((n, n)))[0] for _ in range(d)]
        terms = [_diag_term(d, n, r, l * r, Q) for l in range(K)]
        items.append((terms, [1.0, -1.0 if seed else 1.0, 1e-9, -1e-9]))
    norms = [[tt.tt_norm(t) for t in terms] for terms, _ in items]
    batch = [([dev(t, nr) for t, nr in zip(terms, nb)], coeffs) for (terms, coeffs), nb in zip(items, norms)]
    outs = P.tt_round_batch(ctx(), batch, 1e-6)
    for (terms, coeffs), nb, o in zip(items, norms, outs):
        assert list(o.ranks) == [1] + [2 * r] * (d - 1) + [1]
        _check_item(o.to_numpy(), o.ranks, terms, coeffs, 1e-6, rounding.DEFAULT_FLOOR_C, norms=nb)
    # delta = 0 keeps all 4 r values: the full Jacobi on clustered values at two scales
    outs = P.tt_round_batch(ctx(), batch, 0.0, floor_c=0.0)
    for (terms, coeffs), nb, o in zip(items, norms, outs):
        _check_item(o.to_numpy(), o.ranks, terms, coeffs, 0.0, 0.0, norms=nb)


@pytest.mark.parametrize("e", [-120, -90, -60, 75, 90, 140])
def test_batch_scaled_inputs(e):
    """The value range of the path (include/tt_b200.h): the same sum scaled by 10^e must round to
    the same ranks with the same relative error -- the Jacobi's tests on products of squared
    norms run in units of ||A||_F^2 (exact power-of-two scaling)."""
    import paper_2211_08770_b200 as P
    rng = _rng(4242)
    d, n = 5, [12, 20, 16, 20, 12]
    ranks = [[1, 6, 9, 9, 6, 1], [1, 5, 8, 7, 5, 1], [1, 6, 9, 9, 6, 1]]
    base = [make_random_tt(d, n, r, rng) for r in ranks]
    base[2] = base[0]                      # near cancellation of terms 1 and 3
    coeffs = [1.0, 0.5, -1.0 + 1e-9]
    f = 10.0 ** e
    terms = [[c * (f if k == 0 else 1.0) for k, c in enumerate(t)] for t in base]
    norms = [tt.tt_norm(t) for t in terms]
    batch = [([dev(t, nr) for t, nr in zip(terms, norms)], coeffs)] * 2
    for o in P.tt_round_batch(ctx(), batch, 1e-6):
        _check_item(o.to_numpy(), o.ranks, terms, coeffs, 1e-6, rounding.DEFAULT_FLOOR_C, norms=norms)


def test_batch_overflowing_input_fails_loudly():
    import paper_2211_08770_b200 as P
    from paper_2211_08770_b200._native import TTError
    rng = _rng(4243)
    d, n = 3, [8, 8, 8]
    t = make_random_tt(d, n, [1, 4, 4, 1], rng)
    t[0] = t[0] * 1e200
    with pytest.raises(TTError):
        P.tt_round_batch(ctx(), [([dev(t, float("nan"))], [1.0])] * 2, 1e-6)


# Configurations of the randomised sweep (tools/fuzz_batch.py, ttinputs.make_fuzz_batch) that earlier
# trees got wrong: delta = 0.1 on gapless / graded spectra (the QRCP-truncated SVD dropped the
# first-order term E U~ of the next core's target: differences of 1e-7 .. 1e-4 s(x)), a short wide
# first split (cp > rows: the mass of the unrotated small columns beyond the rank bound was left out
# of the tail, rank 12 for 13), tau at the noise level of a cancelling sum (skipped small-small
# pairs made the Jacobi linear: TT_ENOCONV), and sums the older rotation formula did not converge on.
_FUZZ_REGRESSIONS = [31, 40, 70, 104, 107, 195, 206, 242, 247, 333, 382, 440, 462, 573, 576, 587, 591, 943]


@pytest.mark.parametrize("seed", _FUZZ_REGRESSIONS)
def test_batch_fuzz_regressions(seed):
    import paper_2211_08770_b200 as P
    from ttinputs import make_fuzz_batch
    items, delta, fc, desc = make_fuzz_batch(seed)
    floor_c = rounding.DEFAULT_FLOOR_C if fc is None else fc
    norms = [[tt.tt_norm(t) for t in terms] for terms, _ in items]
    batch = [([dev(t, nr) for t, nr in zip(terms, nb)], coeffs) for (terms, coeffs), nb in zip(items, norms)]
    outs = P.tt_round_batch(ctx(), batch, delta, floor_c=floor_c)
    for (terms, coeffs), nb, o in zip(items, norms, outs):
        assert_round_parity(o.to_numpy(), o.ranks, terms, coeffs, delta, floor_c, nb, tag=desc)
