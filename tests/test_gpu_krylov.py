"""The paper's own workload on the GPU: TT-matvec, the Krylov
TT-Laplacian sets and the memory metrics Eqs. (1)-(2), against oracle/krylov.py.

Each side builds its own Krylov set (GPU: tt_matvec + rank-1 tt_round; oracle: numpy), so the
two sets agree to rounding (checked as |<a_j, a_j'>| = 1 up to sign).  The orthogonalizations
run paper-pure (floor off) on each side's own set; they are compared like the free-running
driver runs of test_gpu_orth.py, with the amplification A_k = (64 u + delta) m kappa_k^p.
"""
import numpy as np
import pytest

from oracle import krylov, orth, tt
from oracle.dense import U_ROUND

from gpu_util import ctx, cuda_ok, dev, diff_norm

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

POWER = {"cgs": 2, "gram": 2, "mgs": 1, "cgs2": 1, "mgs2": 1, "householder": 1}


def _rng(s):
    return np.random.Generator(np.random.PCG64(s))


@pytest.mark.parametrize("d,n", [(3, 5), (4, 3), (2, 7)])
def test_matvec_matches_oracle(d, n):
    import paper_2211_08770_b200 as P
    rng = _rng(10 + d)
    r = [1] + [int(v) for v in rng.integers(1, 5, size=d - 1)] + [1]
    x = [rng.standard_normal((r[k], n, r[k + 1])) for k in range(d)]
    ra = [1] + [int(v) for v in rng.integers(1, 4, size=d - 1)] + [1]
    A = [rng.standard_normal((ra[k], n, n, ra[k + 1])) for k in range(d)]
    for op in (A, krylov.laplacian_ttm(d, n)):
        y = P.tt_matvec(ctx(), P.ttm_device(op), dev(x))
        ref = krylov.matvec(op, x)
        assert y.ranks == tt.ranks(ref)
        g = y.to_numpy()
        for gk, ck in zip(g, ref):
            np.testing.assert_allclose(gk, ck, rtol=0, atol=1e-13 * max(1.0, np.abs(ck).max()))


def test_matvec_shape_errors():
    import paper_2211_08770_b200 as P
    from paper_2211_08770_b200._native import TTError
    x = [np.ones((1, 3, 1))] * 2
    bad = [np.ones((1, 3, 4, 1))] * 2  # 3 x 4 blocks: not n x n
    with pytest.raises(TTError):
        P.tt_matvec(ctx(), dev([c.reshape(1, 12, 1) for c in bad]), dev(x))


def test_laplacian_cores_match_oracle():
    import paper_2211_08770_b200 as P
    for d, n in [(2, 4), (3, 5), (6, 15)]:
        a, b = P.laplacian_cores(d, n), krylov.laplacian_ttm(d, n)
        assert len(a) == len(b)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


def _kappas(S):
    A = np.stack([tt.densify(a) for a in S], axis=1)
    return np.array([np.linalg.cond(A[:, :k]) if k > 1 else 1.0 for k in range(1, len(S) + 1)])


@pytest.mark.parametrize("d,n,m", [(3, 15, 20), (3, 6, 12)])
def test_krylov_set_matches_oracle(d, n, m):
    import paper_2211_08770_b200 as P
    G = P.krylov_set(ctx(), d, n, m)
    S = krylov.krylov_set(d, n, m)
    kap = _kappas(S)
    for j, (g, c) in enumerate(zip(G, S)):
        assert g.ranks == [1] * (d + 1)
        gc = g.to_numpy()
        assert abs(tt.tt_norm(gc) - 1.0) <= 1e-13
        # the rank-1 truncation is smooth where the leading singular value is separated:
        # forward error ~ j u (plus the kappa growth of the recursion)
        assert abs(abs(tt.tt_dot(gc, c)) - 1.0) <= max(1e-12, 1e-14 * j * kap[j]), (j, tt.tt_dot(gc, c))
    # memory metrics (Eqs. (1)-(2)) on the GPU ranks equal the oracle's
    for g, c in zip(G, S):
        assert P.storage_count(g.ranks, g.modes) == tt.storage_count(c)
        assert P.compression_ratio(g.ranks, g.modes) == tt.compression_ratio(c)


@pytest.mark.parametrize("kind", ["cgs", "mgs", "cgs2", "mgs2", "gram", "householder"])
@pytest.mark.parametrize("delta", [1e-5, 1e-8])
def test_krylov_orth_paper_pure(kind, delta):
    """d = 3, n = 15, m = 20 (Fig. 1's setting), floor off: Table 1 counts, LOO within
    2x where it exceeds the amplified noise, and the memory metrics of the outputs."""
    import paper_2211_08770_b200 as P
    d, n, m = 3, 15, 20
    from oracle.dense import SingularGram
    from paper_2211_08770_b200._native import TTError
    G = P.krylov_set(ctx(), d, n, m)
    S = krylov.krylov_set(d, n, m)
    try:
        ref = orth.orth(kind, S, delta, floor_c=0.0)
    except SingularGram:  # Gram + Cholesky breaks down on the ill-conditioned Krylov set
        with pytest.raises(TTError, match="ESINGULAR_GRAM"):
            P.tt_orth(ctx(), kind, G, delta, floor_c=0.0, want_loo=True)
        return
    Q, R, rep = P.tt_orth(ctx(), kind, G, delta, floor_c=0.0, want_loo=True)
    assert rep["rounding_calls"] == ref.rounding_calls
    kap = _kappas(S)
    amp = lambda k: (64 * U_ROUND + delta) * m * kap[k] ** POWER[kind]
    loo_c, loo_g = ref.loo_per_step(), rep["loo_per_step"]
    for k in range(m):
        if max(loo_c[k], loo_g[k]) > max(1e-14, amp(k)):
            assert 0.5 <= loo_g[k] / max(loo_c[k], 1e-300) <= 2.0, (kind, k, loo_g[k], loo_c[k])
        else:
            assert loo_g[k] <= max(2e-14, 2 * amp(k)), (kind, k, loo_g[k], amp(k))
    for i in range(m):
        if amp(i) < 1e-8:  # while the inputs agree, the basis vectors agree (up to sign for HH)
            qg, qc = Q[i].to_numpy(), ref.Q[i]
            sg = 1.0 if tt.tt_dot(qg, qc) >= 0 else -1.0
            assert diff_norm(tt.tt_scale(qg, sg), qc) <= max(1e-10, amp(i)), (kind, i)
    for q, qc in zip(Q, ref.Q):  # Eq. (1) of each basis vector (TT storage may exceed dense: Fig. 3)
        assert P.compression_ratio(q.ranks, q.modes) > 0.0
