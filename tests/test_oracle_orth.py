"""Pins for oracle/orth.py (§2, Algorithms 1-8, Table 1).

Pins: Table 1 rounding counts (golden), the closed forms of the shared-tail construction
(R = R_M, Gram = M^T M, q_i = B Q_M[:, i]), the orthonormal-input fixed point, dense
Gram-Schmidt / Householder QR on the densified vectors, the Householder hand cases and
identities of PAPER.md:286-303, literal == lazy, breakdown behaviour, and the paper's
order-of-magnitude LOO statements (Eqs. (10)-(12)).
"""
import json
import os

import numpy as np
import pytest

from oracle import dense, orth, rounding, tt
from ttinputs import CONFIGS, make_shared_tail_set

HERE = os.path.dirname(__file__)
TABLE1 = json.load(open(os.path.join(HERE, "golden", "table1_rounding_counts.json")))
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))
KINDS = ["cgs", "mgs", "cgs2", "mgs2", "gram", "householder"]


def _sign_fix(R):
    s = np.sign(np.diag(R))
    s[s == 0] = 1
    return s[:, None] * R, s


def _tt_diff_norm(x, y):
    """||x - y|| by an exact (delta = 0) rounding of the difference: the sweep norm ||C_1||_F
    (never sqrt(<a,a> - 2<a,b> + <b,b>))."""
    _, info = rounding.tt_round(tt.tt_sum([x, y], [1.0, -1.0]), 0.0)
    return info.norm


@pytest.fixture(scope="module")
def well_conditioned():
    return make_shared_tail_set(4, 8, 3, 10, 1e2, seed=991)


@pytest.mark.parametrize("kind", KINDS)
def test_rounding_counts_table1(kind, well_conditioned):
    A = well_conditioned.tensors[:5]
    a, b = TABLE1["per_m"][kind]
    for literal in (False, True):
        res = orth.orth(kind, A, 1e-10, literal=literal)
        assert res.rounding_calls == a * 5 + b


@pytest.mark.parametrize("kind", KINDS)
def test_closed_form_well_conditioned(kind, well_conditioned):
    st = well_conditioned
    res = orth.orth(kind, st.tensors, 1e-12)
    qm, rm = st.qr_exact()
    R = res.R
    s = np.ones(st.m)
    if kind == "householder":
        R, s = _sign_fix(R)   # R(i,i) sign is set by Alg. 6's rule
    assert np.linalg.norm(R - rm) <= 1e-9 * np.linalg.norm(rm)
    assert np.all(R[np.tril_indices(st.m, -1)] == 0.0)  # structural zeros
    for i in range(st.m):
        assert _tt_diff_norm(tt.tt_scale(res.Q[i], s[i]), st.q_exact(i)) <= 1e-9
    assert res.loo_per_step()[-1] <= 1e-9


def test_gram_closed_form_c3_shape():
    """Gram(A) = M^T M exactly for the shared-tail construction (C3 shape, reduced m)."""
    c = CONFIGS["C3"]
    st = make_shared_tail_set(c.d, c.n, c.r, 6, c.kappa, c.seed)
    G = orth.gram_matrix(st.tensors)
    assert np.linalg.norm(G - st.gram_exact()) <= 1e-13 * np.linalg.norm(st.gram_exact())


@pytest.mark.parametrize("kind", KINDS)
def test_literal_equals_lazy(kind, well_conditioned):
    A = well_conditioned.tensors[:6]
    r1 = orth.orth(kind, A, 1e-10, literal=True)
    r2 = orth.orth(kind, A, 1e-10, literal=False)
    assert np.linalg.norm(r1.R - r2.R) <= 1e-12 * np.linalg.norm(r1.R)
    assert [i.ranks for i in r1.infos] == [i.ranks for i in r2.infos]
    for q1, q2 in zip(r1.Q, r2.Q):
        assert _tt_diff_norm(q1, q2) <= 1e-12


@pytest.mark.parametrize("kind", KINDS)
def test_orthonormal_input_fixed_point(kind):
    """canonical inputs -> Q = input, R = I."""
    n = [4, 3, 5]
    A = [tt.canonical_tt(i, n) for i in (1, 2, 3, 4, 5)]
    res = orth.orth(kind, A, 1e-8)
    R, s = _sign_fix(res.R)
    assert np.allclose(R, np.eye(5), atol=1e-12)
    for i in range(5):
        np.testing.assert_allclose(s[i] * tt.densify(res.Q[i]), tt.densify(A[i]), atol=1e-12)


def _dense_gs(Ad, kind):
    """Plain dense Gram-Schmidt family on the unfolded vectors (matrix framework of §2.1,
    PAPER.md:80-82, 135, 141-142) and Cholesky-QR (Gram)."""
    n, m = Ad.shape
    Q = np.zeros((n, m))
    R = np.zeros((m, m))
    if kind == "gram":
        L = np.linalg.cholesky(Ad.T @ Ad)
        R = L.T
        return Ad @ np.linalg.inv(R), R
    passes = 2 if kind.endswith("2") else 1
    for i in range(m):
        v = Ad[:, i].copy()
        for _ in range(passes):
            w = v.copy()
            for j in range(i):
                c = Q[:, j] @ (w if kind.startswith("mgs") else v)
                R[j, i] += c
                w -= c * Q[:, j]
            v = w
        R[i, i] = np.linalg.norm(v)
        Q[:, i] = v / R[i, i]
    return Q, R


@pytest.mark.parametrize("kind", KINDS)
def test_dense_equivalence_unfolded(kind):
    """d=3, n=5, m=8, tiny delta: TT kernels == dense counterparts on the
    densified vectors (Householder: numpy QR, i.e. LAPACK Householder, up to column signs)."""
    st = make_shared_tail_set(3, 5, 3, 8, 1e3, seed=77)
    Ad = np.stack([tt.densify(a) for a in st.tensors], axis=1)
    res = orth.orth(kind, st.tensors, 1e-14)
    Qt = np.stack([tt.densify(q) for q in res.Q], axis=1)
    if kind == "householder":
        Qd, Rd = np.linalg.qr(Ad)
        Rd, s = _sign_fix(Rd)
        Qd = Qd * s[None, :]
        Rt, st_ = _sign_fix(res.R)
        Qt = Qt * st_[None, :]
    else:
        Qd, Rd = _dense_gs(Ad, kind)
        Rt = res.R
    assert np.linalg.norm(Rt - Rd) <= 1e-10 * np.linalg.norm(Rd)
    assert np.max(np.abs(np.abs(np.sum(Qt * Qd, axis=0)) - 1.0)) <= 1e-9


def test_tth_vec_hand_cases():
    g_e2, g_e1 = GOLD["householder_2d"]
    n = g_e2["n"]
    u, r, _, _ = orth.tth_vec_literal(tt.canonical_tt(2, n), 1, 1e-12, 0.0)
    assert r[0] == g_e2["r1"]
    v = tt.densify(u)
    assert v[0] == pytest.approx(g_e2["u_entries"]["1"], abs=1e-15)
    assert v[1] == pytest.approx(g_e2["u_entries"]["2"], abs=1e-15)
    u, r, _, _ = orth.tth_vec_literal(tt.canonical_tt(1, n), 1, 1e-12, 0.0)
    assert u is None and r[0] == g_e1["r1"]


def test_householder_maps_w_into_span():
    """with u from Eq. (5), H x = ||x|| y; here H_i w_i = sum_{j<=i} r(j) e_j."""
    st = make_shared_tail_set(3, 4, 2, 4, 10.0, seed=5)
    w = st.tensors[0]
    for i in (1, 2, 3):
        u, r, _, _ = orth.tth_vec_literal(w, i, 1e-14, 0.0)
        hw, _ = orth.apply_h_vec(w, u)
        v = tt.densify(hw)
        target = np.zeros_like(v)
        target[:i] = r
        assert np.linalg.norm(v - target) <= 1e-12 * np.linalg.norm(v)
        # apply-H-vec is an involution
        back, _ = orth.apply_h_vec(hw, u)
        np.testing.assert_allclose(tt.densify(back), tt.densify(w), atol=1e-13)


def test_breakdowns():
    st = make_shared_tail_set(3, 4, 2, 3, 10.0, seed=6)
    A = [st.tensors[0], st.tensors[0]]
    with pytest.raises(dense.SingularGram):
        orth.orth("gram", A, 1e-8)
    with pytest.raises(orth.LinearDependence) as ei:
        orth.orth("mgs", A, 1e-8)
    assert ei.value.index == 1


def test_paper_loo_statements_c1():
    """Order-of-magnitude statements of PAPER.md:509-510 / Eqs. (10)-(12) on C1
    (kappa = 1e8, delta = 1e-8): Householder LOO ~ delta, MGS ~ u kappa, CGS2/MGS2 ~ u,
    CGS and Gram far above MGS (kappa^2)."""
    c = CONFIGS["C1"]
    st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed)
    loo = {k: orth.orth(k, st.tensors, c.delta).loo_per_step() for k in KINDS}
    assert np.max(loo["householder"]) <= 100 * c.delta
    assert np.max(loo["mgs2"]) <= 1e-11 and np.max(loo["cgs2"]) <= 1e-11
    assert np.max(loo["mgs"]) <= 1e3 * dense.U_ROUND * c.kappa
    assert np.max(loo["cgs"]) >= 1e3 * np.max(loo["mgs"])
    assert np.max(loo["gram"]) >= 1e3 * np.max(loo["mgs"])


def test_oracle_self_spread():
    """Evidence for the LOO parity rule: two runs of the SAME oracle on inputs perturbed at
    the unit round-off (first core x (1 + u xi)) give LOO values that differ by more than a
    factor 2 where LOO is rounding noise (TT-Gram on C1, u kappa^2 regime), while both stay
    under the noise bound 64 m u kappa_k^2 that the GPU parity test uses there."""
    c = CONFIGS["C1"]
    st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed)
    rng = np.random.Generator(np.random.PCG64(3))
    pert = []
    for a in st.tensors:
        b = [x.copy() for x in a]
        b[0] = b[0] * (1.0 + dense.U_ROUND * rng.standard_normal(b[0].shape))
        pert.append(b)
    l1 = orth.orth("gram", st.tensors, c.delta).loo_per_step()
    l2 = orth.orth("gram", pert, c.delta).loo_per_step()
    kap = np.array([np.linalg.cond(st.M[:, :k]) if k > 1 else 1.0 for k in range(1, st.m + 1)])
    ratio = np.maximum(l1, l2) / np.maximum(np.minimum(l1, l2), 1e-300)
    noisy = (np.maximum(l1, l2) > 1e-14)
    assert np.any(ratio[noisy] > 2.0)
    assert np.all(np.maximum(l1, l2) <= np.maximum(64 * st.m * dense.U_ROUND * kap ** 2, 1e-14))


# ---- hh_beta = "literal": Alg. 6 line 10 as printed, beta = sqrt(||a||^2 - s)
def test_literal_beta_defect_rule_hand_values():
    """||a||^2 - s < -1e-12 ||a||^2 -> NumericalDefect (0-based step); within the
    tolerance it clamps to 0; otherwise the plain square root."""
    assert orth._literal_beta(1.0, 1.0 + 1e-13, 1) == 0.0
    with pytest.raises(orth.NumericalDefect) as ei:
        orth._literal_beta(1.0, 1.0 + 1e-11, 3)
    assert ei.value.index == 2
    assert orth._literal_beta(5.0, 16.0, 2) == 3.0   # sqrt(25 - 16)


def test_literal_beta_closed_form_and_dense_householder():
    """Well-conditioned input (kappa = 1e2): the literal beta gives R = R_M up to D = diag(sign)
    (closed form of the shared-tail construction) and the dense Householder R of the densified
    vectors; literal == lazy."""
    st = make_shared_tail_set(4, 8, 3, 10, 1e2, seed=991)
    lit = orth.orth("householder", st.tensors, 1e-12, literal=True, hh_beta="literal")
    laz = orth.orth("householder", st.tensors, 1e-12, hh_beta="literal")
    qm, rm = st.qr_exact()
    for res in (lit, laz):
        R, s = _sign_fix(res.R)
        assert np.linalg.norm(R - rm) <= 1e-9 * np.linalg.norm(rm)
    assert np.linalg.norm(lit.R - laz.R) <= 1e-12 * np.linalg.norm(lit.R)
    small = make_shared_tail_set(3, 4, 2, 5, 1e2, seed=17)
    res = orth.orth("householder", small.tensors, 1e-14, hh_beta="literal")
    Ad = np.stack([tt.densify(a) for a in small.tensors], axis=1)
    _, Rd = np.linalg.qr(Ad)
    Rd, _ = _sign_fix(Rd)
    Rt, _ = _sign_fix(res.R)
    assert np.linalg.norm(Rt - Rd) <= 1e-10 * np.linalg.norm(Rd)


def test_literal_beta_cancels_at_high_kappa_reading_a9():
    """Reading A9: the literal beta = sqrt(||a||^2 - s) cancels when a_i is nearly in
    span(e_1..e_{i-1}); at kappa = 1e8 its R(i,i) carry ~1e-3 relative error where the
    rounding-norm beta keeps ~2e-5 (both forms stay normwise backward stable: ||R - R_M||_F
    at the rounding noise)."""
    st = make_shared_tail_set(4, 8, 3, 10, 1e8, seed=991)
    qm, rm = st.qr_exact()
    err = {}
    for hb in ("literal", "round_norm"):
        R, _ = _sign_fix(orth.orth("householder", st.tensors, 1e-14, hh_beta=hb).R)
        assert np.linalg.norm(R - rm) <= 1e-9 * np.linalg.norm(rm)
        err[hb] = np.max(np.abs(np.diag(R) - np.diag(rm)) / np.abs(np.diag(rm)))
    assert err["round_norm"] <= 1e-4
    assert err["literal"] >= 1e-4 and err["literal"] >= 10 * err["round_norm"]


# ---------------------------------------------------------------- TTH-vec masking variant (§8(f) 3)
def test_mask_geq_brute_force():
    """mask_geq(n, L) densified is the indicator of psi-order linear index >= L,
    for every L on small mixed-radix shapes (brute force over all multi-indices)."""
    from oracle.tt import densify, mask_geq, psi
    import itertools
    for n in ([3], [2, 3], [3, 2, 4], [2, 2, 2, 3]):
        total = int(np.prod(n))
        for L in range(total + 1 if total < 30 else 30):
            if L == total:
                continue
            D = densify(mask_geq(n, L))  # psi order: entry lin = psi(i) - 1
            for idx in itertools.product(*[range(v) for v in n]):
                lin = psi([i + 1 for i in idx], n) - 1
                assert D[lin] == (1.0 if lin >= L else 0.0), (n, L, idx)
            ranks = [c.shape[0] for c in mask_geq(n, L)] + [1]
            assert max(ranks) <= 2


def test_hadamard_dense():
    from oracle.tt import densify, tt_hadamard
    rng = np.random.Generator(np.random.PCG64(71))
    n = [3, 4, 2]
    x = [rng.standard_normal((1, 3, 2)), rng.standard_normal((2, 4, 3)), rng.standard_normal((3, 2, 1))]
    y = [rng.standard_normal((1, 3, 3)), rng.standard_normal((3, 4, 2)), rng.standard_normal((2, 2, 1))]
    z = tt_hadamard(x, y)
    assert np.allclose(densify(z), densify(x) * densify(y), rtol=1e-13, atol=1e-13)
    assert [c.shape[2] for c in z] == [6, 6, 1]


def test_masked_first_rounding_input_equals_subtraction():
    """w (x) mask_geq(n, i-1) equals w - sum_{j<i} w(phi(j)) e_j (Alg. 6 lines 4-9) entry by entry
    on a densified tensor; the masked form has no cancellation: the zeroed entries are exactly 0."""
    from oracle.tt import canonical_tt, densify, element, mask_geq, phi, tt_hadamard, tt_sum
    from ttinputs import make_random_tt
    rng = np.random.Generator(np.random.PCG64(72))
    n = [4, 3, 3]
    w = make_random_tt(3, n, [1, 3, 2, 1], rng)
    for i in (1, 2, 5, 13, 36):
        masked = densify(tt_hadamard(w, mask_geq(n, i - 1)))
        terms = [w] + [canonical_tt(j, n) for j in range(1, i)]
        coefs = [1.0] + [-element(w, [t - 1 for t in phi(j, n)]) for j in range(1, i)]
        sub = densify(tt_sum(terms, coefs))
        assert np.max(np.abs(masked - sub)) <= 1e-14 * np.max(np.abs(densify(w)))
        for j in range(1, i):
            assert masked[j - 1] == 0.0  # densify is in psi order: entry j - 1 is phi(j)


def test_householder_masked_closed_form():
    """The masked variant (hh_mask) keeps Alg. 8's Table 1 count (4m-1) and the shared-tail
    closed form R = R_M (up to the signs D) on a well-conditioned set."""
    from oracle import orth
    st = make_shared_tail_set(4, 6, 3, 8, 1e2, seed=991)
    res = orth.orth("householder", st.tensors, 1e-12, hh_mask=True)
    assert res.rounding_calls == 4 * 8 - 1
    rm = st.qr_exact()[1]
    sg = np.sign(np.diag(res.R))
    sg[sg == 0] = 1
    assert np.linalg.norm(sg[:, None] * res.R - rm) <= 1e-10 * np.linalg.norm(rm)
