"""Pins for oracle/tt.py: psi/phi, element, densify, TT-sum, scale, TT-dot, norms, Eqs. (1)-(2).

Each pin fixes the oracle against something other than itself: hand values printed in
tests/golden (cited), brute force over all indices, dense numpy arithmetic on densified
tensors, or exact algebraic identities.
"""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import tt
from ttinputs import make_random_tt

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rng(s):
    return np.random.Generator(np.random.PCG64(s))


def test_psi_golden():
    for case in GOLD["psi"]:
        assert tt.psi(case["idx1"], case["n"]) == case["value"], case["cite"]


def test_psi_phi_roundtrip_exhaustive():
    n = [4, 3, 5]
    seen = set()
    for idx in itertools.product(*[range(1, v + 1) for v in n]):
        lin = tt.psi(list(idx), n)
        assert tt.phi(lin, n) == list(idx)
        seen.add(lin)
    assert seen == set(range(1, 61))  # psi is a bijection onto 1..prod n


def test_element_matches_brute_force_sum():
    """x(i) = sum over rank indices of the core product, brute force."""
    rng = _rng(1)
    x = make_random_tt(3, [3, 2, 4], [1, 2, 3, 1], rng)
    for idx in itertools.product(range(3), range(2), range(4)):
        brute = 0.0
        for j1 in range(2):
            for j2 in range(3):
                brute += x[0][0, idx[0], j1] * x[1][j1, idx[1], j2] * x[2][j2, idx[2], 0]
        assert abs(tt.element(x, idx) - brute) <= 1e-14 * (1 + abs(brute))


def test_densify_psi_order():
    rng = _rng(2)
    n = [3, 4, 2]
    x = make_random_tt(3, n, [1, 2, 2, 1], rng)
    v = tt.densify(x)
    for idx in itertools.product(*[range(k) for k in n]):
        lin = tt.psi([i + 1 for i in idx], n) - 1
        assert v[lin] == pytest.approx(tt.element(x, idx), abs=1e-13)


def test_canonical_basis():
    n = [3, 4, 2]
    N = 24
    for i in range(1, N + 1):
        v = tt.densify(tt.canonical_tt(i, n))
        e = np.zeros(N)
        e[i - 1] = 1.0
        assert np.array_equal(v, e)
    for i in range(1, 9):
        for j in range(1, 9):
            assert tt.tt_dot(tt.canonical_tt(i, n), tt.canonical_tt(j, n)) == (1.0 if i == j else 0.0)


def test_sum_ranks_and_linearity():
    g = GOLD["sum_ranks"]
    rng = _rng(3)
    n = [3, 4, 5]
    x = make_random_tt(3, n, g["x_ranks"], rng)
    y = make_random_tt(3, n, g["y_ranks"], rng)
    s = tt.tt_sum([x, y], [0.7, -1.3])
    assert tt.ranks(s) == g["sum_ranks"], g["cite"]
    np.testing.assert_allclose(tt.densify(s), 0.7 * tt.densify(x) - 1.3 * tt.densify(y), atol=1e-13)
    z = tt.tt_sum([x, x], [1.0, -1.0])
    assert np.max(np.abs(tt.densify(z))) <= 1e-14


def test_scale_first_core():
    rng = _rng(4)
    x = make_random_tt(4, 3, [1, 2, 3, 2, 1], rng)
    y = tt.tt_scale(x, -2.5)
    assert tt.ranks(y) == tt.ranks(x)
    for k in range(1, 4):
        assert np.array_equal(y[k], x[k])
    np.testing.assert_allclose(tt.densify(y), -2.5 * tt.densify(x), rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("seed", range(6))
def test_dot_equals_dense_dot(seed):
    rng = _rng(10 + seed)
    d = 2 + seed % 3
    n = [int(v) for v in rng.integers(2, 5, size=d)]
    rx = [1] + [int(v) for v in rng.integers(1, 4, size=d - 1)] + [1]
    ry = [1] + [int(v) for v in rng.integers(1, 4, size=d - 1)] + [1]
    x = make_random_tt(d, n, rx, rng)
    y = make_random_tt(d, n, ry, rng)
    ref = float(np.dot(tt.densify(x), tt.densify(y)))
    scale = np.linalg.norm(tt.densify(x)) * np.linalg.norm(tt.densify(y))
    assert abs(tt.tt_dot(x, y) - ref) <= 1e-13 * scale
    assert abs(tt.tt_dot(x, y) - tt.tt_dot(y, x)) <= 1e-14 * scale


def test_ones_norm_golden():
    g = GOLD["ones_norm"]
    o = tt.ones_tt(g["d"], g["n"])
    assert tt.tt_dot(o, o) == g["norm_sq"], g["cite"]
    assert tt.tt_norm(o) == pytest.approx(np.sqrt(3375.0), rel=1e-15)


def test_storage_and_compression_golden():
    for case in GOLD["storage_count"]:
        x = [np.zeros((case["ranks"][k], case["n"][k], case["ranks"][k + 1])) for k in range(len(case["n"]))]
        assert tt.storage_count(x) == case["value"], case["cite"]
    for case in GOLD["compression_ratio"]:
        x = [np.zeros((case["ranks"][k], case["n"][k], case["ranks"][k + 1])) for k in range(len(case["n"]))]
        assert tt.compression_ratio(x) == pytest.approx(case["num"] / case["den"], rel=1e-15), case["cite"]
    g = GOLD["compression_gain"]
    b = [np.zeros((g["before_ranks"][k], g["n"], g["before_ranks"][k + 1])) for k in range(6)]
    a = [np.zeros((g["after_ranks"][k], g["n"], g["after_ranks"][k + 1])) for k in range(6)]
    assert tt.compression_gain(b, a) == pytest.approx(g["num"] / g["den"], rel=1e-15), g["cite"]
    assert tt.compression_gain(b, a) * tt.storage_count(a) == pytest.approx(tt.storage_count(b))
