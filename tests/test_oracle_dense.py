"""Pins for oracle/dense.py (Cholesky, triangular inverse, LOO, truncation rule)."""
import json
import os

import numpy as np
import pytest
import scipy.linalg

from oracle import dense, tt

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_cholesky_golden():
    ok, bad = GOLD["cholesky"]
    np.testing.assert_array_equal(dense.cholesky(np.array(ok["G"], float)), np.array(ok["L"], float))
    with pytest.raises(dense.SingularGram) as ei:
        dense.cholesky(np.array(bad["G"], float))
    assert ei.value.index == bad["singular_at"], bad["cite"]


def test_cholesky_reconstructs_and_matches_lapack():
    rng = np.random.Generator(np.random.PCG64(5))
    B = rng.standard_normal((40, 12))
    G = B.T @ B
    L = dense.cholesky(G)
    assert np.allclose(np.tril(L), L)
    assert np.linalg.norm(L @ L.T - G) <= 1e-13 * np.linalg.norm(G)
    np.testing.assert_allclose(L, scipy.linalg.cholesky(G, lower=True), rtol=1e-12, atol=1e-13)


def test_invert_upper_golden_and_identity():
    case = GOLD["invert_upper"][0]
    np.testing.assert_array_equal(dense.invert_upper(np.array(case["R"], float)), np.array(case["Rinv"]))
    rng = np.random.Generator(np.random.PCG64(6))
    R = np.triu(rng.standard_normal((15, 15))) + 5 * np.eye(15)
    X = dense.invert_upper(R)
    assert np.allclose(np.triu(X), X)
    assert np.linalg.norm(R @ X - np.eye(15)) <= 1e-13
    with pytest.raises(dense.SingularTriangular):
        dense.invert_upper(np.array([[1.0, 0.0], [0.0, 0.0]]))


def test_truncation_rule_golden():
    for case in GOLD["truncation"]:
        assert dense.truncation_rank(np.array(case["sigma"], float), case["tau"]) == case["rho"], case["cite"]


def test_loo_golden_and_invariants():
    n = [2, 2]
    e1 = tt.canonical_tt(1, n)
    e2 = tt.canonical_tt(2, n)
    q2 = tt.tt_sum([e1, e2], [1 / np.sqrt(2), 1 / np.sqrt(2)])
    G = np.array([[tt.tt_dot(a, b) for b in (e1, q2)] for a in (e1, q2)])
    assert dense.loo(G) == pytest.approx(np.sqrt(GOLD["loo"][0]["value_sq"]), rel=1e-14)
    # canonical set -> exactly 0; permutation invariance
    assert dense.loo(np.eye(5)) == 0.0
    rng = np.random.Generator(np.random.PCG64(7))
    B = rng.standard_normal((30, 6))
    Gq = B.T @ B
    P = np.eye(6)[rng.permutation(6)]
    assert dense.loo(P @ Gq @ P.T) == pytest.approx(dense.loo(Gq), rel=1e-13)
    # equals the largest singular value of I - G (2-norm definition, Eq. (9))
    assert dense.loo(Gq) == pytest.approx(np.linalg.norm(np.eye(6) - Gq, 2), rel=1e-12)
