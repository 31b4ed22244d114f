"""The seeded C4 input generator (ttinputs.make_batch_sums_stacked) against its construction:
per-item view = same bytes, terms of unit norm with right-orthonormal cores 2..d, the
coefficient pattern (1, w_b, 1e-9, 1e-10), and reproducible slices of the stream."""
import numpy as np

from oracle import tt
from ttinputs import make_batch_sums, make_batch_sums_stacked


def test_stacked_equals_per_item_view_and_slices():
    cores, coeffs = make_batch_sums_stacked(5, d=4, n=6, r=3, start=2)
    items = make_batch_sums(5, d=4, n=6, r=3, start=2)
    for b, (terms, cf) in enumerate(items):
        assert cf == list(coeffs[b])
        for s in range(4):
            for k in range(4):
                assert np.array_equal(terms[s][k], cores[s][k][b])
    full, _ = make_batch_sums_stacked(7, d=4, n=6, r=3)
    for s in range(4):
        for k in range(4):
            assert np.array_equal(full[s][k][2:7], cores[s][k])


def test_terms_unit_norm_right_orthonormal_and_coefficients():
    cores, coeffs = make_batch_sums_stacked(4, d=5, n=4, r=3)
    for b in range(4):
        assert coeffs[b, 0] == 1.0 and coeffs[b, 2] == 1e-9 and coeffs[b, 3] == 1e-10
        assert coeffs[b, 1] == (1.0 if b % 2 == 0 else 1e-9)
        for s in range(4):
            y = [cores[s][k][b] for k in range(5)]
            assert abs(tt.tt_norm(y) - 1.0) <= 1e-14
            for k in range(1, 5):
                G = y[k].reshape(y[k].shape[0], -1)
                assert np.abs(G @ G.T - np.eye(G.shape[0])).max() <= 1e-14


def test_fuzz_batch_generator_is_deterministic_and_in_range():
    """ttinputs.make_fuzz_batch: same seed, same bytes; formal ranks <= 64 (a cancelling item repeats
    its first term as its last, so the items of a batch may differ in shape)."""
    from ttinputs import make_fuzz_batch
    for seed in (0, 31, 576, 943):
        a, da, fa, desc = make_fuzz_batch(seed)
        b, db, fb, _ = make_fuzz_batch(seed)
        assert (da, fa) == (db, fb) and len(a) == len(b) >= 1
        for (ta, ca), (tb, cb) in zip(a, b):
            assert ca == cb
            for x, y in zip(ta, tb):
                assert all(np.array_equal(u, v) for u, v in zip(x, y))
            d = len(ta[0])
            for k in range(1, d):
                assert sum(t[k].shape[0] for t in ta) <= 64
