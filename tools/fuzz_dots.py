#!/usr/bin/env python
"""Randomised parity sweep of the contraction kernels against the oracle: tt_gram (equal shapes:
tiled DMMA kernel for ranks <= 32, pair kernel above), tt_gram_blocks, tt_dot_batch (ragged rank
profiles, two-profile batches), tt_norm and tt_element, over random orders, mode sizes (1 .. 40),
ranks (1 .. 48, odd and even) and term scales.  Bars: |<x, y> - oracle| <= 1e-12 ||x|| ||y||,
elements 1e-13 of the core-norm product.

  python tools/fuzz_dots.py [--seeds 300] [--start 0]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=300)
    ap.add_argument("--start", type=int, default=0)
    args = ap.parse_args()
    import numpy as np
    import paper_2211_08770_b200 as P
    from gpu_util import ctx, dev
    from oracle import tt
    from ttinputs import make_random_tt
    fails = 0
    for seed in range(args.start, args.start + args.seeds):
        rng = np.random.Generator(np.random.PCG64(70000 + seed))
        d = int(rng.integers(1, 10))
        n = [int(v) for v in rng.integers(1, 41, size=d)]
        rmax = int(rng.choice([3, 8, 20, 32, 48]))
        m = int(rng.integers(1, 8))
        equal = rng.random() < 0.5
        prof = [1] + [int(v) for v in rng.integers(1, rmax + 1, size=d - 1)] + [1]
        A = []
        for _ in range(m):
            r = prof if equal else [1] + [int(v) for v in rng.integers(1, rmax + 1, size=d - 1)] + [1]
            t = make_random_tt(d, n, r, rng)
            if rng.random() < 0.3:
                t[0] = t[0] * 10.0 ** float(rng.integers(-60, 61))
            A.append(t)
        tag = f"seed {seed} d={d} n={n} rmax={rmax} m={m} equal={equal}"
        try:
            nr = [tt.tt_norm(a) for a in A]
            D = [dev(a) for a in A]
            want = np.array([[tt.tt_dot(A[i], A[j]) for j in range(m)] for i in range(m)])
            bar = 1e-12 * np.outer(nr, nr) + 1e-300
            pairs = [(i, j) for i in range(m) for j in range(m)]
            got = P.tt_dot_batch(ctx(), [D[i] for i, _ in pairs], [D[j] for _, j in pairs]).cpu().numpy().reshape(m, m)
            assert np.all(np.abs(got - want) <= bar), ("tt_dot_batch", float(np.max(np.abs(got - want) / bar)))
            for i in range(m):
                gn = P.tt_norm(ctx(), D[i])
                assert abs(gn - nr[i]) <= 1e-12 * nr[i] + 1e-300, ("tt_norm", gn, nr[i])
            if equal:
                G = P.tt_gram(ctx(), D).cpu().numpy()
                assert np.all(np.abs(G - want) <= bar), ("tt_gram", float(np.max(np.abs(G - want) / bar)))
                if m >= 2:
                    bi = int(rng.integers(1, m + 1))
                    bj = int(rng.integers(1, m + 1))
                    i0, j0 = int(rng.integers(0, m - bi + 1)), int(rng.integers(0, m - bj + 1))
                    gb = P.tt_gram_blocks(ctx(), D, [(i0, j0, bi, bj)]).cpu().numpy().reshape(bi, bj)
                    assert np.all(np.abs(gb - want[i0:i0 + bi, j0:j0 + bj]) <= bar[i0:i0 + bi, j0:j0 + bj]), "tt_gram_blocks"
            N = 1
            for v in n:
                N *= v
            N = min(N, 2 ** 62)
            lins = [1, N] + [int(rng.integers(1, N + 1)) for _ in range(4)]
            ge = P.tt_element(ctx(), D[0], lins).cpu().numpy()
            for lin, g in zip(lins, ge):
                w = tt.element(A[0], [i - 1 for i in tt.phi(lin, n)])
                scale = float(np.prod([np.linalg.norm(c) for c in A[0]]))
                assert abs(g - w) <= 1e-13 * scale + 1e-300, ("tt_element", lin, g, w)
        except Exception as ex:  # noqa: BLE001
            fails += 1
            print(f"FAIL {tag}\n     {type(ex).__name__}: {str(ex)[:300]}", flush=True)
    print(f"fuzz_dots: {args.seeds} configurations, {fails} failure(s)")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
