#!/usr/bin/env python
"""Randomised parity sweep of the batched engine (tt_round_batch) against the oracle, beyond the
fixed cases of tests/test_gpu_batch.py: random d, mode sizes, term counts and ranks (formal rank
<= 64), graded core scalings (singular values over many decades), mixed term scales, loose and
tight tolerances, floor on / off.  Same parity rule as the tests (tests/gpu_util.py).  Prints one
line per failure and a summary; exit code 1 on any failure.

  python tools/fuzz_batch.py [--seeds 200] [--start 0]
"""
import argparse
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=200)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--only", default="", help="comma-separated seeds (verbose)")
    ap.add_argument("--unknown-norms", action="store_true", help="term norms passed as NaN (computed on the device)")
    ap.add_argument("--max-rank", type=int, default=0, help="cap every rank (tt_round_opts.max_rank)")
    ap.add_argument("--serial", action="store_true", help="each item through tt_round's sweep (TT_B200_SERIAL_BATCH=0)")
    args = ap.parse_args()
    import numpy as np
    import paper_2211_08770_b200 as P
    from gpu_util import assert_round_parity, ctx, dev, WINDOW_HITS, WINDOW_CHECKS
    from oracle import rounding, tt
    from ttinputs import make_fuzz_batch
    fails = 0
    seeds = [int(v) for v in args.only.split(",")] if args.only else range(args.start, args.start + args.seeds)
    for seed in seeds:
        items, delta, fc, tag = make_fuzz_batch(seed)
        floor_c = rounding.DEFAULT_FLOOR_C if fc is None else fc
        if args.only:
            print(f"  coeffs of item 0: {items[0][1]}")
        try:
            norms = [[tt.tt_norm(t) for t in terms] for terms, _ in items]
            un = float("nan") if args.unknown_norms else None
            batch = [([dev(t, nr if un is None else un) for t, nr in zip(terms, nb)], coeffs)
                     for (terms, coeffs), nb in zip(items, norms)]
            mr = args.max_rank if args.max_rank > 0 else None
            if args.serial:
                os.environ["TT_B200_SERIAL_BATCH"] = "0"
                outs = [P.tt_round(ctx(), bt, bc, delta, floor_c=floor_c, max_rank=args.max_rank)[0] for bt, bc in batch]
            else:
                outs = P.tt_round_batch(ctx(), batch, delta, floor_c=floor_c, max_rank=args.max_rank)
            for (terms, coeffs), nb, o in zip(items, norms, outs):
                if args.only:
                    ref, info = rounding.tt_round_sum(terms, coeffs, delta, floor_c=floor_c, term_norms=nb)
                    sx = sum(abs(c) * v for c, v in zip(coeffs, nb))
                    _, di = rounding.tt_round(tt.tt_sum([o.to_numpy(), ref], [1.0, -1.0]), 0.0)
                    print(f"  seed {seed}: gpu ranks {list(o.ranks)} oracle {list(info.ranks)} ||x|| {info.norm:.3e} "
                          f"s(x) {sx:.3e} scale {info.scale:.3e} tau {info.tau:.3e} |dx| {di.norm:.3e} "
                          f"|dx|/s {di.norm / sx:.2e}", flush=True)
                    for k, S in enumerate(info.sigmas):
                        r = info.ranks[k + 1]
                        lo, hi = max(0, r - 2), min(len(S), r + 2)
                        print(f"     split {k + 1}: sigma[{lo}:{hi}] = {S[lo:hi]}, tail(r) {np.sqrt(np.sum(S[r:] ** 2)):.3e}")
                assert_round_parity(o.to_numpy(), o.ranks, terms, coeffs, delta, floor_c, nb, max_rank=mr, tag=f"fuzz{seed}")
        except Exception as ex:  # noqa: BLE001
            fails += 1
            print(f"FAIL {tag}\n     {type(ex).__name__}: {str(ex)[:300]}", flush=True)
            if os.environ.get("FUZZ_TRACE"):
                traceback.print_exc()
    print(f"fuzz: {args.seeds} configurations, {fails} failure(s), {WINDOW_CHECKS[0]} rank comparisons, "
          f"{len(WINDOW_HITS)} window hit(s)")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
