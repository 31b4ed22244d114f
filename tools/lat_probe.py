#!/usr/bin/env python
"""Per-call latency of one small TT-rounding (C1-shaped sum: K terms of rank r, d, n) through
tt_round, serial sweep vs the one-item batch route (TT_B200_SERIAL_BATCH), host wall clock per call.

  python tools/lat_probe.py [--K 10 --d 4 --n 8 --r 3 --calls 200]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=10)
    ap.add_argument("--d", type=int, default=4)
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--r", type=int, default=3)
    ap.add_argument("--calls", type=int, default=200)
    ap.add_argument("--tol", type=float, default=1e-8)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_random_tt
    rng = np.random.Generator(np.random.PCG64(7))
    ranks = [1] + [a.r] * (a.d - 1) + [1]
    terms = [P.DeviceTT.from_numpy(make_random_tt(a.d, [a.n] * a.d, ranks, rng)) for _ in range(a.K)]
    coeffs = list(rng.standard_normal(a.K))
    ctx = P.Context(0)
    for _ in range(5):
        P.tt_round(ctx, terms, coeffs, a.tol)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.calls):
        out, info = P.tt_round(ctx, terms, coeffs, a.tol)
    torch.cuda.synchronize()
    us = 1e6 * (time.perf_counter() - t0) / a.calls
    ctx.profile(True)
    for _ in range(20):
        P.tt_round(ctx, terms, coeffs, a.tol)
    torch.cuda.synchronize()
    rep = ctx.profile_report()
    ctx.profile(False)
    ker = ", ".join(f"{k} {v['launches'] // 20}x {1e3 * v['ms'] / 20:.1f}us" for k, v in
                    sorted(rep.items(), key=lambda kv: -kv[1]["ms"]))
    print(f"K={a.K} d={a.d} n={a.n} r={a.r} serial_batch={os.environ.get('TT_B200_SERIAL_BATCH', '1')}: "
          f"{us:.1f} us/call, ranks {out.ranks}, launches/call {ctx.launches / (a.calls + 5):.1f}\n  per call: {ker}")


if __name__ == "__main__":
    main()
