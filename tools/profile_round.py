#!/usr/bin/env python
"""Per-kernel-class timing of ONE TT-rounding of a C2-shaped MGS sum (single stream).

  python tools/profile_round.py [--terms K] [--reps R]

Builds the TT-sum a_K + sum_{j<K} c_j a_j (d = 8, n = 32, r = 10: formal interior rank 10 K),
rounds it R times at delta = 1e-10 with the library's event profiler on, and prints the
per-class launches / time / average launch time.  Small enough to run under ncu."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--terms", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--d", type=int, default=8)
    ap.add_argument("--r", type=int, default=10)
    ap.add_argument("--delta", type=float, default=1e-10)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2211_08770_b200 import _build
    _build.build_library()
    import paper_2211_08770_b200 as P
    from ttinputs import make_shared_tail_set
    st = make_shared_tail_set(args.d, args.n, args.r, args.terms, 1e4, seed=5)
    rng = np.random.Generator(np.random.PCG64(1))
    coeffs = [1.0] + list(rng.standard_normal(args.terms - 1) * 0.3)
    ctx = P.Context(0)
    terms = [P.DeviceTT.from_numpy(a, norm=1.0) for a in st.tensors]
    out, info = P.tt_round(ctx, terms, coeffs, args.delta)  # warm-up
    torch.cuda.synchronize()
    ctx.profile(True)
    t0 = time.perf_counter()
    for _ in range(args.reps):
        out, info = P.tt_round(ctx, terms, coeffs, args.delta)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.reps
    rep = ctx.profile_report()
    ctx.profile(False)
    tot = sum(v["ms"] for v in rep.values())
    print(json.dumps({"ranks": out.ranks, "wall_ms_per_round": 1e3 * wall, "kernel_ms_per_round": tot / args.reps,
                      "launches_per_round": sum(v["launches"] for v in rep.values()) / args.reps}))
    for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"{k:26s} launches/round={v['launches'] / args.reps:7.1f} ms/round={v['ms'] / args.reps:8.3f} "
              f"avg_us={1e3 * v['ms'] / max(v['launches'], 1):8.2f} TF={v['flops'] / max(v['ms'], 1e-9) / 1e9:7.3f}")


if __name__ == "__main__":
    main()
