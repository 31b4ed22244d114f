#!/usr/bin/env python
"""Time tt_round_batch_strided on C4 items (d=10, n=32, 4 x rank 16, delta 1e-6).

  python tools/bench_batch.py [--B 512] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=512)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-profile", action="store_true",
                    help="no per-launch events: the wave runs split over the streams as in bench.py")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2211_08770_b200 import _build
    _build.build_library()
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked
    t0 = time.time()
    cores, coeffs = make_batch_sums_stacked(args.B)
    print(f"generated {args.B} items in {time.time() - t0:.1f} s", flush=True)
    ctx = P.Context(0)
    dc = [[torch.from_numpy(c).cuda() for c in term] for term in cores]
    norms = np.ones((args.B, 4))
    res = P.tt_round_batch_strided(ctx, dc, coeffs, 1e-6, norms=norms)
    torch.cuda.synchronize()
    ranks = res.ranks[:4].tolist()
    del res
    ctx.profile(not args.no_profile)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        res = P.tt_round_batch_strided(ctx, dc, coeffs, 1e-6, norms=norms)
        del res
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    rep = ctx.profile_report() if not args.no_profile else {}
    ctx.profile(False)
    print(json.dumps({"B": args.B, "ms_per_batch": ms, "roundings_per_s": args.B / ms * 1e3, "ranks": ranks}))
    for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"{k:20s} launches={v['launches']:6d} ms/batch={v['ms'] / args.reps:9.3f} "
              f"TF={v['flops'] / max(v['ms'], 1e-9) / 1e9:7.3f}")


if __name__ == "__main__":
    main()
