#!/usr/bin/env python
"""The paper's experiments on the GPU (Section 3, Figs. 1-4):
Krylov TT-Laplacian sets (d = 3, m = 20 and d = 6, m = 35, n = 15), the six schemes at
delta in {1e-3, 1e-5, 1e-8}, floor off (paper-pure).  One JSON line per (experiment, scheme,
delta): LOO per step (Fig. 1-2), max ranks and compression ratios of the basis (Figs. 3-4),
GPU time.

  python tools/run_krylov.py [--exp 1,2] [--kinds cgs,...] [--deltas 1e-3,1e-5,1e-8]
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
    ap.add_argument("--exp", default="1,2")
    ap.add_argument("--kinds", default="cgs,mgs,cgs2,mgs2,gram,householder")
    ap.add_argument("--deltas", default="1e-3,1e-5,1e-8")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2211_08770_b200 as P
    ctx = P.Context(0)
    exps = {"1": (3, 15, 20), "2": (6, 15, 35)}
    for e in args.exp.split(","):
        d, n, m = exps[e]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A = P.krylov_set(ctx, d, n, m)
        torch.cuda.synchronize()
        gen_ms = 1e3 * (time.perf_counter() - t0)
        for kind in args.kinds.split(","):
            for delta in [float(x) for x in args.deltas.split(",")]:
                line = {"experiment": int(e), "d": d, "n": n, "m": m, "scheme": kind, "delta": delta,
                        "floor_c": 0.0, "krylov_gen_ms": round(gen_ms, 2)}
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                try:
                    Q, R, rep = P.tt_orth(ctx, kind, A, delta, floor_c=0.0, want_loo=True, keep_u=(kind == "householder"))
                    torch.cuda.synchronize()
                    line["gpu_ms"] = round(1e3 * (time.perf_counter() - t0), 2)
                    line["rounding_calls"] = rep["rounding_calls"]
                    line["max_rank_per_call"] = max(rep["max_rank_per_call"])
                    line["loo_per_step"] = [float(v) for v in rep["loo_per_step"]]
                    line["q_max_rank"] = [max(q.ranks) for q in Q]
                    line["q_compression_ratio"] = [P.compression_ratio(q.ranks, q.modes) for q in Q]
                    line["basis_storage_ratio"] = float(sum(P.storage_count(q.ranks, q.modes) for q in Q) /
                                                        (m * float(np.prod([n] * d))))
                    if rep.get("u"):
                        us = [u for u in rep["u"] if u is not None]
                        line["u_max_rank"] = [max(u.ranks) for u in us]
                        line["u_compression_ratio"] = [P.compression_ratio(u.ranks, u.modes) for u in us]
                except P._native.TTError as err:
                    torch.cuda.synchronize()
                    line["gpu_ms"] = round(1e3 * (time.perf_counter() - t0), 2)
                    line["error"] = str(err)
                print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
