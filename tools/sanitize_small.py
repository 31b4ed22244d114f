#!/usr/bin/env python
"""Tiny invocations of the batched rounding engine and the tiled Gram for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

  compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked, make_random_tt
    ctx = P.Context(0)
    # several stacks per panel (n r > 192), a ragged tail, a short left-to-right split
    cores, coeffs = make_batch_sums_stacked(3, d=4, n=20, r=12)
    res = P.tt_round_batch_strided(ctx, [[torch.from_numpy(c).cuda() for c in t] for t in cores], coeffs, 1e-6,
                                   norms=np.ones((3, 4)))
    print("batch ranks", res.ranks.tolist())
    rng = np.random.Generator(np.random.PCG64(3))
    A = [P.DeviceTT.from_numpy(make_random_tt(4, [5, 7, 3, 6], [1, 9, 12, 5, 1], rng)) for _ in range(5)]
    G = P.tt_gram(ctx, A)
    torch.cuda.synchronize()
    print("gram ok", float(G.diagonal().sum()))


if __name__ == "__main__":
    main()
