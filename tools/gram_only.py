#!/usr/bin/env python
"""C3 Gram (m=50, d=16, n=64, r=20) through tt_gram, timed with CUDA events (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import CONFIGS, make_shared_tail_set
    c = CONFIGS["C3"]
    st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed)
    ctx = P.Context(0)
    A = [P.DeviceTT.from_numpy(a) for a in st.tensors]
    G = P.tt_gram(ctx, A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        G = P.tt_gram(ctx, A)
    e1.record()
    torch.cuda.synchronize()
    import numpy as np
    Gx = st.gram_exact()
    err = float(np.linalg.norm(G.cpu().numpy() - Gx) / np.linalg.norm(Gx))
    print(f"gram {e0.elapsed_time(e1) / 3:.3f} ms  rel err vs M^T M {err:.2e}  "
          f"(v1={os.environ.get('TT_B200_GRAM_V1', '0')}, CS={os.environ.get('TT_B200_GRAM_CS', 'auto')})")


if __name__ == "__main__":
    main()
