#!/usr/bin/env python
"""C5 prefix (m' = 20) through tt_orth Householder with and without the TTH-vec masking variant
(hh_mask): time, max rank, R against the closed form R_M, LOO per step.
Measured (B200): both 6.2-6.3 s, R error 1.17e-13, LOO 2.0e-13 / 2.1e-13 at step 20."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2211_08770_b200 as P
from ttinputs import CONFIGS, make_shared_tail_set
c = CONFIGS["C5"]; st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed)
ctx = P.Context(0)
A = [P.DeviceTT.from_numpy(a) for a in st.tensors[:20]]
rm = st.qr_exact()[1][:20, :20]
for mask in (False, True):
    t0 = time.perf_counter()
    Q, R, rep = P.tt_orth(ctx, "householder", A, c.delta, want_loo=True, hh_mask=mask)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    sg = np.sign(np.diag(R)); sg[sg == 0] = 1
    print(json.dumps({"hh_mask": mask, "s": t, "max_rank": int(max(rep["max_rank_per_call"])),
                      "R_err": float(np.linalg.norm(sg[:, None] * R - rm) / np.linalg.norm(rm)),
                      "loo": [float(x) for x in rep["loo_per_step"][[0, 9, 19]]]}))
