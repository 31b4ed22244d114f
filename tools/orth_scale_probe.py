#!/usr/bin/env python
"""tt_orth on a C1-shaped shared-tail set scaled by powers of ten: R must scale with the inputs
(R = f R_M up to signs) and Q must stay orthonormal (value range of the drivers).

  python tools/orth_scale_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import paper_2211_08770_b200 as P
    from ttinputs import CONFIGS, make_shared_tail_set
    ctx = P.Context(0)
    c = CONFIGS["C1"]
    st = make_shared_tail_set(c.d, c.n, c.r, c.m, 1e4, c.seed)
    qm, rm = st.qr_exact()
    for e in (0, -60, -100, -140, 60, 100, 140):
        f = 10.0 ** e
        A = [P.DeviceTT.from_numpy([x * (f if k == 0 else 1.0) for k, x in enumerate(a)]) for a in st.tensors]
        for kind in ("cgs2", "mgs2", "gram", "householder"):
            try:
                Q, R, rep = P.tt_orth(ctx, kind, A, 1e-10, want_loo=True)
                R = np.asarray(R)
                sg = np.sign(np.diag(R))
                err = np.linalg.norm(sg[:, None] * R / f - rm) / np.linalg.norm(rm)
                loo = float(rep["loo_per_step"][-1])
                print(f"scale 1e{e:+d} {kind:11s}: |R/f - R_M| / |R_M| = {err:.2e}, loo_last = {loo:.2e}", flush=True)
            except Exception as ex:  # noqa: BLE001
                print(f"scale 1e{e:+d} {kind:11s}: {type(ex).__name__}: {str(ex)[:140]}", flush=True)


if __name__ == "__main__":
    main()
