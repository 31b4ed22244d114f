#!/usr/bin/env python
"""Batched and serial TT-rounding on inputs scaled by powers of ten (value range of the path:
the engines form products of squared norms).  Prints, per scale, the rank agreement with the
oracle and the relative reconstruction error.

  python tools/scale_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import paper_2211_08770_b200 as P
    from oracle import rounding, tt
    from ttinputs import make_random_tt
    ctx = P.Context(0)
    rng = np.random.Generator(np.random.PCG64(99))
    d, n = 5, [12, 20, 16, 20, 12]
    ranks = [[1, 6, 9, 9, 6, 1], [1, 5, 8, 7, 5, 1], [1, 6, 9, 9, 6, 1]]
    base = [make_random_tt(d, n, r, rng) for r in ranks]
    base[2] = base[0]
    coeffs = [1.0, 0.5, -1.0 + 1e-9]
    for e in (0, -60, -75, -90, -120, -140, -150, 60, 75, 90, 120, 140, 150):
        f = 10.0 ** e
        terms = [[c * (f if k == 0 else 1.0) for k, c in enumerate(t)] for t in base]
        norms = [tt.tt_norm(t) for t in terms]
        ref, info = rounding.tt_round_sum(terms, coeffs, 1e-6, floor_c=rounding.DEFAULT_FLOOR_C, term_norms=norms)
        for name in ("batch", "serial"):
            try:
                dt = [P.DeviceTT.from_numpy(t, norm=nr) for t, nr in zip(terms, norms)]
                if name == "batch":
                    o = P.tt_round_batch(ctx, [(dt, coeffs), (dt, coeffs)], 1e-6)[1]
                else:
                    os.environ["TT_B200_SERIAL_BATCH"] = "0"
                    o, _ = P.tt_round(ctx, dt, coeffs, 1e-6)
                g = o.to_numpy()
                _, di = rounding.tt_round(tt.tt_sum([g, ref], [1.0, -1.0]), 0.0)
                print(f"scale 1e{e:+d} {name:6s}: ranks {'==' if list(o.ranks) == list(info.ranks) else '!='} oracle "
                      f"({list(o.ranks)} / {list(info.ranks)}), |dx| / s = {di.norm / info.scale:.2e}")
            except Exception as ex:  # noqa: BLE001
                print(f"scale 1e{e:+d} {name:6s}: {type(ex).__name__}: {str(ex)[:120]}")


if __name__ == "__main__":
    main()
