#!/usr/bin/env python
"""Batched engine A/B on small cases: reconstruction error of tt_round_batch_strided against the
oracle for shapes that exercise the output-core paths (U = Y V S^-1 DMMA GEMM when the kept
singular values are well separated, the Q_Y application otherwise), partial reflector blocks
(ranks not multiples of 8) and panels with fewer rows than columns.  Run with TT_B200_BR_WY=0/1.

  python tools/wy_debug.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch
    import paper_2211_08770_b200 as P
    from gpu_util import diff_norm
    from oracle import rounding, tt
    from ttinputs import make_random_tt

    ctx = P.Context(0)
    rng = np.random.Generator(np.random.PCG64(77))
    cases = [
        ("d2 n40 r(8,8)", 2, [40, 40], [[1, 8, 1], [1, 8, 1]], [1.0, 0.5]),
        ("d3 n30 r(12,12) spread", 3, [30, 30, 30], [[1, 12, 12, 1], [1, 12, 12, 1]], [1.0, 1e-5]),
        ("d3 n30 r(10,6)", 3, [30, 30, 30], [[1, 10, 10, 1], [1, 6, 6, 1]], [1.0, -0.3]),
        ("d4 n(25,33,2,21)", 4, [25, 33, 2, 21], [[1, 3, 1, 6, 1], [1, 8, 2, 2, 1]], [1.0, 0.7]),
        ("d3 n50 r16x4", 3, [50, 50, 50], [[1, 16, 16, 1]] * 4, [1.0, 1e-3, 1e-6, 2.0]),
        ("rank64 n(7,1,30,9)", 4, [7, 1, 30, 9], [[1, 7, 1, 9, 1], [1, 40, 1, 30, 1], [1, 17, 1, 25, 1]], [1.0, 2.0, -1.0]),
        ("rank64 n(7,2,30,9)", 4, [7, 2, 30, 9], [[1, 7, 1, 9, 1], [1, 40, 1, 30, 1], [1, 17, 1, 25, 1]], [1.0, 2.0, -1.0]),
        ("d3 n(7,30,9) R64", 3, [7, 30, 9], [[1, 7, 9, 1], [1, 40, 30, 1], [1, 17, 25, 1]], [1.0, 2.0, -1.0]),
        ("d2 n(7,9) R64", 2, [7, 9], [[1, 7, 1], [1, 40, 1], [1, 17, 1]], [1.0, 2.0, -1.0]),
        ("d3 n(7,1,9) R64", 3, [7, 1, 9], [[1, 7, 9, 1], [1, 40, 30, 1], [1, 17, 25, 1]], [1.0, 2.0, -1.0]),
        ("d3 n(7,30,9) R(3,64)", 3, [7, 30, 9], [[1, 1, 9, 1], [1, 1, 30, 1], [1, 1, 25, 1]], [1.0, 2.0, -1.0]),
        ("d3 n(7,30,9) R(3,24)", 3, [7, 30, 9], [[1, 1, 9, 1], [1, 1, 8, 1], [1, 1, 7, 1]], [1.0, 2.0, -1.0]),
        ("d3 n(7,30,40) R(3,64)", 3, [7, 30, 40], [[1, 1, 9, 1], [1, 1, 30, 1], [1, 1, 25, 1]], [1.0, 2.0, -1.0]),
        ("d4 n(7,2,30,40)", 4, [7, 2, 30, 40], [[1, 7, 1, 9, 1], [1, 40, 1, 30, 1], [1, 17, 1, 25, 1]], [1.0, 2.0, -1.0]),
        ("d4 n(7,2,30,9) r2", 4, [7, 2, 30, 9], [[1, 7, 2, 9, 1], [1, 40, 2, 30, 1], [1, 17, 2, 25, 1]], [1.0, 2.0, -1.0]),
    ]
    for name, d, n, ranks, coeffs in cases:
        for delta in (0.0, 1e-10):
            B = 3
            items = [[make_random_tt(d, n, r, rng) for r in ranks] for _ in range(B)]
            K = len(ranks)
            cores = [[torch.from_numpy(np.stack([items[b][l][k] for b in range(B)])).cuda() for k in range(d)]
                     for l in range(K)]
            cf = np.array([coeffs] * B)
            fc = 0.0 if delta == 0.0 else rounding.DEFAULT_FLOOR_C
            res = P.tt_round_batch_strided(ctx, cores, cf, delta, floor_c=fc)
            for b in range(B):
                ref, info = rounding.tt_round_sum(items[b], coeffs, delta, floor_c=fc)
                g = res.item_numpy(b)
                same = list(res.ranks[b]) == info.ranks
                if not same:
                    ref, _ = rounding.tt_round_sum(items[b], coeffs, delta, floor_c=fc, force_ranks=list(res.ranks[b]))
                dn = diff_norm(g, ref) / info.scale
                orth = max(float(np.linalg.norm(g[k].reshape(-1, g[k].shape[2]).T @ g[k].reshape(-1, g[k].shape[2])
                                                - np.eye(g[k].shape[2]))) for k in range(d - 1))
                print(f"{name:28s} delta={delta:g} item {b}: ranks {list(res.ranks[b])} oracle {info.ranks} "
                      f"diff/s {dn:.2e} orth {orth:.1e} {'OK' if dn < 1e-10 else 'BAD'}", flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def dump_check():
    """TT_B200_BR_DUMP: compare item 0's right-to-left R factors with numpy's QR of the same
    panels (|R| is unique given the panel, whose row signs do not change |R|)."""
    import numpy as np
    import torch
    import paper_2211_08770_b200 as P
    from ttinputs import make_random_tt
    os.environ["TT_B200_BR_DUMP"] = "/tmp/brdump.bin"
    ctx = P.Context(0)
    rng = np.random.Generator(np.random.PCG64(5))
    for name, d, n, ranks, coeffs in [
            ("d4 n(7,2,30,9) r2", 4, [7, 2, 30, 9], [[1, 7, 2, 9, 1], [1, 40, 2, 30, 1], [1, 17, 2, 25, 1]], [1.0, 1.0, 1.0]),
            ("d4 n(30,30,30,30)", 4, [30] * 4, [[1, 7, 2, 9, 1], [1, 40, 2, 30, 1], [1, 17, 2, 25, 1]], [1.0, 1.0, 1.0])]:
        items = [[make_random_tt(d, n, r, rng) for r in ranks]]
        K = len(ranks)
        cores = [[torch.from_numpy(np.stack([items[0][l][k]])).cuda() for k in range(d)] for l in range(K)]
        P.tt_round_batch_strided(ctx, cores, np.array([coeffs]), 0.0, floor_c=0.0)
        Lg = np.fromfile("/tmp/brdump.bin").reshape(-1, 64, 64)
        # numpy right-to-left sweep of the materialised sum
        from oracle import tt
        x = tt.tt_sum(items[0], coeffs)
        Lprev = None
        for i, k in enumerate(range(d - 1, 0, -1)):
            C = x[k] if Lprev is None else np.tensordot(x[k], Lprev.T, axes=([2], [0]))
            r0, nk, r1 = C.shape
            Q, R = np.linalg.qr(C.reshape(r0, nk * r1).T)
            Lprev = R  # R'_{k-1} x R_{k-1}; core k-1 gets x_3 R^T
            rr, cc = R.shape
            g = Lg[i][:rr, :cc]
            print(f"{name} panel core {k + 1}: |R| diff {np.abs(np.abs(g) - np.abs(R)).max():.2e} (R {rr}x{cc})", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "dump":
    dump_check()
