#!/usr/bin/env python
"""C5 (BASELINE.json configs[4]: TT-Householder, m = 100, d = 50, n = 16, r = 30, kappa = 1e12,
delta = 1e-12) against the oracle -- SURVEY.md §8(c) C6 / §8(d) D5 protocol for the config whose
full oracle run is out of reach (hours):

A. free-running prefix m' = 20 (PAPER.md:479-484 per-step curves are prefixes of one run, A17):
   GPU tt_orth and oracle.orth on a_1..a_20: Table 1 counts, per-call max ranks, R (up to
   D = diag(sign R(i,i)), A8) against the oracle and against R_M, LOO per step (factor 2 where
   above max(1e-14, A_k)), and every q_i through an exact oracle rounding of the difference;
B. teacher-forced spot steps i in {1, 2, 50, 100} of the full m = 100 run: the GPU's own rounding
   inputs at those steps (tt_ctx_round_hook: TTH-vec roundings 1 and 2 of step i, the w_{i+1}
   update, and the phase-2 q_i rounding) are replayed through oracle.rounding.tt_round_sum and
   through tt_round (the GPU primitive, same inputs): ranks identical or inside the C6 window
   (1e-12 tau + c_floor u s(x)) and reconstructions within 1e-10 s(x) (where ranks differ, of
   the oracle's rounding forced to the GPU's ranks).

  python tools/c5_parity.py [--prefix 20] [--steps 1,2,50,100] [--out gpurun_out/c5_parity.json]

Result committed as profiles/c5_parity_r02.json.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prefix", type=int, default=20)
    ap.add_argument("--steps", default="1,2,50,100")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c5_parity.json"))
    ap.add_argument("--skip-prefix", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2211_08770_b200 as P
    from gpu_util import diff_norm, window
    from oracle import orth, rounding
    from oracle.dense import U_ROUND
    from ttinputs import CONFIGS, make_shared_tail_set

    c = CONFIGS["C5"]
    st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed)
    ctx = P.Context(0)
    A = [P.DeviceTT.from_numpy(a) for a in st.tensors]
    report = {"config": "C5", "m": c.m, "d": c.d, "n": c.n, "r": c.r, "kappa": c.kappa, "delta": c.delta,
              "floor_c": rounding.DEFAULT_FLOOR_C, "host_threads": os.cpu_count()}
    rm_full = st.qr_exact()[1]

    def signs(R):
        s = np.sign(np.diag(R))
        s[s == 0] = 1.0
        return s

    # ---------------------------------------------------------------- A. free-running prefix
    if not args.skip_prefix:
        mp = args.prefix
        t0 = time.perf_counter()
        Q, R, rep = P.tt_orth(ctx, "householder", A[:mp], c.delta, want_loo=True)
        torch.cuda.synchronize()
        t_gpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref = orth.orth("householder", st.tensors[:mp], c.delta)
        t_orc = time.perf_counter() - t0
        Rg = signs(R)[:, None] * R
        Ro = signs(ref.R)[:, None] * ref.R
        rm = rm_full[:mp, :mp]
        # LOO of each side's Q through the oracle's routine, and each side's own
        from oracle.orth import OrthResult
        loo_o = np.array(ref.loo_per_step())
        Qg_np = [q.to_numpy() for q in Q]
        loo_g = OrthResult(Qg_np, R).loo_per_step()
        loo_g_own = rep["loo_per_step"]
        qd = []
        for i in range(mp):
            # q_i is unique up to the sign of R(i,i) (A8): align before differencing
            qo = [cc.copy() for cc in ref.Q[i]]
            sgn = signs(R)[i] * signs(ref.R)[i]
            qo[0] = qo[0] * sgn
            qd.append(diff_norm(Q[i].to_numpy(), qo))
        kap = [np.linalg.cond(st.M[:, :k + 1]) if k > 0 else 1.0 for k in range(mp)]
        amp = [(rounding.DEFAULT_FLOOR_C * U_ROUND + c.delta) * mp * kk for kk in kap]
        ratio = [float(max(a, b) / min(a, b)) for a, b in zip(loo_g, loo_o) if min(a, b) > 0 and max(a, b) > 1e-14]
        report["prefix"] = {
            "m": mp, "gpu_s": t_gpu, "oracle_s": t_orc,
            "calls": [int(rep["rounding_calls"]), int(ref.rounding_calls)],
            "calls_table1": 4 * mp - 1,
            "max_rank_per_call_equal": list(map(int, rep["max_rank_per_call"])) == [int(max(x.ranks)) for x in ref.infos],
            "max_rank_per_call_gpu": list(map(int, rep["max_rank_per_call"])),
            "max_rank_per_call_oracle": [int(max(x.ranks)) for x in ref.infos],
            "max_rank": int(max(rep["max_rank_per_call"])),
            "R_rel_err_vs_oracle": float(np.linalg.norm(Rg - Ro) / np.linalg.norm(Ro)),
            "R_rel_err_vs_R_M": float(np.linalg.norm(Rg - rm) / np.linalg.norm(rm)),
            "R_oracle_rel_err_vs_R_M": float(np.linalg.norm(Ro - rm) / np.linalg.norm(rm)),
            "loo_gpu": [float(x) for x in loo_g], "loo_oracle": [float(x) for x in loo_o],
            "loo_gpu_own_dots": [float(x) for x in loo_g_own],
            "loo_ratio_max": max(ratio) if ratio else None,
            "q_diff": [float(x) for x in qd], "q_diff_max": float(max(qd)),
            "amplified_noise_bound": [float(x) for x in amp],
        }
        print(json.dumps({k: v for k, v in report["prefix"].items() if not isinstance(v, list)}), flush=True)

    # ---------------------------------------------------------------- B. teacher-forced spot steps
    steps = [int(s) for s in args.steps.split(",") if s]
    m = c.m
    sel = {}
    for i in steps:
        sel[3 * (i - 1)] = (i, "tthvec_round1")
        sel[3 * (i - 1) + 1] = (i, "tthvec_round2")
        if i < m:
            sel[3 * (i - 1) + 2] = (i, "w_update")
        sel[3 * m - 1 + (i - 1)] = (i, "q_phase2")
    t0 = time.perf_counter()
    with P.RoundTrace(ctx, select=sel.keys()) as tr:
        Qf, Rf, repf = P.tt_orth(ctx, "householder", A, c.delta, want_loo=True)
    torch.cuda.synchronize()
    report["full_run"] = {"gpu_s": time.perf_counter() - t0, "calls": int(repf["rounding_calls"]),
                          "max_rank": int(max(repf["max_rank_per_call"])),
                          "R_rel_err_vs_R_M": float(np.linalg.norm(signs(Rf)[:, None] * Rf - rm_full) /
                                                    np.linalg.norm(rm_full)),
                          "loo_last": float(repf["loo_per_step"][-1])}
    print(json.dumps(report["full_run"]), flush=True)
    del Qf
    spot = []
    for call in sorted(tr.calls):
        coeffs, cores, norms, delta, floor_c = tr.calls[call]
        i, what = sel[call]
        # the oracle materialises the TT-sum (its plain definition): skip a replay that would not
        # fit in half the host's free memory (a host out of memory would take the box down)
        import psutil
        R = [1] + [sum(cs[k].shape[2] for cs in cores) for k in range(len(cores[0]) - 1)] + [1]
        need = 8.0 * 1.3 * sum(R[k] * cores[0][k].shape[1] * R[k + 1] for k in range(len(cores[0])))
        avail = psutil.virtual_memory().available
        if need > 0.5 * avail:
            row = {"step": i, "call": call, "what": what, "K": len(coeffs), "formal_rank_max": int(max(R)),
                   "skipped": f"oracle replay needs ~{need / 1e9:.0f} GB, host has {avail / 1e9:.0f} GB free"}
            spot.append(row)
            print(json.dumps(row), flush=True)
            tr.calls[call] = None
            continue
        terms = [P.DeviceTT.from_numpy(cs, norm=nr) for cs, nr in zip(cores, norms)]
        g, gi = P.tt_round(ctx, terms, coeffs, delta, floor_c=floor_c)
        gn = g.to_numpy()
        del terms
        t0 = time.perf_counter()
        ref, info = rounding.tt_round_sum(cores, coeffs, delta, floor_c=floor_c, term_norms=norms)
        t_o = time.perf_counter() - t0
        same = list(g.ranks) == list(info.ranks)
        win = window(info, floor_c)
        gaps = []
        if not same:
            for k, (a, b) in enumerate(zip(g.ranks[1:-1], info.ranks[1:-1])):
                if a != b:
                    S = info.sigmas[k]
                    lo, hi = min(a, b), max(a, b)
                    gaps.append(min(abs(np.sqrt(np.sum(S[rho:] ** 2)) - info.tau) for rho in range(lo, hi + 1)) / win)
            ref, _ = rounding.tt_round_sum(cores, coeffs, delta, floor_c=floor_c, term_norms=norms,
                                           force_ranks=list(g.ranks))
        dn = diff_norm(gn, ref)
        row = {"step": i, "call": call, "what": what, "K": len(coeffs), "formal_rank_max": int(max(info.formal_ranks)),
               "ranks_equal": same, "max_rank_gpu": int(max(g.ranks)), "max_rank_oracle": int(max(info.ranks)),
               "window_gaps_over_window": gaps, "within_window": all(x <= 1.0 for x in gaps),
               "diff_over_scale": float(dn / info.scale), "pass": (same or all(x <= 1.0 for x in gaps))
               and dn <= 1e-10 * info.scale, "oracle_s": t_o, "norm_gpu": gi["norm"], "norm_oracle": info.norm}
        spot.append(row)
        print(json.dumps(row), flush=True)
        del ref, cores
        tr.calls[call] = None
    report["teacher_forced"] = spot
    report["teacher_forced_all_pass"] = all(r.get("pass", False) for r in spot if "skipped" not in r)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(report, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
