#!/usr/bin/env python
"""Benchmark of the TT-rounding hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[3], "C4" -- the configuration the metric "TT-roundings/sec ...
vs B200 peak" is quoted on): a batch of 4096 independent TT-roundings, item b the TT-sum
y1 + w_b y2 + 1e-9 y3 + 1e-10 y4 of four unit-norm rank-16 TT-vectors (d = 10, n = 32; formal
rank 64), relative tolerance 1e-6 (ranks 32 / 16).  One
step = one tt_round_batch_strided call over the batch (right-to-left Householder sweep, norm and
threshold, left-to-right truncated SVDs, for every item).  The TT-dot Gram matrix of C3
(configs[2], 50 TT-vectors d = 16, n = 64, r = 20: 1275 pairs) and the C2 (configs[1])
TT-MGS + TT-MGS2 drivers are timed alongside and reported in their own keys.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--batch B]

N > 1 (torchrun, one process per GPU): every rank rounds its own 4096-item C4 batch (items
rank*4096 .. rank*4096 + 4095 of the seeded stream; no data-path collective: the roundings are
independent); time = max over ranks; value = all ranks' items / that time; "scaling": "weak".  --impl reference times the CPU oracle (oracle/, the slow fp64 reference written from
the paper) on a bounded sample of the same items.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TT-roundings/sec (fp64 TFLOP/s vs B200 FP64 peak; TT-dot Gram pairs/sec alongside)"
# measured on this pool's B200 by tools/fp64_peak.cu (profiles/fp64_peak_r01.json): FP64 FMA
# pipe (DFMA, what the batched rounding kernels issue) and FP64 tensor (DMMA m8n8k4)
FP64_DFMA_PEAK_TFLOPS = 34.18
FP64_DMMA_PEAK_TFLOPS = 37.07
C4_DELTA = 1e-6
C4_BATCH = 4096
CPU_SAMPLE_SECONDS = 15.0


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi sampling during the timed region (the recipe's clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        cmd = ["nvidia-smi", "-i", str(self.index),
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
               "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
               "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _slice(batch: int, rank: int, world: int):
    """(start, count) of this rank's shard: a whole `batch`-item batch per GPU (weak scaling),
    rank r taking items [r * batch, (r + 1) * batch) of the seeded stream."""
    return rank * batch, batch


def _blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:
        return os.cpu_count() or 1


def _config(batch: int, world: int):
    return {"workload": f"C4 (BASELINE.json configs[3]): batch of {batch} independent TT-roundings, "
                        "each the TT-sum of 4 unit-norm rank-16 TT-vectors (d=10, n=32, formal rank 64)",
            "batch": batch, "global_batch": batch * world, "d": 10, "n": 32, "terms": 4, "term_rank": 16,
            "delta": C4_DELTA, "floor_c": 2048.0,
            "parallelism": f"batch shard x{world} ({batch} independent roundings per GPU, no collective)",
            "l2": "inputs (8.7 GB at B=4096) exceed L2; L2 also flushed (256 MB write) between timed steps"}


def oracle_sample(seconds: float, offset: int = 0):
    """The CPU oracle (as it stands) on C4 items in order until `seconds` have elapsed."""
    from oracle import rounding
    from ttinputs import make_batch_sums
    done, t0 = 0, time.perf_counter()
    while True:
        items = make_batch_sums(4, start=offset + done)
        for terms, coeffs in items:
            rounding.tt_round_sum(terms, coeffs, C4_DELTA, floor_c=rounding.DEFAULT_FLOOR_C, term_norms=[1.0] * 4)
        done += len(items)
        if time.perf_counter() - t0 >= seconds:
            break
    # generation of the 4-item blocks is timed too but is < 1 % of the oracle's time
    return done, time.perf_counter() - t0


def run_reference(args, rank: int, world: int):
    """Reference arm: the CPU oracle on a bounded sample of the C4 items (rank 0 only)."""
    if rank != 0:
        return
    times, counts = [], []
    for it in range(args.warmup + args.steps):
        n, t = oracle_sample(CPU_SAMPLE_SECONDS / max(args.steps, 1) if it >= args.warmup else 1.0)
        if it >= args.warmup:
            times.append(t)
            counts.append(n)
    T = sum(times)
    value = sum(counts) / T
    cores = _blas_threads()
    sample = (f"oracle (numpy/LAPACK fp64) TT-rounding of the first {max(counts)} C4 items per step, "
              f"{T:.1f} s over {args.steps} steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(args.batch, world),
            "cpu_baseline": {"value": value, "unit": "roundings/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "roundings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=C4_BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the Gram / driver side measurements")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="pipelined slices of the host-to-host call")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2211_08770_b200 import _build
    _build.build_library()
    import paper_2211_08770_b200 as P
    from ttinputs import make_batch_sums_stacked

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stream = torch.cuda.current_stream(local_rank)
    ctx = P.Context(local_rank, stream=stream)

    start, B = _slice(args.batch, rank, world)
    cores_h, coeffs = make_batch_sums_stacked(B, start=start)
    norms = np.ones((B, 4))
    cores = [[torch.from_numpy(c).to(dev) for c in term] for term in cores_h]
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def step(inp):
        return P.tt_round_batch_strided(ctx, inp, coeffs, C4_DELTA, norms=norms)

    for _ in range(args.warmup):
        res = step(cores)
        del res
    torch.cuda.synchronize()

    # ------------------------------------------------------------ timed (device-resident inputs)
    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = ctx.launches
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step(cores)
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        ranks = res.ranks
        del res
    barrier()
    launches = ctx.launches - launches0
    clocks = sampler.stop()
    t_local = sum(step_ms) / 1e3
    if world > 1:
        t = torch.tensor([t_local], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    else:
        t_max = t_local
    value = args.batch * world * args.steps / t_max  # all ranks' items / max-over-ranks time
    rank_ok = bool(np.all(ranks[:, 1:-1] == np.where((np.arange(start, start + B) % 2 == 0), 32, 16)[:, None]))

    # ------------------------------------------------------------ per-kernel profile (one extra step)
    ctx.profile(True)
    res = step(cores)
    prof = ctx.profile_report()
    ctx.profile(False)
    out_doubles = res.total_doubles()
    del res

    # ------------------------------------------------------------ end to end (pinned host buffers)
    # the public host-to-host call: inputs copied from pinned memory and results copied back
    # inside the timed region, pipelined over --e2e-chunks slices (tt_round_batch_host)
    host = [[torch.from_numpy(c).pin_memory() for c in term] for term in cores_h]
    h2d = sum(x.numel() * 8 for term in host for x in term)
    out_host = torch.empty(out_doubles + 4096, dtype=torch.float64).pin_memory()
    e2e_ms, d2h = [], 0
    # untimed calls first (the torch caching allocator sizes the slice buffers)
    for _ in range(2):
        out_host, _, _, _ = P.tt_round_batch_host(ctx, host, coeffs, C4_DELTA, norms=norms, chunks=args.e2e_chunks, out_host=out_host)
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out_host, rk_h, nr_h, cnt = P.tt_round_batch_host(ctx, host, coeffs, C4_DELTA, norms=norms, chunks=args.e2e_chunks,
                                                          out_host=out_host, start_event=e0)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        d2h = cnt * 8 + rk_h.nbytes + nr_h.nbytes
    te = sum(e2e_ms) / 1e3
    if world > 1:
        t = torch.tensor([te], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    e2e_value = args.batch * world * args.steps / te

    # ------------------------------------------------------------ roofline of the dominant kernel
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    total_ms = sum(v["ms"] for v in prof.values())
    achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
    traffic = None
    try:  # DRAM bytes per launch of this kernel class from the committed ncu --set full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic_r01.json"))).get(dom_name)
        traffic = tr["dram_bytes_per_launch"] if tr else None
    except Exception:
        traffic = None
    roof = {"bound": "alu", "achieved": achieved, "peak": FP64_DFMA_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_DFMA_PEAK_TFLOPS, "traffic": traffic,
            "traffic_source": "profiles/ncu_traffic_r01.json (dram__bytes_read.sum + dram__bytes_write.sum, one launch)",
            "peak_source": "measured FP64 FMA (DFMA) throughput, tools/fp64_peak.cu -> profiles/fp64_peak_r01.json "
                           "(nominal 148 SM x 64 FMA/clk x 2 x 1.965 GHz = 37.2 TF)",
            "kernel": dom_name, "launches": dom["launches"], "avg_launch_us": 1e3 * dom["ms"] / dom["launches"],
            "share_of_kernel_time": dom["ms"] / total_ms,
            "work_model": "LAPACK-standard flop counts of the operations each launch performs (DESIGN.md §7)"}
    all_flops = sum(v["flops"] for v in prof.values())
    kernel_classes = {k: {"launches": v["launches"], "ms": round(v["ms"], 3), "share": round(v["ms"] / total_ms, 4),
                          "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 else 0.0}
                      for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}

    # ------------------------------------------------------------ alongside: Gram (C3), drivers (C2)
    extras = {}
    if not args.no_extras:
        from ttinputs import CONFIGS, make_shared_tail_set
        c3 = CONFIGS["C3"]
        st3 = make_shared_tail_set(c3.d, c3.n, c3.r, c3.m, c3.kappa, c3.seed)  # same set on every rank (sharded parts)
        A3 = [P.DeviceTT.from_numpy(a) for a in st3.tensors]
        G = P.tt_gram(ctx, A3)
        torch.cuda.synchronize()
        gms = []
        for _ in range(3):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            G = P.tt_gram(ctx, A3)
            e1.record(stream)
            torch.cuda.synchronize()
            gms.append(e0.elapsed_time(e1))
        pairs = c3.m * (c3.m + 1) // 2
        gerr = float(np.linalg.norm(G.cpu().numpy() - st3.gram_exact()) / np.linalg.norm(st3.gram_exact()))
        extras["gram_pairs_per_s"] = pairs / (statistics.median(gms) * 1e-3)
        extras["gram"] = {"workload": "C3 (configs[2]) TT-dot Gram matrix, m=50, d=16, n=64, r=20",
                          "pairs": pairs, "ms": statistics.median(gms), "rel_err_vs_MtM": gerr}
        if world > 1:  # C3 Gram sharded by pair blocks over the ranks (one NCCL all-gather)
            from paper_2211_08770_b200 import parallel
            blockfn = lambda blocks: P.tt_gram_blocks(ctx, A3, blocks)  # noqa: E731
            Gs = parallel.sharded_gram(c3.m, blockfn, block=4)
            torch.cuda.synchronize()
            sms = []
            for _ in range(3):
                barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                Gs = parallel.sharded_gram(c3.m, blockfn, block=4)
                e1.record(stream)
                torch.cuda.synchronize()
                sms.append(e0.elapsed_time(e1))
            tg = torch.tensor([statistics.median(sms)], device=dev, dtype=torch.float64)
            dist.all_reduce(tg, op=dist.ReduceOp.MAX)
            # CGS2 with the projection dots of every step split over the ranks (one NCCL
            # all-gather per pass), C3 prefix m = 10; roundings replicated on every rank
            A3p = A3[:10]
            parallel.cgs_sharded(ctx, "cgs2", A3p[:2], c3.delta)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, Rsh, ncalls = parallel.cgs_sharded(ctx, "cgs2", A3p, c3.delta)
            e1.record(stream)
            torch.cuda.synchronize()
            tc = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
            dist.all_reduce(tc, op=dist.ReduceOp.MAX)
            rm = st3.qr_exact()[1][:10, :10]
            extras["cgs2_sharded"] = {"ranks": world, "m": 10, "roundings": ncalls, "ms": float(tc.item()),
                                      "R_rel_err_vs_R_M": float(np.linalg.norm(Rsh - rm) / np.linalg.norm(rm)),
                                      "collective": "NCCL all_gather_into_tensor of the projection dots, per pass"}
            extras["gram_sharded"] = {"ranks": world, "ms": float(tg.item()), "pairs_per_s": pairs / (float(tg.item()) * 1e-3),
                                      "rel_err_vs_MtM": float(np.linalg.norm(Gs - st3.gram_exact()) / np.linalg.norm(st3.gram_exact())),
                                      "collective": "NCCL all_gather_into_tensor of padded pair blocks"}
        c2 = CONFIGS["C2"]
        st2 = make_shared_tail_set(c2.d, c2.n, c2.r, c2.m, c2.kappa, c2.seed + rank)
        A2 = [P.DeviceTT.from_numpy(a) for a in st2.tensors]
        P.tt_orth(ctx, "mgs", A2, c2.delta)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, _, r1 = P.tt_orth(ctx, "mgs", A2, c2.delta)
        _, _, r2 = P.tt_orth(ctx, "mgs2", A2, c2.delta)
        e1.record(stream)
        torch.cuda.synchronize()
        calls = r1["rounding_calls"] + r2["rounding_calls"]
        extras["drivers_c2"] = {"workload": "C2 (configs[1]) TT-MGS + TT-MGS2, m=30, d=8, n=32, r=10",
                                "roundings": calls, "ms": e0.elapsed_time(e1),
                                "roundings_per_s": calls / (e0.elapsed_time(e1) * 1e-3)}
        # the paper's own workload (Section 3, experiment 1): Krylov TT-Laplacian set
        # d=3, n=15, m=20, five schemes (Gram breaks down on it) at delta=1e-5, floor off
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        K1 = P.krylov_set(ctx, 3, 15, 20)
        kcalls, kloo = 0, {}
        for kind in ("cgs", "mgs", "cgs2", "mgs2", "householder"):
            _, _, rk = P.tt_orth(ctx, kind, K1, 1e-5, floor_c=0.0, want_loo=True)
            kcalls += rk["rounding_calls"]
            kloo[kind] = float(rk["loo_per_step"][-1])
        e1.record(stream)
        torch.cuda.synchronize()
        extras["krylov_exp1"] = {"workload": "PAPER.md Sec. 3 experiment 1: Krylov TT-Laplacian set d=3, n=15, m=20 "
                                             "(rank-1 rounded), CGS/MGS/CGS2/MGS2/Householder at delta=1e-5, floor off",
                                 "roundings": kcalls, "ms": e0.elapsed_time(e1),
                                 "roundings_per_s": kcalls / (e0.elapsed_time(e1) * 1e-3), "loo_last": kloo}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(args.batch, world),
            "e2e": {"value": e2e_value, "unit": "roundings/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_steps": [round(x, 2) for x in e2e_ms], "api": f"tt_round_batch_host ({args.e2e_chunks} pipelined slices)"},
            "gpu_launches": launches,
            "roofline": roof,
            "kernel_profile": "CUDA events around every launch of one extra step (ctx stream)",
            "fp64_tflops_step": all_flops / (t_local / args.steps) / 1e12,
            "kernel_classes": kernel_classes,
            "ranks_closed_form_ok": rank_ok,
            "clocks": clocks,
        }
        line.update(extras)
        if world == 1 and not args.no_cpu_baseline:
            n, t = oracle_sample(CPU_SAMPLE_SECONDS)
            line["cpu_baseline"] = {"value": n / t, "unit": "roundings/s", "cores": _blas_threads(), "kind": "oracle",
                                    "sample": f"oracle TT-rounding of the first {n} C4 items, {t:.1f} s "
                                              "(numpy/LAPACK fp64, BLAS threads = cores)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
