#!/usr/bin/env python
"""Benchmark of the TT-orthogonalization hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], "C2"): MGS and MGS2 on m = 30 TT-vectors, d = 8, n = 32,
ranks 10, kappa = 1e10 (shared-tail mixing), rounding tolerance
1e-10, plus the TT-dot Gram matrix of the 30 inputs.  One step = tt_orth(MGS) +
tt_orth(MGS2) + tt_gram: 90 TT-roundings, 2 x 465 + 435 + ... TT-dots.  Metric: TT-roundings
per second (whole job), with fp64 TFLOP/s of the dominant kernel against the measured FP64
DMMA peak and Gram pairs/s reported alongside.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): every rank runs an independent replica (its own seed) -- the MGS chain
does not shard; scaling "weak", time = max over ranks.
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
FP64_PEAK_TFLOPS = 37.07   # measured: tools/fp64_peak.cu on this pool's B200 (profiles/fp64_peak_r01.json)
CPU_SAMPLE_M = 16          # oracle sample: MGS on the first 16 C2 vectors


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


def build_inputs(seed_offset: int):
    from ttinputs import CONFIGS, make_shared_tail_set
    c = CONFIGS["C2"]
    st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed + seed_offset)
    return c, st


def run_reference(args, rank: int, world: int):
    """Reference arm: the CPU oracle (as it stands) on a bounded sample of the workload."""
    if rank != 0:
        return
    import numpy as np
    from oracle import orth, tt
    c, st = build_inputs(0)
    A = st.tensors[:CPU_SAMPLE_M]
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orth.orth("mgs", A, c.delta)
        t1 = time.perf_counter()
        if it >= args.warmup:
            times.append(t1 - t0)
    T = sum(times)
    value = CPU_SAMPLE_M * len(times) / T
    sample = f"oracle TT-MGS on the first {CPU_SAMPLE_M} of the 30 C2 vectors ({CPU_SAMPLE_M} roundings per step)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 (BASELINE.json configs[1]) MGS sample", "m": c.m, "d": c.d, "n": c.n,
                       "r": c.r, "kappa": c.kappa, "delta": c.delta},
            "cpu_baseline": {"value": value, "unit": "roundings/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "roundings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline():
    from oracle import orth
    c, st = build_inputs(0)
    A = st.tensors[:CPU_SAMPLE_M]
    t0 = time.perf_counter()
    orth.orth("mgs", A, c.delta)
    t = time.perf_counter() - t0
    return {"value": CPU_SAMPLE_M / t, "unit": "roundings/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"oracle TT-MGS on the first {CPU_SAMPLE_M} of the 30 C2 vectors, {t:.1f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2211_08770_b200 import _build
    _build.build_library()
    import paper_2211_08770_b200 as P

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stream = torch.cuda.current_stream(local_rank)
    # the three independent parts of a step (MGS chain, MGS2 chain, Gram matrix) run
    # concurrently, one library context + CUDA stream + host thread each
    ctxs = [P.Context(local_rank, stream=torch.cuda.Stream(local_rank)) for _ in range(3)]
    c, st = build_inputs(rank)
    A = [P.DeviceTT.from_numpy(a) for a in st.tensors]
    rounds_per_step = 3 * c.m
    gram_pairs = c.m * (c.m + 1) // 2

    def step(inputs):
        fork = torch.cuda.Event()
        fork.record(stream)
        res = [None, None, None]
        err = []

        def part(i):
            try:
                cx = ctxs[i]
                cx.stream.wait_event(fork)
                with torch.cuda.stream(cx.stream):
                    if i == 0:
                        res[0] = P.tt_orth(cx, "mgs", inputs, c.delta)
                    elif i == 1:
                        res[1] = P.tt_orth(cx, "mgs2", inputs, c.delta)
                    else:
                        res[2] = P.tt_gram(cx, inputs)
            except Exception as e:  # surfaced after join
                err.append(e)

        th = [threading.Thread(target=part, args=(i,)) for i in range(3)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if err:
            raise err[0]
        for cx in ctxs:  # join: the caller's stream waits for all three
            ev = torch.cuda.Event()
            ev.record(cx.stream)
            stream.wait_event(ev)
        (Q1, R1, r1), (Q2, R2, r2), G = res
        return Q1, Q2, R1, R2, G, r1["rounding_calls"] + r2["rounding_calls"]

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=f"cuda:{local_rank}")

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        out = step(A)
        del out
    torch.cuda.synchronize()

    # ------------------------------------------------------------ timed (device-resident inputs)
    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = sum(cx.launches for cx in ctxs)
    step_ms = []
    calls = 0
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (256 MB > 126 MB L2), not timed
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = step(A)
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        calls += out[-1]
        del out
    barrier()
    launches = sum(cx.launches for cx in ctxs) - launches0
    clocks = sampler.stop()
    for cx in ctxs:
        cx.profile(False)
    # Per-kernel durations: events around every launch of one extra step run on ONE stream
    # (under the 3-stream overlap an event pair would also time the other streams' work).
    cx0 = ctxs[0]
    cx0.profile(True)
    with torch.cuda.stream(cx0.stream):
        P.tt_orth(cx0, "mgs", A, c.delta)
        P.tt_orth(cx0, "mgs2", A, c.delta)
        P.tt_gram(cx0, A)
    prof = cx0.profile_report()
    cx0.profile(False)
    t_local = sum(step_ms) / 1e3
    if world > 1:
        t = torch.tensor([t_local], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    else:
        t_max = t_local
    assert calls == rounds_per_step * args.steps, (calls, rounds_per_step)
    value = rounds_per_step * args.steps * world / t_max

    # ------------------------------------------------------------ end to end (host buffers)
    host = [[torch.from_numpy(x).pin_memory() for x in a] for a in st.tensors]
    h2d = sum(x.numel() * 8 for a in host for x in a)
    e2e_ms = []
    d2h = 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dev_in = [P.DeviceTT([x.to(f"cuda:{local_rank}", non_blocking=True) for x in a]) for a in host]
        Q1, Q2, R1, R2, G, _ = step(dev_in)
        outs = [q.to_numpy() for q in Q1 + Q2]
        Gh = G.cpu()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        d2h = sum(x.nbytes for q in outs for x in q) + Gh.numel() * 8 + R1.nbytes + R2.nbytes
        del Q1, Q2, outs
    te = sum(e2e_ms) / 1e3
    if world > 1:
        t = torch.tensor([te], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    e2e_value = rounds_per_step * args.steps * world / te

    # ------------------------------------------------------------ roofline of the dominant kernel
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    total_ms = sum(v["ms"] for v in prof.values())
    peaks = _peaks()
    if dom["flops"] > 0:
        achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                "peak_source": "measured FP64 DMMA (tools/fp64_peak.cu, profiles/fp64_peak_r01.json)"}
    else:
        achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if peaks.get("_fallback") else "")}
    roof.update({"kernel": dom_name, "launches": dom["launches"], "avg_launch_us": 1e3 * dom["ms"] / dom["launches"],
                 "share_of_kernel_time": dom["ms"] / total_ms})
    all_flops = sum(v["flops"] for v in prof.values())
    kernel_classes = {k: {"launches": v["launches"], "ms": round(v["ms"], 3), "share": round(v["ms"] / total_ms, 4),
                          "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 else 0.0}
                      for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 (BASELINE.json configs[1]): TT-MGS + TT-MGS2 + TT-dot Gram",
                       "m": c.m, "d": c.d, "n": c.n, "r": c.r, "kappa": c.kappa, "delta": c.delta,
                       "floor_c": 2048.0, "roundings_per_step": rounds_per_step, "gram_pairs_per_step": gram_pairs,
                       "l2": "flushed between timed steps (256 MB write)", "parallelism": f"replicas x{world}",
                       "streams": "MGS | MGS2 | Gram concurrently on 3 CUDA streams"},
            "e2e": {"value": e2e_value, "unit": "roundings/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": roof,
            "kernel_profile": "CUDA events around every launch of one extra step on a single stream",
            "fp64_tflops_step": all_flops / t_local / 1e12,
            "gram_pairs_per_s": gram_pairs * args.steps * world / t_max,
            "kernel_classes": kernel_classes,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
