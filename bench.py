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

N > 1 (one process per GPU: under torchrun, or `--gpus N` alone re-launches itself under
torch.distributed.run): BASELINE's "batch split across 1/2/4/8 GPUs" -- the one 4096-item batch is
cut into contiguous slices (tt_plan_slice), rank r rounds its slice, no data-path collective (the
roundings are independent); time = max over ranks; value = 4096 / that time; "scaling": "strong".
Alongside at N > 1: every rank rounding its own 4096 items (weak scaling), the C3 Gram matrix and
the C3 TT-Gram driver with the library's NCCL communicator (pair blocks + all-gather, LPT phase-2
roundings).  --impl reference times the CPU oracle (oracle/, the slow fp64 reference written from
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
    """(start, count) of this rank's shard of the one `batch`-item batch (strong scaling,
    BASELINE configs[3] "batch split across 1/2/4/8 GPUs"): the library's contiguous balanced
    slice (tt_plan_slice; the same formula in Python when the library is not built)."""
    base, rem = divmod(batch, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def _weak_slice(batch: int, rank: int, world: int):
    """(start, count) for the weak-scaling extra: a whole `batch` per GPU, rank r taking items
    [r * batch, (r + 1) * batch) of the seeded stream."""
    return rank * batch, batch


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------- D3 work model
def d3_round_flops(n, term_ranks, out_ranks):
    """SURVEY.md §8(d) D3 flops of one TT-rounding of the TT-sum with per-term ranks
    term_ranks[l][0..d] and output ranks out_ranks[0..d] (the algorithmic work, not what any
    implementation does): right-to-left, per k = d..2, QR + explicit Q of the m x c panel
    (m = n_k R'_k, c = R_{k-1}) 2(2mc^2 - 2c^3/3) (or with m, c swapped) plus the core x L product
    2 R'_{k-1} nnz(X_{k-1}) over the nonzero diagonal blocks; left-to-right, per k = 1..d-1, the
    nominal R-SVD 6ab^2 + 11b^3 of Y_k ((rho_{k-1} n_k) x R'_k) plus 2 rho_k R'_k n_{k+1} R'_{k+1}.
    Returns (right-to-left QR part, right-to-left explicit-Q part, core x L part, left-to-right part)."""
    d = len(n)
    R = [sum(t[k] for t in term_ranks) for k in range(d + 1)]
    R[0] = R[d] = 1
    Rp = [1] * (d + 1)
    qr = expq = cxl = 0.0
    for k in range(d, 1, -1):  # core k (1-based): panel (n_k R'_k) x R_{k-1}
        m, c = n[k - 1] * Rp[k], R[k - 1]
        half = (2 * m * c * c - 2 * c ** 3 / 3) if m >= c else (2 * c * m * m - 2 * m ** 3 / 3)
        qr += half
        expq += half
        Rp[k - 1] = min(m, c)
        nnz = sum(t[k - 2] * n[k - 2] * t[k - 1] for t in term_ranks)
        cxl += 2 * Rp[k - 1] * nnz
    l2r = 0.0
    for k in range(1, d):
        rows, cols = out_ranks[k - 1] * n[k - 1], Rp[k]
        a, b = max(rows, cols), min(rows, cols)
        l2r += 6 * a * b * b + 11 * b ** 3 + 2 * out_ranks[k] * Rp[k] * n[k] * Rp[k + 1]
    return qr, expq, cxl, l2r


def c4_work(batch_ranks, d=10, n=32, r=16, K=4):
    """D3 flops of the C4 step split by phase, and its algorithmic bytes (term cores read once,
    output cores written once), from the output ranks of every item."""
    import numpy as np
    nn = [n] * d
    term = [1] + [min(r, n ** k, n ** (d - k)) for k in range(1, d)] + [1]
    terms = [term] * K
    tot = np.zeros(4)
    cache = {}
    out_doubles = 0
    for rk in batch_ranks:
        key = tuple(int(v) for v in rk)
        if key not in cache:
            cache[key] = np.array(d3_round_flops(nn, terms, list(key)))
        tot += cache[key]
        out_doubles += sum(key[k] * n * key[k + 1] for k in range(d))
    in_doubles = len(batch_ranks) * K * sum(term[k] * n * term[k + 1] for k in range(d))
    return {"r2l_qr": tot[0], "r2l_explicit_q": tot[1], "core_x_L": tot[2], "l2r": tot[3],
            "total": float(tot.sum()), "bytes": 8.0 * (in_doubles + out_doubles)}


def _blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:
        return os.cpu_count() or 1


def _config(batch: int, world: int):
    return {"workload": f"C4 (BASELINE.json configs[3]): batch of {batch} independent TT-roundings, "
                        "each the TT-sum of 4 unit-norm rank-16 TT-vectors (d=10, n=32, formal rank 64)",
            "batch": batch, "global_batch": batch, "d": 10, "n": 32, "terms": 4, "term_rank": 16,
            "delta": C4_DELTA, "floor_c": 2048.0,
            "parallelism": f"batch split x{world} (contiguous slices of the {batch}-item batch, tt_plan_slice; "
                           "no collective)",
            "l2": "inputs (8.7 GB at B=4096) exceed L2; L2 also flushed (256 MB write) between timed steps"}


_ORACLE_ITEMS = []


def oracle_sample(seconds: float, offset: int = 0):
    """The CPU oracle (as it stands) on C4 items in order until `seconds` have elapsed.  The
    items are generated once, before the clock starts (round 1 regenerated them inside the
    timed loop, advancing the seeded stream from item 0 every time: that cost grew with the
    sample and made the bench's 124-item figure 1.5x lower than the reference arm's 12-item one)."""
    from oracle import rounding
    from ttinputs import make_batch_sums
    need = offset + max(8, int(seconds * 40) + 8)
    if len(_ORACLE_ITEMS) < need:
        _ORACLE_ITEMS.extend(make_batch_sums(need - len(_ORACLE_ITEMS), start=len(_ORACLE_ITEMS)))
    done, t0 = 0, time.perf_counter()
    while True:
        if offset + done >= len(_ORACLE_ITEMS):
            _ORACLE_ITEMS.extend(make_batch_sums(64, start=len(_ORACLE_ITEMS)))
        terms, coeffs = _ORACLE_ITEMS[offset + done]
        rounding.tt_round_sum(terms, coeffs, C4_DELTA, floor_c=rounding.DEFAULT_FLOOR_C, term_norms=[1.0] * 4)
        done += 1
        if time.perf_counter() - t0 >= seconds:
            break
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
              f"{T:.1f} s over {args.steps} steps; host {_cpu_model()}, nproc {os.cpu_count()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(args.batch, world),
            "cpu_baseline": {"value": value, "unit": "roundings/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": _cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": "roundings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _relaunch(n: int) -> int:
    """`bench.py --gpus N` outside a launcher: run the same command under torch.distributed.run
    with N processes (one per GPU) and pass its output through."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _event_ms(fn, stream):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def _driver_extras(P, ctx, stream, rank):
    """C1, C3 (TT-Gram, TT-CGS2) and a C5 prefix through tt_orth at full config sizes (C5: m' = 20
    of m = 100), each with its closed-form check (shared-tail construction: R = R_M)."""
    import numpy as np
    from ttinputs import CONFIGS, make_shared_tail_set
    out = {}

    def run(name, kind, m=None):
        c = CONFIGS[name]
        mm = c.m if m is None else m
        st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed)
        A = [P.DeviceTT.from_numpy(a) for a in st.tensors[:mm]]
        ms, (Q, R, rep) = _event_ms(lambda: P.tt_orth(ctx, kind, A, c.delta, want_loo=True), stream)
        rm = st.qr_exact()[1][:mm, :mm]
        if kind == "householder":
            sg = np.sign(np.diag(R))
            sg[sg == 0] = 1
            R = sg[:, None] * R
        key = f"{name.lower()}_{kind}" + (f"_m{mm}" if m is not None else "")
        out[key] = {"workload": f"{name} ({c.note}) TT-{kind}, m={mm}, d={c.d}, n={c.n}, r={c.r}, "
                                f"kappa={c.kappa:g}, delta={c.delta:g}",
                    "roundings": rep["rounding_calls"], "ms": ms,
                    "roundings_per_s": rep["rounding_calls"] / (ms * 1e-3),
                    "max_rank": int(max(rep["max_rank_per_call"])),
                    "R_rel_err_vs_R_M": float(np.linalg.norm(R - rm) / np.linalg.norm(rm)),
                    "loo_last": float(rep["loo_per_step"][-1])}
    run("C1", "cgs")
    run("C3", "gram")
    run("C3", "cgs2")
    run("C5", "householder", m=20)
    return out


def _oracle_driver_extras():
    """the oracle (as it stands) on C1 with all host threads and with 1 thread,
    and on C2 MGS with all threads -- the same inputs as the GPU drivers."""
    from oracle import orth
    from ttinputs import CONFIGS, make_shared_tail_set
    out = {}
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    for name, kind, one in (("C1", "cgs", False), ("C1", "cgs", True), ("C2", "mgs", False)):
        c = CONFIGS[name]
        st = make_shared_tail_set(c.d, c.n, c.r, c.m, c.kappa, c.seed)
        t0 = time.perf_counter()
        if one and threadpool_limits is not None:
            with threadpool_limits(1):
                res = orth.orth(kind, st.tensors, c.delta)
        else:
            res = orth.orth(kind, st.tensors, c.delta)
        t = time.perf_counter() - t0
        out[f"{name.lower()}_{kind}" + ("_1thread" if one else "")] = {
            "s": t, "roundings": int(res.rounding_calls), "roundings_per_s": res.rounding_calls / t,
            "threads": 1 if one else _blas_threads()}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=C4_BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the Gram / driver side measurements")
    ap.add_argument("--e2e-slices", type=int, default=4, help="pipelined slices of the host-to-host call")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2211_08770_b200 import _build
    _build.build_library()
    import paper_2211_08770_b200 as P
    from paper_2211_08770_b200 import parallel
    from ttinputs import make_batch_sums_stacked

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stream = torch.cuda.current_stream(local_rank)
    ctx = P.Context(local_rank, stream=stream)

    start, B = parallel.plan_slice(args.batch, world, rank)
    cores_h, coeffs = make_batch_sums_stacked(B, start=start)
    norms = np.ones((B, 4))
    cores = [[torch.from_numpy(c).to(dev) for c in term] for term in cores_h]
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def tmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step(inp, cf, nr):
        return P.tt_round_batch_strided(ctx, inp, cf, C4_DELTA, norms=nr)

    for _ in range(args.warmup):
        res = step(cores, coeffs, norms)
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
        ms, res = _event_ms(lambda: step(cores, coeffs, norms), stream)
        step_ms.append(ms)
        ranks = res.ranks
        del res
    barrier()
    launches = ctx.launches - launches0
    clocks = sampler.stop()
    t_local = sum(step_ms) / 1e3
    t_max = tmax(t_local)
    value = args.batch * args.steps / t_max  # the whole batch over the max-over-ranks time
    rank_ok = bool(np.all(ranks[:, 1:-1] == np.where((np.arange(start, start + B) % 2 == 0), 32, 16)[:, None]))

    # ------------------------------------------------------------ per-kernel profile (one extra step)
    ctx.profile(True)
    res = step(cores, coeffs, norms)
    prof = ctx.profile_report()
    ctx.profile(False)
    out_doubles = res.total_doubles()
    prof_ranks = res.ranks
    del res

    # ------------------------------------------------------------ end to end (pinned host buffers)
    # the public host-to-host C-ABI call tt_round_batch_host: inputs copied from pinned memory and
    # results copied back inside the timed region, pipelined by the library over its own streams
    host = [[torch.from_numpy(c).pin_memory() for c in term] for term in cores_h]
    h2d = sum(x.numel() * 8 for term in host for x in term)
    out_host = torch.empty(out_doubles + 4096, dtype=torch.float64).pin_memory()
    e2e_ms, d2h = [], 0
    for _ in range(2):  # untimed: the context's copy streams and staging buffers are created
        P.tt_round_batch_host(ctx, host, coeffs, C4_DELTA, norms=norms, slices=args.e2e_slices, out_host=out_host)
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        ms, (out_host, rk_h, nr_h, cnt) = _event_ms(
            lambda: P.tt_round_batch_host(ctx, host, coeffs, C4_DELTA, norms=norms, slices=args.e2e_slices,
                                          out_host=out_host), stream)
        e2e_ms.append(ms)
        d2h = cnt * 8 + rk_h.nbytes + nr_h.nbytes
    te = tmax(sum(e2e_ms) / 1e3)
    e2e_value = args.batch * args.steps / te

    # ------------------------------------------------------------ roofline
    peak = max(FP64_DFMA_PEAK_TFLOPS, FP64_DMMA_PEAK_TFLOPS)
    hbm = float(_peaks().get("hbm_gbs", 6552.3))
    work = c4_work(prof_ranks)
    total_ms = sum(v["ms"] for v in prof.values())
    r2l = prof.get("batch_r2l_qr", {"ms": float("nan"), "launches": 1})
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    # the right-to-left kernel performs D3's QR (R + reflectors) and core x L terms; D3's
    # explicit-Q half is done here as reflector applications inside batch_l2r_apply
    r2l_alg = work["r2l_qr"] + work["core_x_L"]
    achieved = r2l_alg / (r2l["ms"] * 1e-3) / 1e12
    traffic = None
    try:  # DRAM bytes per launch of this kernel class from the committed ncu --set full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json"))).get("batch_r2l_qr")
        traffic = tr["dram_bytes_per_launch"] if tr else None
    except Exception:
        traffic = None
    step_s = t_local / args.steps
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "batch_r2l_qr (br_r2l_wy_kernel)",
            "launches": r2l["launches"], "avg_launch_us": 1e3 * r2l["ms"] / max(r2l["launches"], 1),
            "algorithmic_flops_per_launch": r2l_alg / max(r2l["launches"], 1),
            "share_of_kernel_time": r2l["ms"] / total_ms,
            "work_model": "SURVEY.md §8(d) D3: right-to-left QR 2mc^2-2c^3/3 per panel + core x L over the nonzero "
                          "blocks, summed over the batch's items and the 9 panels (one launch per panel)",
            "peak_source": "max(FP64 DFMA 34.18, FP64 DMMA 37.07) TFLOP/s measured by tools/fp64_peak.cu "
                           "(profiles/fp64_peak_r01.json), SURVEY.md §8(d) D2",
            "traffic_source": "profiles/ncu_traffic_r02.json (dram__bytes_read.sum + dram__bytes_write.sum, one launch)",
            "step": {"d3_flops": work["total"], "tflops": work["total"] / step_s / 1e12,
                     "frac": work["total"] / step_s / 1e12 / peak,
                     "d3_split": {k: work[k] for k in ("r2l_qr", "r2l_explicit_q", "core_x_L", "l2r")}},
            "hbm": {"algorithmic_bytes": work["bytes"], "gbs": work["bytes"] / step_s / 1e9,
                    "peak_gbs": hbm, "frac": work["bytes"] / step_s / 1e9 / hbm},
            "dominant_kernel": dom_name}
    kernel_classes = {k: {"launches": v["launches"], "ms": round(v["ms"], 3), "share": round(v["ms"] / total_ms, 4),
                          "lapack_tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 else 0.0}
                      for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}

    # ------------------------------------------------------------ alongside
    extras = {}
    if not args.no_extras:
        from ttinputs import CONFIGS, make_shared_tail_set
        c3 = CONFIGS["C3"]
        st3 = make_shared_tail_set(c3.d, c3.n, c3.r, c3.m, c3.kappa, c3.seed)  # same set on every rank
        A3 = [P.DeviceTT.from_numpy(a) for a in st3.tensors]
        pairs = c3.m * (c3.m + 1) // 2
        G = P.tt_gram(ctx, A3)
        torch.cuda.synchronize()
        gms = []
        for _ in range(5):
            flush.zero_()
            ms, G = _event_ms(lambda: P.tt_gram(ctx, A3), stream)
            gms.append(ms)
        gerr = float(np.linalg.norm(G.cpu().numpy() - st3.gram_exact()) / np.linalg.norm(st3.gram_exact()))
        r3 = [1] + [min(c3.r, c3.n ** k, c3.n ** (c3.d - k)) for k in range(1, c3.d)] + [1]
        # SURVEY §8(a) a6 per pair and core: 2n(a_{k-1} b_{k-1} b_k + a_{k-1} a_k b_k)
        gflops = pairs * sum(2 * c3.n * (r3[k] * r3[k] * r3[k + 1] + r3[k] * r3[k + 1] * r3[k + 1])
                             for k in range(c3.d))
        gmed = statistics.median(gms)
        extras["gram_pairs_per_s"] = pairs / (gmed * 1e-3)
        extras["gram"] = {"workload": "C3 (configs[2]) TT-dot Gram matrix, m=50, d=16, n=64, r=20",
                          "pairs": pairs, "ms": gmed, "ms_min": min(gms), "rel_err_vs_MtM": gerr,
                          "d3_flops": gflops, "tflops": gflops / (gmed * 1e-3) / 1e12,
                          "frac_of_dmma_peak": gflops / (gmed * 1e-3) / 1e12 / FP64_DMMA_PEAK_TFLOPS}
        if world > 1:
            # the library's own NCCL communicator: C3 Gram by LPT pair blocks + one all-gather, and
            # the C3 TT-Gram driver with its 50 phase-2 roundings LPT-sharded (owner rounds, ranks
            # all-gathered, q_i broadcast)
            parallel.attach_nccl(ctx)
            P.tt_gram(ctx, A3)
            sms = []
            for _ in range(5):
                barrier()
                ms, Gs = _event_ms(lambda: P.tt_gram(ctx, A3), stream)
                sms.append(ms)
            tg = tmax(statistics.median(sms))
            extras["gram_sharded"] = {"ranks": world, "ms": tg, "pairs_per_s": pairs / (tg * 1e-3),
                                      "rel_err_vs_MtM": float(np.linalg.norm(Gs.cpu().numpy() - st3.gram_exact())
                                                              / np.linalg.norm(st3.gram_exact())),
                                      "collective": "library-owned NCCL all-gather of LPT-assigned 4x4 pair blocks"}
            barrier()
            ms, (_, Rg, repg) = _event_ms(lambda: P.tt_orth(ctx, "gram", A3, c3.delta), stream)
            tgd = tmax(ms)
            rm = st3.qr_exact()[1]
            extras["gram_driver_sharded"] = {
                "ranks": world, "ms": tgd, "roundings": repg["rounding_calls"],
                "R_rel_err_vs_R_M": float(np.linalg.norm(Rg - rm) / np.linalg.norm(rm)),
                "collective": "NCCL all-gather of dot slices and of phase-2 ranks, grouped broadcasts of q_i"}
            parallel.detach(ctx)
            # weak scaling: every rank rounds its own whole batch
            ws, wb = _weak_slice(args.batch, rank, world)
            wc_h, wcf = make_batch_sums_stacked(wb, start=ws)
            wc = [[torch.from_numpy(c).to(dev) for c in term] for term in wc_h]
            step(wc, wcf, np.ones((wb, 4)))
            wms = []
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                barrier()
                ms, _r = _event_ms(lambda: step(wc, wcf, np.ones((wb, 4))), stream)
                wms.append(ms)
            tw = tmax(sum(wms) / 1e3)
            extras["weak_scaling"] = {"per_gpu_batch": args.batch, "global_batch": args.batch * world,
                                      "value": args.batch * world * args.steps / tw, "unit": "roundings/s",
                                      "ms_per_step": 1e3 * tw / args.steps}
            del wc
        if rank == 0:
            extras["drivers"] = _driver_extras(P, ctx, stream, rank)
            c2 = CONFIGS["C2"]
            st2 = make_shared_tail_set(c2.d, c2.n, c2.r, c2.m, c2.kappa, c2.seed)
            A2 = [P.DeviceTT.from_numpy(a) for a in st2.tensors]
            P.tt_orth(ctx, "mgs", A2, c2.delta)
            ms, (r1, r2) = _event_ms(lambda: (P.tt_orth(ctx, "mgs", A2, c2.delta)[2],
                                              P.tt_orth(ctx, "mgs2", A2, c2.delta)[2]), stream)
            calls = r1["rounding_calls"] + r2["rounding_calls"]
            extras["drivers_c2"] = {"workload": "C2 (configs[1]) TT-MGS + TT-MGS2, m=30, d=8, n=32, r=10",
                                    "roundings": calls, "ms": ms, "roundings_per_s": calls / (ms * 1e-3)}
            # the paper's own workload (Section 3, experiment 1): Krylov TT-Laplacian set
            # d=3, n=15, m=20, five schemes (Gram breaks down on it) at delta=1e-5, floor off
            def krylov():
                K1 = P.krylov_set(ctx, 3, 15, 20)
                kcalls, kloo = 0, {}
                for kind in ("cgs", "mgs", "cgs2", "mgs2", "householder"):
                    _, _, rk = P.tt_orth(ctx, kind, K1, 1e-5, floor_c=0.0, want_loo=True)
                    kcalls += rk["rounding_calls"]
                    kloo[kind] = float(rk["loo_per_step"][-1])
                return kcalls, kloo
            ms, (kcalls, kloo) = _event_ms(krylov, stream)
            extras["krylov_exp1"] = {"workload": "PAPER.md Sec. 3 experiment 1: Krylov TT-Laplacian set d=3, n=15, "
                                                 "m=20 (rank-1 rounded), CGS/MGS/CGS2/MGS2/Householder at delta=1e-5, "
                                                 "floor off", "roundings": kcalls, "ms": ms,
                                     "roundings_per_s": kcalls / (ms * 1e-3), "loo_last": kloo}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(args.batch, world),
            "e2e": {"value": e2e_value, "unit": "roundings/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_steps": [round(x, 2) for x in e2e_ms],
                    "api": f"tt_round_batch_host (C ABI, host buffers, {args.e2e_slices} pipelined slices)"},
            "gpu_launches": launches,
            "roofline": roof,
            "kernel_profile": "CUDA events around every launch of one extra step (ctx stream); lapack_tflops = "
                              "the library's LAPACK-standard counts of what each kernel computes",
            "kernel_classes": kernel_classes,
            "ranks_closed_form_ok": rank_ok,
            "clocks": clocks,
        }
        line.update(extras)
        if world == 1 and not args.no_cpu_baseline:
            n, t = oracle_sample(CPU_SAMPLE_SECONDS)
            line["cpu_baseline"] = {"value": n / t, "unit": "roundings/s", "cores": _blas_threads(), "kind": "oracle",
                                    "sample": f"oracle TT-rounding of the first {n} C4 items, {t:.1f} s "
                                              "(numpy/LAPACK fp64, BLAS threads = cores; items generated before "
                                              "the clock starts)",
                                    "cpu_model": _cpu_model(), "nproc": os.cpu_count()}
            if not args.no_extras:
                line["cpu_baseline"]["drivers"] = _oracle_driver_extras()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
