#!/usr/bin/env python
"""Per-kernel summary of one `ncu --set full` report: duration, issue activity, occupancy, FP64 /
tensor pipe use, DRAM traffic, and the top stall sites (SASS) with their share of samples.

  python tools/ncu_stalls.py REPORT.ncu-rep [N]
"""
import collections
import csv
import subprocess
import sys


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    want = ["Duration", "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Achieved Occupancy",
            "Registers Per Thread", "Theoretical Occupancy", "DRAM Throughput", "L2 Hit Rate", "Memory Throughput"]
    res = {}
    for row in csv.reader(out.splitlines()):
        if len(row) > 3 and row[-3] in want:
            res[row[-3]] = row[-1] + " " + row[-2]
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2] if len(rows) > 2 else rows[1]
    d = dict(zip(h, zip(v, u)))
    return {n: (" ".join(d[n]) if n in d else None) for n in names}


def sass(rep, top):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, x in enumerate(rows) if len(x) > 3 and x[0] == "Address"][0]
    h = rows[hi]
    k = h.index("Warp Stall Sampling (All Samples)")
    body = [x for x in rows[hi + 1:] if len(x) == len(h)]
    tot = sum(int(x[k]) for x in body) or 1
    byop = collections.Counter()
    for x in body:
        ins = x[1].split()
        byop[ins[1] if ins and ins[0].startswith("@") else (ins[0] if ins else "?")] += int(x[k])
    body.sort(key=lambda x: -int(x[k]))
    lines = [f"stall samples {tot}; by opcode: " + ", ".join(f"{o} {100 * c / tot:.1f}%" for o, c in byop.most_common(8))]
    for x in body[:top]:
        lines.append(f"  {100 * int(x[k]) / tot:5.1f}%  {x[0][-6:]}  {x[1][:80]}")
    return "\n".join(lines)


if __name__ == "__main__":
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    for kk, vv in details(rep).items():
        print(f"{kk}: {vv}")
    r = raw(rep, ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
                  "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
                  "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
                  "smsp__inst_executed.sum",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__cycles_elapsed.avg",
                  "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__warps_issue_stalled_barrier_per_warp_active.pct"])
    for kk, vv in r.items():
        print(f"{kk}: {vv}")
    print(sass(rep, top))
