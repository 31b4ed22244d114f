#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: a launch list (--metrics gpu__time_duration.sum
--csv) and optionally one `--set full` report.  Usage:

  python tools/ncu_summary.py LAUNCHES.csv [REPORT.ncu-rep] > profiles/ncu_<round>.md
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("<unnamed>", "anon").split("(")[0].split("<")[0].split("::")[-1]
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        us = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.1f} | {v / T:.3f} | {v / cnt[k]:.2f} |")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_barrier", "sm__cycles_elapsed.avg"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    idx = [(w, h.index(w)) for w in WANT if w in h]
    out = ["| kernel | " + " | ".join(f"{w} [{units[i]}]" for w, i in idx) + " |",
           "|---" * (len(idx) + 1) + "|"]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("::")[-1]
        out.append(f"| {name} | " + " | ".join(r[i] for _, i in idx) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)\n")
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print("\n## Full-set capture (ncu --set full --clock-control none)\n")
        print(report(sys.argv[2]))
