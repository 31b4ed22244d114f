#!/usr/bin/env python
"""Host<->device copy bandwidth of this box (pinned memory, 1 GiB transfers): H2D alone, D2H
alone, both directions at once -- the bound of the host-to-host (e2e) bench number."""
import json

import torch


def main():
    n = (1 << 30) // 8
    h_src = torch.empty(n, dtype=torch.float64).pin_memory()
    h_dst = torch.empty(n, dtype=torch.float64).pin_memory()
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        s1.synchronize(); s2.synchronize()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)

    def both():
        h2d(); d2h()

    gb = n * 8 / 1e9
    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"h2d_GBps": gb / t1, "d2h_GBps": gb / t2, "both_GBps_aggregate": 2 * gb / t3,
                      "bytes_per_copy": n * 8}))


if __name__ == "__main__":
    main()
