#!/usr/bin/env python
"""Pinned host <-> device copy bandwidth on this box (the ceiling of bench.py's
e2e number): H2D alone, D2H alone, and both directions at once on two streams.
python tools/pcie_bw.py [MiB]"""
import json
import sys

import torch

n = (int(sys.argv[1]) if len(sys.argv) > 1 else 512) << 20
h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    s1.wait_stream(torch.cuda.current_stream())
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)


def d2h():
    with torch.cuda.stream(s1):
        h_dst.copy_(d_b, non_blocking=True)


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"bytes": n, "h2d_GBps": round(n / t1 / 1e6, 2), "d2h_GBps": round(n / t2 / 1e6, 2),
                  "bidir_total_GBps": round(2 * n / t3 / 1e6, 2)}))
