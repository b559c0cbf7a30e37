#!/usr/bin/env python
"""Summarise ncu reports: key throughput/occupancy metrics and top stall reasons.
  python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Compute (SM) Throughput",
        "L2 Hit Rate", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "No Eligible", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem", "Grid Size", "Block Size"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = d.get("Kernel Name", "")[:70]
        if d.get("Metric Name") in WANT:
            res.setdefault(k, {})[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'
    return res


def raw(rep, pats):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            if any(p in h for p in pats):
                d[h] = (v, u)
        res.append(d)
    return res


for rep in sys.argv[1:]:
    print("=" * 8, rep)
    for k, m in details(rep).items():
        print(" ", k)
        for w in WANT:
            if w in m:
                print(f"    {w:34s} {m[w]}")
    for d in raw(rep, ["pipe"]):
        pipes = []
        for h, (v, u) in d.items():
            if "pct_of_peak_sustained_active" in h and ("inst_executed_pipe" in h or "pipe_" in h):
                try:
                    pipes.append((float(v.replace(",", "")), h))
                except ValueError:
                    pass
        for v, h in sorted(pipes, reverse=True)[:10]:
            print(f"    {h:70s} {v:.1f} %")
    for d in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum",
                       "smsp__average_warp_latency_issue_stalled", "smsp__pcsamp_warps_issue_stalled"]):
        st = [(h, v) for h, (v, u) in d.items() if "stalled" in h]
        try:
            st = sorted(st, key=lambda t: -float(t[1].replace(",", "")))[:8]
        except ValueError:
            st = st[:8]
        for h, (v, u) in d.items():
            if "dram__bytes" in h:
                print(f"    {h:50s} {v} {u}")
        for h, v in st:
            print(f"    {h:70s} {v}")
