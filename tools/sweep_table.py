#!/usr/bin/env python
"""Render tools/sweep.py JSON lines as the fixed-width table kept in profiles/.
  python tools/sweep_table.py gpurun_out/sweep.jsonl > profiles/rNN_sweep.txt"""
import json
import sys

print("# tools/sweep.py: device time per call (CUDA-graph replay), algorithmic GB/s, % of the "
      "measured copy peak; ref = same-traffic torch kernel in the same mode")
for line in open(sys.argv[1]):
    d = json.loads(line)
    if "config" not in d:
        print("#", line.strip())
        continue
    ref = d.get("copy_same_bytes_us", d.get("torch_add_same_traffic_us"))
    print(f"{d['config']:<14} {d['op']:<19} {d['dtype']:<4} {str(d['shape']):<22} "
          f"{'ragged' if d['ragged'] else 'full':<10} {d['us']:>7.2f} us {d['GBps']:>9.1f} GB/s "
          f"{d['pct_peak']:>5.1f}%  ref {ref} us  {d['tier']}")
