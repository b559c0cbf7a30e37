#!/usr/bin/env python
"""Render tools/sweep.py JSON lines as the fixed-width table kept in profiles/.
  python tools/sweep_table.py gpurun_out/sweep.jsonl > profiles/rNN_sweep.txt"""
import json
import sys

print("# tools/sweep.py: device time per call (CUDA-graph replay), algorithmic GB/s, % of the "
      "measured copy peak, % of nominal 8 TB/s; ref = same-traffic torch SM kernel (neg / add) in "
      "the same mode, moving the op's algorithmic bytes, and (ref/ours) its time over ours; err = max "
      "abs error vs the fp64 oracle on 256 sampled rows")
for line in open(sys.argv[1]):
    d = json.loads(line)
    if "config" not in d:
        print("#", line.strip())
        continue
    ref = d.get("ref_same_traffic_us", d.get("copy_same_bytes_us", d.get("torch_add_same_traffic_us")))
    nom = d.get("pct_nominal")
    err = d.get("max_abs_err")
    print(f"{d['config']:<14} {d['op']:<19} {d['dtype']:<4} {str(d['shape']):<22} "
          f"{'ragged' if d['ragged'] else 'full':<10} {d['us']:>7.2f} us {d['GBps']:>9.1f} GB/s "
          f"{d['pct_peak']:>5.1f}% " + (f"({nom:>5.1f}% nom) " if nom is not None else "") +
          f" ref {ref} us ({100 * float(ref) / d['us']:.0f}%) " +
          (f" err {err:.2e} " if err is not None else "") + f" {d['tier']}")
