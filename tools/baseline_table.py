#!/usr/bin/env python
"""Join the BASELINE.md §4 evidence into one markdown table:
  python tools/baseline_table.py gpurun_out/bl > profiles/r02_baseline_table.md
Inputs (tools/gpu_r02_baseline.sh): sweep.jsonl (CUDA-graph device time, algorithmic GB/s,
% of the measured copy peak / nominal 8 TB/s, max error), ncu.csv + ncu_cases.jsonl (one
launch per case: DRAM bytes and duration), oracle.jsonl (fp64 oracle rows/s, 1 / all threads)."""
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3}


def k(d):
    return (d["config"], d["op"], d["dtype"], tuple(d["shape"]), bool(d["ragged"]))


def main(dirp):
    sweep, orc, ncu = {}, {}, {}
    for l in open(os.path.join(dirp, "sweep.jsonl")):
        d = json.loads(l)
        if "config" in d:
            sweep[k(d)] = d
    for l in open(os.path.join(dirp, "oracle.jsonl")):
        if l.startswith("{"):
            d = json.loads(l)
            orc[k(d)] = d
    cases = [json.loads(l) for l in open(os.path.join(dirp, "ncu_cases.jsonl")) if l.startswith("{")]
    rows = [r for r in csv.reader(open(os.path.join(dirp, "ncu.csv"))) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        try:
            kid = int(r[ix["ID"]])
        except ValueError:
            continue
        v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1.0)
        per.setdefault(kid, {})[r[ix["Metric Name"]]] = v
    for c, kid in zip(cases, sorted(per)):
        ncu[k(c)] = per[kid]
    print("| config | op | dtype | shape | lengths | µs / call | rows/s | alg. GB/s | ncu DRAM GB/s "
          "| % of 8 TB/s | % of measured peak | max abs err | oracle rows/s (1 thread / all) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for key, s in sweep.items():
        n = ncu.get(key, {})
        dram = (n.get("dram__bytes_read.sum", 0) + n.get("dram__bytes_write.sum", 0))
        dur = n.get("gpu__time_duration.sum")
        o = orc.get(key, {})
        shape = s["shape"]
        rows_ = shape[0] * shape[1] * shape[2] if s["op"] == "softmax" else shape[0]
        print(f"| {s['config']} | {s['op']} | {s['dtype']} | {'×'.join(map(str, shape))} | "
              f"{'ragged' if s['ragged'] else 'full'} | {s['us']:.2f} | {rows_ / s['us'] / 1e3:.3g} G | "
              f"{s['GBps']:.0f} | {dram / dur / 1e9 if dur else float('nan'):.0f} | "
              f"{s.get('pct_nominal', float('nan')):.1f} | {s['pct_peak']:.1f} | "
              f"{s.get('max_abs_err', float('nan')):.1e} | "
              f"{o.get('oracle_1t_rows_per_s', float('nan')):.3g} / {o.get('oracle_all_rows_per_s', float('nan')):.3g} |")


if __name__ == "__main__":
    main(sys.argv[1])
