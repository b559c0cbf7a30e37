#!/usr/bin/env python
"""Copy the evidence worth judging from gpurun_out/ (scratch) into profiles/
(tracked), named per round.

  python tools/make_profiles.py r01

Writes:
  profiles/<round>_launches.csv        ncu --metrics gpu__time_duration.sum,dram__bytes_*
                                       launch list of the bench.py command (C4)
  profiles/<round>_ncu_full.txt        key metrics + stall reasons of each kernel in
                                       prof_c4.ncu-rep (ncu --set full)
  profiles/<round>_sass_<kernel>.txt   per-opcode instruction mix from the same report
  profiles/<round>_tune.txt            tier sweep (tools/tune.py) summaries
  profiles/<round>_bench.json          the bench.py line of the same round
  profiles/traffic.json                dram read+write bytes per launch, per kernel,
                                       read by bench.py for roofline.traffic
"""
import csv
import glob
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(rnd):
    src = os.path.join(OUT, "launches.csv")
    if not os.path.exists(src):
        return {}
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    I = hdr.index
    with open(os.path.join(PROF, f"{rnd}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "metric", "unit", "value"])
        agg = defaultdict(lambda: defaultdict(list))
        for r in rows[start + 1:]:
            if len(r) < len(hdr):
                continue
            k = r[I("Kernel Name")]
            w.writerow([r[I("ID")], k, r[I("Grid Size")], r[I("Block Size")], r[I("Metric Name")],
                        r[I("Metric Unit")], r[I("Metric Value")]])
            agg[k][r[I("Metric Name")]].append(float(r[I("Metric Value")].replace(",", "")))
    return agg


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    agg = launches(rnd)
    bpath = os.path.join(OUT, "bench.json")
    bench = json.load(open(bpath)) if os.path.exists(bpath) else {}
    plans = bench.get("kernels", {})
    traffic = {}
    total_ns = sum(sum(m.get("gpu__time_duration.sum", [])) for m in agg.values())
    lines = []
    for k, m in agg.items():
        rd, wr = m.get("dram__bytes_read.sum", [0]), m.get("dram__bytes_write.sum", [0])
        t = m.get("gpu__time_duration.sum", [0])
        per = (sum(rd) + sum(wr)) / max(1, len(rd))
        name = plans.get("softmax") if "softmax" in k else plans.get("layernorm")
        traffic[f"C4:{name}"] = {"dram_bytes_per_launch": per, "kernel": k,
                                 "launches": len(t), "avg_ns_cold": sum(t) / max(1, len(t)),
                                 "share_of_launch_time": sum(t) / total_ns if total_ns else None,
                                 "source": f"profiles/{rnd}_launches.csv (ncu --metrics, "
                                           "--clock-control none)"}
        lines.append(f"{k}: launches={len(t)} avg_ns={sum(t)/max(1,len(t)):.0f} "
                     f"share={sum(t)/total_ns:.3f} dram_read={sum(rd)/max(1,len(rd)):.4g} "
                     f"dram_write={sum(wr)/max(1,len(wr)):.4g}")
    if traffic:  # only from a fresh launch list (never overwrite with nothing)
        json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    rep = os.path.join(OUT, "prof_c4.ncu-rep")
    rep_exists = os.path.exists(os.path.join(OUT, "prof_c4.ncu-rep"))
    with open(os.path.join(PROF, f"{rnd}_ncu_full.txt"), "w") if (lines or rep_exists) \
            else open(os.devnull, "w") as f:
        f.write("# ncu --set full --clock-control none, bench.py C4 step (tools/gpu_check.sh NCU=1)\n")
        f.write("# launch-list summary (cold-cache, serialised; compare shares):\n")
        for l in lines:
            f.write("#   " + l + "\n")
        if os.path.exists(rep):
            f.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                                    rep], capture_output=True, text=True).stdout)
    if os.path.exists(rep):
        s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_sass.py"), rep, "20"],
                           capture_output=True, text=True).stdout
        open(os.path.join(PROF, f"{rnd}_sass_c4.txt"), "w").write(s)
    tune = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "show_tune.py"), "8"],
                          capture_output=True, text=True, cwd=ROOT).stdout
    if tune.strip():
        open(os.path.join(PROF, f"{rnd}_tune.txt"), "w").write(
            "# tools/tune.py sweeps (GB/s algorithmic, CUDA events, inputs > 4x L2); * = automatic tier\n"
            + tune)
    if bench:
        shutil.copy(bpath, os.path.join(PROF, f"{rnd}_bench.json"))
    for src, dst, title in (("sweep.jsonl", f"{rnd}_sweep.txt", "tools/sweep.py"),
                            ("sweep_next2.jsonl", f"{rnd}_sweep_next2.txt",
                             "tools/sweep.py --next2 (NEXT-2 kernels)")):
        p = os.path.join(OUT, src)
        if not os.path.exists(p):
            continue
        rows = [json.loads(l) for l in open(p) if l.strip()]
        out = [f"# {title}: device time per call (CUDA-graph replay), algorithmic GB/s, "
               "% of the measured copy peak; ref = same-traffic torch kernel in the same mode"]
        for r in rows:
            if "op" not in r:
                out.append("# " + json.dumps(r))
                continue
            ref = r.get("copy_same_bytes_us") or r.get("torch_add_same_traffic_us")
            out.append(f"{r['config']:14s} {r['op']:19s} {r['dtype']:4s} {str(r['shape']):22s} "
                       f"{'ragged' if r['ragged'] else 'full  '} {r['us']:9.2f} us "
                       f"{r['GBps']:8.1f} GB/s {r['pct_peak']:5.1f}%  ref {ref} us  {r['tier']}")
        open(os.path.join(PROF, dst), "w").write("\n".join(out) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
