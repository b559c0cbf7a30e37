#!/usr/bin/env python
"""Per-instruction SASS profile from an ncu report: instructions executed and
stall samples, top-N and totals by opcode.  python tools/ncu_sass.py REP [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
I = hdr.index
recs = []
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    try:
        recs.append((r[I("Address")], r[I("Source")].strip(), int(r[I("Instructions Executed")]),
                     int(r[I("Warp Stall Sampling (All Samples)")])))
    except ValueError:
        pass
tot = sum(x[2] for x in recs)
samp = sum(x[3] for x in recs)
print(f"total warp instructions executed {tot:,}  stall samples {samp:,}")
byop = collections.Counter()
for a, s, e, st in recs:
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    byop[op.split(".")[0]] += e
for op, e in byop.most_common(25):
    print(f"  {op:10s} {e:>14,} {100*e/tot:5.1f}%")
print("hottest by stall samples:")
for a, s, e, st in sorted(recs, key=lambda x: -x[3])[:n]:
    print(f"  {st:6d} {e:>12,}  {s[:90]}")
