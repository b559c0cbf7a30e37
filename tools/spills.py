#!/usr/bin/env python
"""List kernels with register spills from the ptxas logs of the last build
(paper_2010_05680_b200/_build/*.ptxas.log).   python tools/spills.py [filter]"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
flt = sys.argv[1] if len(sys.argv) > 1 else ""
n = 0
for f in sorted(glob.glob(os.path.join(ROOT, "paper_2010_05680_b200/_build/*.ptxas.log"))):
    for b in re.split(r"ptxas info\s+: Compiling entry function '", open(f).read())[1:]:
        name = b.split("'")[0]
        m = re.search(r"(\d+) bytes spill stores", b)
        r = re.search(r"Used (\d+) registers", b)
        if m and int(m.group(1)) > 0:
            dn = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            n += 1
            if flt in dn:
                print(f"{int(m.group(1)):5d} B spill  {r.group(1) if r else '?':>3} regs  {dn[:140]}")
print("kernels with spills:", n)
