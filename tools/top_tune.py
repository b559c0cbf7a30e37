#!/usr/bin/env python
"""Print the fastest tiers of tools/tune.py JSON-line outputs.
  python tools/top_tune.py FILE.jsonl [FILE2 ...] [-n 6]"""
import json
import sys

args = [a for a in sys.argv[1:] if not a.startswith("-n")]
n = 6
for a in sys.argv[1:]:
    if a.startswith("-n"):
        n = int(a[2:])
for f in args:
    rows = [json.loads(l) for l in open(f) if l.startswith("{")]
    if not rows:
        continue
    print("==", f, rows[0].get("dims"), "ragged" if rows[0].get("ragged") else "")
    rows.sort(key=lambda d: d["us"])
    for d in rows[:n]:
        print(" ", "*" if d["auto"] else " ", d["tier"], d["us"], d["GBps"])
    a = [d for d in rows if d["auto"]]
    if a:
        print("   auto:", a[0]["tier"], a[0]["us"])
