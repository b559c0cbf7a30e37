import glob, json, sys
for f in sorted(glob.glob("gpurun_out/tune_*.jsonl")):
    rows = []
    for l in open(f):
        try:
            rows.append(json.loads(l))
        except Exception:
            print("  !", l.strip()[:160])
    rows.sort(key=lambda d: -d["GBps"])
    print("==", f)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    auto = [d for d in rows if d["auto"]][:1]
    for d in rows[:n] + [d for d in auto if d not in rows[:n]]:
        print(("*" if d["auto"] else " "), d["tier"], d["us"], d["GBps"])
