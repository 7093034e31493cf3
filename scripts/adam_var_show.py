"""Per-table fold+Adam kernel time (us, median over traced steps) and step
ms for each SKB_ADAM_VARIANT run of scripts/adam_var_ab.sh."""
import glob
import json
import os
import statistics

for d in sorted(glob.glob("gpurun_out/av/v*/")):
    v = os.path.basename(d.rstrip("/"))
    try:
        tr = json.load(open(os.path.join(d, "trace_c5.json")))
        line = json.loads(open(d.rstrip("/") + ".jsonl").read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(v, "missing", e)
        continue
    ev = sorted((e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"
                 and "fused_adam" in e["name"]), key=lambda e: e["ts"])
    per = [[] for _ in range(5)]
    for i, e in enumerate(ev):
        per[i % 5].append(e["dur"])
    name = ev[0]["name"][:45] if ev else "?"
    print(f"{v:4s} step {line['ms_per_step']:.3f} ms  adam us per D8..128:",
          [round(statistics.median(p), 1) if p else None for p in per], name)
