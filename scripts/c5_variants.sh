#!/bin/bash
# per-table fold+Adam kernel times of one warm C5 step under each fold variant
for v in 0 1 2 3 4 5; do
  SKB_ADAM_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c5v_$v.csv python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  python - "$v" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/c5v_{sys.argv[1]}.csv")))
hdr = None; seq = []
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    x = dict(zip(hdr, r))
    if x.get("Metric Name") != "gpu__time_duration.sum": continue
    if "k_fused_adam" in x["Kernel Name"]:
        seq.append(float(x["Metric Value"].replace(",", "")) / 1e3)
print("variant", sys.argv[1], "fold per table (dims 8..128) us:", [round(v) for v in seq[-5:]])
PY
done
