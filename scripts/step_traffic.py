"""Per-step DRAM traffic of a timed region from an ncu --csv list taken with
`--nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum` (bench.py's NVTX range around its
timed steps).  ncu serialises and cold-starts every kernel, so the sums are
the step's kernel work without overlap: bytes are meaningful, times are an
upper bound.

  python scripts/step_traffic.py list.csv STEPS [ALGO_BYTES_PER_STEP]
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2])
algo = float(sys.argv[3]) if len(sys.argv) > 3 else None
hdr, per = None, collections.defaultdict(dict)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    x = dict(zip(hdr, r))
    per[x["ID"]]["name"] = x["Kernel Name"].split("(")[0].replace("void ", "")[:70]
    per[x["ID"]][x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
byk = collections.defaultdict(lambda: [0, 0.0, 0.0])
tb = tt = 0.0
for v in per.values():
    b = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    k = byk[v["name"]]
    k[0] += 1
    k[1] += b
    k[2] += t
    tb += b
    tt += t
out = {"launches_per_step": len(per) / steps, "dram_bytes_per_step": tb / steps, "serial_kernel_us_per_step": tt / steps}
if algo:
    out["algorithmic_bytes_per_step"] = algo
    out["dram_over_algorithmic"] = tb / steps / algo
out["kernels"] = {k: {"launches_per_step": c / steps, "dram_bytes_per_step": b / steps, "us_per_step": t / steps}
                  for k, (c, b, t) in sorted(byk.items(), key=lambda kv: -kv[1][1])}
print(json.dumps(out, indent=1))
