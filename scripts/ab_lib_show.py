"""Summarise gpurun_out/ablib.jsonl (variant, config -> ms per step)."""
import collections
import json

out = collections.defaultdict(list)
for line in open("gpurun_out/ablib.jsonl"):
    v, c, j = line.split(" ", 2)
    out[(c, v)].append(round(json.loads(j)["ms_per_step"], 3))
for k in sorted(out):
    print(k, out[k])
