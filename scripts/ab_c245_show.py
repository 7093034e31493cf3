"""Print ms/step per config from gpurun_out/ab_<tag>.jsonl files."""
import json
import sys

for tag in sys.argv[1:]:
    out = {}
    for line in open(f"gpurun_out/ab_{tag}.jsonl"):
        k, j = line.split(" ", 1)
        d = json.loads(j)
        out.setdefault(k, []).append(round(d["ms_per_step"], 3))
    print(tag, out)
