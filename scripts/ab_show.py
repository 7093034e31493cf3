"""Print `<label...> {json}` lines written by the A/B scripts."""
import json
import sys

for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.jsonl"):
    i = line.find("{")
    if i < 0:
        continue
    d = json.loads(line[i:])
    print(f"{line[:i].strip():32s} ms/step {d['ms_per_step']:.4f}")
