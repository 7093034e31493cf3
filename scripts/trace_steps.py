"""Per-step kernel timeline of a Chrome trace written by bench.py's SKB_TRACE
hook: kernels grouped into steps by a marker kernel (the first launch of each
step), printed as start / end offsets from the step start with their stream,
so the critical path of a step can be read off.

  python scripts/trace_steps.py gpurun_out/trace/trace_c4.json k_fused_tile [steps]
"""
import json
import sys

tr = json.load(open(sys.argv[1]))
marker = sys.argv[2]
nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
starts = [e["ts"] for e in ev if marker in e["name"]]
print(f"{len(starts)} marker launches; step lengths (us):",
      [round(b - a, 1) for a, b in zip(starts[:-1], starts[1:])])
for k in range(min(nsteps, len(starts) - 1)):
    a, b = starts[k], starts[k + 1]
    print(f"--- step {k}: {b - a:.1f} us")
    for e in ev:
        if e["ts"] + e["dur"] < a - 50 or e["ts"] >= b:
            continue
        s = e["args"].get("stream", e.get("tid"))
        print(f"  {e['ts'] - a:9.1f} {e['ts'] + e['dur'] - a:9.1f}  s{s:<4} {e['name'][:90]}")
