"""List the kernels of a SKB_TRACE timeline (start ms, duration ms, stream, name)."""
import json
import sys

tr = json.load(open(sys.argv[1]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev[:n]:
    if e["dur"] > 20:
        print(f'{(e["ts"] - t0) / 1e3:8.3f} {e["dur"] / 1e3:7.3f} s{e["args"].get("stream")} {e["name"][:60]}')
