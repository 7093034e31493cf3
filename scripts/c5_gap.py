"""Largest idle gap of the compute stream in a C5 trace and what ran in it."""
import collections
import json
import sys

tr = json.load(open(sys.argv[1]))
ev = sorted((e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")),
            key=lambda e: e["ts"])
t0 = ev[0]["ts"]
busy = collections.Counter()
for e in ev:
    busy[e["args"].get("stream")] += e["dur"]
main = busy.most_common(1)[0][0]
m = [e for e in ev if e["args"].get("stream") == main]
gaps = sorted(((b["ts"] - (a["ts"] + a["dur"]), a["ts"] + a["dur"], b["ts"]) for a, b in zip(m, m[1:])), reverse=True)
g, s, e_ = gaps[0]
print(f"main stream {main}: busy {busy[main] / 1e3:.3f} ms of {(ev[-1]['ts'] - t0) / 1e3:.3f}; largest gap {g:.1f} us")
agg = collections.defaultdict(lambda: [0, 0.0, 1e18, 0])
for e in ev:
    if e["ts"] + e["dur"] >= s and e["ts"] <= e_:
        k = (e["args"].get("stream"), e["name"][:50])
        r = agg[k]
        r[0] += 1
        r[1] += e["dur"]
        r[2] = min(r[2], e["ts"])
        r[3] = max(r[3], e["ts"] + e["dur"])
for (st, nm), (c, d, a, b) in sorted(agg.items(), key=lambda kv: kv[1][2]):
    print(f"  s{st} {c:4d} x {nm:50s} sum {d:7.1f} us  span {(a - s):7.1f} .. {(b - s):7.1f} us")
