"""Per-stream busy time, union busy time and idle gaps of a Chrome trace
written by bench.py's SKB_TRACE hook (torch.profiler / CUPTI kernel records).

  python scripts/trace_gaps.py gpurun_out/trace/trace_c5.json [top]
"""
import collections
import json
import sys

tr = json.load(open(sys.argv[1]))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
by_stream = collections.defaultdict(list)
for e in ev:
    by_stream[e["args"].get("stream", e.get("tid"))].append(e)
print(f"{len(ev)} device records over {(t1 - t0) / 1e3:.3f} ms")
for s, es in sorted(by_stream.items(), key=lambda kv: -sum(e["dur"] for e in kv[1])):
    print(f"  stream {s}: {len(es)} records, busy {sum(e['dur'] for e in es) / 1e3:.3f} ms")
# union of busy intervals
busy, cur_s, cur_e = 0.0, None, None
gaps = []
for e in ev:
    s, en = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, cur_e, e["name"][:70]))
        cur_s, cur_e = s, en
    else:
        cur_e = max(cur_e, en)
busy += cur_e - cur_s
print(f"union busy {busy / 1e3:.3f} ms, idle {(t1 - t0 - busy) / 1e3:.3f} ms in {len(gaps)} gaps")
for g, at, name in sorted(gaps, reverse=True)[:10]:
    print(f"  gap {g:8.1f} us at +{(at - t0) / 1e3:8.3f} ms before {name}")
tot = collections.Counter()
cnt = collections.Counter()
for e in ev:
    tot[e["name"][:80]] += e["dur"]
    cnt[e["name"][:80]] += 1
print("top kernels (sum of durations):")
for k, v in tot.most_common(top):
    print(f"  {cnt[k]:5d} x {v / cnt[k]:8.1f} us = {v / 1e3:8.3f} ms  {k}")
