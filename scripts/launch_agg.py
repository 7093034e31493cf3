"""Aggregate an ncu --csv launch list: per-kernel count, mean and total time.
Optional second arg: only the last K launches (the timed steps)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, L = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    x = dict(zip(hdr, r))
    if x.get("Metric Name") == "gpu__time_duration.sum":
        L.append((x["Kernel Name"][:90], float(x["Metric Value"].replace(",", "")) / 1000))
if last:
    L = L[-last:]
tot, cnt = collections.Counter(), collections.Counter()
for k, t in L:
    tot[k] += t
    cnt[k] += 1
print(f"{len(L)} launches, {sum(tot.values()):.1f} us total")
for k, t in tot.most_common(30):
    print(f"{cnt[k]:5d} {t / cnt[k]:9.1f} us  tot {t:9.1f}  {k}")
