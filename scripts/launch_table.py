"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, d = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    x = dict(zip(hdr, r))
    if x.get("Metric Name") != "gpu__time_duration.sum":
        continue
    d.setdefault(x["Kernel Name"][:90], []).append(float(x["Metric Value"].replace(",", "")))
for k, v in d.items():
    print(f"{len(v):5d} {sum(v) / len(v) / 1000:9.2f} us  {k}")
