"""Per-kernel metrics (last capture of each kernel) of an ncu --set full
report as JSON (run here, no GPU):
  python scripts/ncu_kernels.py report.ncu-rep TAG WORKLOAD > profiles/ncu_<x>.json"""
import json
import sys

sys.path.insert(0, "scripts")
from ncu_summary import WANT, raw  # noqa: E402

rep, tag, workload = sys.argv[1:4]
hdr, units, rows = raw(rep)
ki = hdr.index("Kernel Name")
out = {}
for r in rows:
    name = r[ki].split("(")[0].replace("void ", "")
    rec = {}
    for w in WANT:
        if w in hdr:
            v = r[hdr.index(w)].replace(",", "")
            try:
                rec[w] = float(v)
            except ValueError:
                rec[w] = v
    B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    S = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}
    u = lambda w: units[hdr.index(w)] if w in hdr else ""
    rd, wr = rec.get("dram__bytes_read.sum"), rec.get("dram__bytes_write.sum")
    if isinstance(rd, float) and isinstance(wr, float):
        rec["dram_bytes"] = rd * B.get(u("dram__bytes_read.sum"), 1) + wr * B.get(u("dram__bytes_write.sum"), 1)
        t = rec.get("gpu__time_duration.sum")
        if isinstance(t, float) and t > 0:
            rec["seconds"] = t * S.get(u("gpu__time_duration.sum"), 1e-9)
            rec["dram_tb_per_s"] = rec["dram_bytes"] / rec["seconds"] / 1e12
    rec["units"] = {w: units[hdr.index(w)] for w in WANT if w in hdr}
    out[name] = rec
print(json.dumps({"tag": tag, "workload": workload, "kernels": out}, indent=1))
