"""Summarise an ncu --set full report + launch list into profiles/ (run here, no GPU)."""
import csv, io, json, subprocess, sys, collections

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "lts__t_sector_hit_rate.pct",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]

def main(rep, launches, tag):
    hdr, units, rows = raw(rep)
    ki = hdr.index("Kernel Name")
    per = collections.OrderedDict()
    for r in rows:
        name = r[ki].split("(")[0].replace("void ", "")
        rec = {w: (r[hdr.index(w)] + " " + units[hdr.index(w)]).strip() for w in WANT if w in hdr}
        per.setdefault(name, []).append(rec)
    summary = {}
    for name, recs in per.items():
        rec = recs[-1]
        def num(k):
            v = rec.get(k, "").split()[0].replace(",", "")
            try: return float(v)
            except: return None
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        unit = rec.get("dram__bytes_read.sum", "").split()[-1] if rec.get("dram__bytes_read.sum") else ""
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        summary[name] = {"metrics": rec, "dram_bytes_per_launch": (rd + wr) * scale if rd is not None else None,
                         "launches_captured": len(recs)}
    # launch list: per-kernel time shares of the last steps
    rows = list(csv.reader(open(launches)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi])) for r in rows[i + 1:] if len(r) > vi]
    agg = collections.OrderedDict()
    for n, v in data[-60:]:
        agg[n] = agg.get(n, 0.0) + v
    tot = sum(agg.values())
    shares = {n: {"ns": v, "share": v / tot} for n, v in sorted(agg.items(), key=lambda x: -x[1])}
    json.dump({"tag": tag, "kernels": summary, "launch_shares_last_steps": shares}, open(f"profiles/ncu_{tag}.json", "w"), indent=1)
    # bench.py reads the dominant kernel's dram bytes per launch from here
    simple = {}
    for key, pat in (("fold_adam", "k_fused_adam_tma"), ("pool", "k_fused_pool_s"), ("probe", "k_fused_probe")):
        for name, v in summary.items():
            if pat in name:
                simple[key] = {"kernel": name, "dram_bytes_per_launch": v["dram_bytes_per_launch"], "tag": tag}
    json.dump(simple, open("profiles/ncu_summary.json", "w"), indent=1)
    print(json.dumps(simple, indent=1))
    for n, v in shares.items():
        print(f"{v['ns']/1e3:9.1f} us {100*v['share']:5.1f}%  {n}")

if __name__ == "__main__":
    main(*sys.argv[1:4])
