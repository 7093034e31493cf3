#!/usr/bin/env python
"""ops_bench.py — the paper's Table-1 operator set on B200.

Runs the eight operators of `run_benchmarks` (reference bench.py:165-212) at
their Table-1 shapes through this repo's public API, times
each on the device (CUDA events, median of repeats, inputs resident in HBM),
and reports MBU = algorithmic bytes / time / peak with the reference's own
traffic formulas (bench.py:48-85), next to RecIS's published H20 MBU
(PAPER.md:337-344).  Prints one JSON line per operator and a markdown table.

  python ops_bench.py [--repeats 20]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

I64, F32 = 8, 4
# RecIS on H20, PAPER.md:337-344 (TensorFlow / PyTorch / RecIS MBU %)
PAPER_H20 = {
    "bucketize": (0.40, 0.40, 0.88), "mod": (0.45, 0.70, 1.68), "ids partition": (None, 34.60, 55.10),
    "sequence tile": (2.43, 4.58, 18.25), "reduce hard": (0.48, 0.93, 2.25), "reduce easy": (1.38, 2.75, 13.75),
    "gather": (1.70, 15.00, 47.50), "scatter": (None, 20.75, 58.00),
}


def traffic(kind, **k):
    """Reference bench.py:48-85 formulas (algorithmic minimum bytes)."""
    if kind == "bucketize":
        return k["n"] * F32 + k["cols"] * k["edges"] * F32 + k["n"] * I64
    if kind == "mod":
        return 2 * k["n"] * I64
    if kind == "partition":
        return k["n"] * I64 + k["u"] * I64 + 2 * k["n"] * I64
    if kind == "reduce":
        return k["n"] * k["d"] * F32 + (k["g"] + 1) * I64 + k["g"] * k["d"] * F32
    if kind == "tile":
        return k["taken"] * k["d"] * F32 + (k["g"] + 1) * I64 + k["g"] * k["k"] * k["d"] * F32
    if kind in ("gather", "scatter"):
        return k["n"] * I64 + 2 * k["n"] * k["d"] * F32
    raise ValueError(kind)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeats", type=int, default=20)
    ap.add_argument("--rows", action="store_true", help="also measure the other SURVEY §8(a) rows")
    args = ap.parse_args()
    import torch
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200 import _native as N

    torch.cuda.set_device(0)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
        peak_kind = "measured"
    except Exception:
        peak, peak_kind = 6.65e12, "fallback"
    rng = np.random.Generator(np.random.PCG64(0))
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2: flush between repeats

    def timed(fn):
        ts = []
        for r in range(args.repeats + 3):
            scrub.fill_(r & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(e0.elapsed_time(e1) / 1e3)
        return statistics.median(ts)

    results = []

    def report(name, nbytes, sec, shape, dispatches=1):
        mbu = nbytes / sec / peak
        results.append({"op": name, "shape": shape, "bytes": int(nbytes), "time_us": sec * 1e6,
                        "achieved_gbs": nbytes / sec / 1e9, "mbu_pct": 100 * mbu, "peak_kind": peak_kind,
                        "dispatches": dispatches, "recis_h20_mbu_pct": PAPER_H20[name][2]})
        print(json.dumps(results[-1]), flush=True)

    # bucketize / mod: 100 columns x 10,000 values, one fused dispatch (bench.py:119-162)
    C, V = 100, 10_000
    vals = [torch.from_numpy(rng.random(V, dtype=np.float32)).cuda() for _ in range(C)]
    offs = np.array([0, V], np.int64)
    cols = [skb.RaggedTensor(v, torch.from_numpy(offs).cuda()) for v in vals]
    edges = np.linspace(0.05, 0.95, 10, dtype=np.float32)
    plan = skb.FusedPlan.for_bucketize([edges] * C)
    # the fused kernel over pre-concatenated columns (what one dispatch moves)
    cat = torch.cat(vals)
    col_offs = torch.arange(0, C * V + 1, V, dtype=torch.int64, device="cuda")
    e_dev, eo_dev = plan._params_dev()
    out = torch.empty(C * V, dtype=torch.int64, device="cuda")
    sec = timed(lambda: N.call("skb_bucketize_multi", N.ptr(cat), N.ptr(col_offs), C, N.ptr(e_dev), N.ptr(eo_dev),
                               N.ptr(out), C * V, N.stream_ptr()))
    report("bucketize", traffic("bucketize", n=C * V, cols=C, edges=10), sec, "100 cols x 10,000")
    ivals = torch.from_numpy(rng.integers(0, 1 << 40, C * V, dtype=np.int64)).cuda()
    mods = torch.tensor([1_000_003 + 2 * c for c in range(C)], dtype=torch.int64, device="cuda")
    sec = timed(lambda: N.call("skb_mod_multi", N.ptr(ivals), N.ptr(col_offs), C, N.ptr(mods), N.ptr(out), C * V,
                               N.stream_ptr()))
    report("mod", traffic("mod", n=C * V), sec, "100 cols x 10,000")

    # ids partition: 1M ids over 8 shards (bench.py:174-179)
    n = 1_000_000
    ids = torch.from_numpy(rng.integers(0, n, n, dtype=np.int64)).cuda()
    u = int(torch.unique(ids).numel())
    uq = torch.empty(n, dtype=torch.int64, device="cuda")
    cnt = torch.empty(8, dtype=torch.int64, device="cuda")
    ish = torch.empty(n, dtype=torch.int64, device="cuda")
    ipo = torch.empty(n, dtype=torch.int64, device="cuda")
    sec = timed(lambda: N.call("skb_unique_partition", N.ptr(ids), n, 8, N.ptr(uq), N.ptr(cnt), N.ptr(ish),
                               N.ptr(ipo), N.stream_ptr()))
    report("ids partition", traffic("partition", n=n, u=u), sec, "1M ids, 8 shards")

    # sequence tile / reduce hard / reduce easy at 1M x 16 (bench.py:182-195)
    R, D = 1_000_000, 16
    rows = torch.from_numpy(rng.random((R, D), dtype=np.float32)).cuda()
    k = 8
    toffs = np.append(np.arange(0, R, k + 2, dtype=np.int64), R)
    taken = int(np.minimum(np.diff(toffs), k).sum())
    td = torch.from_numpy(toffs).cuda()
    G = len(toffs) - 1
    tout = torch.empty((G, k * D), device="cuda")
    sec = timed(lambda: N.call("skb_segment_tile", N.ptr(rows), R, D, N.ptr(td), G, k, 0.0, N.ptr(tout),
                               N.stream_ptr()))
    report("sequence tile", traffic("tile", taken=taken, g=G, k=k, d=D), sec, "1M x 16, len 10, k 8")
    for name, L in (("reduce hard", 1000), ("reduce easy", 2)):
        o = np.append(np.arange(0, R, L, dtype=np.int64), R)
        od = torch.from_numpy(o).cuda()
        G = len(o) - 1
        strat = skb.segments.resolve_strategy("auto", R, G)
        sid = 0 if strat == "sequential" else 1
        rout = torch.empty((G, D), device="cuda")
        sec = timed(lambda: N.call("skb_segment_reduce", N.ptr(rows), R, D, N.ptr(od), G, 0, sid, N.ptr(rout),
                                   N.stream_ptr()))
        report(name, traffic("reduce", n=R, g=G, d=D), sec, f"1M x 16, segment length {L} ({strat})")

    # gather / scatter over a populated table, 1M x 16 (bench.py:198-210)
    table = skb.EmbeddingTable("bench", D, seed=0, capacity_hint=R)
    all_ids = torch.arange(R, dtype=torch.int64, device="cuda")
    offsets = table.lookup_or_insert(all_ids, 1)
    gidx = offsets[torch.from_numpy(rng.integers(0, R, R)).cuda()]
    gout = torch.empty((R, D), device="cuda")
    sec = timed(lambda: N.call("skb_table_gather", table.handle, N.ptr(gidx), R, N.ptr(gout), N.stream_ptr()))
    report("gather", traffic("gather", n=R, d=D), sec, "1M x 16 (liveness-checked)")
    sidx = offsets[torch.from_numpy(rng.permutation(R)).cuda()]
    newr = torch.from_numpy(rng.random((R, D), dtype=np.float32)).cuda()
    sec = timed(lambda: N.call("skb_table_scatter_update", table.handle, N.ptr(sidx), R, N.ptr(newr),
                               N.stream_ptr()))
    report("scatter", traffic("scatter", n=R, d=D), sec, "1M x 16 (distinct + liveness checked)")
    # the same checked operators inside deferred_checks(): every check still
    # runs (on the device) and raises at the context's exit; the call itself
    # neither synchronises nor reads back
    # (the C-ABI entries EmbeddingTable.gather / scatter_update call there,
    # with a caller-owned flag array, like the other rows of this table)
    dflags = torch.full((4,), -1, dtype=torch.int64, device="cuda")
    sec = timed(lambda: N.call("skb_table_gather_deferred", table.handle, N.ptr(gidx), R, N.ptr(gout), N.ptr(dflags),
                               N.stream_ptr()))
    report("gather", traffic("gather", n=R, d=D), sec, "1M x 16 (liveness-checked, deferred check)")
    sec = timed(lambda: N.call("skb_table_scatter_update_deferred", table.handle, N.ptr(sidx), R, N.ptr(newr),
                               N.ptr(dflags), N.stream_ptr()))
    report("scatter", traffic("scatter", n=R, d=D), sec, "1M x 16 (distinct + liveness checked, deferred check)")
    assert dflags.cpu().tolist() == [-1] * 4, "deferred checks flagged valid inputs"
    # the same two operators without the reference's per-call validation
    # (callers that own the offsets, e.g. the fused step / the exchange)
    sec = timed(lambda: N.call("skb_table_gather_unchecked", table.handle, N.ptr(gidx), R, N.ptr(gout),
                               N.stream_ptr()))
    report("gather", traffic("gather", n=R, d=D), sec, "1M x 16 (trusted offsets)")
    sec = timed(lambda: N.call("skb_table_write_rows", table.handle, N.ptr(sidx), R, 0, N.ptr(newr), N.stream_ptr()))
    report("scatter", traffic("scatter", n=R, d=D), sec, "1M x 16 (BlockStore.write, range-checked)")

    # ---- the remaining SURVEY §8(a) rows through the public API (device tensors;
    # bytes = each input read once + each output written once)
    if args.rows:
        rows_out = []

        def row(tag, name, nbytes, fn, shape):
            sec = timed(fn)
            rows_out.append({"row": tag, "op": name, "shape": shape, "bytes": int(nbytes), "time_us": sec * 1e6,
                             "achieved_gbs": nbytes / sec / 1e9, "mbu_pct": 100 * nbytes / sec / peak})
            print(json.dumps(rows_out[-1]), flush=True)

        n = 1_000_000
        ids1 = torch.from_numpy(rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)).cuda()
        plan8 = skb.ShardPlan(8)
        row("a1", "shard_of (mix64 % S)", 16 * n, lambda: plan8.shard_of(ids1), "1M ids, 8 shards")
        lt = skb.LogicalTable("dim16", 16, 1, seed=0, members=["m0"], namespaced=True)
        row("a2", "keys_for (namespaced key)", 16 * n, lambda: lt.keys_for("m0", ids1), "1M ids")
        row("a4", "initial_rows", 8 * n + 64 * n, lambda: skb.initial_rows(3, ids1, 16), "1M ids x 16")
        t2 = skb.EmbeddingTable("a5", 16, seed=0, capacity_hint=2 * n)
        uniq = torch.arange(n, dtype=torch.int64, device="cuda") * 7919
        t2.lookup_or_insert(uniq, 1)
        # warm: every id present -> probe + offsets + last_step (duplicate check included)
        row("a5", "lookup_or_insert (warm, dup-checked)", 8 * n + 16 * n + 8 * n + 8 * n,
            lambda: t2.lookup_or_insert(uniq, 2), "1M unique ids, all present")
        offs_u = t2.lookup_or_insert(uniq, 2)
        gsrc = torch.randn((n, 16), device="cuda")
        cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
        row("a13", "sparse_adam_step (distinct-checked)", 8 * n + 64 * n + 2 * 192 * n,
            lambda: skb.sparse_adam_step(t2.store, offs_u, gsrc, cfg, 3), "1M rows x 16, AdamW")
        pos = torch.from_numpy(rng.integers(0, n // 4, n, dtype=np.int64)).cuda()
        pr = skb.unique_partition(pos, skb.ShardPlan(4))
        per = [torch.randn((len(x), 16), device="cuda") for x in pr.shard_ids]
        row("a8", "PartitionResult.restore", 16 * n + 64 * n + 64 * pr.num_unique, lambda: pr.restore(per),
            "1M positions x 16, 4 shards")
        grads = torch.randn((n, 16), device="cuda")
        inv = pr.inverse_pos + torch.tensor(pr._bases(), device="cuda")[pr.inverse_shard]
        fout = torch.empty((pr.num_unique, 16), device="cuda")
        row("a12", "grad pre-aggregation (ordered fold)", 8 * n + 64 * n + 64 * pr.num_unique,
            lambda: N.call("skb_grad_fold", N.ptr(grads), n, 16, N.ptr(inv.contiguous()), pr.num_unique, N.ptr(fout),
                           N.stream_ptr()), "1M positions x 16 -> ~250K rows")
        row("a19", "load_stats", 8 * n + 64, lambda: skb.load_stats(ids1, plan8), "1M ids, 8 shards")
        tok = rng.integers(0, 1_000_000, n).astype("S7")
        ln = np.char.str_len(tok).astype(np.int64)
        so = np.zeros(n + 1, np.int64)
        np.cumsum(ln, out=so[1:])
        blob = tok.view(np.uint8).reshape(n, 7)[np.arange(7)[None, :] < ln[:, None]]
        bd, sd = torch.from_numpy(blob).cuda(), torch.from_numpy(so).cuda()
        row_offs = torch.arange(0, n + 1, 4, dtype=torch.int64, device="cuda")
        row("a15", "hash_feature (FNV-1a, packed strings)", len(blob) + 8 * (n + 1) + 8 * n,
            lambda: skb.hash_feature_packed(bd, sd, row_offs), "1M strings (~6 B)")
        R = 65536
        la, lb = rng.integers(0, 6, R), rng.integers(0, 6, R)
        oa = np.concatenate([[0], np.cumsum(la)]).astype(np.int64)
        ob = np.concatenate([[0], np.cumsum(lb)]).astype(np.int64)
        A = skb.RaggedTensor(torch.from_numpy(rng.integers(0, 1 << 40, oa[-1])).cuda(), torch.from_numpy(oa).cuda())
        Bt = skb.RaggedTensor(torch.from_numpy(rng.integers(0, 1 << 40, ob[-1])).cuda(), torch.from_numpy(ob).cuda())
        tot = int((la * lb).sum())
        row("a18", "cross (pairwise FNV)", 8 * (oa[-1] + ob[-1]) + 24 * R + 8 * tot,
            lambda: skb.cross_many([(A, Bt)], sizes=[tot]), f"64K rows, {tot} outputs")
        seq_o = torch.arange(0, n + 1, 250, dtype=torch.int64, device="cuda")
        RT = skb.RaggedTensor(ids1, seq_o)
        row("a20", "RaggedTensor.truncate(100, tail)", 8 * n + 8 * (n // 250 + 1) * 2 + 8 * 100 * (n // 250),
            lambda: RT.truncate(100, "tail"), "4000 rows x 250 -> 100")
        t3 = skb.EmbeddingTable("a14", 16, seed=0, evict_threshold=1, capacity_hint=2 * n)

        def evict_cycle():
            t3.lookup_or_insert(uniq, 10)
            t3.evict(20)  # every row stale

        row("a14", "admit 1M + evict 1M (cycle)", 2 * (8 * n + 16 * n + 192 * n), evict_cycle,
            "1M ids admitted then evicted")
        print("\n| §8 row | op | shape | time (us) | GB/s | % of peak |")
        print("|---|---|---|---|---|---|")
        for r in rows_out:
            print(f"| {r['row']} | {r['op']} | {r['shape']} | {r['time_us']:.1f} | {r['achieved_gbs']:.0f} | "
                  f"{r['mbu_pct']:.1f} |")

    print(f"\n| op | shape | time (us) | GB/s | MBU on B200 (% of {peak_kind} peak) | RecIS MBU on H20 (paper) |")
    print("|---|---|---|---|---|---|")
    for r in results:
        print(f"| {r['op']} | {r['shape']} | {r['time_us']:.1f} | {r['achieved_gbs']:.0f} | {r['mbu_pct']:.2f} | "
              f"{r['recis_h20_mbu_pct']} |")


if __name__ == "__main__":
    main()
