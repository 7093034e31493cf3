"""bench_configs.py — bench.py's legs for SURVEY §8d's configs other than the
headline C2 (`python bench.py --workload c1|c3|c4|c5`).  Part of bench.py
(imported only by it); each workload prints ONE JSON line with the same
keys as the headline (value, roofline, cpu_baseline, clocks), measured on
one GPU with CUDA events over the timed steps.

  c1  dim16, B=4096, one feature, bag length 1, sum, SparseAdamW — the
      launch-bound config (fits in L2); CUDA-graph mode of the fused step.
  c3  the per-GPU owner side of C3: zipf(alpha=1.1) ids, 26 features x dim16
      merged namespaced table, B=65536, sum, grown from empty to 1e9/8 rows
      (the share of one of 8 GPUs).  Zipf's tail keeps admitting new ids;
      each step shifts ids >= 2^20 by a per-step offset so every step's tail
      is fresh while the hot head repeats (growth without regenerating
      1.7M zipf draws per step).  Reports the growth curve.
  c4  B=8192 sequences of length 1000 (zipf ids), dim 64, tile combiner
      k=1000 -> [8192, 64000] per step, backward = the tile gradient of
      every position + SparseAdamW on the touched rows.
  c5  200 features (dims 8/16/32/64/128 -> 5 logical tables of 40 members),
      B=16384, mean combiner, bags min(geometric(.25), 64) with 10% empty and
      1% at 64; feature engine inside the step: 20 byte-string columns ->
      hash_feature, 20 float columns -> fused bucketize (10 edges), 20
      crosses of id-column pairs -> fused mod 1_000_003, 140 raw id columns.

The CPU baselines run the reference algorithm (the oracle port) on a
bounded sample of the same workload on this host's cores.
"""

from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np

import bench as B

DIMS5 = (8, 16, 32, 64, 128)


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


_CLK = {"summary": None, "gc": None}


def _timed(run, steps):
    """The timed region every config shares: CUDA events on the current
    stream around `run(steps)`, an NVTX "timed" range (ncu/CUPTI filters),
    and nvidia-smi clocks sampled while it runs (the sampler starts before
    e0 so the first samples land inside the region).  Returns ms per step."""
    import torch
    e0, e1 = _events()
    B.GcPauses.freeze()
    with B.ClockSampler(torch.cuda.current_device()) as clk, B.GcPauses() as gcp:
        time.sleep(0.25)  # the sampler's first rows
        e0.record()
        torch.cuda.nvtx.range_push("timed")
        run(steps)
        torch.cuda.nvtx.range_pop()
        e1.record()
        torch.cuda.synchronize()
    _CLK["summary"] = clk.summary()
    _CLK["gc"] = gcp.summary()
    return e0.elapsed_time(e1) / steps


class _Watch:
    """Diagnostics (SKB_C5_WATCH=1): a thread samples the main thread's Python
    stack every ms while a watched block runs; blocks longer than 10 ms print
    the stacks seen after the 10 ms mark (and the sampling gaps: a gap means
    the main thread held the GIL inside a C call)."""

    def __init__(self):
        import sys
        import threading
        import traceback
        self.sys, self.tb = sys, traceback
        self.main = threading.get_ident()
        self.t0 = None
        self.samples = []
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        while True:
            time.sleep(0.001)
            t0 = self.t0
            if t0 is not None:
                dt = time.perf_counter() - t0
                if dt > 0.010:
                    f = self.sys._current_frames().get(self.main)
                    st = "".join(self.tb.format_stack(f, limit=6)[-4:]) if f else "?"
                    self.samples.append((round(dt * 1e3, 2), st))

    def __enter__(self):
        self.samples = []
        self.t0 = time.perf_counter()

    def __exit__(self, *a):
        dt = time.perf_counter() - self.t0
        self.t0 = None
        if dt > 0.010:
            import sys
            print(f"[watch] block {dt * 1e3:.1f} ms; {len(self.samples)} samples", file=sys.stderr)
            last = None
            for t, st in self.samples:
                if st != last:
                    print(f"[watch] t={t} ms\n{st}", file=sys.stderr)
                    last = st


def _settle(run, warmup: int, chunk: int = 10, cap: int = 300) -> int:
    """Warm-up until the torch caching allocator stops growing: `warmup`
    steps, then chunks of `chunk` steps until two chunks in a row make no new
    device allocation (at most `cap` extra steps).  Blocks the step's tensors pin
    across streams (record_stream) are freed late, so the pool keeps adding
    segments for a few dozen steps; each addition is a cudaMalloc, which in
    a process holding ~150 GB of mapped tables took 20-100 ms at random on
    the host — long enough for the device to drain its queue and idle.
    Returns the warm-up steps run."""
    import torch
    run(warmup)
    done, clean = warmup, 0
    while done < warmup + cap and clean < 2:
        a0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
        run(chunk)
        done += chunk
        clean = clean + 1 if torch.cuda.memory_stats().get("num_device_alloc", 0) == a0 else 0
    return done


def _worst(steps_ms, host_t):
    """The slowest timed step: its device ms and the host ms of each phase
    of it and of the step before (a host stall shows up in one of those)."""
    i = max(range(len(steps_ms)), key=steps_ms.__getitem__)
    ph = ("forward", "backward", "build", "prefetch")
    out = {"index": i, "ms": round(steps_ms[i], 3)}
    for j, tag in ((i - 1, "host_prev"), (i, "host")):
        if 0 <= j < len(host_t):
            out[tag] = {nm: round(host_t[j][q] * 1e3, 3) for q, nm in enumerate(ph)}
    return out


def _line(args, workload, value, ms, ids_per_step, samples_per_step, algo_bytes, cpu, config, extra=None):
    peak, peak_kind = B.load_peaks()
    achieved = algo_bytes / (ms / 1e3) / 1e9
    line = {
        "metric": B.METRIC, "value": value, "unit": "IDs/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "workload_key": workload,
        "config": config, "samples_per_s": samples_per_step / (ms / 1e3), "ids_per_step": ids_per_step,
        "roofline": {"bound": "hbm", "kernel": "whole step (SURVEY §8d B_step)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                     "peak_kind": peak_kind, "algorithmic_bytes": int(algo_bytes)},
        "cpu_baseline": cpu, "clocks": _CLK["summary"], "gc_in_timed": _CLK["gc"],
        "fold": getattr(args, "fold", "exact") + (" (tolerance mode: hot-id runs > 32 positions reduced as a two-level "
                                                  "tree, not bit-exact)" if getattr(args, "fold", "exact") == "tree"
                                                  else " (bit-exact np.add.at order)"),
    }
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)


def _cpu(fn, sample: str, steps: int = 3, warm: int = 1):
    """Time the oracle leg: `fn(step)` runs one sampled step; returns the
    median seconds per step and the effective cores (process / wall)."""
    for w in range(warm):
        fn(w + 1)
    ts = []
    c0, w0 = time.process_time(), time.perf_counter()
    for s in range(steps):
        t0 = time.perf_counter()
        fn(warm + 1 + s)
        ts.append(time.perf_counter() - t0)
    wall = time.perf_counter() - w0
    return statistics.median(ts), round((time.process_time() - c0) / wall, 2) if wall > 0 else 1.0


# ---------------------------------------------------------------------------
# C1
# ---------------------------------------------------------------------------

def c1(args):
    import torch
    import paper_2509_20883_b200 as skb
    Bn, D = 4096, 16
    lt = skb.LogicalTable("f0", D, 1, seed=0, members=["f0"], namespaced=False, capacity_hint=200_000)
    rng = np.random.default_rng(0)
    offs = np.arange(Bn + 1, dtype=np.int64)
    pool_ids = [torch.from_numpy(rng.integers(0, 100_000, Bn)).cuda() for _ in range(8)]
    batch = skb.PackedBatch(lt, ["f0"], [rng.integers(0, 100_000, Bn)], [offs])
    dp = torch.randn((Bn, D), device="cuda") * 1e-2
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    pooled = torch.empty((Bn, D), device="cuda")
    skb.use_graphs(lt, True)
    step = [0]

    def run(count):
        for _ in range(count):
            step[0] += 1
            batch.ids.copy_(pool_ids[step[0] % 8], non_blocking=True)  # fixed buffer: graph replay
            skb.lookup_pool(lt, batch, step[0], "sum", out=pooled)
            skb.pool_grad_adam(lt, dp, cfg, step[0])

    run(max(args.warmup, 3) + 20)  # admits the id space; graphs captured on the 2nd call
    torch.cuda.synchronize()
    steps = max(args.steps, 200)  # ~50 us steps: time enough of them to amortise graph re-captures
    ms = _timed(run, steps)
    B.maybe_trace("c1", lambda: run(20))
    u, unew = skb.last_step_stats(lt)
    sb = B.step_bytes(Bn, Bn, u, unew, D)

    cpu = None
    if not args.no_cpu_baseline:
        from oracle import sparse_oracle as O
        olt = O.OracleLogical("f0", D, 1, seed=0, members=["f0"], namespaced=False)
        host_ids = [p.cpu().numpy() for p in pool_ids]
        g = dp.cpu().numpy()

        def one(k):
            ids = host_ids[k % 8]
            rows = O.lookup(olt, ids, k)
            O.pool(rows, offs, "sum")
            O.grad_update(olt, ids, g, k, lr=1e-3, weight_decay=0.01, variant="adamw")

        for k in range(8):  # same warm state: the sampled ids admitted
            one(k + 1)
        sec, cores = _cpu(lambda k: one(100 + k), "C1 full", steps=10, warm=2)
        cpu = {"value": Bn / sec, "unit": "IDs/s", "cores": 1, "kind": "port",
               "sample": f"C1 full size (4096 ids/step), warm, 10 steps median; effective cores {cores}"}
    _line(args, "c1", Bn / (ms / 1e3), ms, Bn, Bn, sb, cpu,
          {"workload": "C1: table f0 dim16, batch 4096, 1 feature, bag length 1, sum, SparseAdamW; ids "
                       "integers(0,1e5); fused step in CUDA-graph mode", "global_batch": Bn, "dim": D,
           "parallelism": "single shard", "l2": "fits in L2 (latency-bound config)"},
          {"note": "C1's working set (~2.5 MB/step) is L2-resident; the roofline fraction is not meaningful "
                   "here, step latency is the figure of merit",
           "us_per_step": ms * 1e3, "unique_rows_per_step": u, "steps": steps})


# ---------------------------------------------------------------------------
# C3 (one GPU's owner share, growth to 1e9/8 rows)
# ---------------------------------------------------------------------------

def _zipf_batch(seed_base, Bn, F):
    return [np.random.Generator(np.random.PCG64(seed_base + f)).zipf(1.1, Bn).astype(np.int64) for f in range(F)]


def c3(args):
    import torch
    import paper_2509_20883_b200 as skb
    F, Bn, D = 26, 65536, 16
    mem = [f"C{f}" for f in range(F)]
    # the IDMap is sized for the target up front (no rehash on the way: 15%
    # headroom, the last 20-step chunk overshoots the target by ~10%); the
    # row arena starts empty and grows copy-free (VMM) as rows are admitted
    lt = skb.LogicalTable("dim16", D, 1, seed=0, members=mem, namespaced=True,
                          capacity_hint=int(args.c3_rows * 1.15))
    skb.set_fold_mode(lt, args.fold)
    offs = [np.arange(Bn + 1, dtype=np.int64)] * F
    P = 4
    base = []
    for k in range(P):
        b = skb.PackedBatch(lt, mem, _zipf_batch(1000 * k, Bn, F), offs)
        base.append(b.ids.clone())
    bufs = [skb.PackedBatch(lt, mem, _zipf_batch(0, Bn, F), offs) for _ in range(2)]
    n = F * Bn
    dp = torch.randn((n, D), device="cuda") * 1e-2
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    pooled = torch.empty((n, D), device="cuda")
    hot = torch.tensor(1 << 20, dtype=torch.int64, device="cuda")
    step = [0]

    def fill(k):
        # head (< 2^20) repeats; the tail is shifted into a fresh range every step
        ids = base[k % P]
        torch.where(ids < hot, ids, ids + (k + 1) * (1 << 44), out=bufs[k % 2].ids)

    pending = set()

    def run(count):
        # cross-step pipeline: step k+1's ids are produced and its index phase
        # (probe, admission of ~0.4M new rows, sort) issued before step k's
        # backward, on the table's index stream
        for _ in range(count):
            step[0] += 1
            k = step[0]
            if k not in pending:
                fill(k)
                skb.prefetch(lt, bufs[k % 2], k, "sum")
            pending.discard(k)
            skb.lookup_pool(lt, bufs[k % 2], k, "sum", out=pooled)
            fill(k + 1)
            skb.prefetch(lt, bufs[(k + 1) % 2], k + 1, "sum")
            pending.add(k + 1)
            skb.pool_grad_adam(lt, dp, cfg, k)

    target = int(args.c3_rows)
    run(args.warmup)
    torch.cuda.synchronize()
    curve = []
    t_all = 0.0
    ids_all = 0
    chunk = max(1, args.steps)
    t_start = time.perf_counter()
    while True:
        # an event after every step: the slowest step of the chunk (a growth
        # stall would show here, not only in the chunk's mean)
        evs = [_events()[0] for _ in range(chunk + 1)]
        host_ms = []
        evs[0].record()
        for i in range(chunk):
            h0 = time.perf_counter()
            run(1)
            host_ms.append((time.perf_counter() - h0) * 1e3)
            evs[i + 1].record()
        torch.cuda.synchronize()
        steps_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(chunk)]
        ms = sum(steps_ms)
        t_all += ms
        ids_all += chunk * n
        rows = lt.num_rows
        u, unew = skb.last_step_stats(lt)
        curve.append({"rows": int(rows), "ms_per_step": ms / chunk, "max_step_ms": max(steps_ms),
                      "max_host_call_ms": max(host_ms),
                      "ids_per_s": chunk * n / (ms / 1e3), "last_step_unique": u, "last_step_new": unew})
        if rows >= target or time.perf_counter() - t_start > 240:
            break
    # steady state at the final size: same batches, new tails still admitted
    ms = _timed(run, args.steps)
    B.maybe_trace("c3", lambda: run(6))
    u, unew = skb.last_step_stats(lt)
    sb = B.step_bytes(n, n, u, unew, D)

    cpu = None
    if not args.no_cpu_baseline:
        from oracle import sparse_oracle as O
        cb = 1024
        olt = O.OracleLogical("dim16", D, 1, seed=0, members=mem, namespaced=True)
        samples = [_zipf_batch(1000 * k, cb, F) for k in range(2)]
        g = np.random.default_rng(3).normal(0, 1e-2, (F * cb, D)).astype(np.float32)

        def one(k):
            ids = [np.where(x < (1 << 20), x, x + (k + 1) * (1 << 44)) for x in samples[k % 2]]
            keys = np.concatenate([olt.keys_for(m, x) for m, x in zip(mem, ids)])
            rows_ = O.lookup(olt, keys, k)
            for f in range(F):
                O.pool(rows_[f * cb:(f + 1) * cb], np.arange(cb + 1, dtype=np.int64), "sum")
            O.grad_update(olt, keys, g, k, lr=1e-3, weight_decay=0.01, variant="adamw")

        sec, cores = _cpu(one, "", steps=3, warm=1)
        cpu = {"value": F * cb / sec, "unit": "IDs/s", "cores": 1, "kind": "port",
               "sample": f"C3 scaled to batch {cb}/feature ({F * cb} ids/step), growing table, 3 steps median; "
                         f"effective cores {cores}"}
    _line(args, "c3", n / (ms / 1e3), ms, n, Bn, sb, cpu,
          {"workload": "C3 per-GPU owner share: zipf(1.1) ids, 26 x dim16 merged namespaced table, batch "
                       "65536, bag length 1, sum, SparseAdamW; table grown from empty inside the timed steps (IDMap "
                       "sized from the capacity hint, row arena mapped copy-free as rows arrive)", "global_batch": Bn, "features": F, "dim": D,
           "target_rows": target, "parallelism": "single shard (one GPU's share of 8)",
           "l2": "inputs larger than L2 (table grows to GBs)"},
          {"growth_curve": curve, "table_rows": int(lt.num_rows), "growth_ids_per_s": ids_all / (t_all / 1e3),
           "growth_max_step_ms": max(c["max_step_ms"] for c in curve),
           "unique_rows_per_step": u, "new_rows_per_step": unew})


# ---------------------------------------------------------------------------
# C4
# ---------------------------------------------------------------------------

def c4(args):
    import torch
    import paper_2509_20883_b200 as skb
    G, L, D = 8192, 1000, 64
    n = G * L
    # capacity: the table's ~2.35M rows plus three steps of positions, the
    # host's no-sync admission bound (every in-flight position a possible new
    # row); a tighter arena makes every step synchronise to refresh counters
    lt = skb.LogicalTable("seq", D, 1, seed=4, members=["seq"], namespaced=False, capacity_hint=2_400_000 + 3 * n)
    skb.set_fold_mode(lt, args.fold)
    offs_d = torch.arange(0, n + 1, L, dtype=torch.int64, device="cuda")
    P = 2
    ids = [torch.from_numpy(np.random.Generator(np.random.PCG64(4 + k)).zipf(1.1, n).astype(np.int64)).cuda()
           for k in range(P)]
    dtile = torch.randn((G, L * D), device="cuda") * 1e-2
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    step = [0]
    fused = not args.no_pipeline  # --no-pipeline: the drop-in API path instead of the fused step
    if fused:
        # truncate(1000, "tail") keeps every length-1000 sequence whole: the
        # fused tile combiner then reads each bag's first k = 1000 rows
        batches = []
        for k in range(P):
            x = skb.RaggedTensor(ids[k], offs_d).truncate(L, "tail")
            batches.append(skb.PackedBatch(lt, ["seq"], [x.values], [x.row_offsets]))
        tiles = torch.empty((G, L * D), device="cuda")
    plan = skb.ShardPlan(1)

    pending = set()

    def run(count):
        for _ in range(count):
            step[0] += 1
            if fused:
                # cross-step pipeline: step k+1's index phase (probe,
                # admission, sort of 8.2M positions) is issued before step
                # k's backward and runs under its long fold
                k = step[0]
                if k not in pending:
                    skb.prefetch(lt, batches[k % P], k, "tile", k=L, pad=0.0)
                pending.discard(k)
                skb.lookup_pool(lt, batches[k % P], k, "tile", out=tiles, k=L, pad=0.0)
                skb.prefetch(lt, batches[(k + 1) % P], k + 1, "tile", k=L, pad=0.0)
                pending.add(k + 1)
                skb.pool_grad_adam(lt, dtile, cfg, k)
                continue
            x = skb.RaggedTensor(ids[step[0] % P], offs_d).truncate(L, "tail")
            rows = skb.all_to_all_lookup(lt, x.values, plan, step[0])
            skb.segment_tile(rows, x.row_offsets, L, pad=0.0)
            # every kept position maps to one tile row: its gradient is that row
            skb.all_to_all_grad_update(lt, x.values, dtile.view(n, D), plan, cfg, step[0])

    _settle(run, max(args.warmup, 3))
    torch.cuda.synchronize()
    import ctypes
    from paper_2509_20883_b200 import _native as N
    if fused:
        N.call("skb_fused_profile", lt.local_table.handle, args.steps, N.stream_ptr())
    ms = _timed(run, args.steps)
    phase_ms = {}
    if fused:
        buf = (ctypes.c_float * args.steps)()
        for p_, name in enumerate(B.PHASES):
            cnt = ctypes.c_int64()
            N.call("skb_fused_profile_read", lt.local_table.handle, p_, buf, args.steps, ctypes.byref(cnt))
            vals = list(buf)[: cnt.value]
            phase_ms[name] = [round(v, 3) for v in vals]
        N.call("skb_fused_profile", lt.local_table.handle, 0, N.stream_ptr())
    B.maybe_trace("c4", lambda: run(3))
    u = int(torch.unique(ids[step[0] % P]).numel())
    sb = B.step_bytes(n, n, u, 0, D)  # G' = G*k = n tile rows

    cpu = None
    if not args.no_cpu_baseline:
        from oracle import sparse_oracle as O
        cg = 64
        olt = O.OracleLogical("seq", D, 1, seed=4, members=["seq"], namespaced=False)
        hid = ids[0][: cg * L].cpu().numpy()
        hoffs = np.arange(0, cg * L + 1, L, dtype=np.int64)
        g = dtile[:cg].reshape(cg * L, D).cpu().numpy()

        def one(k):
            rows_ = O.lookup(olt, hid, k)
            O.tile(rows_, hoffs, L)
            O.grad_update(olt, hid, g, k, lr=1e-3, weight_decay=0.01, variant="adamw")

        sec, cores = _cpu(one, "", steps=2, warm=1)
        cpu = {"value": cg * L / sec, "unit": "IDs/s", "cores": 1, "kind": "port",
               "sample": f"C4 scaled to batch {cg} ({cg * L} ids/step), 2 steps median; effective cores {cores}"}
    _line(args, "c4", n / (ms / 1e3), ms, n, G, sb, cpu,
          {"workload": "C4: 8192 sequences x length 1000, zipf(1.1) ids, dim64, truncate(1000,'tail') + "
                       "segment_tile(k=1000) -> [8192, 64000], tile-gradient backward + SparseAdamW; "
                       + ("fused step, tile combiner" if fused else
                          "drop-in API path: all_to_all_lookup -> segment_tile -> all_to_all_grad_update"),
           "global_batch": G, "seq_len": L, "dim": D, "parallelism": "single shard",
           "l2": "inputs larger than L2 (2.1 GB tile per step)"},
          {"unique_rows_per_step": u, "kernels_ms_per_step": phase_ms})


# ---------------------------------------------------------------------------
# C5
# ---------------------------------------------------------------------------

def _c5_lens(rng, rows, p=0.25, cap=64):
    lens = np.minimum(rng.geometric(p, rows), cap).astype(np.int64)
    u = rng.random(rows)
    lens[u < 0.10] = 0
    lens[u > 0.99] = cap
    return lens


def _c5_batch(k, Bn):
    """Host inputs of one C5 batch: per feature kind, ragged columns."""
    out = {"str": [], "flt": [], "cross": [], "raw": []}
    for i in range(200):
        rng = np.random.Generator(np.random.PCG64([5000 + i, k]))
        if 40 <= i < 60:  # cross of two short id columns (mean crossed bag ~ the others')
            la, lb = _c5_lens(rng, Bn, 0.5, 8), _c5_lens(rng, Bn, 0.5, 8)
            oa, ob = np.zeros(Bn + 1, np.int64), np.zeros(Bn + 1, np.int64)
            np.cumsum(la, out=oa[1:])
            np.cumsum(lb, out=ob[1:])
            out["cross"].append((rng.integers(0, 1_000_000, oa[-1]), oa, rng.integers(0, 1_000_000, ob[-1]), ob))
            continue
        lens = _c5_lens(rng, Bn)
        o = np.zeros(Bn + 1, np.int64)
        np.cumsum(lens, out=o[1:])
        m = int(o[-1])
        if i < 20:
            tok = rng.integers(0, 1_000_000, m).astype("S7")  # b"123456" style byte strings
            ln = np.char.str_len(tok).astype(np.int64)
            so = np.zeros(m + 1, np.int64)
            np.cumsum(ln, out=so[1:])
            raw = tok.view(np.uint8).reshape(m, 7)
            blob = raw[np.arange(7)[None, :] < ln[:, None]]
            out["str"].append((blob, so, o))
        elif i < 40:
            out["flt"].append((rng.random(m, dtype=np.float32), o))
        else:
            out["raw"].append((rng.integers(0, 1_000_000, m), o))
    return out


def c5(args):
    import torch
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200.hashing import fnv1a64_packed
    Bn = 16384
    kinds = ["str"] * 20 + ["flt"] * 20 + ["cross"] * 20 + ["raw"] * 140
    members = {d: [f"f{i}" for i in range(200) if DIMS5[i % 5] == d] for d in DIMS5}
    # warm (default): every key the stream can produce is admitted before timing
    # (36M rows per table, 109 GB of rows in all; the arena keeps headroom for
    # the positions of the steps in flight — the host's no-sync admission
    # bound — else every step would synchronize to refresh the counters);
    # --cold: tables start empty
    # with rows pre-reserved (no growth copies), admission in every step
    lts = {d: skb.LogicalTable(f"dim{d}", d, 1, seed=0, members=members[d], namespaced=True,
                               capacity_hint=24_000_000 if args.cold else int(os.environ.get("SKB_C5_HINT", 45_000_000))) for d in DIMS5}
    for lt_ in lts.values():
        skb.set_fold_mode(lt_, args.fold)
    # per-table kernel overrides for A/B runs: SKB_C5_VARIANTS="8:1:-1/16:2:-1" (dim:adam:pool)
    for spec in filter(None, os.environ.get("SKB_C5_VARIANTS", "").split("/")):
        d_, a_, p_ = (int(x) for x in spec.split(":"))
        skb.set_variants(lts[d_], a_, p_)
    prepop_s = None
    if not args.cold:
        t0 = time.perf_counter()
        raw = torch.arange(1_000_000, dtype=torch.int64, device="cuda")
        tok = np.arange(1_000_000).astype("S7")
        ln = np.char.str_len(tok).astype(np.int64)
        so = np.zeros(len(tok) + 1, np.int64)
        np.cumsum(ln, out=so[1:])
        blob = tok.view(np.uint8).reshape(-1, 7)[np.arange(7)[None, :] < ln[:, None]]
        space = {"str": fnv1a64_packed(torch.from_numpy(blob).cuda(), torch.from_numpy(so).cuda()),
                 "flt": torch.arange(11, dtype=torch.int64, device="cuda"),
                 "cross": torch.arange(1_000_003, dtype=torch.int64, device="cuda"), "raw": raw}
        for i in range(200):
            lt = lts[DIMS5[i % 5]]
            lt.local_table._admit_unique(lt.keys_for(f"f{i}", space[kinds[i]]), 0)
        torch.cuda.synchronize()
        for lt in lts.values():
            lt.num_rows  # exact counters on the host (the growth bound starts from them)
        prepop_s = time.perf_counter() - t0
    edges = np.linspace(0.05, 0.95, 10, dtype=np.float32)
    bplan = skb.FusedPlan.for_bucketize([edges] * 20)
    mplan = skb.FusedPlan.for_mod([1_000_003] * 20)
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    P = 2
    t0 = time.perf_counter()
    host = [_c5_batch(k, Bn) for k in range(P)]
    gen_s = time.perf_counter() - t0

    def dev(b):
        d = {}
        blob = np.concatenate([x[0] for x in b["str"]])
        so, base = [], 0
        nstr = []
        for x in b["str"]:
            so.append(x[1][:-1] + base)
            base += int(x[1][-1])
            nstr.append(len(x[1]) - 1)
        so.append(np.array([base], np.int64))
        d["blob"] = torch.from_numpy(blob).cuda()
        d["so"] = torch.from_numpy(np.concatenate(so)).cuda()
        d["nstr"] = nstr
        d["str_offs"] = [torch.from_numpy(x[2]).cuda() for x in b["str"]]
        d["flt"] = [skb.RaggedTensor(torch.from_numpy(v).cuda(), torch.from_numpy(o).cuda()) for v, o in b["flt"]]
        d["cross"] = [(skb.RaggedTensor(torch.from_numpy(a).cuda(), torch.from_numpy(oa).cuda()),
                       skb.RaggedTensor(torch.from_numpy(c).cuda(), torch.from_numpy(ob).cuda()))
                      for a, oa, c, ob in b["cross"]]
        d["raw"] = [(torch.from_numpy(v).cuda(), torch.from_numpy(o).cuda()) for v, o in b["raw"]]
        d["cross_sizes"] = [int((np.diff(oa) * np.diff(ob)).sum()) for _, oa, _, ob in b["cross"]]
        return d

    devs = [dev(b) for b in host]
    grads = {}
    step = [0]
    stats = {}

    def features(d):
        """feature engine -> (ids, offsets) per feature index 0..199"""
        cols = [None] * 200
        h = fnv1a64_packed(d["blob"], d["so"])  # 20 string columns in one launch
        base = 0
        for j in range(20):
            cols[j] = (h[base:base + d["nstr"][j]], d["str_offs"][j])
            base += d["nstr"][j]
        for j, r in enumerate(skb.fused_bucketize(bplan, d["flt"])):
            cols[20 + j] = (r.values, r.row_offsets)
        # sizes from the host-side offsets the input pipeline holds: no sync in the step
        crossed = skb.cross_many(d["cross"], sizes=d["cross_sizes"])
        for j, r in enumerate(skb.fused_mod(mplan, crossed)):
            cols[40 + j] = (r.values, r.row_offsets)
        for j, (v, o) in enumerate(d["raw"]):
            cols[60 + j] = (v, o)
        return cols

    def build(k):
        """feature engine + one packed batch per table for step k"""
        cols = features(devs[k % P])
        out = {}
        for di, dd in enumerate(DIMS5):
            idx = [i for i in range(200) if i % 5 == di]
            out[dd] = skb.PackedBatch(lts[dd], members[dd], [cols[i][0] for i in idx], [cols[i][1] for i in idx])
        return out

    pending = {}
    # default priority: at high priority (like the tables' index streams) the
    # feature engine of step k+1 ran under step k's fold+Adam, but the step
    # was no faster (6.36 vs 6.28 ms): the kernels it overlapped slowed down
    side = torch.cuda.Stream()
    watch = _Watch() if os.environ.get("SKB_C5_WATCH") else None
    if watch:
        _build = build

        def build(k):  # noqa: F811
            with watch:
                return _build(k)
    host_t = []  # host seconds per step: (forward calls, backward calls, build, prefetch)

    def run(count, marks=None):
        # cross-step pipeline: step k's forward AND backward are enqueued first
        # (several ms of device work), then the host builds step k+1 (feature
        # engine launches, packed batches) and issues its index phase (probe,
        # admission, sort; per table on its high-priority index stream), which
        # runs underneath the fold+Adam of step k — the host's per-step work
        # hides behind the device's instead of leaving it idle
        first = step[0] + 1
        if first not in pending:
            pending[first] = build(first)
            for dd in DIMS5:
                skb.prefetch(lts[dd], pending[first][dd], first, "mean")
        for _ in range(count):
            step[0] += 1
            k = step[0]
            tp = time.perf_counter()
            cur = pending.pop(k)
            per = {}
            main = torch.cuda.current_stream()
            for dd in DIMS5:
                batch = cur[dd]
                key = (dd, batch.num_bags)
                if key not in grads:
                    grads[key] = torch.randn((batch.num_bags, dd), device="cuda") * 1e-2
                per[dd] = (batch.num_ids, batch.num_bags)
                skb.lookup_pool(lts[dd], batch, k, "mean")
            tf = time.perf_counter()
            for dd in DIMS5:
                skb.pool_grad_adam(lts[dd], grads[(dd, cur[dd].num_bags)], cfg, k)
            tb = time.perf_counter()
            if marks is not None:
                marks.append(_events()[0])
                marks[-1].record()
            # step k+1's feature engine and packed batches depend only on its
            # inputs: on a side stream they run under step k's backward instead
            # of queueing behind it (the prefetch orders itself after them)
            with torch.cuda.stream(side):
                nxt = build(k + 1)
                for b in nxt.values():  # read later on the compute stream
                    b.ids.record_stream(main)
                    b.bag_offs.record_stream(main)
                tn = time.perf_counter()
                for dd in DIMS5:
                    skb.prefetch(lts[dd], nxt[dd], k + 1, "mean")
            pending[k + 1] = nxt
            host_t.append((tf - tp, tb - tf, tn - tb, time.perf_counter() - tn))
            stats["per"] = per
        torch.cuda.current_stream().wait_stream(side)  # the last step's build counts in the timed region

    # the feature engine's data checks (bucketize NaN) are read once per run
    # instead of once per call: no host synchronisation inside a step
    with skb.deferred_checks():
        warm_run = _settle(run, max(args.warmup, 3))
    torch.cuda.synchronize()
    marks = []

    def timed_run(count):
        # one event per step boundary on the compute stream: the per-step
        # spread (a slow step shows as an outlier, not as a shifted mean)
        marks.append(_events()[0])
        marks[-1].record()
        run(count, marks)

    wall_s = []

    def timed_run(count, _inner=timed_run):
        w0 = time.perf_counter()
        _inner(count)
        torch.cuda.synchronize()
        wall_s.append(time.perf_counter() - w0)

    m0 = torch.cuda.memory_stats()
    with skb.deferred_checks():
        ms = _timed(timed_run, args.steps)
    wall = wall_s[0] / args.steps * 1e3
    m1 = torch.cuda.memory_stats()
    alloc = {k: m1.get(k, 0) - m0.get(k, 0) for k in ("num_alloc_retries", "num_device_alloc", "num_device_free",
                                                      "num_sync_all_streams")}
    alloc["reserved_gb"] = m1.get("reserved_bytes.all.current", 0) / 2**30
    alloc["free_gb"] = torch.cuda.mem_get_info()[0] / 2**30
    steps_ms = [a.elapsed_time(b) for a, b in zip(marks[:-1], marks[1:])]
    ht = host_t[-args.steps:]
    host_ms = {nm: statistics.median(x[i] for x in ht) * 1e3 for i, nm in enumerate(("forward", "backward", "build",
                                                                                        "prefetch"))}
    with skb.deferred_checks():
        B.maybe_trace("c5", lambda: run(3))
    per = stats["per"]
    n, g = sum(v[0] for v in per.values()), sum(v[1] for v in per.values())
    sb = 0
    per_table = {}
    for dd in DIMS5:
        u, unew = skb.last_step_stats(lts[dd])
        sb += B.step_bytes(per[dd][0], per[dd][1], u, unew, dd)
        per_table[f"dim{dd}"] = {"ids": per[dd][0], "bags": per[dd][1], "unique": u, "new": unew}

    cpu = None
    if not args.no_cpu_baseline:
        from oracle import sparse_oracle as O
        cb = 256
        hb = _c5_batch(0, cb)
        olts = {d: O.OracleLogical(f"dim{d}", d, 1, seed=0, members=members[d], namespaced=True) for d in DIMS5}

        def one(k):
            cols = [None] * 200
            for j, (blob, so, o) in enumerate(hb["str"]):
                strs = [bytes(blob[so[q]:so[q + 1]]) for q in range(len(so) - 1)]
                cols[j] = (O.hash_strings(strs), o)
            for j, (v, o) in enumerate(hb["flt"]):
                cols[20 + j] = (O.bucketize_values(v, edges), o)
            for j, (a, oa, c, ob) in enumerate(hb["cross"]):
                cv, co = O.cross_rows(a, oa, c, ob)
                cols[40 + j] = (O.floor_mod(cv, 1_000_003), co)
            for j, (v, o) in enumerate(hb["raw"]):
                cols[60 + j] = (v, o)
            for di, dd in enumerate(DIMS5):
                idx = [i for i in range(200) if i % 5 == di]
                keys = np.concatenate([olts[dd].keys_for(f"f{i}", cols[i][0]) for i in idx])
                rows_ = O.lookup(olts[dd], keys, k)
                grads_ = []
                base = 0
                for i in idx:
                    o = cols[i][1]
                    m = int(o[-1])
                    O.pool(rows_[base:base + m], o, "mean")
                    dpo = np.full((len(o) - 1, dd), 1e-3, np.float32)
                    lens = np.diff(o)
                    per = np.repeat(dpo / np.maximum(lens, 1)[:, None].astype(np.float32), lens, axis=0)
                    grads_.append(per.astype(np.float32))
                    base += m
                O.grad_update(olts[dd], keys, np.concatenate(grads_), k, lr=1e-3, weight_decay=0.01,
                              variant="adamw")

        sec, cores = _cpu(one, "", steps=2, warm=1)
        ncpu = sum(int(o[-1]) for o in [x[2] for x in hb["str"]] + [x[1] for x in hb["flt"]] +
                   [x[1] for x in hb["raw"]])
        ncpu += sum(int((np.diff(oa) * np.diff(ob)).sum()) for _, oa, _, ob in hb["cross"])
        cpu = {"value": ncpu / sec, "unit": "IDs/s", "cores": 1, "kind": "port",
               "sample": f"C5 scaled to batch {cb} ({ncpu} ids/step incl. feature engine), 2 steps median; "
                         f"effective cores {cores}"}
    _line(args, "c5", n / (ms / 1e3), ms, n, Bn, sb, cpu,
          {"workload": "C5: 200 features (dims 8-128 -> 5 merged namespaced tables), batch 16384, mean "
                       "combiner, geometric(.25) bags capped at 64 (10% empty, 1% at 64); feature engine in "
                       "the step: 20 hash_feature, 20 fused bucketize, 20 cross + fused mod, 140 raw id columns",
           "global_batch": Bn, "features": 200, "dims": list(DIMS5), "parallelism": "single shard",
           "l2": "inputs larger than L2"},
          {"bags_per_step": g, "host_wall_ms_per_step": wall, "host_batch_gen_s": gen_s,
           "step_ms": {"median": statistics.median(steps_ms), "min": min(steps_ms), "max": max(steps_ms)},
           "host_issue_ms": host_ms, "torch_alloc_in_timed": alloc, "warmup_steps_run": warm_run,
           "per_table": per_table,
           "worst_step": _worst(steps_ms, ht),
           "table_rows": {f"dim{d}": int(lts[d].num_rows) for d in DIMS5}, "prepopulate_s": prepop_s,
           "arena_rows": {f"dim{d}": int(lts[d].local_table._h.stats()[4]) for d in DIMS5},
           "state": "cold (growing)" if args.cold else "warm (all stream keys admitted)"})


def run_config(args):
    import os
    import torch
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"workload_key": args.workload, "unavailable": "one-GPU config leg"}))
        return
    torch.cuda.set_device(0)
    {"c1": c1, "c3": c3, "c4": c4, "c5": c5}[args.workload](args)
