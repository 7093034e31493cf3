#!/usr/bin/env python
"""bench.py — sparse-step throughput of the B200 hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1], SURVEY §8d "C2"): Criteo-shape DLRM
sparse step — 26 sparse features C0..C25 of dim 64 merged into one
namespaced logical table `dim64`, batch 65,536 per GPU, bag length 1 (sum
combiner), ids uniform in [0, 1e6) per feature, SparseAdamW (lr 1e-3, wd
0.01).  Warm steady state: the table is pre-populated with all 26M keys
before timing (the stream's limit), so a step is probe + gather + pool +
grad fold + AdamW on ~1.65M unique rows.  Synthetic data; the pooled
gradient (the dense tower's output) is a resident N(0, 1e-2) tensor.

One "step" = lookup_pool (keys_for + dedup/admission + gather + pooling)
+ pool_grad_adam (ordered grad fold + AdamW) for one batch.

Arms
  default           our sm_100a path; prints the JSON line (rank 0).
  --impl reference  the reference algorithm's CPU implementation (the
                    oracle port — the reference is Python; it cannot be
                    compiled) on this host's cores, same metric/config, each
                    step a bounded sample (batch 4096 per feature).
Multi-GPU (torchrun, N > 1): weak scaling — every rank runs its own batch of
65,536 samples through the row-sharded logical table (one shard per GPU,
NCCL all-to-all exchange; paper_2509_20883_b200/distributed.py).
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-step IDs/sec & samples/sec at 1/2/4/8 B200; % HBM roofline vs CPU ref"
F_FEATURES, DIM, BATCH, ID_SPACE = 26, 64, 65536, 1_000_000
CPU_SAMPLE_BATCH = 4096
PHASES = ("probe", "miss", "pool", "sort", "fold_adam")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--batch", type=int, default=BATCH)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cold", action="store_true", help="do not pre-populate the table")
    p.add_argument("--no-pipeline", action="store_true", help="no cross-step prefetch of the index phase")
    p.add_argument("--prefetch-late", action="store_true",
                   help="issue step k+1's index phase after step k's pool (default: before it)")
    p.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                   help="c2 (default) is the headline line; c1/c3/c4/c5 measure SURVEY §8d's other configs "
                        "on one GPU (their own JSON line each, not the headline)")
    p.add_argument("--fold", default="exact", choices=["exact", "tree"],
                   help="hot-id gradient fold: exact np.add.at order (default) or the opt-in tolerance-mode tree "
                        "(c3/c4/c5 legs)")
    p.add_argument("--c3-rows", type=float, default=1.25e8,
                   help="c3: grow the shard to this many rows (1e9 rows / 8 GPUs per GPU)")
    return p.parse_args()


# ---------------------------------------------------------------------------
# synthetic inputs (host, numpy PCG64 — identical for both arms)
# ---------------------------------------------------------------------------

def make_batch(rank: int, k: int, batch: int):
    """ids per feature for batch k of rank r: integers(0, 1e6), seed 100+f."""
    ids = []
    for f in range(F_FEATURES):
        rng = np.random.Generator(np.random.PCG64([100 + f, rank, k]))
        ids.append(rng.integers(0, ID_SPACE, batch, dtype=np.int64))
    return ids


def members():
    return [f"C{f}" for f in range(F_FEATURES)]


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# Python garbage-collector pauses in the timed region
# ---------------------------------------------------------------------------

class GcPauses:
    """Records every collector pass (generation, ms) while active.  A full
    (generation 2) pass walks every live container object — with torch
    imported that is ~0.5M objects, tens of ms — and the host issuing the
    step stops for that long, so the device drains its queue and idles.
    `freeze()` (the default; SKB_BENCH_GC_FREEZE=0 turns it off) does what a
    long-running trainer does once its setup is done: one full collection,
    then gc.freeze() moves the survivors to the permanent generation, so
    later passes only walk the step's own short-lived objects."""

    def __init__(self):
        self.passes = []
        self._t0 = None

    def _cb(self, phase, info):
        if phase == "start":
            self._t0 = time.perf_counter()
        elif self._t0 is not None:
            self.passes.append((info.get("generation", -1), (time.perf_counter() - self._t0) * 1e3))
            self._t0 = None

    def __enter__(self):
        gc.callbacks.append(self._cb)
        return self

    def __exit__(self, *a):
        gc.callbacks.remove(self._cb)

    @staticmethod
    def freeze() -> bool:
        if os.environ.get("SKB_BENCH_GC_FREEZE", "1") == "0":
            return False
        gc.collect()
        gc.freeze()
        return True

    def summary(self):
        return {"frozen": gc.get_freeze_count() > 0, "passes": len(self.passes),
                "full_passes": sum(1 for g, _ in self.passes if g == 2),
                "max_ms": round(max((d for _, d in self.passes), default=0.0), 3),
                "total_ms": round(sum(d for _, d in self.passes), 3)}


# ---------------------------------------------------------------------------
# algorithmic bytes (SURVEY §8d convention)
# ---------------------------------------------------------------------------

def maybe_trace(tag, fn):
    """SKB_TRACE=<dir>: after the timed region, run fn() (a few more steps)
    under torch.profiler (CUPTI kernel timeline) and write
    <dir>/trace_<tag>.json (Chrome trace) for per-stream busy time and gaps
    (scripts/trace_gaps.py).  Never part of a reported number."""
    d = os.environ.get("SKB_TRACE")
    if not d:
        return
    import torch
    from torch.profiler import ProfilerActivity, profile
    os.makedirs(d, exist_ok=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        fn()
        torch.cuda.synchronize()
    p.export_chrome_trace(os.path.join(d, f"trace_{tag}.json"))


def phase_bytes(n, g, u, unew, d, mode_mean=False):
    """Algorithmic minimum bytes per launch of each fused phase."""
    return {
        # ids read, IDMap probe (16 B entry), slot written, miss flag
        "probe": 8 * n + 16 * n + 4 * n + n,
        # admission of unew rows: IDMap insert + w/m/v init write + metadata
        "miss": unew * (16 + 12 * d + 8 * 3 + 1),
        # slot read, one row gather per position, bag offsets, pooled write, bag-of-position write
        "pool": 4 * n + 4 * d * n + 8 * (g + 1) + 4 * d * g + 4 * n + 8 * u,
        # stable sort of (slot, bag) u32 pairs: read + write once, run heads
        "sort": 16 * n + 4 * u,
        # sorted pairs + heads read, dpooled row per position, w/m/v read + write
        "fold_adam": 8 * n + 4 * u + 4 * d * n + (16 * n if mode_mean else 0) + 24 * d * u,
    }


def step_bytes(n, g, u, unew, d):
    """B_step = 8N + 24U + 28D·U + 8D·G' + 16(G+1) + Unew·(16+12D)."""
    return 8 * n + 24 * u + 28 * d * u + 8 * d * g + 16 * (g + 1) + unew * (16 + 12 * d)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# CPU reference (oracle port; only the cpu_baseline / --impl reference legs)
# ---------------------------------------------------------------------------

def cpu_reference_steps(steps: int, warmup: int, batch: int, rank: int = 0):
    """train.py call sequence on the oracle port: keys_for -> lookup ->
    segment_reduce(sum) -> per-row grads -> grad_update (SparseAdamW)."""
    from oracle import sparse_oracle as O
    mem = members()
    olt = O.OracleLogical("dim64", DIM, 1, seed=0, members=mem, namespaced=True)
    batches = [make_batch(rank, k, batch) for k in range(max(2, min(steps, 4)))]
    dps = [np.random.Generator(np.random.PCG64(7 + k)).normal(0, 1e-2, (F_FEATURES * batch, DIM)).astype(np.float32)
           for k in range(len(batches))]
    offs = np.arange(batch + 1, dtype=np.int64)

    def one(step, k):
        ids = batches[k % len(batches)]
        keys = np.concatenate([olt.keys_for(m, x) for m, x in zip(mem, ids)])
        rows = O.lookup(olt, keys, step)
        for f in range(F_FEATURES):
            O.pool(rows[f * batch:(f + 1) * batch], offs, "sum")
        grads = dps[k % len(dps)]  # bag length 1, sum: per-row grad = dpooled row
        O.grad_update(olt, keys, grads, step, lr=1e-3, weight_decay=0.01, variant="adamw")

    # warm the table with every sample batch first (warm steady state, like the GPU arm)
    for k in range(len(batches)):
        one(k + 1, k)
    for w in range(warmup):
        one(len(batches) + 1 + w, w)
    times = []
    c0 = time.process_time()
    w0 = time.perf_counter()
    for s in range(steps):
        t0 = time.perf_counter()
        one(len(batches) + warmup + 1 + s, s)
        times.append(time.perf_counter() - t0)
    wall = time.perf_counter() - w0
    cores = (time.process_time() - c0) / wall if wall > 0 else 1.0
    n = F_FEATURES * batch
    med = statistics.median(times)
    return {"ids_per_s": n / med, "samples_per_s": batch / med, "ms_per_step": med * 1e3, "steps": steps,
            "ids_per_step": n, "effective_cores": round(cores, 2)}


def host_info():
    """What the CPU numbers ran on."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except AttributeError:
        affinity = os.cpu_count() or 1
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity_cores": affinity, "numpy": np.__version__}


def _cpu_worker(a):
    wid, steps, warmup, batch, barrier, out = a
    import time as _t
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[wid % len(os.sched_getaffinity(0))]})
    except (AttributeError, OSError):
        pass
    barrier.wait()
    t0 = _t.perf_counter()
    r = cpu_reference_steps(steps, warmup, batch, rank=wid)
    out.put((wid, r, t0, _t.perf_counter()))


def cpu_reference_parallel(steps: int, warmup: int, batch: int, procs: int):
    """`procs` independent replicas of the oracle's train.py step, one
    process per host core (the reference is numpy + the GIL: its only
    parallelism is a per-shard thread pool, sharding.py:222-227, so one
    process per core is the most it can use).  Each replica owns its own
    table and its own sample batches (rank-seeded); aggregate = total ids of
    the timed steps / the slowest replica's timed time."""
    import multiprocessing as mp
    if procs <= 1:
        r = cpu_reference_steps(steps, warmup, batch)
        return r, 1
    ctx = mp.get_context("fork")
    barrier, out = ctx.Barrier(procs), ctx.Queue()
    ps = [ctx.Process(target=_cpu_worker, args=((w, steps, warmup, batch, barrier, out),)) for w in range(procs)]
    for p in ps:
        p.start()
    res = [out.get() for _ in ps]
    for p in ps:
        p.join()
    per = [r for _, r, _, _ in res]
    slowest = max(r["ms_per_step"] for r in per)
    agg = sum(r["ids_per_step"] for r in per) / (slowest / 1e3)
    return {"ids_per_s": agg, "samples_per_s": agg / F_FEATURES, "ms_per_step": slowest, "steps": steps,
            "ids_per_step": sum(r["ids_per_step"] for r in per),
            "effective_cores": round(sum(r["effective_cores"] for r in per), 2),
            "per_process_ids_per_s": [round(r["ids_per_s"]) for r in per]}, procs


def cpu_procs() -> int:
    env = os.environ.get("BENCH_CPU_PROCS")
    if env:
        return max(1, int(env))
    return max(1, min(host_info()["affinity_cores"], 64))


def cpu_baseline_line(steps, warmup):
    procs = cpu_procs()
    r, procs = cpu_reference_parallel(steps, warmup, CPU_SAMPLE_BATCH, procs)
    sample = (f"C2 at batch {CPU_SAMPLE_BATCH}/feature ({F_FEATURES * CPU_SAMPLE_BATCH} ids per replica-step), "
              f"warm tables; {procs} independent oracle-port replicas, one process per core, each {steps} timed "
              f"steps after {warmup} warm-up; value = all replicas' ids / the slowest replica's median step")
    return r, {"value": r["ids_per_s"], "unit": "IDs/s", "cores": procs, "kind": "port", "sample": sample,
               "effective_cores": r["effective_cores"], **host_info()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = max(1, min(args.steps, 5))
    warm = min(args.warmup, 5)  # each step ~0.35 s: the whole arm stays within seconds
    r, cpu = cpu_baseline_line(steps, warm)
    line = {"metric": METRIC, "value": r["ids_per_s"], "unit": "IDs/s", "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 Criteo-shape: 26 x dim64, uniform ids, sum, SparseAdamW (warm)",
                       "global_batch": CPU_SAMPLE_BATCH * cpu["cores"], "per_process_batch": CPU_SAMPLE_BATCH,
                       "features": F_FEATURES, "dim": DIM},
            "impl": "reference", "samples_per_s": r["samples_per_s"], "cpu_baseline": cpu,
            "e2e": {"value": r["ids_per_s"], "unit": "IDs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200 import _native as N

    B = args.batch
    mem = members()
    n_ids = F_FEATURES * B
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    # capacity: the 26M rows plus four steps of positions — the host's no-sync
    # admission bound counts every in-flight position as a possible new row;
    # with less slack every prefetch waits for the previous index phase's
    # counter snapshot (a host sync per step)
    lt = skb.LogicalTable("dim64", DIM, 1, seed=0, members=mem, namespaced=True,
                          capacity_hint=(F_FEATURES * ID_SPACE + 4 * F_FEATURES * B) if not args.cold else 0)
    table = lt.local_table

    # warm steady state: every key of the stream admitted before timing
    prepop_ms = None
    if not args.cold:
        t0 = time.perf_counter()
        all_ids = torch.arange(ID_SPACE, dtype=torch.int64, device="cuda")
        for m in mem:
            table._admit_unique(lt.keys_for(m, all_ids), 0)
        torch.cuda.synchronize()
        prepop_ms = (time.perf_counter() - t0) * 1e3
        del all_ids

    # P rotating batches (host pinned + device resident) and resident dpooled
    P = 4
    offs = [np.arange(B + 1, dtype=np.int64)] * F_FEATURES
    host_batches, dev_batches, dps = [], [], []
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234 + rank)
    for k in range(P):
        ids = make_batch(rank, k, B)
        batch = skb.PackedBatch(lt, mem, ids, offs)
        dev_batches.append(batch)
        host_batches.append((torch.from_numpy(batch.ids.cpu().numpy()).pin_memory(),
                             torch.from_numpy(batch.bag_offs.cpu().numpy()).pin_memory()))
        dps.append(torch.empty((batch.num_bags, DIM), device="cuda").normal_(0.0, 1e-2, generator=gen))
    G = dev_batches[0].num_bags
    pooled = torch.empty((G, DIM), device="cuda")
    # two device batch buffers refilled from pinned host memory in the e2e arm
    e2e_batches = [skb.PackedBatch(lt, mem, make_batch(rank, 0, B), offs) for _ in range(3)]
    copy_stream = torch.cuda.Stream()
    buf_free = [torch.cuda.Event() for _ in range(3)]
    stats_host = torch.empty((args.steps, 4), dtype=torch.int64).pin_memory()
    step_no = [0]

    def run_steps(get, count, after_backward=None, before_step=None, input_stream=None):
        """`count` pipelined steps: the index phase (probe, admission, sort) of
        step k+1 is prefetched before the pool of step k, so it runs on the
        table's index stream underneath step k's pool and fold+Adam.
        `input_stream`: the stream the step's inputs arrive on (the prefetch
        orders itself after that stream instead of the compute stream)."""
        first = step_no[0] + 1

        def pre(k):
            if input_stream is None:
                skb.prefetch(lt, get(k)[0], first + k, "sum")
            else:
                with torch.cuda.stream(input_stream):
                    skb.prefetch(lt, get(k)[0], first + k, "sum")

        if not args.no_pipeline:
            pre(0)
        pipelined = not args.no_pipeline
        for k in range(count):
            batch, dp = get(k)
            if pipelined and not args.prefetch_late and k + 1 < count:
                pre(k + 1)
                if before_step:  # after the prefetch: it must not queue behind later copies
                    before_step(k)
            skb.lookup_pool(lt, batch, first + k, "sum", out=pooled)
            if pipelined and args.prefetch_late and k + 1 < count:
                pre(k + 1)
            if before_step and (args.prefetch_late or not pipelined or k + 1 >= count):
                before_step(k)
            skb.pool_grad_adam(lt, dp, cfg, first + k)
            if after_backward:
                after_backward(k)
        step_no[0] += count

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clk = ClockSampler(local).__enter__()
    t_wait = time.perf_counter()
    while not clk.rows and time.perf_counter() - t_wait < 5.0:
        time.sleep(0.02)
    run_steps(lambda k: (dev_batches[k % P], dps[k % P]), args.warmup)
    barrier()
    # untimed soak so clocks settle and the sampler sees the GPU under load
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 0.4:
        run_steps(lambda k: (dev_batches[k % P], dps[k % P]), 8)
        barrier()
    u_touched, u_new = skb.last_step_stats(lt)

    # ---- timed region: inputs resident in HBM --------------------------------
    lib = N.lib()
    N.call("skb_fused_profile", table.handle, args.steps, N.stream_ptr())
    launches0 = lib.skb_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/: the timed steps' kernels only
    run_steps(lambda k: (dev_batches[k % P], dps[k % P]), args.steps)
    torch.cuda.nvtx.range_pop()
    ev1.record()
    barrier()
    launches = lib.skb_launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    phase_ms = {}
    buf = (ctypes.c_float * args.steps)()
    for p, name in enumerate(PHASES):
        cnt = ctypes.c_int64()
        N.call("skb_fused_profile_read", table.handle, p, buf, args.steps, ctypes.byref(cnt))
        vals = list(buf)[: cnt.value]
        phase_ms[name] = sum(vals) / len(vals) if vals else 0.0
    N.call("skb_fused_profile", table.handle, 0, N.stream_ptr())
    maybe_trace("c2", lambda: run_steps(lambda k: (dev_batches[k % P], dps[k % P]), 6))
    u_touched, u_new = skb.last_step_stats(lt)

    # ---- e2e: public API with host buffers, H2D + result D2H inside ----------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    staged = {}

    copy_ev = []
    # H2D of step k's inputs from pinned host memory on a copy stream, two
    # steps ahead, into one of three device batch buffers; a buffer is
    # refilled only after the backward of the step that last read it.
    main_stream = torch.cuda.current_stream()

    def stage(k):
        if k >= args.steps or k in staged:
            return
        eb = e2e_batches[k % 3]
        copy_stream.wait_event(buf_free[k % 3])
        with torch.cuda.stream(copy_stream):
            hid, hoff = host_batches[k % P]
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(copy_stream)
            eb.ids.copy_(hid, non_blocking=True)
            eb.bag_offs.copy_(hoff, non_blocking=True)
            c1.record(copy_stream)
            copy_ev.append((c0, c1))
        staged[k] = eb

    def get_e2e(k):
        stage(k)
        return staged[k], dps[k % P]

    def before_step(k):
        # stage step k+2's inputs once step k+1's prefetch has been issued on
        # the copy stream (so that prefetch does not wait for this copy)
        stage(k + 2)

    stats_stream = torch.cuda.Stream()

    def after_e2e(k):
        buf_free[k % 3].record(main_stream)
        # the step's metrics (misses, new rows, unique rows) back to the host,
        # on a side stream: a copy on the compute stream delays the next
        # step's pool launch past the next index phase's probe (measured
        # ~40 us/step: the high-priority probe then takes the SMs first)
        with torch.cuda.stream(stats_stream):  # (the copy waits for the step's backward itself)
            N.call("skb_fused_stats_async", table.handle, ctypes.c_void_p(stats_host[k].data_ptr()), N.stream_ptr())

    # the compute stream sees the copied inputs through the prefetch's
    # ready event (index stream waited on the copy stream)
    w_e2e = time.perf_counter()
    if os.environ.get("SKB_TRACE"):  # diagnostic: the whole e2e loop under the kernel timeline
        maybe_trace("c2_e2e", lambda: run_steps(get_e2e, args.steps, after_e2e, before_step,
                                                input_stream=copy_stream))
    else:
        run_steps(get_e2e, args.steps, after_e2e, before_step, input_stream=copy_stream)
    host_e2e_ms = (time.perf_counter() - w_e2e) * 1e3 / args.steps  # host time to issue a step
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    h2d_ms = statistics.median(a.elapsed_time(b) for a, b in copy_ev) if copy_ev else None
    clk.__exit__(None, None, None)
    h2d = int(host_batches[0][0].numel() * 8 + host_batches[0][1].numel() * 8)

    # max over ranks
    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_total, e2e_ms = allmax(ms_total), allmax(e2e_ms)
    ms_step = ms_total / args.steps
    value = world * n_ids / (ms_step / 1e3)
    e2e_value = world * n_ids / (e2e_ms / args.steps / 1e3)

    peak, peak_kind = load_peaks()
    pb = phase_bytes(n_ids, G, u_touched, u_new, DIM)
    # dominant kernel = the phase moving the most algorithmic bytes (fold+Adam);
    # phase wall times overlap across the two streams, so not max(phase_ms)
    dom = max((k for k in phase_ms if k in pb), key=lambda k: pb[k])
    achieved = pb[dom] / (phase_ms[dom] / 1e3) / 1e9
    tr = load_traffic().get(dom, {})
    traffic = tr.get("dram_bytes_per_launch")
    traffic_src = (f"ncu --set full capture of {tr.get('kernel')} (profiles/ncu_summary.json, tag {tr.get('tag')}); "
                   "not measured in this run") if tr else None
    sb = step_bytes(n_ids, G, u_touched, u_new, DIM)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline_line(3, 0)[1]
        line = {
            "metric": METRIC, "value": value, "unit": "IDs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 Criteo-shape DLRM sparse step: 26 x dim64 merged table, uniform ids "
                                   "[0,1e6) per feature, bag length 1, sum, SparseAdamW, "
                                   + ("cold table" if args.cold else "warm table (26M rows pre-admitted)"),
                       "global_batch": B * world, "per_gpu_batch": B, "features": F_FEATURES, "dim": DIM,
                       "ids_per_step_per_gpu": n_ids, "table_rows": int(table.num_rows),
                       "parallelism": f"independent replicas x{world}" if world > 1 else "single shard",
                       "l2": "inputs larger than L2: 20 GB row arena + 4 rotating 0.46 GB batches"},
            "samples_per_s": world * B / (ms_step / 1e3),
            "unique_rows_per_step": u_touched, "new_rows_per_step": u_new,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_kind": peak_kind, "algorithmic_bytes": pb[dom]},
            "step_roofline": {"algorithmic_bytes": sb, "achieved": sb / (ms_step / 1e3) / 1e9,
                              "frac": sb / (ms_step / 1e3) / 1e9 / peak},
            "kernels_ms": phase_ms,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "IDs/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 32,
                    "host_issue_ms_per_step": host_e2e_ms,
                    "note": "each step's ids + bag offsets copied H2D from pinned host memory (copy stream, two "
                            "steps ahead) and the step's stats D2H; pooled / dpooled stay on the device (the "
                            "dense tower runs on the GPU)",
                    "h2d_ms_per_step": h2d_ms},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "prepopulate_ms": prepop_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_dist(args):
    """N > 1: weak scaling over the row-sharded table (one shard per GPU, NCCL
    all-to-all exchange of ids, rows and grads; distributed.DistSparseStep)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_DIST_BACKEND=gloo lets several ranks share one GPU (functional check only)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local if backend == "nccl" else 0
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200 import _native as N
    from paper_2509_20883_b200.distributed import DistSparseStep

    B, mem = args.batch, members()
    n_ids = F_FEATURES * B
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    per_rank = (F_FEATURES * ID_SPACE) // world
    lt = skb.LogicalTable("dim64", DIM, world, seed=0, members=mem, namespaced=True, dist=True,
                          capacity_hint=0 if args.cold else per_rank + per_rank // 10)
    table = lt.local_table
    if not args.cold:  # warm: each rank admits the keys it owns
        all_ids = torch.arange(ID_SPACE, dtype=torch.int64, device="cuda")
        plan = skb.ShardPlan(world)
        for m in mem:
            keys = lt.keys_for(m, all_ids)
            table._admit_unique(keys[plan.shard_of(keys) == rank].contiguous(), 0)
        torch.cuda.synchronize()
    P = 4
    offs = [np.arange(B + 1, dtype=np.int64)] * F_FEATURES
    batches, dps = [], []
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234 + rank)
    for k in range(P):
        b = skb.PackedBatch(lt, mem, make_batch(rank, k, B), offs)
        batches.append(b)
        dps.append(torch.empty((b.num_bags, DIM), device="cuda").normal_(0.0, 1e-2, generator=gen))
    # ids, rows and grads over peer memory (CUDA IPC windows, NVLink P2P
    # stores from the producing kernels); the owner side is the fused step
    stepper = DistSparseStep(lt)
    pooled = torch.empty((batches[0].num_bags, DIM), device="cuda")
    step_no = [0]

    def run(count):
        # cross-step pipeline: step k+1's requester prepare + count exchange
        # are enqueued between forward(k) and backward(k); the count readback
        # (the step's one host sync) happens in forward(k+1), under backward(k)
        for k in range(count):
            step_no[0] += 1
            t = step_no[0]
            if stepper._pre is None:
                stepper.prefetch(batches[t % P], t)
            stepper.forward(batches[t % P], t, "sum", out=pooled)
            if k + 1 < count:
                stepper.prefetch(batches[(t + 1) % P], t + 1)
            stepper.backward(dps[t % P], cfg, t)

    clk = ClockSampler(local).__enter__()
    run(args.warmup)
    dist.barrier()
    torch.cuda.synchronize()
    lib = N.lib()
    l0 = lib.skb_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    run(args.steps)
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    launches = lib.skb_launch_count() - l0
    # per-rank traffic of the last step: local unique rows U, owner rows U2,
    # bytes sent to peers per direction (ids + rows back + grads)
    ctx_counts = stepper.last_counts
    U = int(sum(ctx_counts["send"]))
    U2 = stepper.owner_unique()
    sent_remote = sum(c for j, c in enumerate(ctx_counts["send"]) if j != rank)
    recv_remote = sum(c for j, c in enumerate(ctx_counts["recv"]) if j != rank)
    xbytes = sent_remote * (8 + 4 * DIM) + recv_remote * 4 * DIM

    # e2e: each step's ids + offsets copied H2D from pinned host memory, the
    # step's pooled checksum row read back
    host = [(torch.from_numpy(b.ids.cpu().numpy()).pin_memory(),
             torch.from_numpy(b.bag_offs.cpu().numpy()).pin_memory()) for b in batches]
    e2e_b = [skb.PackedBatch(lt, mem, make_batch(rank, 0, B), offs) for _ in range(2)]
    res = torch.empty((args.steps, DIM), dtype=torch.float32).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        step_no[0] += 1
        eb = e2e_b[k % 2]
        eb.ids.copy_(host[k % P][0], non_blocking=True)
        eb.bag_offs.copy_(host[k % P][1], non_blocking=True)
        stepper.forward(eb, step_no[0], "sum", out=pooled)
        stepper.backward(dps[k % P], cfg, step_no[0])
        res[k].copy_(pooled[0], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk.__exit__(None, None, None)
    stepper.win.close_all()
    t = torch.tensor([ev0.elapsed_time(ev1), e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t[0].item()) / args.steps
    e2e_ms = float(t[1].item()) / args.steps
    if rank == 0:
        peak, peak_kind = load_peaks()
        G = batches[0].num_bags
        sb = step_bytes(n_ids, G, U2, 0, DIM)
        h2d = int(host[0][0].numel() * 8 + host[0][1].numel() * 8)
        line = {
            "metric": METRIC, "value": world * n_ids / (ms_step / 1e3), "unit": "IDs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 Criteo-shape DLRM sparse step, row-sharded over GPUs: 26 x dim64, "
                                   "uniform ids [0,1e6) per feature, bag length 1, sum, SparseAdamW, warm",
                       "global_batch": B * world, "per_gpu_batch": B, "features": F_FEATURES, "dim": DIM,
                       "parallelism": f"row-sharded x{world}: ids, rows and grads stored into peers' IPC "
                                      "windows by the producing kernels (NVLink P2P); owner side = fused step",
                       "l2": "inputs larger than L2"},
            "samples_per_s": world * B / (ms_step / 1e3),
            "roofline": {"bound": "hbm", "kernel": "step (rank-0 local HBM bytes)", "achieved": sb / ms_step / 1e6,
                         "peak": peak, "unit": "GB/s", "frac": sb / ms_step / 1e6 / peak, "traffic": None,
                         "peak_kind": peak_kind, "algorithmic_bytes": sb},
            "exchange": {"bytes_per_step_per_direction": xbytes, "GB_per_s": xbytes / ms_step / 1e6,
                         "nvlink_peak_GB_per_s": 900.0, "local_unique": U, "owner_unique": U2},
            "cpu_baseline": None,
            "e2e": {"value": world * n_ids / (e2e_ms / 1e3), "unit": "IDs/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 4 * DIM},
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_threads(args):
    """BENCH_SHARED_GPU=1 with --gpus N on one GPU: the N ranks of the
    row-sharded step as N threads of this process (distributed.ThreadRanks),
    each with its own stream, table shard, windows and batch — the full
    multi-GPU protocol (P2P stores, stream-ordered peer barriers, one count
    readback per step) with every rank's kernels sharing one device.  A
    functional + protocol-overhead measurement, not an N-GPU number: the
    line's n_gpus is 1 and `emulated_ranks` says N."""
    import threading
    import torch
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200.distributed import DistSparseStep, ThreadRanks

    W, B, mem = args.gpus, args.batch, members()
    n_ids = F_FEATURES * B
    world = ThreadRanks(W)
    res = [None] * W
    errs = []
    start = threading.Barrier(W)
    torch.cuda.set_device(0)

    def body(rank):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                g = world.group(rank)
                per_rank = (F_FEATURES * ID_SPACE) // W
                lt = skb.LogicalTable("dim64", DIM, W, seed=0, members=mem, namespaced=True, dist=True, group=g,
                                      capacity_hint=0 if args.cold else per_rank + per_rank // 10)
                if not args.cold:
                    all_ids = torch.arange(ID_SPACE, dtype=torch.int64, device="cuda")
                    plan = skb.ShardPlan(W)
                    for m in mem:
                        keys = lt.keys_for(m, all_ids)
                        lt.local_table._admit_unique(keys[plan.shard_of(keys) == rank].contiguous(), 0)
                P = 4
                offs = [np.arange(B + 1, dtype=np.int64)] * F_FEATURES
                gen = torch.Generator(device="cuda")
                gen.manual_seed(1234 + rank)
                batches = [skb.PackedBatch(lt, mem, make_batch(rank, k, B), offs) for k in range(P)]
                dps = [torch.empty((b.num_bags, DIM), device="cuda").normal_(0.0, 1e-2, generator=gen)
                       for b in batches]
                stepper = DistSparseStep(lt)
                cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
                pooled = torch.empty((batches[0].num_bags, DIM), device="cuda")
                step_no = [0]

                def run(count):
                    for k in range(count):
                        step_no[0] += 1
                        t = step_no[0]
                        if stepper._pre is None:
                            stepper.prefetch(batches[t % P], t)
                        stepper.forward(batches[t % P], t, "sum", out=pooled)
                        if k + 1 < count:
                            stepper.prefetch(batches[(t + 1) % P], t + 1)
                        stepper.backward(dps[t % P], cfg, t)

                run(args.warmup)
                st.synchronize()
                start.wait()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                syncs0 = stepper.syncs
                w0 = time.perf_counter()
                e0.record(st)
                run(args.steps)
                e1.record(st)
                st.synchronize()
                wall = time.perf_counter() - w0
                if os.environ.get("SKB_TRACE"):  # every rank steps; rank 0 records the timeline
                    start.wait()
                    if rank == 0:
                        maybe_trace(f"n{W}_shared", lambda: run(4))
                    else:
                        run(4)
                        st.synchronize()
                res[rank] = {"ms": e0.elapsed_time(e1) / args.steps, "wall_ms": wall * 1e3 / args.steps,
                             "syncs_per_step": (stepper.syncs - syncs0) / args.steps,
                             "counts": stepper.last_counts, "owner_unique": stepper.owner_unique()}
                stepper.win.close_all()
        except BaseException as e:  # surface thread failures
            errs.append(repr(e))
            world._barrier.abort()
            start.abort()

    ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(W)]
    clk = ClockSampler(0).__enter__()
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    if any(t.is_alive() for t in ths):
        errs.append("thread ranks did not finish within 600 s")
    clk.__exit__(None, None, None)
    if errs:
        raise RuntimeError("; ".join(errs))
    ms = max(r["ms"] for r in res)
    line = {"metric": METRIC, "value": W * n_ids / (ms / 1e3), "unit": "IDs/s", "n_gpus": 1, "emulated_ranks": W,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"C2 row-sharded over {W} ranks emulated on ONE GPU (threads of one process): "
                                   "26 x dim64, uniform ids, bag length 1, sum, SparseAdamW, warm",
                       "per_rank_batch": B, "features": F_FEATURES, "dim": DIM,
                       "parallelism": f"row-sharded x{W} (ThreadRanks): P2P window stores, stream-ordered peer "
                                      "barriers, owner side = fused step"},
            "per_rank": res, "wall_ms_per_step": max(r["wall_ms"] for r in res),
            "clocks": clk.summary(), "gpu_launches": None}
    print(json.dumps(line), flush=True)


def launch_cmd(args_argv, n: int, port: int):
    """The torchrun command `bench.py --gpus N` re-executes itself under when
    it was started as a plain process (one rank per GPU, 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(args_argv)


def self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: spawn N ranks.  Needs N
    visible GPUs; BENCH_SHARED_GPU=1 runs the N ranks on one GPU with gloo
    control (a functional check of the multi-rank path, not a measurement)."""
    import socket
    import torch
    shared = os.environ.get("BENCH_SHARED_GPU") == "1"
    if shared and os.environ.get("BENCH_SHARED_PROCS") != "1":
        run_threads(args)  # ranks as threads of this process on one GPU
        return 0
    have = torch.cuda.device_count()
    if have < args.gpus and not shared:
        print(json.dumps({"metric": METRIC, "n_gpus": args.gpus, "error":
                          f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have} "
                          "(BENCH_SHARED_GPU=1 runs the ranks on one GPU for a functional check)"}), flush=True)
        return 2
    env = dict(os.environ)
    if shared:
        env["BENCH_DIST_BACKEND"] = "gloo"
    # communicator setup lines (one per rank) go to stderr: the JSON line stays alone on stdout
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    return subprocess.call(launch_cmd(sys.argv[1:], args.gpus, port), env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        sys.exit(self_launch(args))
    if args.workload != "c2":
        from bench_configs import run_config
        run_config(args)
    elif args.impl == "reference":
        run_reference(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_dist(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
