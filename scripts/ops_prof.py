#!/usr/bin/env python
"""Run the Table-1 partition / gather / scatter operators a few times each so
an `ncu` launch list (or `--set full` capture) shows their per-kernel cost.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv python scripts/ops_prof.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200 import _native as N

    which = sys.argv[1:] or ["partition", "gather", "scatter"]
    torch.cuda.set_device(0)
    rng = np.random.Generator(np.random.PCG64(0))
    n = 1_000_000
    if "partition" in which:
        ids = torch.from_numpy(rng.integers(0, n, n, dtype=np.int64)).cuda()
        uq = torch.empty(n, dtype=torch.int64, device="cuda")
        cnt = torch.empty(8, dtype=torch.int64, device="cuda")
        ish = torch.empty(n, dtype=torch.int64, device="cuda")
        ipo = torch.empty(n, dtype=torch.int64, device="cuda")
        for _ in range(3):
            N.call("skb_unique_partition", N.ptr(ids), n, 8, N.ptr(uq), N.ptr(cnt), N.ptr(ish), N.ptr(ipo),
                   N.stream_ptr())
    D = 16
    if "gather" in which or "scatter" in which:
        table = skb.EmbeddingTable("bench", D, seed=0, capacity_hint=n)
        offsets = table.lookup_or_insert(torch.arange(n, dtype=torch.int64, device="cuda"), 1)
        gidx = offsets[torch.from_numpy(rng.integers(0, n, n)).cuda()]
        gout = torch.empty((n, D), device="cuda")
        sidx = offsets[torch.from_numpy(rng.permutation(n)).cuda()]
        newr = torch.from_numpy(rng.random((n, D), dtype=np.float32)).cuda()
        for _ in range(3):
            if "gather" in which:
                N.call("skb_table_gather", table.handle, N.ptr(gidx), n, N.ptr(gout), N.stream_ptr())
                N.call("skb_table_gather_unchecked", table.handle, N.ptr(gidx), n, N.ptr(gout), N.stream_ptr())
            if "scatter" in which:
                N.call("skb_table_scatter_update", table.handle, N.ptr(sidx), n, N.ptr(newr), N.stream_ptr())
                N.call("skb_table_write_rows", table.handle, N.ptr(sidx), n, 0, N.ptr(newr), N.stream_ptr())
    torch.cuda.synchronize()


if __name__ == "__main__" and not os.environ.get("OPS_TIMING"):
    main()


def timing():
    """Per-op: device time of one call (events around it, as ops_bench),
    back-to-back throughput of 50 calls, and host submission time."""
    import time
    import torch
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200 import _native as N
    torch.cuda.set_device(0)
    rng = np.random.Generator(np.random.PCG64(0))
    n, D = 1_000_000, 16
    ids = torch.from_numpy(rng.integers(0, n, n, dtype=np.int64)).cuda()
    uq, ish, ipo = (torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(3))
    cnt = torch.empty(8, dtype=torch.int64, device="cuda")
    table = skb.EmbeddingTable("bench", D, seed=0, capacity_hint=n)
    offsets = table.lookup_or_insert(torch.arange(n, dtype=torch.int64, device="cuda"), 1)
    gidx = offsets[torch.from_numpy(rng.integers(0, n, n)).cuda()]
    gout = torch.empty((n, D), device="cuda")
    sidx = offsets[torch.from_numpy(rng.permutation(n)).cuda()]
    newr = torch.from_numpy(rng.random((n, D), dtype=np.float32)).cuda()
    ops = {
        "partition": lambda: N.call("skb_unique_partition", N.ptr(ids), n, 8, N.ptr(uq), N.ptr(cnt), N.ptr(ish),
                                    N.ptr(ipo), N.stream_ptr()),
        "gather_checked": lambda: N.call("skb_table_gather", table.handle, N.ptr(gidx), n, N.ptr(gout),
                                         N.stream_ptr()),
        "gather": lambda: N.call("skb_table_gather_unchecked", table.handle, N.ptr(gidx), n, N.ptr(gout),
                                 N.stream_ptr()),
        "scatter_update": lambda: N.call("skb_table_scatter_update", table.handle, N.ptr(sidx), n, N.ptr(newr),
                                         N.stream_ptr()),
        "write_rows": lambda: N.call("skb_table_write_rows", table.handle, N.ptr(sidx), n, 0, N.ptr(newr),
                                     N.stream_ptr()),
        "noop_ctypes": lambda: N.call("skb_version") if False else None,
    }
    for name, fn in ops.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record()
        for _ in range(50):
            fn()
        h1 = time.perf_counter()
        e1.record(); torch.cuda.synchronize()
        print(f"{name:16s} single {np.median(ts):7.1f} us  back-to-back {e0.elapsed_time(e1) * 1e3 / 50:7.1f} us"
              f"  host submit {(h1 - h0) / 50 * 1e6:7.1f} us", flush=True)


if __name__ == "__main__" and os.environ.get("OPS_TIMING"):
    timing()
