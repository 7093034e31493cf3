"""cudaMalloc latency with and without large VMM-mapped tables resident
(diagnostics for the C5 host stalls).  Each sample frees the caching
allocator's cache first, so torch.empty reaches cudaMalloc."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")


def probe(tag):
    out = {}
    for mb in (2, 20, 64, 256):
        ts = []
        for _ in range(10):
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            t0 = time.perf_counter()
            x = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
            ts.append((time.perf_counter() - t0) * 1e3)
            del x
        out[mb] = (round(statistics.median(ts), 3), round(max(ts), 3))
    print(tag, "MB -> (median ms, max ms)", out, "free GB", round(torch.cuda.mem_get_info()[0] / 2**30, 1), flush=True)


torch.cuda.init()
probe("no tables")
import paper_2509_20883_b200 as skb  # noqa: E402

for hint in (5_000_000, 45_000_000):
    lts = [skb.LogicalTable(f"t{d}_{hint}", d, 1, seed=0, capacity_hint=hint) for d in (8, 16, 32, 64, 128)]
    torch.cuda.synchronize()
    probe(f"5 tables hint {hint}")
    # the same with the device busy (a long kernel queued): does cudaMalloc wait?
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    for _ in range(20):
        a.add_(1)
    t0 = time.perf_counter()
    x = torch.empty(48 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.empty_cache()
    y = torch.empty(50 << 20, dtype=torch.uint8, device="cuda")
    print("  alloc while busy ms", round((time.perf_counter() - t0) * 1e3, 3), flush=True)
    torch.cuda.synchronize()
    del a, x, y
    del lts
    import gc
    gc.collect()
    torch.cuda.synchronize()
