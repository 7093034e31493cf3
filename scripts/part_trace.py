"""ids partition (Table 1: 1M ids, 8 shards): in-situ kernel times from a
CUPTI trace (L2 scrubbed before each call, as ops_bench does)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_20883_b200 import _native as N  # noqa: E402

torch.cuda.set_device(0)
n = int(os.environ.get("N", 1_000_000))
S = int(os.environ.get("S", 8))
rng = np.random.Generator(np.random.PCG64(0))
ids = torch.from_numpy(rng.integers(0, n, n, dtype=np.int64)).cuda()
uq = torch.empty(n, dtype=torch.int64, device="cuda")
cnt = torch.empty(S, dtype=torch.int64, device="cuda")
ish = torch.empty(n, dtype=torch.int64, device="cuda")
ipo = torch.empty(n, dtype=torch.int64, device="cuda")
scrub = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def call():
    N.call("skb_unique_partition", N.ptr(ids), n, S, N.ptr(uq), N.ptr(cnt), N.ptr(ish), N.ptr(ipo), N.stream_ptr())


for _ in range(5):
    call()
torch.cuda.synchronize()
ts = []
for r in range(20):
    scrub.fill_(r)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print("event us median", sorted(ts)[len(ts) // 2])
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for r in range(10):
        scrub.fill_(r)
        call()
    torch.cuda.synchronize()
tot = collections.defaultdict(list)
for e in prof.events():
    if e.device_type.name == "CUDA":
        tot[e.name[:60]].append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
for k, v in tot.items():
    print(f"{k:60s} n={len(v):3d} median {sorted(v)[len(v) // 2]:8.2f} us")
