"""ids partition (Table 1: 1M ids, 8 shards) kernel breakdown under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_20883_b200 import _native as N
torch.cuda.set_device(0)
n = 1_000_000
rng = np.random.Generator(np.random.PCG64(0))
ids = torch.from_numpy(rng.integers(0, n, n, dtype=np.int64)).cuda()
uq = torch.empty(n, dtype=torch.int64, device="cuda")
cnt = torch.empty(8, dtype=torch.int64, device="cuda")
ish = torch.empty(n, dtype=torch.int64, device="cuda")
ipo = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(5):
    N.call("skb_unique_partition", N.ptr(ids), n, 8, N.ptr(uq), N.ptr(cnt), N.ptr(ish), N.ptr(ipo), N.stream_ptr())
torch.cuda.synchronize()
