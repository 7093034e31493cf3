"""Long-run fold microbenchmark: grad_fold over n positions of which a
fraction belongs to one hot id (the rest distinct), dim D."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20883_b200 as skb
from paper_2509_20883_b200 import _native as N

n, D = int(float(os.environ.get("LF_N", 1e6))), int(os.environ.get("LF_D", 64))
hot = float(os.environ.get("LF_HOT", 1.0))
torch.cuda.set_device(0)
rng = np.random.default_rng(0)
inv = np.where(rng.random(n) < hot, 0, np.arange(1, n + 1)).astype(np.int64)
_, inv = np.unique(inv, return_inverse=True)
U = int(inv.max()) + 1
inv_d = torch.from_numpy(inv).cuda()
g = torch.randn((n, D), device="cuda")
out = torch.empty((U, D), device="cuda")
for _ in range(2):
    N.call("skb_grad_fold", N.ptr(g), n, D, N.ptr(inv_d), U, N.ptr(out), N.stream_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    N.call("skb_grad_fold", N.ptr(g), n, D, N.ptr(inv_d), U, N.ptr(out), N.stream_ptr())
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
hot_rows = int((inv == 0).sum())
print(f"grad_fold n={n} D={D} hot run={hot_rows}: {ms:.3f} ms, hot-run bytes/ms = {hot_rows * D * 4 / ms / 1e6:.1f} GB/s")
