import sys, os, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2509_20883_b200 as skb
from paper_2509_20883_b200 import _native as N, fused as FZ
from paper_2509_20883_b200.optim import adam_scalars
torch.cuda.init()
def bench(name, fn, n=2000):
    fn(); t0 = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:40s} {(time.perf_counter()-t0)/n*1e6:8.2f} us")
bench("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
bench("N.stream_ptr()", N.stream_ptr)
bench("torch.cuda.is_available()", torch.cuda.is_available)
bench("torch.cuda.device_count()", torch.cuda.device_count)
bench("torch.cuda.current_device()", torch.cuda.current_device)
lt = skb.LogicalTable("f0", 16, 1, seed=0, members=["f0"], capacity_hint=200000)
B = 4096
b = skb.PackedBatch(lt, ["f0"], [np.random.randint(0, 100000, B)], [np.arange(B + 1)])
cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
bench("adam_scalars", lambda: adam_scalars(cfg, 5))
bench("_batch_args", lambda: FZ._batch_args(lt, b, 5, "sum"))
dp = torch.zeros((B, 16), device="cuda")
bench("N.to_dev(dp)", lambda: N.to_dev(dp, "float32"))
bench("N.ptr(dp)", lambda: N.ptr(dp))
pooled = torch.empty((B, 16), device="cuda")
step = [1]
def stepfn():
    k = step[0]; step[0] += 1
    skb.lookup_pool(lt, b, k, "sum", out=pooled)
    skb.pool_grad_adam(lt, dp, cfg, k)
bench("full step (serial)", stepfn, 500)
skb.use_graphs(lt, True)
bench("full step (serial, graphs)", stepfn, 500)
torch.cuda.synchronize()
