"""C1 (dim16, B=4096, one feature, bag length 1, sum, AdamW) step time:
the launch-bound regime the CUDA-graph path targets."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20883_b200 as skb

B, D, steps = 4096, 16, int(os.environ.get('C1_STEPS', 200))
lt = skb.LogicalTable("f0", D, 1, seed=0, members=["f0"], namespaced=False, capacity_hint=200_000)
rng = np.random.default_rng(0)
batches = [skb.PackedBatch(lt, ["f0"], [rng.integers(0, 100_000, B)], [np.arange(B + 1, dtype=np.int64)])
           for _ in range(2)]
pool_ids = [torch.from_numpy(rng.integers(0, 100_000, B)).cuda() for _ in range(8)]
dp = torch.randn((B, D), device="cuda") * 1e-2
cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
pooled = torch.empty((B, D), device="cuda")
mode = sys.argv[1] if len(sys.argv) > 1 else "pipelined"
graphs = "graphs" in sys.argv[2:]
skb.use_graphs(lt, graphs)

def batch(k):
    # two device batch buffers refilled in place (fixed pointers: graph replay)
    b = batches[k % 2]
    b.ids.copy_(pool_ids[k % 8], non_blocking=True)
    return b

def run(first, count):
    if mode == "pipelined":
        skb.prefetch(lt, batch(first), first, "sum")
    for k in range(first, first + count):
        if mode == "pipelined" and k + 1 < first + count:
            skb.prefetch(lt, batch(k + 1), k + 1, "sum")
        skb.lookup_pool(lt, batches[k % 2] if mode == "pipelined" else batch(k), k, "sum", out=pooled)
        skb.pool_grad_adam(lt, dp, cfg, k)

run(1, 20); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
run(21, steps)
e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"C1 {mode}{' graphs' if graphs else ''}: {e0.elapsed_time(e1)/steps*1e3:.1f} us/step device, {(t1-t0)/steps*1e6:.1f} us/step host wall")
