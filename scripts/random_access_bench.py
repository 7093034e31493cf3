"""DRAM cost of one random aligned read of W bytes on this GPU (used to set
the probe's algorithmic-bytes convention): index_select of 4M random rows of
W bytes from a 4 GiB buffer.  Run under ncu with dram__bytes_read.sum to get
bytes per access; prints CUDA-event times per width."""
import torch

torch.cuda.set_device(0)
buf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
n = 4 << 20
for w in (8, 16, 32, 64, 128, 256):
    rows = buf.view(torch.int64).view(-1, w // 8)
    idx = torch.randint(0, rows.shape[0], (n,), device="cuda")
    out = torch.index_select(rows, 0, idx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.index_select(rows, 0, idx, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"W={w} B: {e0.elapsed_time(e1) / 5 * 1e3:.1f} us per {n} random reads")
