import torch, time
for mb in (13.6, 27.3, 256):
    n = int(mb * 1e6 / 8)
    h = torch.empty(n, dtype=torch.int64).pin_memory()
    d = torch.empty(n, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    print(f"H2D {mb} MB: {t:.3f} ms  {n*8/t/1e6:.1f} GB/s")
