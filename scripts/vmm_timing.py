"""Host cost of the VMM growth calls (cuMemCreate / cuMemMap / cuMemSetAccess)
per chunk size on this GPU — sizes the table's growth chunks (csrc/vmm.cu)."""
import time

import torch
from cuda.bindings import driver as d

torch.cuda.init()
torch.zeros(1, device="cuda")
dev = torch.cuda.current_device()
prop = d.CUmemAllocationProp()
prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
prop.location.id = dev
acc = d.CUmemAccessDesc()
acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
acc.location.id = dev
acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
err, va = d.cuMemAddressReserve(64 << 30, 0, 0, 0)
off = 0
for mb in (2, 64, 256, 1024, 2048, 256, 64):
    size = mb << 20
    t0 = time.perf_counter()
    err, h = d.cuMemCreate(size, prop, 0)
    t1 = time.perf_counter()
    err, = d.cuMemMap(int(va) + off, size, 0, h, 0)
    t2 = time.perf_counter()
    err, = d.cuMemSetAccess(int(va) + off, size, [acc], 1)
    t3 = time.perf_counter()
    off += size
    print(f"{mb:5d} MB: create {1e3 * (t1 - t0):7.3f} ms  map {1e3 * (t2 - t1):7.3f} ms  access {1e3 * (t3 - t2):7.3f} ms")
