// vmm.cu — see vmm.cuh.  Driver entry points are resolved through the
// runtime (cudaGetDriverEntryPoint): no link-time dependency on libcuda.
#include <mutex>

#include <cuda.h>

#include "vmm.cuh"

namespace skb {

namespace {
typedef CUresult (*PfnReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PfnFreeVA)(CUdeviceptr, size_t);
typedef CUresult (*PfnCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
typedef CUresult (*PfnRelease)(CUmemGenericAllocationHandle);
typedef CUresult (*PfnMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PfnUnmap)(CUdeviceptr, size_t);
typedef CUresult (*PfnSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
typedef CUresult (*PfnGran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);

struct Api {
  PfnReserve reserve = nullptr;
  PfnFreeVA free_va = nullptr;
  PfnCreate create = nullptr;
  PfnRelease release = nullptr;
  PfnMap map = nullptr;
  PfnUnmap unmap = nullptr;
  PfnSetAccess access = nullptr;
  PfnGran gran = nullptr;
  bool ok = false;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** f) {
      cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
      return cudaGetDriverEntryPoint(name, f, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *f != nullptr;
    };
    a.ok = get("cuMemAddressReserve", (void**)&a.reserve) && get("cuMemAddressFree", (void**)&a.free_va) &&
           get("cuMemCreate", (void**)&a.create) && get("cuMemRelease", (void**)&a.release) &&
           get("cuMemMap", (void**)&a.map) && get("cuMemUnmap", (void**)&a.unmap) &&
           get("cuMemSetAccess", (void**)&a.access) && get("cuMemGetAllocationGranularity", (void**)&a.gran);
    cudaGetLastError();
    if (getenv("SKB_NO_VMM")) a.ok = false;
  });
  return a;
}

CUmemAllocationProp prop_for_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = dev;
  return p;
}

void check(CUresult r, const char* what) {
  if (r == CUDA_ERROR_OUT_OF_MEMORY) raise(SKB_E_NOMEM, 0, "%s: out of device memory", what);
  if (r != CUDA_SUCCESS) raise(SKB_E_CUDA, r, "%s failed (CUresult %d)", what, (int)r);
}

size_t round_up(size_t x, size_t g) { return (x + g - 1) / g * g; }
}  // namespace

bool vmm_available() { return api().ok; }

size_t vmm_granularity() {
  static size_t g = 0;
  if (!g) {
    CUmemAllocationProp p = prop_for_current();
    check(api().gran(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    if (!g) g = 2u << 20;
  }
  return g;
}

static void map_chunk(uint64_t va, size_t bytes, unsigned long long h) {
  Api& A = api();
  check(A.map((CUdeviceptr)va, bytes, 0, (CUmemGenericAllocationHandle)h, 0), "cuMemMap");
  int dev = 0;
  cudaGetDevice(&dev);
  CUmemAccessDesc d = {};
  d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d.location.id = dev;
  d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  check(A.access((CUdeviceptr)va, bytes, &d, 1), "cuMemSetAccess");
}

void vmm_prepare(VmmArray& a, size_t bytes, int device) {
  Api& A = api();
  if (!a.base || a.prep_bytes) return;
  SKB_CUDA(cudaSetDevice(device));
  const size_t g = vmm_granularity();
  size_t add = round_up(bytes > 0 ? bytes : 1, g);
  if (a.mapped + add > a.reserved) add = (a.reserved - a.mapped) / g * g;
  if (!add) return;
  CUmemAllocationProp p = prop_for_current();
  CUmemGenericAllocationHandle h = 0;
  if (A.create(&h, add, &p, 0) != CUDA_SUCCESS) {  // out of memory ahead of need: growth will retry (and raise)
    cudaGetLastError();
    return;
  }
  map_chunk(a.base + a.mapped, add, (unsigned long long)h);
  a.prep_handle = (unsigned long long)h;
  a.prep_bytes = add;
}

bool vmm_grow(VmmArray& a, size_t bytes, size_t reserve_hint, cudaStream_t s) {
  Api& A = api();
  const size_t g = vmm_granularity();
  const size_t want = round_up(bytes > 0 ? bytes : 1, g);
  if (want <= a.mapped) return false;
  if (a.prep_bytes) {  // adopt the chunk prepared ahead: only the zero-fill is left
    a.chunks.push_back(VmmArray::Chunk{a.prep_handle, a.mapped, a.prep_bytes});
    SKB_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(a.base + a.mapped), 0, a.prep_bytes, s));
    a.mapped += a.prep_bytes;
    a.prep_handle = 0;
    a.prep_bytes = 0;
    if (want <= a.mapped) return false;
  }
  bool moved = false;
  if (want > a.reserved) {
    // (re)reserve: the requested hint, or 4x what is needed now
    size_t res = round_up(reserve_hint > want ? reserve_hint : 4 * want, g);
    CUdeviceptr nb = 0;
    check(A.reserve(&nb, res, 0, 0, 0), "cuMemAddressReserve");
    if (a.base) {
      // the same physical chunks behind the new range: no data moves, but
      // kernels must be done with the old addresses before they are unmapped
      SKB_CUDA(cudaDeviceSynchronize());
      for (const auto& c : a.chunks) map_chunk(nb + c.offset, c.bytes, c.handle);
      for (const auto& c : a.chunks) check(A.unmap((CUdeviceptr)(a.base + c.offset), c.bytes), "cuMemUnmap");
      check(A.free_va((CUdeviceptr)a.base, a.reserved), "cuMemAddressFree");
      moved = true;
    }
    a.base = nb;
    a.reserved = res;
  }
  const size_t add = want - a.mapped;
  CUmemAllocationProp p = prop_for_current();
  CUmemGenericAllocationHandle h = 0;
  check(A.create(&h, add, &p, 0), "cuMemCreate");
  map_chunk(a.base + a.mapped, add, (unsigned long long)h);
  a.chunks.push_back(VmmArray::Chunk{(unsigned long long)h, a.mapped, add});
  SKB_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(a.base + a.mapped), 0, add, s));
  a.mapped = want;
  return moved;
}

void vmm_free(VmmArray& a) {
  if (!a.base) return;
  Api& A = api();
  if (a.prep_bytes) {
    A.unmap((CUdeviceptr)(a.base + a.mapped), a.prep_bytes);
    A.release((CUmemGenericAllocationHandle)a.prep_handle);
  }
  for (const auto& c : a.chunks) {
    A.unmap((CUdeviceptr)(a.base + c.offset), c.bytes);
    A.release((CUmemGenericAllocationHandle)c.handle);
  }
  A.free_va((CUdeviceptr)a.base, a.reserved);
  a = VmmArray();
}

}  // namespace skb
