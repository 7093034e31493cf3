// runtime.cu — error plumbing, device facts, stream-ordered scratch.
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace skb {

static thread_local std::string t_err;
static thread_local int64_t t_err_arg = 0;

void raise(int code, int64_t arg, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw SkbError(code, buf, arg);
}

int set_error(int code, const char* msg, int64_t arg) {
  t_err = msg ? msg : "";
  t_err_arg = arg;
  return code;
}

void clear_error() {
  t_err.clear();
  t_err_arg = 0;
}

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static std::mutex g_mu;
static std::vector<int> g_sm;            // per device
static std::vector<bool> g_pool_ready;   // per device

int sm_count() {
  int dev = 0;
  SKB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  if ((int)g_sm.size() <= dev) g_sm.resize(dev + 1, 0);
  if (!g_sm[dev]) {
    int v = 0;
    SKB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    g_sm[dev] = v;
  }
  return g_sm[dev];
}

static void ensure_pool() {
  int dev = 0;
  SKB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  if ((int)g_pool_ready.size() <= dev) g_pool_ready.resize(dev + 1, false);
  if (g_pool_ready[dev]) return;
  cudaMemPool_t pool;
  SKB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  // keep freed scratch cached in the pool: per-step scratch is then free
  uint64_t thr = 8ull << 30;
  SKB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  // never let an allocation on one stream wait for another stream's pending
  // free: the index stream's scratch (CUB sort temp storage) reusing a block
  // the main stream freed made it wait behind fold+Adam (C4/C5 step times
  // 8 -> 100 ms at random); without internal dependencies the pool takes
  // fresh (cached) memory instead
  int no = 0;
  SKB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no));
  // optional L2 fetch-granularity hint (random 16 B probes vs 128 B lines)
  if (const char* g = getenv("SKB_L2_FETCH")) SKB_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, atoi(g)));
  g_pool_ready[dev] = true;
}

void* scratch_alloc(size_t bytes, cudaStream_t s) {
  ensure_pool();
  void* p = nullptr;
  // round up to 256 B so vector access is always aligned
  bytes = (bytes + 255) & ~size_t(255);
  SKB_CUDA(cudaMallocAsync(&p, bytes, s));
  return p;
}

void scratch_free(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

HostMailbox::HostMailbox(int count) : n(count) {
  SKB_CUDA(cudaMallocHost(&h, sizeof(int64_t) * count));
}
HostMailbox::~HostMailbox() {
  if (h) cudaFreeHost(h);
}

__global__ void k_init_flag(unsigned long long* f) {
  f[0] = ~0ull;
  f[1] = 0;
}

DevFlag::DevFlag(cudaStream_t st) : buf(16, st), s(st) {
  k_init_flag<<<1, 1, 0, s>>>(ptr());
  SKB_LAUNCH_CHECK();
}

int64_t* pinned_mailbox() {  // per host thread; a D2H into pageable memory is staged and slower
  thread_local HostMailbox box(4);
  return box.h;
}

int64_t DevFlag::read() {
  int64_t* h = pinned_mailbox();
  SKB_CUDA(cudaMemcpyAsync(h, buf.p, 16, cudaMemcpyDeviceToHost, s));
  SKB_CUDA(cudaStreamSynchronize(s));
  return (uint64_t)h[0] == ~0ull ? -1 : h[0];
}

__global__ void k_ht_fill(HEntry* t, int64_t count, long long init_val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    reinterpret_cast<longlong2*>(t)[i] = make_longlong2(kEmptyKey, init_val);
  }
}

void ht_fill(HEntry* t, int64_t count, long long init_val, cudaStream_t s) {
  if (count <= 0) return;
  k_ht_fill<<<grid_for(count, 256), 256, 0, s>>>(t, count, init_val);
  SKB_LAUNCH_CHECK();
}

}  // namespace skb

using namespace skb;

extern "C" {

const char* skb_version(void) { return "sparsekit_b200 0.1.0 (sm_100a)"; }
const char* skb_last_error(void) { return t_err.c_str(); }
int64_t skb_last_error_arg(void) { return t_err_arg; }

int64_t skb_launch_count(void) { return g_launches.load(); }

int skb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  SKB_API_BEGIN
  if (bytes > 0) SKB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, skb::as_stream(stream)));
  SKB_API_END
}

int skb_device_sm_count(int device, int* out_host) {
  SKB_API_BEGIN
  int v = 0;
  SKB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  *out_host = v;
  SKB_API_END
}

}  // extern "C"
