// hashing.cu — L0 integer hashing on device: SplitMix64 finalizer, owner
// shard, namespaced storage keys, FNV-1a over byte strings and id pairs.
// Bit-exact with hashing.py:27-86 / sharding.py:41-43,160,170-178.
#include "common.cuh"

namespace skb {

__global__ void k_mix64(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)mix64((uint64_t)in[i]);
}

__global__ void k_shard_of(const int64_t* __restrict__ in, int64_t n, uint64_t S, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)owner_of(in[i], S);
}

__global__ void k_keys_for(const int64_t* __restrict__ in, int64_t n, uint64_t salt, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)mix64((uint64_t)in[i] ^ salt);
}

// One thread per string; strings are short (feature values).  Bytes are read
// with byte loads from L2-resident blobs.
__global__ void k_fnv_strings(const uint8_t* __restrict__ blob, const int64_t* __restrict__ offs, int64_t n,
                              int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = offs[i], e = offs[i + 1];
    uint64_t h = kFnvBasis;
    for (int64_t j = b; j < e; ++j) h = (h ^ (uint64_t)blob[j]) * kFnvPrime;
    out[i] = (int64_t)h;
  }
}

__device__ __forceinline__ uint64_t fnv_pair(uint64_t x, uint64_t y) {
  uint64_t h = kFnvBasis;
#pragma unroll
  for (int k = 0; k < 8; ++k) h = (h ^ ((x >> (8 * k)) & 0xFF)) * kFnvPrime;
#pragma unroll
  for (int k = 0; k < 8; ++k) h = (h ^ ((y >> (8 * k)) & 0xFF)) * kFnvPrime;
  return h;
}

__global__ void k_fnv_pairs(const int64_t* __restrict__ x, const int64_t* __restrict__ y, int64_t n,
                            int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)fnv_pair((uint64_t)x[i], (uint64_t)y[i]);
}

// cross: one thread per output element; row found by binary search over the
// output offsets (x-major product, features.py:65-89).
__global__ void k_cross(const int64_t* __restrict__ a, const int64_t* __restrict__ aoff,
                        const int64_t* __restrict__ b, const int64_t* __restrict__ boff, int64_t rows,
                        const int64_t* __restrict__ ooff, int64_t total, int64_t* __restrict__ out,
                        int64_t* size_flag) {
  const int64_t true_total = ooff[rows];
  if (size_flag && blockIdx.x == 0 && threadIdx.x == 0 && true_total != total) *size_flag = true_total;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    if (t >= true_total) {  // a caller-supplied size larger than the products: never read past the inputs
      out[t] = 0;
      continue;
    }
    int64_t lo = 0, hi = rows;  // find r with ooff[r] <= t < ooff[r+1]
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (ooff[mid] <= t) lo = mid; else hi = mid;
    }
    int64_t r = lo;
    int64_t within = t - ooff[r];
    int64_t lb = boff[r + 1] - boff[r];
    int64_t i = within / lb, j = within - i * lb;
    out[t] = (int64_t)fnv_pair((uint64_t)a[aoff[r] + i], (uint64_t)b[boff[r] + j]);
  }
}

__global__ void k_cross_lens(const int64_t* __restrict__ aoff, const int64_t* __restrict__ boff, int64_t rows,
                             int64_t* __restrict__ lens) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    lens[r] = (aoff[r + 1] - aoff[r]) * (boff[r + 1] - boff[r]);
}

// ---------------------------------------------------------------------------
// cross_many: every column pair of a step in two launches (features.py:65-89
// per pair).  One descriptor per pair; outputs of all pairs share one buffer
// (out_base = the pair's first output).  Launch 1: one CTA per pair scans its
// row products into out_offs and checks the caller's size; launch 2: one
// thread per output element of all pairs (pair by binary search over the
// descriptors' out_base, row by binary search over the pair's out_offs).
// ---------------------------------------------------------------------------
struct CrossDesc {
  const int64_t* a;
  const int64_t* ao;
  const int64_t* b;
  const int64_t* bo;
  int64_t rows;
  int64_t* oo;       // [rows + 1]
  int64_t total;     // caller size of this pair's output (or the true one)
  int64_t out_base;  // first output of this pair in the shared buffer
  int64_t* flag;     // optional: true product count when it differs from total
  int64_t pad;
};
static_assert(sizeof(CrossDesc) == 80, "descriptor layout is shared with features.py");

constexpr int kCrossScanThreads = 1024;
constexpr int kCrossScanItems = 8;

__global__ void __launch_bounds__(kCrossScanThreads) k_cross_offsets_many(const CrossDesc* __restrict__ descs) {
  const CrossDesc d = descs[blockIdx.x];
  constexpr int W = kCrossScanThreads / 32;
  __shared__ int64_t s_warp[W];
  __shared__ int64_t s_carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  constexpr int64_t kChunk = (int64_t)kCrossScanThreads * kCrossScanItems;
  for (int64_t c0 = 0; c0 < d.rows; c0 += kChunk) {
    int64_t v[kCrossScanItems];
    int64_t loc = 0;
    const int64_t r0 = c0 + (int64_t)threadIdx.x * kCrossScanItems;
#pragma unroll
    for (int q = 0; q < kCrossScanItems; ++q) {
      const int64_t r = r0 + q;
      v[q] = r < d.rows ? (d.ao[r + 1] - d.ao[r]) * (d.bo[r + 1] - d.bo[r]) : 0;
      loc += v[q];
    }
    int64_t inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    int64_t before = s_carry, tot = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int64_t x = s_warp[q];
      if (q < w) before += x;
      tot += x;
    }
    int64_t run = before + inc - loc;
#pragma unroll
    for (int q = 0; q < kCrossScanItems; ++q) {
      const int64_t r = r0 + q;
      if (r < d.rows) d.oo[r] = run;
      run += v[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    d.oo[d.rows] = s_carry;
    if (d.flag && s_carry != d.total) *d.flag = s_carry;
  }
}

constexpr int kCrossMaxPairs = 1024;

__global__ void __launch_bounds__(256) k_cross_many(const CrossDesc* __restrict__ descs, int npairs, int64_t T,
                                                    int64_t* __restrict__ out) {
  __shared__ int64_t s_base[kCrossMaxPairs + 1];
  for (int k = threadIdx.x; k < npairs; k += blockDim.x) s_base[k] = descs[k].out_base;
  if (threadIdx.x == 0) s_base[npairs] = T;
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = npairs;  // pair p with s_base[p] <= t < s_base[p+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_base[mid] <= t) lo = mid; else hi = mid;
    }
    const CrossDesc& d = descs[lo];
    const int64_t tl = t - s_base[lo];
    const int64_t true_total = __ldg(d.oo + d.rows);
    if (tl >= true_total) {  // a caller-supplied size larger than the products: never read past the inputs
      out[t] = 0;
      continue;
    }
    int64_t a = 0, b = d.rows;  // row r with oo[r] <= tl < oo[r+1]
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (__ldg(d.oo + mid) <= tl) a = mid; else b = mid;
    }
    const int64_t within = tl - __ldg(d.oo + a);
    const int64_t lb = __ldg(d.bo + a + 1) - __ldg(d.bo + a);
    const int64_t i = within / lb, j = within - i * lb;
    out[t] = (int64_t)fnv_pair((uint64_t)__ldg(d.a + __ldg(d.ao + a) + i), (uint64_t)__ldg(d.b + __ldg(d.bo + a) + j));
  }
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_mix64(const int64_t* ids, int64_t n, int64_t* out, void* stream) {
  SKB_API_BEGIN
  if (n <= 0) return SKB_OK;
  k_mix64<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(ids, n, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_shard_of(const int64_t* ids, int64_t n, int64_t num_shards, int64_t* out, void* stream) {
  SKB_API_BEGIN
  if (num_shards < 1) raise(SKB_E_VALUE, num_shards, "num_shards must be >= 1");
  if (n <= 0) return SKB_OK;
  k_shard_of<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(ids, n, (uint64_t)num_shards, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_keys_for(const int64_t* ids, int64_t n, uint64_t salt, int64_t* out, void* stream) {
  SKB_API_BEGIN
  if (n <= 0) return SKB_OK;
  k_keys_for<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(ids, n, salt, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

uint64_t skb_fnv1a64_host(const uint8_t* bytes_host, int64_t len) {
  uint64_t h = kFnvBasis;
  for (int64_t i = 0; i < len; ++i) h = (h ^ bytes_host[i]) * kFnvPrime;
  return h;
}

int skb_fnv1a64_strings(const uint8_t* blob, const int64_t* str_offs, int64_t n, int64_t* out, void* stream) {
  SKB_API_BEGIN
  if (n <= 0) return SKB_OK;
  k_fnv_strings<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(blob, str_offs, n, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_fnv1a64_pairs(const int64_t* x, const int64_t* y, int64_t n, int64_t* out, void* stream) {
  SKB_API_BEGIN
  if (n <= 0) return SKB_OK;
  k_fnv_pairs<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, y, n, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_cross_offsets(const int64_t* a_offs, const int64_t* b_offs, int64_t rows, int64_t* out_offs,
                      void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (rows <= 0) {
    SKB_CUDA(cudaMemsetAsync(out_offs, 0, sizeof(int64_t), s));
    return SKB_OK;
  }
  Scratch lens(sizeof(int64_t) * rows, s);
  k_cross_lens<<<grid_for(rows, 256), 256, 0, s>>>(a_offs, b_offs, rows, lens.as<int64_t>());
  SKB_LAUNCH_CHECK();
  scan_exclusive_i64(lens.as<int64_t>(), out_offs, rows, out_offs + rows, s);
  SKB_API_END
}

int skb_cross_offsets_many(const void* descs_dev, int64_t npairs, void* stream) {
  SKB_API_BEGIN
  if (npairs < 0) raise(SKB_E_ARG, npairs, "cross_many: negative pair count");
  if (npairs == 0) return SKB_OK;
  k_cross_offsets_many<<<(unsigned)npairs, kCrossScanThreads, 0, as_stream(stream)>>>(
      static_cast<const CrossDesc*>(descs_dev));
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_cross_many(const void* descs_dev, int64_t npairs, int64_t total, int64_t* out, void* stream) {
  SKB_API_BEGIN
  if (npairs < 0 || npairs > kCrossMaxPairs) raise(SKB_E_ARG, npairs, "cross_many: 0..1024 pairs per launch");
  if (total < 0) raise(SKB_E_VALUE, total, "cross: negative output size");
  if (npairs == 0 || total == 0) return SKB_OK;
  k_cross_many<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(static_cast<const CrossDesc*>(descs_dev),
                                                                     (int)npairs, total, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_cross(const int64_t* a_vals, const int64_t* a_offs, const int64_t* b_vals, const int64_t* b_offs,
              int64_t rows, const int64_t* out_offs, int64_t total, int64_t* out, int64_t* size_flag,
              void* stream) {
  SKB_API_BEGIN
  if (total < 0) raise(SKB_E_VALUE, total, "cross: negative output size");
  // total == 0 still launches one thread when a size flag wants the check
  if (total == 0 && !size_flag) return SKB_OK;
  k_cross<<<total > 0 ? grid_for(total, 256) : 1, 256, 0, as_stream(stream)>>>(a_vals, a_offs, b_vals, b_offs, rows,
                                                                               out_offs, total, out, size_flag);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

}  // extern "C"
