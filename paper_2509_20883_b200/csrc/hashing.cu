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
