// checkpoint.cu — device side of the checkpoint boundary (checkpoint.py:192-313).
//
// save_sharded needs every table's rows globally sorted by stored key
// (checkpoint.py:212-214: stable argsort of the concatenated shard exports);
// load_sharded re-routes rows to a new shard count (checkpoint.py:300-311).
// On the GPU that is one stable radix argsort of the int64 keys plus row
// gathers / scatters of the SoA export buffers — all HBM-bound copies: one
// warp per row, 16-byte vectors when the row width allows.
#include "common.cuh"

namespace skb {

__global__ void k_iota_i64(int64_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

// SCATTER=false: out[i] = src[idx[i]];  SCATTER=true: out[idx[i]] = src[i].
// Rows of W words of type V (V = uint4 / uint2 / uint32_t), one warp per row.
template <class V, bool SCATTER>
__global__ void __launch_bounds__(256) k_move_rows(const V* __restrict__ src, int64_t words, const int64_t* __restrict__ idx,
                                                   int64_t n, V* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int64_t j = __ldg(idx + r);
    const V* s = src + (SCATTER ? r : j) * words;
    V* d = out + (SCATTER ? j : r) * words;
    for (int64_t w = lane; w < words; w += 32) d[w] = s[w];
  }
}

template <bool SCATTER>
static void move_rows(const void* src, int64_t row_bytes, const int64_t* idx, int64_t n, void* out, cudaStream_t s) {
  if (n <= 0) return;
  if (row_bytes <= 0 || row_bytes % 4) raise(SKB_E_ARG, row_bytes, "row_bytes must be a positive multiple of 4");
  const uintptr_t a = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(out);
  const unsigned g = grid_for(n * 32, 256);
  if (row_bytes % 16 == 0 && a % 16 == 0)
    k_move_rows<uint4, SCATTER><<<g, 256, 0, s>>>((const uint4*)src, row_bytes / 16, idx, n, (uint4*)out);
  else if (row_bytes % 8 == 0 && a % 8 == 0)
    k_move_rows<uint2, SCATTER><<<g, 256, 0, s>>>((const uint2*)src, row_bytes / 8, idx, n, (uint2*)out);
  else
    k_move_rows<uint32_t, SCATTER><<<g, 256, 0, s>>>((const uint32_t*)src, row_bytes / 4, idx, n, (uint32_t*)out);
  SKB_LAUNCH_CHECK();
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_argsort_i64(const int64_t* keys, int64_t n, int64_t* sorted_keys, int64_t* perm, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (n < 0) raise(SKB_E_ARG, n, "n must be >= 0");
  if (n == 0) return SKB_OK;
  Scratch iota(sizeof(int64_t) * n, s);
  k_iota_i64<<<grid_for(n, 256), 256, 0, s>>>(iota.as<int64_t>(), n);
  SKB_LAUNCH_CHECK();
  sort_pairs_i64(keys, sorted_keys, iota.as<int64_t>(), perm, n, s);
  SKB_API_END
}

int skb_gather_rows(const void* src, int64_t row_bytes, const int64_t* idx, int64_t n, void* out, void* stream) {
  SKB_API_BEGIN
  move_rows<false>(src, row_bytes, idx, n, out, as_stream(stream));
  SKB_API_END
}

int skb_scatter_rows(const void* src, int64_t row_bytes, const int64_t* idx, int64_t n, void* out, void* stream) {
  SKB_API_BEGIN
  move_rows<true>(src, row_bytes, idx, n, out, as_stream(stream));
  SKB_API_END
}

}  // extern "C"

namespace skb {
__global__ void k_partition_dest(const int64_t* __restrict__ base, const int64_t* __restrict__ inv_s,
                                 const int64_t* __restrict__ inv_p, int64_t n, int64_t* __restrict__ dest) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dest[i] = base[inv_s[i]] + inv_p[i];
}
}  // namespace skb

extern "C" int skb_partition_dest(const int64_t* shard_base, const int64_t* inv_shard, const int64_t* inv_pos,
                                  int64_t n, int64_t* dest, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  k_partition_dest<<<grid_for(n, 256), 256, 0, s>>>(shard_base, inv_shard, inv_pos, n, dest);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}
