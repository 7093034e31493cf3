// rows.cuh — row-granular copy / fold kernels shared by the table, partition
// and fused paths.  Rows are float32[D]; a row is moved by D/VEC consecutive
// lanes with 128-bit accesses (VEC = 4) so every warp instruction touches
// whole 32-byte sectors of one or more rows.
#pragma once
#include "common.cuh"

namespace skb {

// dst[i] = src[idx(i)] for i < n (idx(i) < 0 -> row left untouched, or filled with `fill`)
template <int VEC, class Idx>
__global__ void k_rows_gather(Idx idx, const float* __restrict__ src, int64_t sstride, float* __restrict__ dst,
                              int64_t dstride, int64_t n, int D, bool do_fill, float fill) {
  const int per_row = D / VEC;
  const int64_t total = n * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / per_row;
    int c = (int)(t - i * per_row) * VEC;
    int64_t r = idx(i);
    float* d = dst + i * dstride + c;
    if (r < 0) {
      if (do_fill) {
        if constexpr (VEC == 4) st4(d, make_float4(fill, fill, fill, fill));
        else d[0] = fill;
      }
      continue;
    }
    const float* sp = src + r * sstride + c;
    if constexpr (VEC == 4) st4(d, ldg4(sp));
    else d[0] = __ldg(sp);
  }
}

// dst[idx(i)] = src[i]
template <int VEC, class Idx>
__global__ void k_rows_scatter(Idx idx, const float* __restrict__ src, int64_t sstride, float* __restrict__ dst,
                               int64_t dstride, int64_t n, int D) {
  const int per_row = D / VEC;
  const int64_t total = n * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / per_row;
    int c = (int)(t - i * per_row) * VEC;
    int64_t r = idx(i);
    if (r < 0) continue;
    const float* sp = src + i * sstride + c;
    float* d = dst + r * dstride + c;
    if constexpr (VEC == 4) st4(d, ldg4(sp));
    else d[0] = __ldg(sp);
  }
}

struct IdxArray {
  const int64_t* a;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return a[i]; }
};
struct IdxIdentity {
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return i; }
};

template <class Idx>
void launch_rows_gather(Idx idx, const float* src, int64_t sstride, float* dst, int64_t dstride, int64_t n, int D,
                        cudaStream_t s, bool do_fill = false, float fill = 0.f) {
  if (n <= 0 || D <= 0) return;
  bool v4 = (D % 4 == 0) && (sstride % 4 == 0) && (dstride % 4 == 0) && ((uintptr_t)src % 16 == 0) &&
            ((uintptr_t)dst % 16 == 0);
  if (v4) {
    k_rows_gather<4><<<grid_for(n * (D / 4), 256), 256, 0, s>>>(idx, src, sstride, dst, dstride, n, D, do_fill, fill);
  } else {
    k_rows_gather<1><<<grid_for(n * D, 256), 256, 0, s>>>(idx, src, sstride, dst, dstride, n, D, do_fill, fill);
  }
  SKB_LAUNCH_CHECK();
}

template <class Idx>
void launch_rows_scatter(Idx idx, const float* src, int64_t sstride, float* dst, int64_t dstride, int64_t n, int D,
                         cudaStream_t s) {
  if (n <= 0 || D <= 0) return;
  bool v4 = (D % 4 == 0) && (sstride % 4 == 0) && (dstride % 4 == 0) && ((uintptr_t)src % 16 == 0) &&
            ((uintptr_t)dst % 16 == 0);
  if (v4) {
    k_rows_scatter<4><<<grid_for(n * (D / 4), 256), 256, 0, s>>>(idx, src, sstride, dst, dstride, n, D);
  } else {
    k_rows_scatter<1><<<grid_for(n * D, 256), 256, 0, s>>>(idx, src, sstride, dst, dstride, n, D);
  }
  SKB_LAUNCH_CHECK();
}

}  // namespace skb
