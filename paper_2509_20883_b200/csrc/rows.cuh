// rows.cuh — row-granular copy / fold kernels shared by the table, partition
// and fused paths.  Rows are float32[D]; a row is moved by D/VEC consecutive
// lanes with 128-bit accesses (VEC = 4) so every warp instruction touches
// whole 32-byte sectors of one or more rows.
#pragma once
#include "common.cuh"
#include "pool.cuh"

namespace skb {

// dst[i] = src[idx(i)] for i < n (idx(i) < 0 -> row left untouched, or filled with `fill`).
// Each thread owns U work items spaced one grid-stride apart and issues all U
// index loads, then all U row loads, then the stores: U independent random
// row fetches in flight per thread instead of one dependent chain.
// CHECK: idx(i) outside [0, limit) or !live[idx(i)] -> atomicMin(flag, i),
// row filled (the caller raises before anyone reads it).
constexpr int kRowsUnroll = 4;
template <int VEC, class Idx, bool CHECK = false>
__global__ void __launch_bounds__(256) k_rows_gather(Idx idx, const float* __restrict__ src, int64_t sstride,
                                                     float* __restrict__ dst, int64_t dstride, int64_t n, int D,
                                                     bool do_fill, float fill, const uint8_t* __restrict__ live = nullptr,
                                                     int64_t limit = 0, unsigned long long* flag = nullptr) {
  using V = typename VecT<VEC>::T;
  constexpr int U = kRowsUnroll;
  const int per_row = D / VEC;
  const bool pow2 = (per_row & (per_row - 1)) == 0;
  const int sh = __ffs(per_row) - 1;
  const int64_t total = n * per_row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < total; base += stride * U) {
    int64_t row[U], r[U];
    int col[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = base + u * stride;
      r[u] = -2;  // -2: no item
      if (t < total) {
        row[u] = pow2 ? (t >> sh) : t / per_row;  // no 64-bit division for power-of-two row widths
        col[u] = (int)(t - row[u] * per_row) * VEC;
        r[u] = idx(row[u]);
        if constexpr (CHECK) {
          if (r[u] < 0 || r[u] >= limit) {
            if (col[u] == 0) atomicMin(flag, (unsigned long long)row[u]);
            r[u] = -1;
          }
        }
      }
    }
    V v[U];
    uint8_t lv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (r[u] >= 0) {
        v[u] = vload<VEC>(src + r[u] * sstride + col[u]);  // in range: safe to fetch before the live test
        if constexpr (CHECK) lv[u] = __ldg(live + r[u]);
      }
    }
    if constexpr (CHECK) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r[u] >= 0 && !lv[u]) {
          if (col[u] == 0) atomicMin(flag, (unsigned long long)row[u]);
          r[u] = -1;
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (r[u] == -2) continue;
      float* d = dst + row[u] * dstride + col[u];
      if (r[u] >= 0) {
        vstore<VEC>(d, v[u]);
      } else if (do_fill || CHECK) {
        vstore<VEC>(d, vfill<VEC>(fill));
      }
    }
  }
}

// dst[idx(i)] = src[i]; same U-way independent issue as k_rows_gather
template <int VEC, class Idx>
__global__ void __launch_bounds__(256) k_rows_scatter(Idx idx, const float* __restrict__ src, int64_t sstride,
                                                      float* __restrict__ dst, int64_t dstride, int64_t n, int D) {
  using V = typename VecT<VEC>::T;
  constexpr int U = kRowsUnroll;
  const int per_row = D / VEC;
  const bool pow2 = (per_row & (per_row - 1)) == 0;
  const int sh = __ffs(per_row) - 1;
  const int64_t total = n * per_row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < total; base += stride * U) {
    int64_t r[U];
    int64_t row[U];
    int col[U];
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = base + u * stride;
      r[u] = -1;
      if (t < total) {
        row[u] = pow2 ? (t >> sh) : t / per_row;  // no 64-bit division for power-of-two row widths
        col[u] = (int)(t - row[u] * per_row) * VEC;
        r[u] = idx(row[u]);
        v[u] = vload<VEC>(src + row[u] * sstride + col[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r[u] >= 0) vstore<VEC>(dst + r[u] * dstride + col[u], v[u]);
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
    k_rows_gather<4><<<grid_for((n * (D / 4) + kRowsUnroll - 1) / kRowsUnroll, 256), 256, 0, s>>>(
        idx, src, sstride, dst, dstride, n, D, do_fill, fill);
  } else {
    k_rows_gather<1><<<grid_for((n * D + kRowsUnroll - 1) / kRowsUnroll, 256), 256, 0, s>>>(
        idx, src, sstride, dst, dstride, n, D, do_fill, fill);
  }
  SKB_LAUNCH_CHECK();
}

// gather + liveness check in one pass (gather embedding.py:233-238): flagged
// rows are zero-filled and the caller raises IndexError after reading `flag`
template <class Idx>
void launch_rows_gather_checked(Idx idx, const float* src, int64_t sstride, float* dst, int64_t dstride, int64_t n,
                                int D, const uint8_t* live, int64_t limit, unsigned long long* flag, cudaStream_t s) {
  if (n <= 0 || D <= 0) return;
  bool v4 = (D % 4 == 0) && (sstride % 4 == 0) && (dstride % 4 == 0) && ((uintptr_t)src % 16 == 0) &&
            ((uintptr_t)dst % 16 == 0);
  if (v4) {
    k_rows_gather<4, Idx, true><<<grid_for((n * (D / 4) + kRowsUnroll - 1) / kRowsUnroll, 256), 256, 0, s>>>(
        idx, src, sstride, dst, dstride, n, D, false, 0.f, live, limit, flag);
  } else {
    k_rows_gather<1, Idx, true><<<grid_for((n * D + kRowsUnroll - 1) / kRowsUnroll, 256), 256, 0, s>>>(
        idx, src, sstride, dst, dstride, n, D, false, 0.f, live, limit, flag);
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
    k_rows_scatter<4><<<grid_for((n * (D / 4) + kRowsUnroll - 1) / kRowsUnroll, 256), 256, 0, s>>>(
        idx, src, sstride, dst, dstride, n, D);
  } else {
    k_rows_scatter<1><<<grid_for((n * D + kRowsUnroll - 1) / kRowsUnroll, 256), 256, 0, s>>>(
        idx, src, sstride, dst, dstride, n, D);
  }
  SKB_LAUNCH_CHECK();
}

}  // namespace skb
