// features.cu — multi-column feature-engine kernels (features.py:41-62,
// 165-189).  One launch covers every column of a FusedPlan: a per-element
// column lookup (binary search over the column offsets, L1-resident) selects
// the column's edges / modulus — the GPU form of "many small kernels fused
// into one dispatch" (PAPER §2.2.2).
#include "common.cuh"

namespace skb {

__device__ __forceinline__ int64_t column_of(const int64_t* __restrict__ col_offs, int64_t C, int64_t i) {
  int64_t lo = 0, hi = C;  // col_offs[lo] <= i < col_offs[lo+1]
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (col_offs[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// input element i of column c: one concatenated array, or per-column
// pointers (descriptor table: no concatenation copy before the launch)
template <class T>
struct FlatSrc {
  const T* vals;
  __device__ __forceinline__ T at(int64_t i, int64_t, const int64_t*) const { return vals[i]; }
};
template <class T>
struct ColSrc {
  const T* const* cols;
  __device__ __forceinline__ T at(int64_t i, int64_t c, const int64_t* col_offs) const {
    return cols[c][i - col_offs[c]];
  }
};

// bin = #{edges e : e <= v} (np.searchsorted side="right"); NaN flagged
template <class Src>
__global__ void k_bucketize(Src src, const int64_t* __restrict__ col_offs, int64_t C,
                            const float* __restrict__ edges, const int64_t* __restrict__ edge_offs, int64_t n,
                            int64_t* __restrict__ out, unsigned long long* nan_flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = C == 1 ? 0 : column_of(col_offs, C, i);
    float v = src.at(i, c, col_offs);
    if (v != v) {
      atomicMin(nan_flag, (unsigned long long)i);
      out[i] = 0;
      continue;
    }
    int64_t eb = edge_offs[c], ee = edge_offs[c + 1];
    int64_t lo = eb, hi = ee;  // first edge > v
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (__ldg(edges + mid) <= v) lo = mid + 1; else hi = mid;
    }
    out[i] = lo - eb;
  }
}

// non-negative remainder (np.remainder with m > 0)
template <class Src>
__global__ void k_mod(Src src, const int64_t* __restrict__ col_offs, int64_t C,
                      const int64_t* __restrict__ moduli, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = C == 1 ? 0 : column_of(col_offs, C, i);
    int64_t m = moduli[c];
    int64_t r = src.at(i, c, col_offs) % m;
    out[i] = r < 0 ? r + m : r;
  }
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_bucketize_multi(const float* values, const int64_t* col_offs, int64_t num_cols, const float* edges_cat,
                        const int64_t* edge_offs, int64_t* out, int64_t n_total, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (n_total <= 0) return SKB_OK;
  DevFlag f(s);
  k_bucketize<<<grid_for(n_total, 256), 256, 0, s>>>(FlatSrc<float>{values}, col_offs, num_cols, edges_cat, edge_offs,
                                                     n_total, out, f.ptr());
  SKB_LAUNCH_CHECK();
  if (f.read() >= 0) raise(SKB_E_VALUE, 0, "bucketize input contains NaN");
  SKB_API_END
}

int skb_bucketize_multi_async(const float* values, const int64_t* col_offs, int64_t num_cols, const float* edges_cat,
                              const int64_t* edge_offs, int64_t* out, int64_t n_total, unsigned long long* nan_flag,
                              void* stream) {
  SKB_API_BEGIN
  if (n_total <= 0) return SKB_OK;
  k_bucketize<<<grid_for(n_total, 256), 256, 0, as_stream(stream)>>>(FlatSrc<float>{values}, col_offs, num_cols,
                                                                     edges_cat, edge_offs, n_total, out, nan_flag);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_mod_multi(const int64_t* values, const int64_t* col_offs, int64_t num_cols, const int64_t* moduli,
                  int64_t* out, int64_t n_total, void* stream) {
  SKB_API_BEGIN
  if (n_total <= 0) return SKB_OK;
  k_mod<<<grid_for(n_total, 256), 256, 0, as_stream(stream)>>>(FlatSrc<int64_t>{values}, col_offs, num_cols, moduli,
                                                                n_total, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_bucketize_cols(const float* const* col_ptrs, const int64_t* col_offs, int64_t num_cols,
                       const float* edges_cat, const int64_t* edge_offs, int64_t* out, int64_t n_total,
                       unsigned long long* nan_flag, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (n_total <= 0) return SKB_OK;
  if (nan_flag) {
    k_bucketize<<<grid_for(n_total, 256), 256, 0, s>>>(ColSrc<float>{col_ptrs}, col_offs, num_cols, edges_cat,
                                                       edge_offs, n_total, out, nan_flag);
    SKB_LAUNCH_CHECK();
    return SKB_OK;
  }
  DevFlag f(s);
  k_bucketize<<<grid_for(n_total, 256), 256, 0, s>>>(ColSrc<float>{col_ptrs}, col_offs, num_cols, edges_cat, edge_offs,
                                                     n_total, out, f.ptr());
  SKB_LAUNCH_CHECK();
  if (f.read() >= 0) raise(SKB_E_VALUE, 0, "bucketize input contains NaN");
  SKB_API_END
}

int skb_mod_cols(const int64_t* const* col_ptrs, const int64_t* col_offs, int64_t num_cols, const int64_t* moduli,
                 int64_t* out, int64_t n_total, void* stream) {
  SKB_API_BEGIN
  if (n_total <= 0) return SKB_OK;
  k_mod<<<grid_for(n_total, 256), 256, 0, as_stream(stream)>>>(ColSrc<int64_t>{col_ptrs}, col_offs, num_cols, moduli,
                                                                n_total, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

// PackedBatch (fused.py): F members' ids concatenated and their bag offsets
// shifted by each member's first position — one launch over N + G + 1
// outputs through per-member pointer tables (replaces cat + repeat_interleave)
__global__ void k_pack_members(const int64_t* const* __restrict__ ids, const int64_t* const* __restrict__ offs,
                               const int64_t* __restrict__ mpos, const int64_t* __restrict__ mbag, int64_t F,
                               int64_t* __restrict__ ids_out, int64_t* __restrict__ bag_offs_out) {
  const int64_t N = mpos[F], G = mbag[F];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N + G + 1;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < N) {
      const int64_t f = column_of(mpos, F, t);
      ids_out[t] = __ldg(ids[f] + (t - mpos[f]));
    } else {
      const int64_t g = t - N;
      if (g == G) {
        bag_offs_out[G] = N;
      } else {
        const int64_t f = column_of(mbag, F, g);
        bag_offs_out[g] = mpos[f] + __ldg(offs[f] + (g - mbag[f]));
      }
    }
  }
}

int skb_pack_members(const int64_t* const* ids_ptrs, const int64_t* const* offs_ptrs, const int64_t* member_pos,
                     const int64_t* member_bag, int64_t num_members, int64_t n_total, int64_t num_bags,
                     int64_t* ids_out, int64_t* bag_offs_out, void* stream) {
  SKB_API_BEGIN
  k_pack_members<<<grid_for(n_total + num_bags + 1, 256), 256, 0, as_stream(stream)>>>(
      ids_ptrs, offs_ptrs, member_pos, member_bag, num_members, ids_out, bag_offs_out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

}  // extern "C"
