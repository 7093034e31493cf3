// segments.cu — ragged combiner pooling (segments.py:61-116) and CSR helpers.
//
// Bit-exact with the reference's numpy 2.3.5 float semantics:
//   scatter    = np.add.at: left fold from +0.0 in row order
//   sequential = np.add.reduceat: rows[s] + pairwise(rows[s+1:e]) per column,
//                pairwise = numpy's 8-accumulator blocks of <= 128 with the
//                n/2 (multiple-of-8) recursive split
//   mean       = sum / float32(len), empty segments stay 0
#include <cstring>

#include "common.cuh"
#include "pool.cuh"

namespace skb {

template <int VEC>
__global__ void k_segment_reduce(const float* __restrict__ rows, int D, const int64_t* __restrict__ offs, int64_t G,
                                 int mode, int strategy, float* __restrict__ out) {
  const int per_row = D / VEC;
  const int64_t total = G * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t g = t / per_row;
    int c = (int)(t - g * per_row) * VEC;
    int64_t b = offs[g], e = offs[g + 1];
    RowSrc src{rows, D, c};
    typename VecT<VEC>::T acc = strategy == 0 ? pool_sequential<VEC>(src, b, reduceat_end(b, e, g == G - 1, offs[G]))
                                              : pool_scatter<VEC>(src, b, e);
    if (mode == 1 && e > b) acc = vdiv<VEC>(acc, (float)(e - b));
    vstore<VEC>(out + g * D + c, acc);
  }
}

// Long `sequential` segments: numpy's pairwise tree over rows[b+1:e] has
// leaves of <= 128 rows that are independent; one warp per (segment, column
// vector) folds leaf i on lane i (the 8-accumulator leaf loop, unchanged),
// then every lane evaluates the tree in numpy's order with the leaf values
// fetched by shuffle — the same additions in the same order as pw_sum, with
// up to 32 leaves' loads in flight instead of one thread's.
__device__ __forceinline__ int pw_leaves(int64_t n, int64_t* lb, int64_t* ln, int cap) {
  int64_t sb[24], sn[24];  // DFS stack (depth <= log2(n / 64) + 1)
  int sp = 0, k = 0;
  sb[sp] = 0;
  sn[sp++] = n;
  while (sp > 0) {
    const int64_t b = sb[--sp], m = sn[sp];
    if (m <= 128) {
      if (k < cap) {
        lb[k] = b;
        ln[k] = m;
      }
      ++k;
      continue;
    }
    int64_t n2 = m / 2;
    n2 -= n2 % 8;
    sb[sp] = b + n2;  // right pushed first: the left half is visited first
    sn[sp++] = m - n2;
    sb[sp] = b;
    sn[sp++] = n2;
  }
  return k;
}

// numpy's tree over the leaves of a length-n pairwise sum; leaf i's value
// lives on lane i * cpw + col (uniform control flow: every lane walks the tree)
template <int VEC>
__device__ typename VecT<VEC>::T pw_combine(int64_t n, typename VecT<VEC>::T v, int cpw, int col) {
  using T = typename VecT<VEC>::T;
  struct Frame {
    int64_t n;
    T left;
    int stage;
  };
  Frame st[24];
  int sp = 0, leaf = 0;
  st[sp++] = Frame{n, vfill<VEC>(0.f), 0};
  T result = vfill<VEC>(0.f);
  bool have = false;
  while (sp > 0) {
    Frame& f = st[sp - 1];
    if (!have) {
      if (f.n <= 128) {
        result = vshfl<VEC>(v, leaf++ * cpw + col);
        have = true;
        --sp;
        continue;
      }
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      st[sp++] = Frame{n2, vfill<VEC>(0.f), 0};
    } else {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      if (f.stage == 0) {
        f.left = result;
        f.stage = 1;
        have = false;
        st[sp++] = Frame{f.n - n2, vfill<VEC>(0.f), 0};
      } else {
        result = vadd<VEC>(f.left, result);
        --sp;
      }
    }
  }
  return result;
}

// one warp per (segment, column vector): lane i folds leaf i
template <int VEC>
__global__ void __launch_bounds__(256) k_segment_reduce_warp(const float* __restrict__ rows, int D,
                                                             const int64_t* __restrict__ offs, int64_t G, int mode,
                                                             float* __restrict__ out) {
  using T = typename VecT<VEC>::T;
  const int per_row = D / VEC;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < G * per_row; w += warps) {
    const int64_t g = w / per_row;
    const int c = (int)(w - g * per_row) * VEC;
    const int64_t b = offs[g], e0 = offs[g + 1];
    const int64_t e = reduceat_end(b, e0, g == G - 1, offs[G]);
    RowSrc src{rows, D, c};
    T acc;
    int64_t lb[32], ln[32];
    const int nl = e - b > 129 ? pw_leaves(e - b - 1, lb, ln, 32) : 1;
    if (nl == 1 || nl > 32) {  // one leaf (or a very long tree): lane 0, serial pairwise
      acc = lane == 0 ? pool_sequential<VEC>(src, b, e) : vfill<VEC>(0.f);
    } else {
      T v = vfill<VEC>(0.f);
      if (lane < nl) v = pw_leaf<VEC>(src, b + 1 + lb[lane], ln[lane]);  // all leaves at once
      acc = vadd<VEC>(src.template load<VEC>(b), pw_combine<VEC>(e - b - 1, v, 1, 0));
    }
    if (lane == 0) {
      if (mode == 1 && e0 > b) acc = vdiv<VEC>(acc, (float)(e0 - b));
      vstore<VEC>(out + g * D + c, acc);
    }
  }
}

// float64 rows: one thread per (segment, column), the same fold orders in
// double (numpy's pairwise_sum is one template for float and double)
__global__ void k_segment_reduce_f64(const double* __restrict__ rows, int D, const int64_t* __restrict__ offs,
                                     int64_t G, int mode, int strategy, double* __restrict__ out) {
  const int64_t total = G * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / D;
    const int c = (int)(t - g * D);
    const int64_t b = offs[g], e = offs[g + 1];
    RowSrcD src{rows, D, c};
    double acc = strategy == 0 ? pool_sequential<0>(src, b, reduceat_end(b, e, g == G - 1, offs[G]))
                               : pool_scatter<0>(src, b, e);
    if (mode == 1 && e > b) acc = __ddiv_rn(acc, (double)(e - b));
    out[g * D + c] = acc;
  }
}

// integer rows: wrapping int64 sums (order-independent, so one kernel serves
// both strategies)
__global__ void k_segment_sum_i64(const int64_t* __restrict__ rows, int D, const int64_t* __restrict__ offs,
                                  int64_t G, int64_t* __restrict__ out) {
  const int64_t total = G * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / D;
    const int c = (int)(t - g * D);
    uint64_t acc = 0;
    for (int64_t p = offs[g]; p < offs[g + 1]; ++p) acc += (uint64_t)__ldg(rows + p * D + c);
    out[t] = (int64_t)acc;
  }
}

// 8-byte elements (float64 or int64 rows): a bit copy, pad given as bits
__global__ void k_segment_tile_x64(const uint64_t* __restrict__ rows, int D, const int64_t* __restrict__ offs,
                                   int64_t G, int64_t k, uint64_t pad, uint64_t* __restrict__ out) {
  const int64_t total = G * k * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gj = t / D;
    const int c = (int)(t - gj * D);
    const int64_t g = gj / k, j = gj - g * k;
    const int64_t b = offs[g], len = offs[g + 1] - b;
    out[t] = j < len ? __ldg(rows + (b + j) * D + c) : pad;
  }
}

template <int VEC>
__global__ void k_segment_tile(const float* __restrict__ rows, int D, const int64_t* __restrict__ offs, int64_t G,
                               int64_t k, float pad, float* __restrict__ out) {
  const int per_row = D / VEC;
  const int64_t total = G * k * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t gj = t / per_row;
    int c = (int)(t - gj * per_row) * VEC;
    int64_t g = gj / k, j = gj - g * k;
    int64_t b = offs[g], len = offs[g + 1] - b;
    float* d = out + gj * D + c;
    if (j < len) {
      if constexpr (VEC == 4) st4(d, ldg4(rows + (b + j) * D + c));
      else d[0] = __ldg(rows + (b + j) * D + c);
    } else {
      if constexpr (VEC == 4) st4(d, make_float4(pad, pad, pad, pad));
      else d[0] = pad;
    }
  }
}

// code: 1 = offs[0] != 0, 2 = decreasing, 3 = end != n
__global__ void k_validate(const int64_t* __restrict__ offs, int64_t len, int64_t n, unsigned long long* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 && offs[0] != 0) atomicMin(flag, 1ull);
    if (i + 1 < len && offs[i + 1] < offs[i]) atomicMin(flag, 2ull);
    if (i == len - 1 && offs[i] != n) atomicMin(flag, 3ull);
  }
}

// RaggedTensor.truncate (ragged.py:139-163)
__global__ void k_trunc_lens(const int64_t* __restrict__ offs, int64_t rows, int64_t max_len,
                             int64_t* __restrict__ keep) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = offs[r + 1] - offs[r];
    keep[r] = l < max_len ? l : max_len;
  }
}

__global__ void k_trunc_index(const int64_t* __restrict__ offs, const int64_t* __restrict__ noffs, int64_t rows,
                              int tail, int64_t* __restrict__ src) {
  // one warp per row: rows are long (sequence features), copy index spans
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    int64_t nb = noffs[r], keep = noffs[r + 1] - nb;
    int64_t start = tail ? offs[r + 1] - keep : offs[r];
    for (int64_t j = lane; j < keep; j += 32) src[nb + j] = start + j;
  }
}

template <class E>
__global__ void k_gather_elems(const E* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                               E* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

// one warp per row; element = W bytes-words of type E (width elements)
template <class E>
__global__ void k_pad_dense(const E* __restrict__ vals, int64_t width, const int64_t* __restrict__ offs, int64_t rows,
                            int64_t max_len, E pad, E* __restrict__ out, uint8_t* __restrict__ mask,
                            unsigned long long* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    int64_t b = offs[r], len = offs[r + 1] - b;
    if (len > max_len && lane == 0) atomicMin(flag, (unsigned long long)r);
    for (int64_t j = lane; j < max_len * width; j += 32) {
      int64_t e = j / width;
      out[r * max_len * width + j] = e < len ? vals[b * width + j] : pad;
    }
    for (int64_t j = lane; j < max_len; j += 32) mask[r * max_len + j] = j < len;
  }
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_segment_reduce(const float* rows, int64_t n, int64_t dim, const int64_t* offsets, int64_t num_segments,
                       int32_t mode, int32_t strategy, float* out, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (num_segments <= 0 || dim <= 0) return SKB_OK;
  const int D = (int)dim;
  const bool v4 = D % 4 == 0 && (uintptr_t)rows % 16 == 0 && (uintptr_t)out % 16 == 0;
  if (strategy == 0 && n >= 256 * num_segments) {  // long sequential segments: warp-parallel pairwise leaves
    if (v4)
      k_segment_reduce_warp<4><<<grid_for(num_segments * (D / 4) * 32, 256), 256, 0, s>>>(rows, D, offsets,
                                                                                          num_segments, mode, out);
    else
      k_segment_reduce_warp<1><<<grid_for(num_segments * D * 32, 256), 256, 0, s>>>(rows, D, offsets, num_segments,
                                                                                    mode, out);
    SKB_LAUNCH_CHECK();
    return SKB_OK;
  }
  if (v4)
    k_segment_reduce<4><<<grid_for(num_segments * (D / 4), 128), 128, 0, s>>>(rows, D, offsets, num_segments, mode,
                                                                             strategy, out);
  else
    k_segment_reduce<1><<<grid_for(num_segments * D, 128), 128, 0, s>>>(rows, D, offsets, num_segments, mode, strategy,
                                                                       out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_segment_tile(const float* rows, int64_t n, int64_t dim, const int64_t* offsets, int64_t num_segments,
                     int64_t k, float pad, float* out, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  (void)n;
  if (k < 0) raise(SKB_E_VALUE, k, "k must be >= 0");
  if (num_segments <= 0 || k == 0 || dim <= 0) return SKB_OK;
  const int D = (int)dim;
  if (D % 4 == 0 && (uintptr_t)rows % 16 == 0 && (uintptr_t)out % 16 == 0)
    k_segment_tile<4><<<grid_for(num_segments * k * (D / 4), 256), 256, 0, s>>>(rows, D, offsets, num_segments, k, pad,
                                                                               out);
  else
    k_segment_tile<1><<<grid_for(num_segments * k * D, 256), 256, 0, s>>>(rows, D, offsets, num_segments, k, pad, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_segment_reduce_f64(const double* rows, int64_t n, int64_t dim, const int64_t* offsets, int64_t num_segments,
                           int32_t mode, int32_t strategy, double* out, void* stream) {
  SKB_API_BEGIN
  (void)n;
  if (num_segments <= 0 || dim <= 0) return SKB_OK;
  k_segment_reduce_f64<<<grid_for(num_segments * dim, 128), 128, 0, as_stream(stream)>>>(
      rows, (int)dim, offsets, num_segments, mode, strategy, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_segment_sum_i64(const int64_t* rows, int64_t n, int64_t dim, const int64_t* offsets, int64_t num_segments,
                        int64_t* out, void* stream) {
  SKB_API_BEGIN
  (void)n;
  if (num_segments <= 0 || dim <= 0) return SKB_OK;
  k_segment_sum_i64<<<grid_for(num_segments * dim, 128), 128, 0, as_stream(stream)>>>(rows, (int)dim, offsets,
                                                                                      num_segments, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_segment_tile_x64(const void* rows, int64_t n, int64_t dim, const int64_t* offsets, int64_t num_segments,
                         int64_t k, uint64_t pad_bits, void* out, void* stream) {
  SKB_API_BEGIN
  (void)n;
  if (k < 0) raise(SKB_E_VALUE, k, "k must be >= 0");
  if (num_segments <= 0 || k == 0 || dim <= 0) return SKB_OK;
  k_segment_tile_x64<<<grid_for(num_segments * k * dim, 256), 256, 0, as_stream(stream)>>>(
      static_cast<const uint64_t*>(rows), (int)dim, offsets, num_segments, k, pad_bits, static_cast<uint64_t*>(out));
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_validate_offsets(const int64_t* offsets, int64_t len, int64_t n_expected, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (len < 1) raise(SKB_E_VALUE, 1, "offsets must be a 1-D array of length num_rows+1");
  DevFlag f(s);
  k_validate<<<grid_for(len, 256), 256, 0, s>>>(offsets, len, n_expected, f.ptr());
  SKB_LAUNCH_CHECK();
  int64_t code = f.read();
  if (code == 1) raise(SKB_E_VALUE, 1, "offsets must start at 0");
  if (code == 2) raise(SKB_E_VALUE, 2, "offsets must be nondecreasing");
  if (code == 3) raise(SKB_E_VALUE, 3, "offsets end != number of rows");
  SKB_API_END
}

int skb_ragged_truncate(const int64_t* offs, int64_t rows, int64_t max_len, int32_t tail, int64_t* new_offs,
                        int64_t* src_index, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (max_len < 0) raise(SKB_E_VALUE, max_len, "max_len must be >= 0");
  if (rows <= 0) {
    SKB_CUDA(cudaMemsetAsync(new_offs, 0, sizeof(int64_t), s));
    return SKB_OK;
  }
  Scratch keep(sizeof(int64_t) * rows, s);
  k_trunc_lens<<<grid_for(rows, 256), 256, 0, s>>>(offs, rows, max_len, keep.as<int64_t>());
  SKB_LAUNCH_CHECK();
  scan_exclusive_i64(keep.as<int64_t>(), new_offs, rows, new_offs + rows, s);
  if (src_index) {
    k_trunc_index<<<grid_for(rows * 32, 256), 256, 0, s>>>(offs, new_offs, rows, tail, src_index);
    SKB_LAUNCH_CHECK();
  }
  SKB_API_END
}

int skb_gather_elems(const void* src, int64_t elem_bytes, const int64_t* idx, int64_t n, void* out, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  unsigned g = grid_for(n, 256);
  if (elem_bytes == 8)
    k_gather_elems<<<g, 256, 0, s>>>((const uint64_t*)src, idx, n, (uint64_t*)out);
  else if (elem_bytes == 4)
    k_gather_elems<<<g, 256, 0, s>>>((const uint32_t*)src, idx, n, (uint32_t*)out);
  else if (elem_bytes == 1)
    k_gather_elems<<<g, 256, 0, s>>>((const uint8_t*)src, idx, n, (uint8_t*)out);
  else
    raise(SKB_E_ARG, elem_bytes, "elem_bytes must be 1, 4 or 8");
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_ragged_pad_dense(const void* values, int64_t elem_bytes, int64_t width, const int64_t* offs, int64_t rows,
                         int64_t max_len, const void* pad_host, void* out, uint8_t* mask, void* stream) {
  SKB_API_BEGIN
  cudaStream_t s = as_stream(stream);
  if (rows <= 0 || max_len < 0) return SKB_OK;
  DevFlag f(s);
  unsigned g = grid_for(rows * 32, 256);
  if (elem_bytes == 8) {
    uint64_t pad;
    memcpy(&pad, pad_host, 8);
    k_pad_dense<<<g, 256, 0, s>>>((const uint64_t*)values, width, offs, rows, max_len, pad, (uint64_t*)out, mask,
                                  f.ptr());
  } else if (elem_bytes == 4) {
    uint32_t pad;
    memcpy(&pad, pad_host, 4);
    k_pad_dense<<<g, 256, 0, s>>>((const uint32_t*)values, width, offs, rows, max_len, pad, (uint32_t*)out, mask,
                                  f.ptr());
  } else {
    raise(SKB_E_ARG, elem_bytes, "elem_bytes must be 4 or 8");
  }
  SKB_LAUNCH_CHECK();
  if (f.read() >= 0) raise(SKB_E_VALUE, 0, "row longer than max_len; truncate first");
  SKB_API_END
}

}  // extern "C"
