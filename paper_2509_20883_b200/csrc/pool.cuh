// pool.cuh — bit-exact pooling folds over a row source (direct rows or
// arena rows addressed through slots).  VEC = 4 handles 4 columns per thread
// with 128-bit loads; VEC = 1 is the generic-D fallback.
#pragma once
#include "common.cuh"

namespace skb {

template <int VEC> struct VecT;
template <> struct VecT<4> { using T = float4; };
template <> struct VecT<1> { using T = float; };
template <> struct VecT<0> { using T = double; };  // float64 rows (segments.py keeps the input dtype)

template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T vfill(float x);
template <> __device__ __forceinline__ float4 vfill<4>(float x) { return make_float4(x, x, x, x); }
template <> __device__ __forceinline__ float vfill<1>(float x) { return x; }
template <> __device__ __forceinline__ double vfill<0>(float x) { return (double)x; }

template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T vadd(typename VecT<VEC>::T a, typename VecT<VEC>::T b);
template <> __device__ __forceinline__ float4 vadd<4>(float4 a, float4 b) { return add4(a, b); }
template <> __device__ __forceinline__ float vadd<1>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double vadd<0>(double a, double b) { return __dadd_rn(a, b); }

template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T vshfl(typename VecT<VEC>::T v, int src);
template <> __device__ __forceinline__ float4 vshfl<4>(float4 v, int src) {
  return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                     __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}
template <> __device__ __forceinline__ float vshfl<1>(float v, int src) { return __shfl_sync(0xffffffffu, v, src); }

template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T vload(const float* p);
template <> __device__ __forceinline__ float4 vload<4>(const float* p) { return ldg4(p); }
template <> __device__ __forceinline__ float vload<1>(const float* p) { return __ldg(p); }

template <int VEC> __device__ __forceinline__ void vstore(float* p, typename VecT<VEC>::T v);
template <> __device__ __forceinline__ void vstore<4>(float* p, float4 v) { st4(p, v); }
template <> __device__ __forceinline__ void vstore<1>(float* p, float v) { *p = v; }

template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T vdiv(typename VecT<VEC>::T a, float d);
template <> __device__ __forceinline__ float4 vdiv<4>(float4 a, float d) {
  return make_float4(__fdiv_rn(a.x, d), __fdiv_rn(a.y, d), __fdiv_rn(a.z, d), __fdiv_rn(a.w, d));
}
template <> __device__ __forceinline__ float vdiv<1>(float a, float d) { return __fdiv_rn(a, d); }

// rows[p * D + c]
struct RowSrc {
  const float* rows;
  int D;
  int c;
  template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T load(int64_t p) const {
    return vload<VEC>(rows + p * D + c);
  }
};

// rows[p * D + c] of a float64 matrix (one column per thread)
struct RowSrcD {
  const double* rows;
  int D;
  int c;
  template <int VEC> __device__ __forceinline__ double load(int64_t p) const { return __ldg(rows + p * D + c); }
};

// np.add.at semantics: ((+0 + r_b) + r_{b+1}) + ...
template <int VEC, class Src>
__device__ __forceinline__ typename VecT<VEC>::T pool_scatter(const Src& s, int64_t b, int64_t e) {
  using T = typename VecT<VEC>::T;
  T acc = vfill<VEC>(0.f);
  int64_t p = b;
  // 4 independent loads in flight, folded strictly in order
  for (; p + 4 <= e; p += 4) {
    T x0 = s.template load<VEC>(p), x1 = s.template load<VEC>(p + 1), x2 = s.template load<VEC>(p + 2),
      x3 = s.template load<VEC>(p + 3);
    acc = vadd<VEC>(vadd<VEC>(vadd<VEC>(vadd<VEC>(acc, x0), x1), x2), x3);
  }
  for (; p < e; ++p) acc = vadd<VEC>(acc, s.template load<VEC>(p));
  return acc;
}

// numpy pairwise_sum leaf, n <= 128 elements starting at position b
template <int VEC, class Src>
__device__ __forceinline__ typename VecT<VEC>::T pw_leaf(const Src& s, int64_t b, int64_t n) {
  using T = typename VecT<VEC>::T;
  if (n < 8) {
    T acc = vfill<VEC>(-0.f);
    for (int64_t i = 0; i < n; ++i) acc = vadd<VEC>(acc, s.template load<VEC>(b + i));
    return acc;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = s.template load<VEC>(b + j);
  int64_t i = 8;
  const int64_t lim = n - (n % 8);
  for (; i + 16 <= lim; i += 16) {  // two 8-row blocks' loads in flight; same add order per accumulator
    T x[8], y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = s.template load<VEC>(b + i + j);
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = s.template load<VEC>(b + i + 8 + j);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = vadd<VEC>(vadd<VEC>(r[j], x[j]), y[j]);
  }
  for (; i < lim; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = vadd<VEC>(r[j], s.template load<VEC>(b + i + j));
  }
  T res = vadd<VEC>(vadd<VEC>(vadd<VEC>(r[0], r[1]), vadd<VEC>(r[2], r[3])),
                    vadd<VEC>(vadd<VEC>(r[4], r[5]), vadd<VEC>(r[6], r[7])));
  for (; i < n; ++i) res = vadd<VEC>(res, s.template load<VEC>(b + i));
  return res;
}

// numpy pairwise_sum over [b, b+n): recursion unrolled with an explicit stack
template <int VEC, class Src>
__device__ typename VecT<VEC>::T pw_sum(const Src& s, int64_t b, int64_t n) {
  using T = typename VecT<VEC>::T;
  if (n <= 128) return pw_leaf<VEC>(s, b, n);
  struct Frame {
    int64_t b, n;
    T left;
    int stage;
  };
  Frame st[48];
  int sp = 0;
  st[sp++] = Frame{b, n, vfill<VEC>(0.f), 0};
  T result = vfill<VEC>(0.f);
  bool have = false;
  while (sp > 0) {
    Frame& f = st[sp - 1];
    if (!have) {
      if (f.n <= 128) {
        result = pw_leaf<VEC>(s, f.b, f.n);
        have = true;
        --sp;
        continue;
      }
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      st[sp++] = Frame{f.b, n2, vfill<VEC>(0.f), 0};
    } else {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      if (f.stage == 0) {
        f.left = result;
        f.stage = 1;
        have = false;
        st[sp++] = Frame{f.b + n2, f.n - n2, vfill<VEC>(0.f), 0};
      } else {
        result = vadd<VEC>(f.left, result);
        --sp;
      }
    }
  }
  return result;
}

// segments.py:44-47 clips the reduceat indices to n-1, so a non-final
// segment that ends at row n (only empty segments follow it) is reduced over
// [b, n-1): its last row is dropped.  Reproduced for parity.
__device__ __forceinline__ int64_t reduceat_end(int64_t b, int64_t e, bool last_segment, int64_t n_end) {
  return (!last_segment && e == n_end && e - b >= 2) ? e - 1 : e;
}

// np.add.reduceat semantics: rows[b] + pairwise(rows[b+1:e]); empty -> 0
template <int VEC, class Src>
__device__ __forceinline__ typename VecT<VEC>::T pool_sequential(const Src& s, int64_t b, int64_t e) {
  if (e <= b) return vfill<VEC>(0.f);
  auto first = s.template load<VEC>(b);
  if (e - b == 1) return first;
  return vadd<VEC>(first, pw_sum<VEC>(s, b + 1, e - b - 1));
}

}  // namespace skb
