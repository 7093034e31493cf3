// cubwrap.cu — the only translation unit that instantiates CUB device-wide
// primitives (scan / select / stable radix sort).  Temp storage comes from the
// stream-ordered scratch pool.
#include <cub/cub.cuh>

#include "common.cuh"

namespace skb {

namespace {
template <class F>
void run_cub(F&& f, cudaStream_t s) {
  size_t bytes = 0;
  SKB_CUDA(f(nullptr, bytes));
  Scratch tmp(bytes ? bytes : 16, s);
  SKB_CUDA(f(tmp.p, bytes));
}

__global__ void k_total_i64(const int64_t* excl, const int64_t* in, int64_t n, int64_t* total) {
  *total = n ? excl[n - 1] + in[n - 1] : 0;
}
__global__ void k_total_i32(const int64_t* excl, const int32_t* in, int64_t n, int64_t* total) {
  *total = n ? excl[n - 1] + (int64_t)in[n - 1] : 0;
}

struct HeadOp {
  const uint32_t* k;
  __device__ __forceinline__ bool operator()(const int64_t& i) const {
    return i == 0 || k[i] != k[i - 1];
  }
};
}  // namespace

void scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total, cudaStream_t s) {
  if (n > 0)
    run_cub([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, in, out, n, s); }, s);
  if (total) {
    k_total_i64<<<1, 1, 0, s>>>(out, in, n, total);
    SKB_LAUNCH_CHECK();
  }
}

void scan_exclusive_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, int64_t* total,
                               cudaStream_t s) {
  if (n > 0) {
    run_cub(
        [&](void* t, size_t& b) {
          return cub::DeviceScan::ExclusiveScan(t, b, in, out, cub::Sum(), (int64_t)0, n, s);
        },
        s);
  }
  if (total) {
    k_total_i32<<<1, 1, 0, s>>>(out, in, n, total);
    SKB_LAUNCH_CHECK();
  }
}

__global__ void k_total_u8(const int64_t* excl, const uint8_t* in, int64_t n, int64_t* total) {
  *total = n ? excl[n - 1] + (int64_t)in[n - 1] : 0;
}

void scan_exclusive_u8_to_i64(const uint8_t* in, int64_t* out, int64_t n, int64_t* total, cudaStream_t s) {
  if (n > 0) {
    run_cub(
        [&](void* t, size_t& b) {
          return cub::DeviceScan::ExclusiveScan(t, b, in, out, cub::Sum(), (int64_t)0, n, s);
        },
        s);
  }
  if (total) {
    k_total_u8<<<1, 1, 0, s>>>(out, in, n, total);
    SKB_LAUNCH_CHECK();
  }
}

void select_flagged_index(const uint8_t* flags, int64_t n, int64_t* out, int64_t* d_count,
                          cudaStream_t s) {
  if (n == 0) {
    SKB_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
    return;
  }
  cub::CountingInputIterator<int64_t> it(0);
  run_cub([&](void* t, size_t& b) { return cub::DeviceSelect::Flagged(t, b, it, flags, out, d_count, n, s); },
          s);
}

void select_flagged_index32(const uint8_t* flags, int64_t n, uint32_t* out, int64_t* d_count,
                            cudaStream_t s) {
  if (n == 0) {
    SKB_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
    return;
  }
  cub::CountingInputIterator<uint32_t> it(0);
  run_cub([&](void* t, size_t& b) { return cub::DeviceSelect::Flagged(t, b, it, flags, out, d_count, n, s); },
          s);
}

void sort_pairs_u32(const uint32_t* k_in, uint32_t* k_out, const uint32_t* v_in, uint32_t* v_out,
                    int64_t n, int end_bit, cudaStream_t s) {
  if (n == 0) return;
  run_cub(
      [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, k_in, k_out, v_in, v_out, n, 0, end_bit, s);
      },
      s);
}

size_t sort_pairs_u32_bytes(int64_t n, int end_bit) {
  size_t bytes = 0;
  SKB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                           (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, end_bit, nullptr));
  return bytes;
}

void sort_pairs_u32_ws(const uint32_t* k_in, uint32_t* k_out, const uint32_t* v_in, uint32_t* v_out, int64_t n,
                       int end_bit, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (n == 0) return;
  SKB_CUDA(cub::DeviceRadixSort::SortPairs(ws, ws_bytes, k_in, k_out, v_in, v_out, n, 0, end_bit, s));
}

void sort_pairs_i64(const int64_t* k_in, int64_t* k_out, const int64_t* v_in, int64_t* v_out,
                    int64_t n, cudaStream_t s, int end_bit) {
  if (n == 0) return;
  run_cub(
      [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, k_in, k_out, v_in, v_out, n, 0, end_bit, s);
      },
      s);
}

void select_run_heads_u32(const uint32_t* keys, int64_t n, uint32_t* out, int64_t* d_count,
                          cudaStream_t s) {
  if (n == 0) {
    SKB_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
    return;
  }
  cub::CountingInputIterator<int64_t> it(0);
  HeadOp op{keys};
  run_cub([&](void* t, size_t& b) { return cub::DeviceSelect::If(t, b, it, out, d_count, n, op, s); }, s);
}

}  // namespace skb
