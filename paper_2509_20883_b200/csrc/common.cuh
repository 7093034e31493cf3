// common.cuh — shared device/host helpers for libsparsekit_b200 (sm_100a).
//
// Everything here is integer/byte or IEEE-exact float work: the hot path is
// HBM-bound gather/scatter/probe traffic, so the helpers are about coalesced
// 128-bit access, warp-cooperative row groups and stream-ordered scratch —
// not tensor cores (nothing on this path is a dense contraction).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/sparsekit_b200.h"

namespace skb {

// ---------------------------------------------------------------------------
// errors: internal code throws SkbError; every extern "C" entry catches.
// ---------------------------------------------------------------------------
struct SkbError : std::runtime_error {
  int code;
  int64_t arg;
  SkbError(int c, const std::string& m, int64_t a = 0) : std::runtime_error(m), code(c), arg(a) {}
};

[[noreturn]] void raise(int code, int64_t arg, const char* fmt, ...);
int set_error(int code, const char* msg, int64_t arg);
void clear_error();

#define SKB_CUDA(x)                                                                 \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      if (e_ == cudaErrorMemoryAllocation) {                                        \
        cudaGetLastError();                                                         \
        ::skb::raise(SKB_E_NOMEM, 0, "%s: %s", #x, cudaGetErrorString(e_));         \
      }                                                                             \
      ::skb::raise(SKB_E_CUDA, 0, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_),     \
                   __FILE__, __LINE__);                                             \
    }                                                                               \
  } while (0)

// every launch of one of OUR kernels is followed by SKB_LAUNCH_CHECK(); the
// counter backs the bench's gpu_launches claim (CUB internals not counted)
void count_launch();
#define SKB_LAUNCH_CHECK()            \
  do {                                \
    ::skb::count_launch();            \
    SKB_CUDA(cudaGetLastError());     \
  } while (0)

#define SKB_API_BEGIN \
  try {               \
    ::skb::clear_error();
#define SKB_API_END                                                      \
  return SKB_OK;                                                         \
  }                                                                      \
  catch (const ::skb::SkbError& e) {                                     \
    return ::skb::set_error(e.code, e.what(), e.arg);                    \
  }                                                                      \
  catch (const std::exception& e) {                                      \
    return ::skb::set_error(SKB_E_CUDA, e.what(), 0);                    \
  }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// device facts and grid sizing (148 SMs on B200; grids are SM multiples)
// ---------------------------------------------------------------------------
int sm_count();
inline unsigned grid_for(int64_t work_items, int threads, int waves_per_sm = 8) {
  int64_t want = (work_items + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * waves_per_sm;
  if (want < 1) want = 1;
  return (unsigned)(want < cap ? want : cap);
}

// ---------------------------------------------------------------------------
// stream-ordered scratch (cudaMallocAsync on a retained pool)
// ---------------------------------------------------------------------------
void* scratch_alloc(size_t bytes, cudaStream_t s);
void scratch_free(void* p, cudaStream_t s);

struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(size_t b, cudaStream_t st) : bytes(b), s(st) { p = b ? scratch_alloc(b, st) : nullptr; }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  Scratch(Scratch&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; }
  Scratch& operator=(Scratch&& o) noexcept {
    release();
    p = o.p; bytes = o.bytes; s = o.s; o.p = nullptr;
    return *this;
  }
  ~Scratch() { release(); }
  void release() {
    if (p) scratch_free(p, s);
    p = nullptr;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Pinned host mailbox for small device->host readbacks (flags, counts).
struct HostMailbox {
  int64_t* h = nullptr;
  int n = 0;
  explicit HostMailbox(int count);
  ~HostMailbox();
};

// pinned int64[4] owned by the calling host thread (small synchronous readbacks)
int64_t* pinned_mailbox();

// Device error flag: {code, arg}; kernels record the first (lowest-index)
// offending element with atomicMin on a packed key.
struct DevFlag {
  Scratch buf;  // int64[2]: [0] = min offending index (INT64_MAX = none), [1] = unused
  cudaStream_t s;
  explicit DevFlag(cudaStream_t st);
  unsigned long long* ptr() const { return buf.as<unsigned long long>(); }
  // synchronizes; returns the minimal flagged index or -1
  int64_t read();
};

// ---------------------------------------------------------------------------
// hashing (bit-exact with hashing.py)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kFnvBasis = 0xCBF29CE484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001B3ull;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// Bucket hash for open addressing.  Deliberately independent of mix64 so a
// shard that owns keys with mix64(k) % S == r still spreads over all buckets
// (SURVEY §7.3 hard part 3): Murmur3 fmix64 of the key.
__host__ __device__ __forceinline__ uint64_t bucket_hash(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

__host__ __device__ __forceinline__ uint64_t owner_of(int64_t key, uint64_t S) {
  uint64_t h = mix64((uint64_t)key);
  return (S & (S - 1)) == 0 ? (h & (S - 1)) : (h % S);
}

// ---------------------------------------------------------------------------
// open-addressing hash table entries {key, val}; 16-byte aligned so one probe
// is one 32-byte sector.  EMPTY marks a free bucket; a real key equal to EMPTY
// lives in the side entry at index `cap` (full int64 key space is admissible).
// ---------------------------------------------------------------------------
constexpr long long kEmptyKey = (long long)0x8000000000000000ull;  // INT64_MIN
struct __align__(16) HEntry {
  long long key;
  long long val;
};

// plain 128-bit probe load: tables are never written while a kernel probes them
__device__ __forceinline__ HEntry ld_entry(const HEntry* p) {
  longlong2 v = *reinterpret_cast<const longlong2*>(p);
  return HEntry{v.x, v.y};
}

// Fill cap+1 entries with {EMPTY, init_val}.
void ht_fill(HEntry* t, int64_t count, long long init_val, cudaStream_t s);

__host__ __device__ __forceinline__ int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ---------------------------------------------------------------------------
// vector helpers
// ---------------------------------------------------------------------------
// segment of x in the ascending prefix array pre[0..S] (pre[S] = total)
__device__ __forceinline__ int seg_of(const int64_t* __restrict__ pre, int S, int64_t x) {
  int lo = 0, hi = S;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(pre + mid) <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// Destination of fold-only output row `key`: out + key*D, or (peers set) the
// row's place in the receive window of the rank owning key's segment
// (segments pre[j]..pre[j+1] go to peers[j] from row base[j]) — the
// requester's folded gradients stored straight over NVLink, no staging copy.
struct RowOut {
  const int64_t* pre = nullptr;
  int S = 0;
  float* const* peers = nullptr;
  const int64_t* base = nullptr;
  __device__ __forceinline__ float* row(float* out, uint32_t key, int D) const {
    if (!peers) return out + (int64_t)key * D;
    const int j = seg_of(pre, S, key);
    return peers[j] + (__ldg(base + j) + ((int64_t)key - __ldg(pre + j))) * D;
  }
};

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// streaming (L1 no-allocate) 128-bit load for rows read once
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// CUB wrappers (defined in cubwrap.cu; only that TU instantiates CUB)
// ---------------------------------------------------------------------------
// exclusive scan of int64 flags/values, out[n]; total (device int64*) optional
void scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total, cudaStream_t s);
void scan_exclusive_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, int64_t* total,
                               cudaStream_t s);
void scan_exclusive_u8_to_i64(const uint8_t* in, int64_t* out, int64_t n, int64_t* total, cudaStream_t s);
// ordered compaction of indices i in [0,n) with flags[i] != 0 -> out, count -> *d_count
void select_flagged_index(const uint8_t* flags, int64_t n, int64_t* out, int64_t* d_count,
                          cudaStream_t s);
void select_flagged_index32(const uint8_t* flags, int64_t n, uint32_t* out, int64_t* d_count,
                            cudaStream_t s);
// stable radix sort of (uint32 key, uint32 val) pairs on bits [0, end_bit)
void sort_pairs_u32(const uint32_t* k_in, uint32_t* k_out, const uint32_t* v_in, uint32_t* v_out,
                    int64_t n, int end_bit, cudaStream_t s);
// the same sort with caller-owned temp storage (no allocation per call)
size_t sort_pairs_u32_bytes(int64_t n, int end_bit);
void sort_pairs_u32_ws(const uint32_t* k_in, uint32_t* k_out, const uint32_t* v_in, uint32_t* v_out, int64_t n,
                       int end_bit, void* ws, size_t ws_bytes, cudaStream_t s);
// stable radix sort of (int64 key, int64 val) pairs (signed order); keys
// known to lie in [0, 2^end_bit) may pass end_bit < 64 (fewer passes)
void sort_pairs_i64(const int64_t* k_in, int64_t* k_out, const int64_t* v_in, int64_t* v_out,
                    int64_t n, cudaStream_t s, int end_bit = 64);
// segment heads of a sorted u32 key array: out = indices i where i==0 or k[i]!=k[i-1]
void select_run_heads_u32(const uint32_t* keys, int64_t n, uint32_t* out, int64_t* d_count,
                          cudaStream_t s);

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

}  // namespace skb
