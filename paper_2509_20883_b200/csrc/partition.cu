// partition.cu — fused dedup + owner partition (unique_partition,
// sharding.py:74-100), PartitionResult.restore (sharding.py:58-66) and the
// gradient pre-aggregation fold (sharding.py:283-290).
//
// Dedup: every position inserts its id into an open-addressing scratch table
// with atomicMin(first position); a position is a first occurrence iff the
// table's minimum equals its own index.  An ordered compaction of those flags
// yields the unique ids in global first-occurrence order; for S > 1 a 1-pass
// stable radix sort on the owner shard gives the stable per-shard split.  The
// per-shard rank is written back into the scratch entry so every position's
// inverse is one probe-free lookup (hslot cached from the insert pass).
#include <cstdlib>

#include "common.cuh"
#include "rows.cuh"
#include "partition.cuh"
#include "longfold.cuh"

namespace skb {

__device__ __forceinline__ int64_t ht_insert_min(HEntry* t, uint64_t mask, int64_t cap, long long key,
                                                 long long pos) {
  int64_t i;
  if (key == kEmptyKey) {
    i = cap;
  } else {  // read before any atomic: repeated (hot) keys find their bucket without one
    i = (int64_t)(bucket_hash((uint64_t)key) & mask);
    while (true) {
      long long k = __ldcg(&t[i].key);
      if (k == kEmptyKey)
        k = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&t[i].key), (unsigned long long)kEmptyKey,
                                 (unsigned long long)key);
      if (k == kEmptyKey || k == key) break;
      i = (int64_t)(((uint64_t)i + 1) & mask);
    }
  }
  if (__ldcg(&t[i].val) > pos) atomicMin(&t[i].val, pos);
  return i;
}

__global__ void k_dedup_insert(const int64_t* __restrict__ ids, int64_t n, HEntry* t, uint64_t mask, int64_t cap,
                               int64_t* __restrict__ hslot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    hslot[i] = ht_insert_min(t, mask, cap, ids[i], i);
}

__global__ void k_first_flags(const HEntry* t, const int64_t* __restrict__ hslot, int64_t n,
                              uint8_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (t[hslot[i]].val == i) ? 1 : 0;
}

__global__ void k_emit_single(const int64_t* __restrict__ ids, const int64_t* __restrict__ fpos,
                              const int64_t* __restrict__ d_u, const int64_t* __restrict__ hslot, HEntry* t,
                              int64_t* __restrict__ uniq) {
  const int64_t U = *d_u;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < U; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = fpos[k];
    uniq[k] = ids[p];
    t[hslot[p]].val = k;
  }
}

__global__ void k_owner_keys(const int64_t* __restrict__ ids, const int64_t* __restrict__ fpos,
                             const int64_t* __restrict__ d_u, int64_t n, uint64_t S, uint32_t* __restrict__ sk,
                             uint32_t* __restrict__ kv) {
  const int64_t U = *d_u;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    sk[k] = k < U ? (uint32_t)owner_of(ids[fpos[k]], S) : (uint32_t)S;
    kv[k] = (uint32_t)k;
  }
}

__global__ void k_shard_starts(const uint32_t* __restrict__ sk, const int64_t* __restrict__ d_u, int64_t S,
                               int64_t* __restrict__ starts) {
  const int64_t U = *d_u;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= S; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = U;  // lower_bound of s in sk[0:U]
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sk[mid] < (uint32_t)s) lo = mid + 1; else hi = mid;
    }
    starts[s] = lo;
  }
}

__global__ void k_shard_counts(const int64_t* __restrict__ starts, int64_t S, int64_t* __restrict__ counts) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x)
    counts[s] = starts[s + 1] - starts[s];
}

__global__ void k_emit_sharded(const int64_t* __restrict__ ids, const int64_t* __restrict__ fpos,
                               const int64_t* __restrict__ d_u, const uint32_t* __restrict__ sk,
                               const uint32_t* __restrict__ kv, const int64_t* __restrict__ starts,
                               const int64_t* __restrict__ hslot, HEntry* t, int64_t* __restrict__ uniq) {
  const int64_t U = *d_u;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < U; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = fpos[kv[j]];
    uniq[j] = ids[p];
    t[hslot[p]].val = j - starts[sk[j]];
  }
}

__global__ void k_inverse(const int64_t* __restrict__ ids, const int64_t* __restrict__ hslot, const HEntry* t,
                          int64_t n, uint64_t S, int64_t* __restrict__ inv_shard, int64_t* __restrict__ inv_pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    inv_pos[i] = t[hslot[i]].val;
    if (inv_shard) inv_shard[i] = S == 1 ? 0 : (int64_t)owner_of(ids[i], S);
  }
}

// ---------------------------------------------------------------------------
// Stable multi-split for S <= kSplitMaxS in four launches, no sort, no
// look-back spinning and no host round trip:
//   k_part_init    position table all kNoPos + zeroed tile-done counter
//   k_part_insert  every position claims its key's bucket (one 32-bit CAS)
//                  or lowers the bucket's position to its own index -> the
//                  bucket holds the key's first occurrence
//   k_part_count   tile of kPartTile positions per block: first occurrences
//                  ranked per owner shard inside the tile (__match_any_sync +
//                  per-warp running counts) -> lrank[i]; per-(shard, tile)
//                  counts; the LAST block to finish scans them shard-major
//                  into global offsets (shard base included) and the counts
//   k_part_emit    per position i with first occurrence f (the bucket value):
//                  global rank = off[shard][tile(f)] + lrank[f];
//                  inv_pos = rank - base[shard]; f == i stores the id
// Output order is exactly sharding.py:87-100's (global first-occurrence
// order within each shard, shards concatenated in shard order).
constexpr int kSplitMaxS = 256;
constexpr int kPartThreads = 256;
constexpr int kPartRounds = 4;                             // 32-position rounds per warp
constexpr int kPartTile = kPartThreads * kPartRounds;      // 1024 positions per tile
constexpr int kPartU = 1;  // insert chains per thread (4 in flight measured slower: 30.6 vs 24.4 us, L2 atomics)
constexpr int kScanSmem = 8192;                            // int32 staging of the tile-count scan

// The split path's table holds ONE uint32 per bucket: the first position of
// the key that owns it (the key itself is read back through ids[], which is
// L2-resident).  4 B per bucket instead of a 16-B {key, first} entry: the
// table of 1M positions is 8 MB instead of 32 MB, a claim is one 32-bit CAS,
// and no key value has to be reserved as "empty".
constexpr uint32_t kNoPos = 0xFFFFFFFFu;

// table fill + zeroed counters, one launch (cap is a power of two >= 64)
__global__ void k_part_init(uint32_t* t, int64_t cap, unsigned long long* status, int64_t nstatus) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap / 4; i += stride)
    reinterpret_cast<uint4*>(t)[i] = make_uint4(kNoPos, kNoPos, kNoPos, kNoPos);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nstatus; i += stride) status[i] = 0ull;
}

// every position claims its key's bucket (CAS from kNoPos) or, finding the
// key there, lowers the bucket to its own position: the bucket ends holding
// the key's first occurrence.  The first CAS of each of a thread's kPartU
// positions is issued before any result is used (kPartU round trips in
// flight); CAS first, no plain load before it: most positions of a batch
// carry a key not seen yet, and for them the CAS is the only round trip.
template <int kPartU>
__global__ void __launch_bounds__(kPartThreads) k_part_insert(const int64_t* __restrict__ ids, int64_t n,
                                                              uint32_t* t, uint64_t mask,
                                                              uint32_t* __restrict__ hslot) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n; base += stride * kPartU) {
    long long key[kPartU];
    uint64_t h[kPartU];
    uint32_t v[kPartU];
#pragma unroll
    for (int u = 0; u < kPartU; ++u) {
      const int64_t i = base + u * stride;
      key[u] = i < n ? ids[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < kPartU; ++u) {
      const int64_t i = base + u * stride;
      h[u] = bucket_hash((uint64_t)key[u]) & mask;
      v[u] = i < n ? atomicCAS(t + h[u], kNoPos, (uint32_t)i) : kNoPos;
    }
#pragma unroll
    for (int u = 0; u < kPartU; ++u) {
      const int64_t i = base + u * stride;
      if (i >= n) continue;
      const uint32_t me = (uint32_t)i;
      while (v[u] != kNoPos) {  // kNoPos: claimed, this position is the first so far
        if (__ldg(ids + v[u]) == key[u]) {  // the key's bucket: keep the smaller position
          if (v[u] > me) atomicMin(t + h[u], me);
          break;
        }
        h[u] = (h[u] + 1) & mask;
        v[u] = atomicCAS(t + h[u], kNoPos, me);
      }
      hslot[i] = (uint32_t)h[u];
    }
  }
}

__global__ void __launch_bounds__(kPartThreads) k_part_count(const int64_t* __restrict__ ids, int64_t n,
                                                             const uint32_t* __restrict__ t,
                                                             const uint32_t* __restrict__ hslot, int S,
                                                             int64_t ntiles, int* __restrict__ off,
                                                             uint32_t* __restrict__ lrank_out,
                                                             unsigned long long* done, int64_t* __restrict__ counts) {
  constexpr int W = kPartThreads / 32;
  __shared__ int sbuf[kScanSmem + kScanSmem / 32];  // wc during the tile, scan staging (padded) in the last block
  int (*wc)[kSplitMaxS] = reinterpret_cast<int (*)[kSplitMaxS]>(sbuf);  // per-warp per-shard counts -> warp bases
  __shared__ bool s_last;
  for (int k = threadIdx.x; k < W * kSplitMaxS; k += blockDim.x) sbuf[k] = 0;
  const int64_t tile = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1;
  const int64_t i0 = tile * kPartTile + (int64_t)w * (32 * kPartRounds) + lane;
  uint32_t hs[kPartRounds];
  long long fv[kPartRounds], key[kPartRounds];
  int sh[kPartRounds], lr[kPartRounds];
  // every load of the tile's rounds in flight before any warp intrinsic
#pragma unroll
  for (int r = 0; r < kPartRounds; ++r)
    if (i0 + r * 32 < n) hs[r] = hslot[i0 + r * 32];
#pragma unroll
  for (int r = 0; r < kPartRounds; ++r) {
    fv[r] = -1;
    if (i0 + r * 32 < n) {
      fv[r] = (long long)t[hs[r]];
      key[r] = ids[i0 + r * 32];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kPartRounds; ++r) {
    const bool first = fv[r] == i0 + r * 32;
    sh[r] = first ? (S == 1 ? 0 : (int)owner_of(key[r], (uint64_t)S)) : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, sh[r]);
    const int lower = __popc(grp & lt_mask);
    lr[r] = first ? wc[w][sh[r]] + lower : 0;
    __syncwarp();
    if (first && lower == 0) wc[w][sh[r]] += __popc(grp);
    __syncwarp();
  }
  __syncthreads();
  for (int k = threadIdx.x; k < S; k += blockDim.x) {  // warp bases inside the tile, tile count
    int run = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int c = wc[q][k];
      wc[q][k] = run;
      run += c;
    }
    off[(int64_t)k * ntiles + tile] = run;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kPartRounds; ++r)
    if (sh[r] >= 0) lrank_out[i0 + r * 32] = (uint32_t)(wc[w][sh[r]] + lr[r]);
  __syncthreads();  // sbuf is reused by the scan
  // last block to finish: exclusive scan of the shard-major counts, staged
  // through shared memory kScanSmem values at a time (all loads in flight)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1ull) == (unsigned long long)(gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t m = (int64_t)S * ntiles;
  constexpr int kPer = kScanSmem / kPartThreads;
  __shared__ int s_sum[W];
  int carry = 0;
  for (int64_t b0 = 0; b0 < m; b0 += kScanSmem) {
    const int64_t cnt = m - b0 < kScanSmem ? m - b0 : kScanSmem;
    for (int k = threadIdx.x; k < cnt; k += kPartThreads) sbuf[k + (k >> 5)] = __ldcg(&off[b0 + k]);
    __syncthreads();
    int loc = 0;
#pragma unroll 8
    for (int k = 0; k < kPer; ++k) {
      const int j = threadIdx.x * kPer + k;
      loc += j < cnt ? sbuf[j + (j >> 5)] : 0;
    }
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_sum[w] = inc;
    __syncthreads();
    int run = carry + inc - loc;
    int tot = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int v = s_sum[q];
      if (q < w) run += v;
      tot += v;
    }
#pragma unroll 8
    for (int k = 0; k < kPer; ++k) {
      const int j = threadIdx.x * kPer + k;
      if (j < cnt) {
        const int x = sbuf[j + (j >> 5)];
        off[b0 + j] = run;
        run += x;
      }
    }
    carry += tot;
    __syncthreads();
  }
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    const int b = off[(int64_t)k * ntiles];
    const int e = k + 1 < S ? off[(int64_t)(k + 1) * ntiles] : carry;
    counts[k] = e - b;
  }
}

__global__ void __launch_bounds__(kPartThreads) k_part_emit(const int64_t* __restrict__ ids, int64_t n,
                                                            const uint32_t* __restrict__ t,
                                                            const uint32_t* __restrict__ hslot, int S,
                                                            int64_t ntiles, const int* __restrict__ off,
                                                            const uint32_t* __restrict__ lrank,
                                                            int64_t* __restrict__ uniq,
                                                            int64_t* __restrict__ inv_shard,
                                                            int64_t* __restrict__ inv_pos,
                                                            uint32_t* __restrict__ gidx) {
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b0 < n; b0 += stride * U) {
    long long f[U], key[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = b0 + u * stride;
      if (i < n) {
        key[u] = ids[i];
        f[u] = (long long)t[hslot[i]];
      }
    }
    uint32_t lr[U];
    int sh[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = b0 + u * stride;
      if (i < n) {
        lr[u] = lrank[f[u]];
        sh[u] = S == 1 ? 0 : (int)owner_of(key[u], (uint64_t)S);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = b0 + u * stride;
      if (i >= n) continue;
      const int64_t g = __ldg(&off[(int64_t)sh[u] * ntiles + f[u] / kPartTile]) + lr[u];
      if (inv_pos) inv_pos[i] = g - __ldg(&off[(int64_t)sh[u] * ntiles]);
      if (inv_shard) inv_shard[i] = sh[u];
      if (gidx) gidx[i] = (uint32_t)g;  // index into the owner-concatenated unique list
      if (f[u] == i) uniq[g] = key[u];
    }
  }
}

void dedup_insert(const int64_t* ids, int64_t n, DedupResult& r, cudaStream_t s) {
  r.cap = next_pow2(n * 2 > 64 ? n * 2 : 64);
  r.table = Scratch(sizeof(HEntry) * (r.cap + 1), s);
  r.hslot = Scratch(sizeof(int64_t) * (n ? n : 1), s);
  HEntry* t = r.table.as<HEntry>();
  ht_fill(t, r.cap + 1, (long long)0x7FFFFFFFFFFFFFFFll, s);
  if (n > 0) {
    k_dedup_insert<<<grid_for(n, 256), 256, 0, s>>>(ids, n, t, (uint64_t)(r.cap - 1), r.cap, r.hslot.as<int64_t>());
    SKB_LAUNCH_CHECK();
  }
}

// ---------------------------------------------------------------------------
// Duplicate test (the distinctness precondition of lookup_or_insert,
// embedding.py:196-198, and of the offset checks): a key-only claim table,
// half the bytes of the {key, position} dedup table and no per-position
// output.  A position whose key is already claimed (read first, then one
// 64-bit CAS) flags itself; kEmptyKey counts on a side word.  Any flagged
// position proves a duplicate — which one is not needed by any caller.
// ---------------------------------------------------------------------------
__global__ void k_claim_init(longlong2* t, int64_t count2, unsigned long long* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count2; i += stride)
    t[i] = make_longlong2(kEmptyKey, kEmptyKey);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    flag[0] = ~0ull;  // DevFlag word
    flag[1] = 0ull;   // occurrences of kEmptyKey
  }
}

// COUNT: the position that claims a key also counts it for its owner shard
// (shard histogram in shared memory, S <= kClaimMaxS) — load_stats' per-shard
// unique counts without building the partition
constexpr int kClaimMaxS = 4096;

template <bool COUNT>
__global__ void __launch_bounds__(256) k_claim_keys(const int64_t* __restrict__ ids, int64_t n, long long* t,
                                                    uint64_t mask, unsigned long long* flag, int S,
                                                    unsigned long long* counts) {
  constexpr int U = 4;
  __shared__ unsigned int hist[COUNT ? kClaimMaxS : 1];
  if (COUNT) {
    for (int k = threadIdx.x; k < S; k += blockDim.x) hist[k] = 0u;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n; base += stride * U) {
    long long key[U];
#pragma unroll
    for (int u = 0; u < U; ++u) key[u] = base + u * stride < n ? __ldg(ids + base + u * stride) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * stride;
      if (i >= n) continue;
      bool dup = false;
      if (key[u] == kEmptyKey) {
        dup = atomicAdd(&flag[1], 1ull) != 0ull;
      } else {
        uint64_t slot = bucket_hash((uint64_t)key[u]) & mask;
        while (true) {
          long long k = __ldcg(t + slot);
          if (k == kEmptyKey)
            k = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(t + slot), (unsigned long long)kEmptyKey,
                                     (unsigned long long)key[u]);
          if (k == kEmptyKey) break;
          if (k == key[u]) { dup = true; break; }
          slot = (slot + 1) & mask;
        }
      }
      if (COUNT) {
        if (!dup) atomicAdd(&hist[owner_of(key[u], (uint64_t)S)], 1u);
      } else if (dup) {
        atomicMin(&flag[0], (unsigned long long)i);
      }
    }
  }
  if (COUNT) {
    __syncthreads();
    for (int k = threadIdx.x; k < S; k += blockDim.x)
      if (hist[k]) atomicAdd(&counts[k], (unsigned long long)hist[k]);
  }
}

__global__ void k_zero_u64(unsigned long long* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0ull;
}

bool has_duplicate(const int64_t* ids, int64_t n, cudaStream_t s) {
  if (n < 2) return false;
  const int64_t cap = next_pow2(n * 2 > 64 ? n * 2 : 64);
  Scratch t(sizeof(long long) * cap, s);
  DevFlag f(s);
  k_claim_init<<<grid_for(cap / 2, 256), 256, 0, s>>>(t.as<longlong2>(), cap / 2, f.ptr());
  SKB_LAUNCH_CHECK();
  k_claim_keys<false><<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(ids, n, t.as<long long>(), (uint64_t)(cap - 1),
                                                                 f.ptr(), 1, nullptr);
  SKB_LAUNCH_CHECK();
  return f.read() >= 0;
}

// per-shard unique-id counts (device int64[S]), no host round trip
static void shard_unique_counts(const int64_t* ids, int64_t n, int64_t S, int64_t* counts, cudaStream_t s) {
  k_zero_u64<<<grid_for(S, 256), 256, 0, s>>>(reinterpret_cast<unsigned long long*>(counts), S);
  SKB_LAUNCH_CHECK();
  if (n <= 0) return;
  if (S > kClaimMaxS) {  // rare: many shards — the partition already produces the counts
    Scratch a(sizeof(int64_t) * n, s), b(sizeof(int64_t) * n, s), c(sizeof(int64_t) * n, s);
    unique_partition(ids, n, S, a.as<int64_t>(), counts, b.as<int64_t>(), c.as<int64_t>(), s);
    return;
  }
  const int64_t cap = next_pow2(n * 2 > 64 ? n * 2 : 64);
  Scratch t(sizeof(long long) * cap, s), f(16, s);
  k_claim_init<<<grid_for(cap / 2, 256), 256, 0, s>>>(t.as<longlong2>(), cap / 2, f.as<unsigned long long>());
  SKB_LAUNCH_CHECK();
  k_claim_keys<true><<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(ids, n, t.as<long long>(), (uint64_t)(cap - 1),
                                                                f.as<unsigned long long>(), (int)S,
                                                                reinterpret_cast<unsigned long long*>(counts));
  SKB_LAUNCH_CHECK();
}

void dedup_first_occurrence(const int64_t* ids, int64_t n, DedupResult& r, cudaStream_t s) {
  dedup_insert(ids, n, r, s);
  r.fpos = Scratch(sizeof(int64_t) * (n ? n : 1), s);
  r.d_u = Scratch(sizeof(int64_t) * 2, s);
  HEntry* t = r.table.as<HEntry>();
  if (n > 0) {
    Scratch flags(n, s);
    k_first_flags<<<grid_for(n, 256), 256, 0, s>>>(t, r.hslot.as<int64_t>(), n, flags.as<uint8_t>());
    SKB_LAUNCH_CHECK();
    select_flagged_index(flags.as<uint8_t>(), n, r.fpos.as<int64_t>(), r.d_u.as<int64_t>(), s);
  } else {
    SKB_CUDA(cudaMemsetAsync(r.d_u.p, 0, sizeof(int64_t), s));
  }
}

// the split path's work arrays, carved from one buffer (persistent callers
// keep it; unique_partition takes it from the stream-ordered pool)
static size_t split_ws_layout(int64_t n, int64_t S, size_t* b_t, size_t* b_h, size_t* b_o) {
  const int64_t cap = next_pow2(n * 2 > 64 ? n * 2 : 64);
  const int64_t ntiles = (n + kPartTile - 1) / kPartTile;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  *b_t = al(sizeof(uint32_t) * cap);
  *b_h = al(4 * (n > 0 ? n : 1));
  *b_o = al(sizeof(int) * (ntiles > 0 ? ntiles : 1) * S);
  return *b_t + 2 * *b_h + *b_o + 256;
}

size_t unique_partition_ws_bytes(int64_t n, int64_t S) {
  size_t a, b, c;
  return split_ws_layout(n, S, &a, &b, &c);
}

static void split_partition(const int64_t* ids, int64_t n, int64_t S, int64_t* uniq, int64_t* counts,
                            int64_t* inv_shard, int64_t* inv_pos, uint32_t* gidx, void* ws, cudaStream_t s) {
  const int64_t cap = next_pow2(n * 2 > 64 ? n * 2 : 64);
  const int64_t ntiles = (n + kPartTile - 1) / kPartTile;
  size_t b_t, b_h, b_o;
  split_ws_layout(n, S, &b_t, &b_h, &b_o);
  char* w = static_cast<char*>(ws);
  uint32_t* t = reinterpret_cast<uint32_t*>(w);
  uint32_t* hs = reinterpret_cast<uint32_t*>(w + b_t);
  uint32_t* lr = reinterpret_cast<uint32_t*>(w + b_t + b_h);
  int* off = reinterpret_cast<int*>(w + b_t + 2 * b_h);
  unsigned long long* done = reinterpret_cast<unsigned long long*>(w + b_t + 2 * b_h + b_o);
  k_part_init<<<grid_for(cap / 4, 256), 256, 0, s>>>(t, cap, done, 1);
  SKB_LAUNCH_CHECK();
  k_part_insert<kPartU><<<grid_for((n + kPartU - 1) / kPartU, kPartThreads), kPartThreads, 0, s>>>(
      ids, n, t, (uint64_t)(cap - 1), hs);
  SKB_LAUNCH_CHECK();
  k_part_count<<<(unsigned)ntiles, kPartThreads, 0, s>>>(ids, n, t, hs, (int)S, ntiles, off, lr, done, counts);
  SKB_LAUNCH_CHECK();
  k_part_emit<<<grid_for((n + 3) / 4, kPartThreads), kPartThreads, 0, s>>>(
      ids, n, t, hs, (int)S, ntiles, off, lr, uniq, inv_shard, inv_pos, gidx);
  SKB_LAUNCH_CHECK();
}

void unique_partition_ws(const int64_t* ids, int64_t n, int64_t S, int64_t* uniq, int64_t* counts, uint32_t* gidx,
                         void* ws, cudaStream_t s) {
  if (n == 0) {
    SKB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * S, s));
    return;
  }
  if (S > kSplitMaxS || n >= (1ll << 30)) raise(SKB_E_UNSUPPORTED, S, "persistent partition: S <= 256, n < 2^30");
  split_partition(ids, n, S, uniq, counts, nullptr, nullptr, gidx, ws, s);
}

void unique_partition(const int64_t* ids, int64_t n, int64_t S, int64_t* uniq, int64_t* counts, int64_t* inv_shard,
                      int64_t* inv_pos, cudaStream_t s) {
  if (n == 0) {
    SKB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * S, s));
    return;
  }
  if (S <= kSplitMaxS && n < (1ll << 30)) {  // stable multi-split, no sort
    // one stream-ordered allocation carved into the five work arrays
    Scratch work(unique_partition_ws_bytes(n, S), s);
    split_partition(ids, n, S, uniq, counts, inv_shard, inv_pos, nullptr, work.p, s);
    return;
  }
  DedupResult r;
  dedup_first_occurrence(ids, n, r, s);
  HEntry* t = r.table.as<HEntry>();
  const int64_t* d_u = r.d_u.as<int64_t>();
  if (S == 1) {
    k_emit_single<<<grid_for(n, 256), 256, 0, s>>>(ids, r.fpos.as<int64_t>(), d_u, r.hslot.as<int64_t>(), t, uniq);
    SKB_LAUNCH_CHECK();
    SKB_CUDA(cudaMemcpyAsync(counts, d_u, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  } else {
    if (S >= (1ll << 31)) raise(SKB_E_UNSUPPORTED, S, "num_shards too large");
    Scratch sk(4 * n, s), kv(4 * n, s), sk2(4 * n, s), kv2(4 * n, s);
    k_owner_keys<<<grid_for(n, 256), 256, 0, s>>>(ids, r.fpos.as<int64_t>(), d_u, n, (uint64_t)S, sk.as<uint32_t>(),
                                                  kv.as<uint32_t>());
    SKB_LAUNCH_CHECK();
    sort_pairs_u32(sk.as<uint32_t>(), sk2.as<uint32_t>(), kv.as<uint32_t>(), kv2.as<uint32_t>(), n,
                   bits_for((uint64_t)S), s);
    Scratch starts(sizeof(int64_t) * (S + 1), s);
    k_shard_starts<<<grid_for(S + 1, 128), 128, 0, s>>>(sk2.as<uint32_t>(), d_u, S, starts.as<int64_t>());
    SKB_LAUNCH_CHECK();
    k_shard_counts<<<grid_for(S, 128), 128, 0, s>>>(starts.as<int64_t>(), S, counts);
    SKB_LAUNCH_CHECK();
    k_emit_sharded<<<grid_for(n, 256), 256, 0, s>>>(ids, r.fpos.as<int64_t>(), d_u, sk2.as<uint32_t>(),
                                                    kv2.as<uint32_t>(), starts.as<int64_t>(), r.hslot.as<int64_t>(),
                                                    t, uniq);
    SKB_LAUNCH_CHECK();
  }
  k_inverse<<<grid_for(n, 256), 256, 0, s>>>(ids, r.hslot.as<int64_t>(), t, n, (uint64_t)S, inv_shard, inv_pos);
  SKB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// ordered fold of per-position rows into per-segment sums (left fold from +0,
// input order): the np.add.at semantics of sharding.py:289 / segments.py:57.
// Positions are grouped by a stable sort on the group index.
template <int VEC>
__global__ void k_fold_sorted(const uint32_t* __restrict__ heads, const int64_t* __restrict__ d_nseg, int64_t n,
                              const uint32_t* __restrict__ skey, const uint32_t* __restrict__ spos,
                              const float* __restrict__ rows, int D, float* __restrict__ out,
                              LongRun* __restrict__ longs, int64_t* __restrict__ nlong, int64_t longs_cap) {
  const int per_row = D / VEC;
  const int64_t nseg = *d_nseg;
  const int64_t total = nseg * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t sidx = t / per_row;
    int c = (int)(t - sidx * per_row) * VEC;
    int64_t b = heads[sidx];
    int64_t e = sidx + 1 < nseg ? (int64_t)heads[sidx + 1] : n;
    if (VEC == 4 && longs && e - b > kLongRun) {  // hot id: CTA-per-run long fold
      if (c == 0) push_long_run(longs, nlong, longs_cap, skey[b], (uint32_t)b, (uint32_t)e);
      continue;
    }
    if constexpr (VEC == 4) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t j = b; j < e; ++j) acc = add4(acc, ldg4(rows + (int64_t)spos[j] * D + c));
      st4(out + (int64_t)skey[b] * D + c, acc);
    } else {
      float acc = 0.f;
      for (int64_t j = b; j < e; ++j) acc = __fadd_rn(acc, __ldg(rows + (int64_t)spos[j] * D + c));
      out[(int64_t)skey[b] * D + c] = acc;
    }
  }
}

__global__ void k_iota_keys(const int64_t* __restrict__ inv, int64_t n, uint32_t* __restrict__ k,
                            uint32_t* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    k[i] = (uint32_t)inv[i];
    v[i] = (uint32_t)i;
  }
}

void grad_fold(const float* grads, int64_t n, int D, const int64_t* inverse, int64_t U, float* out, cudaStream_t s) {
  SKB_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * U * D, s));
  if (n == 0 || U == 0) return;
  if (n >= (1ll << 32) || U >= (1ll << 32)) raise(SKB_E_UNSUPPORTED, n, "grad_fold: too many rows");
  Scratch k(4 * n, s), v(4 * n, s), k2(4 * n, s), v2(4 * n, s), heads(4 * n, s), nseg(16, s);
  const int64_t lcap = n / kLongRun + 1;
  Scratch longs(sizeof(LongRun) * lcap, s);
  SKB_CUDA(cudaMemsetAsync(nseg.p, 0, 16, s));
  k_iota_keys<<<grid_for(n, 256), 256, 0, s>>>(inverse, n, k.as<uint32_t>(), v.as<uint32_t>());
  SKB_LAUNCH_CHECK();
  sort_pairs_u32(k.as<uint32_t>(), k2.as<uint32_t>(), v.as<uint32_t>(), v2.as<uint32_t>(), n,
                 bits_for((uint64_t)(U - 1)), s);
  select_run_heads_u32(k2.as<uint32_t>(), n, heads.as<uint32_t>(), nseg.as<int64_t>(), s);
  bool v4 = (D % 4 == 0) && ((uintptr_t)grads % 16 == 0) && ((uintptr_t)out % 16 == 0);
  if (v4)
    k_fold_sorted<4><<<grid_for(n * (D / 4), 256), 256, 0, s>>>(heads.as<uint32_t>(), nseg.as<int64_t>(), n,
                                                               k2.as<uint32_t>(), v2.as<uint32_t>(), grads, D, out,
                                                               longs.as<LongRun>(), nseg.as<int64_t>() + 1, lcap);
  else
    k_fold_sorted<1><<<grid_for(n * D, 256), 256, 0, s>>>(heads.as<uint32_t>(), nseg.as<int64_t>(), n,
                                                         k2.as<uint32_t>(), v2.as<uint32_t>(), grads, D, out, nullptr,
                                                         nullptr, 0);
  SKB_LAUNCH_CHECK();
  if (v4) {
    const int64_t imgs = long_fold_pack_images(n, D);
    Scratch prow(sizeof(float) * imgs * long_fold_stage_f(D), s), pl(sizeof(uint32_t) * lcap, s),
        po(sizeof(uint32_t) * lcap, s), pc(sizeof(int64_t) * 2, s), pr(sizeof(uint32_t) * lcap, s);
    LongFoldPack pk{prow.as<float>(), imgs, pl.as<uint32_t>(), po.as<uint32_t>(), pc.as<int64_t>(), lcap,
                    pr.as<uint32_t>()};
    launch_long_fold<false>(longs.as<LongRun>(), nseg.as<int64_t>() + 1, lcap, v2.as<uint32_t>(), grads, D, nullptr, 0,
                            AdamDev{}, out, nullptr, -1, s, nullptr, &pk);
  }
}

struct IdxRestore {
  const int64_t* base;
  const int64_t* sh;
  const int64_t* pos;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return base[sh[i]] + pos[i]; }
};

}  // namespace skb

using namespace skb;

extern "C" {

int skb_unique_partition(const int64_t* ids, int64_t n, int64_t num_shards, int64_t* uniq_out,
                         int64_t* shard_counts_out, int64_t* inv_shard, int64_t* inv_pos, void* stream) {
  SKB_API_BEGIN
  if (num_shards < 1) raise(SKB_E_VALUE, num_shards, "num_shards must be >= 1");
  if (n < 0) raise(SKB_E_ARG, n, "negative length");
  unique_partition(ids, n, num_shards, uniq_out, shard_counts_out, inv_shard, inv_pos, as_stream(stream));
  SKB_API_END
}

int skb_shard_unique_counts(const int64_t* ids, int64_t n, int64_t num_shards, int64_t* counts_out, void* stream) {
  SKB_API_BEGIN
  if (num_shards < 1) raise(SKB_E_ARG, num_shards, "num_shards must be >= 1");
  if (n < 0) raise(SKB_E_ARG, n, "n must be >= 0");
  shard_unique_counts(ids, n, num_shards, counts_out, as_stream(stream));
  SKB_API_END
}

int skb_partition_restore(const float* rows_cat, int64_t dim, const int64_t* shard_base, const int64_t* inv_shard,
                          const int64_t* inv_pos, int64_t n, float* out, void* stream) {
  SKB_API_BEGIN
  launch_rows_gather(IdxRestore{shard_base, inv_shard, inv_pos}, rows_cat, dim, out, dim, n, (int)dim,
                     as_stream(stream));
  SKB_API_END
}

int skb_grad_fold(const float* grads, int64_t n, int64_t dim, const int64_t* inverse, int64_t num_unique,
                  float* out, void* stream) {
  SKB_API_BEGIN
  grad_fold(grads, n, (int)dim, inverse, num_unique, out, as_stream(stream));
  SKB_API_END
}

}  // extern "C"
