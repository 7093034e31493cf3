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
  } else {
    i = (int64_t)(bucket_hash((uint64_t)key) & mask);
    while (true) {  // one atomic per probe: CAS returns the resident key
      long long prev = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&t[i].key),
                                            (unsigned long long)kEmptyKey, (unsigned long long)key);
      if (prev == kEmptyKey || prev == key) break;
      i = (int64_t)(((uint64_t)i + 1) & mask);
    }
  }
  atomicMin(&t[i].val, pos);
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
// Stable multi-split for S <= kSplitMaxS: per-tile per-shard counts of the
// first occurrences, one-block shard-major scan, then an in-order emit in
// which each warp ranks its first occurrences among same-shard lanes with
// __match_any_sync and the block keeps running per-shard cursors.  Five
// kernels, no sort; the output order is exactly sharding.py:87-100's.
constexpr int kSplitTile = 1024;
constexpr int kSplitMaxS = 256;

__global__ void __launch_bounds__(256) k_split_count(const int64_t* __restrict__ ids, int64_t n, const HEntry* t,
                                                     const int64_t* __restrict__ hslot, int S,
                                                     int64_t* __restrict__ tile_cnt, int64_t ntiles) {
  __shared__ int cnt[kSplitMaxS];
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int k = threadIdx.x; k < S; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    const int64_t b = tile * kSplitTile, e = b + kSplitTile < n ? b + kSplitTile : n;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x)
      if (t[hslot[i]].val == i) atomicAdd(&cnt[S == 1 ? 0 : (int)owner_of(ids[i], (uint64_t)S)], 1);
    __syncthreads();
    for (int k = threadIdx.x; k < S; k += blockDim.x) tile_cnt[(int64_t)k * ntiles + tile] = cnt[k];
    __syncthreads();
  }
}

// exclusive scan of m values in one block (each thread owns kScanItems
// consecutive values per pass); totals of each shard row -> counts
constexpr int kScanItems = 8;
__global__ void __launch_bounds__(1024) k_split_scan(int64_t* __restrict__ v, int64_t m, int64_t ntiles, int S,
                                                    int64_t* __restrict__ counts) {
  __shared__ int64_t s_sum[32];
  __shared__ int64_t s_carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int64_t per_pass = (int64_t)blockDim.x * kScanItems;
  for (int64_t base = 0; base < m; base += per_pass) {
    const int64_t i0 = base + (int64_t)threadIdx.x * kScanItems;
    int64_t x[kScanItems];
    int64_t local = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      x[k] = i0 + k < m ? v[i0 + k] : 0;
      local += x[k];
    }
    int64_t incl = local;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffff, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_sum[w] = incl;
    __syncthreads();
    if (w == 0) {
      int64_t q = lane < (int)(blockDim.x >> 5) ? s_sum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffff, q, o);
        if (lane >= o) q += y;
      }
      s_sum[lane] = q;
    }
    __syncthreads();
    int64_t run = incl - local + (w ? s_sum[w - 1] : 0) + s_carry;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (i0 + k < m) v[i0 + k] = run;
      run += x[k];
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = run;
    __syncthreads();
  }
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    const int64_t start = v[(int64_t)k * ntiles];
    const int64_t end = k + 1 < S ? v[(int64_t)(k + 1) * ntiles] : s_carry;
    counts[k] = end - start;
  }
}

__global__ void __launch_bounds__(256) k_split_emit(const int64_t* __restrict__ ids, int64_t n, HEntry* t,
                                                    const int64_t* __restrict__ hslot, int S,
                                                    const int64_t* __restrict__ tile_off, int64_t ntiles,
                                                    int64_t* __restrict__ uniq) {
  __shared__ int64_t run[kSplitMaxS];    // running output cursor per shard
  __shared__ int64_t base0[kSplitMaxS];  // shard start in the concatenated output
  __shared__ int wcnt[8][kSplitMaxS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int k = threadIdx.x; k < S; k += blockDim.x) {
      run[k] = tile_off[(int64_t)k * ntiles + tile];
      base0[k] = tile_off[(int64_t)k * ntiles];
    }
    const int64_t b = tile * kSplitTile, e = b + kSplitTile < n ? b + kSplitTile : n;
    for (int64_t r0 = b; r0 < e; r0 += blockDim.x) {
      for (int k = threadIdx.x; k < 8 * S; k += blockDim.x) (&wcnt[0][0])[(k / S) * kSplitMaxS + k % S] = 0;
      __syncthreads();
      const int64_t i = r0 + threadIdx.x;
      const bool first = i < e && t[hslot[i]].val == i;
      const int sh = first ? (S == 1 ? 0 : (int)owner_of(ids[i], (uint64_t)S)) : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, sh);
      const int rank = __popc(grp & ((1u << lane) - 1));
      if (first && rank == 0) wcnt[w][sh] = __popc(grp);
      __syncthreads();
      if (first) {
        int64_t off = run[sh] + rank;
        for (int q = 0; q < w; ++q) off += wcnt[q][sh];
        uniq[off] = ids[i];
        t[hslot[i]].val = off - base0[sh];
      }
      __syncthreads();
      for (int k = threadIdx.x; k < S; k += blockDim.x) {
        int64_t tot = 0;
        for (int q = 0; q < 8; ++q) tot += wcnt[q][k];
        run[k] += tot;
      }
      __syncthreads();
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

void unique_partition(const int64_t* ids, int64_t n, int64_t S, int64_t* uniq, int64_t* counts, int64_t* inv_shard,
                      int64_t* inv_pos, cudaStream_t s) {
  if (n == 0) {
    SKB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * S, s));
    return;
  }
  if (S <= kSplitMaxS) {  // stable multi-split, no sort
    DedupResult r;
    dedup_insert(ids, n, r, s);
    HEntry* t = r.table.as<HEntry>();
    const int64_t ntiles = (n + kSplitTile - 1) / kSplitTile;
    Scratch tc(sizeof(int64_t) * S * ntiles, s);
    k_split_count<<<grid_for(ntiles * 256, 256), 256, 0, s>>>(ids, n, t, r.hslot.as<int64_t>(), (int)S,
                                                              tc.as<int64_t>(), ntiles);
    SKB_LAUNCH_CHECK();
    k_split_scan<<<1, 1024, 0, s>>>(tc.as<int64_t>(), S * ntiles, ntiles, (int)S, counts);
    SKB_LAUNCH_CHECK();
    k_split_emit<<<grid_for(ntiles * 256, 256), 256, 0, s>>>(ids, n, t, r.hslot.as<int64_t>(), (int)S,
                                                             tc.as<int64_t>(), ntiles, uniq);
    SKB_LAUNCH_CHECK();
    k_inverse<<<grid_for(n, 256), 256, 0, s>>>(ids, r.hslot.as<int64_t>(), t, n, (uint64_t)S, inv_shard, inv_pos);
    SKB_LAUNCH_CHECK();
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
  if (v4)
    launch_long_fold<false>(longs.as<LongRun>(), nseg.as<int64_t>() + 1, lcap, v2.as<uint32_t>(), grads, D, nullptr, 0,
                            AdamDev{}, out, nullptr, -1, s);
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
