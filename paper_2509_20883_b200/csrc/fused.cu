// fused.cu — the request-merged sparse step for one logical table on one GPU.
//
// Forward (replaces keys_for + unique_partition + lookup_or_insert + gather +
// restore + segment_reduce of train.py:130-176 for S = 1):
//   K1 probe   : per position — namespaced key (sharding.py:178) with the
//                member table staged in shared memory, IDMap probe -> slot
//                (uint32) or miss; misses counted on device.
//   K2..K5 miss: only positions whose key is unknown do work (every launch
//                exits at once when the device miss count is 0): first-
//                occurrence dedup among misses, ordered rank (tile counts ->
//                one-block scan -> tile ranks), admission with the reference's
//                slot order, slot broadcast to duplicate misses.
//   K6 pool    : tiles of 256 bags; bag offsets and the tile's slots are staged
//                in shared memory with coalesced loads so the only global
//                latency per bag is the 128-bit row gather; fold (scatter /
//                pairwise, bit-exact), mean, write pooled and bag-of-position.
// Backward (replaces the per-row grad expansion train.py:181-186 +
// all_to_all_grad_update sharding.py:257-297):
//   K7 stable radix sort of (slot, bag) by slot, K8 run heads,
//   K9 fold + Adam: tiles of 256 unique rows with heads / slots / bags staged
//                in shared memory; w, m, v loads are issued before the dpooled
//                fold so ~4 independent 16-byte loads per lane are in flight;
//                fold in position order from +0 (np.add.at), AdamW, one write
//                of the 12*D-byte row, and the step's last_step (deferred from
//                the forward: one write per unique row instead of per position).
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "fused.cuh"
#include "graph.cuh"
#include "p2p.cuh"
#include "partition.cuh"
#include "longfold.cuh"
#include "tma.cuh"
#include "pool.cuh"
#include "table.cuh"

namespace skb {

constexpr int kSmemMembers = 512;  // member tables up to this size are staged in smem
constexpr int kTileBags = 256;
constexpr int kTilePos = 2048;
constexpr int kTileU = 256;
constexpr int kTileJ = 1024;
constexpr int kRankTile = 4096;    // positions per tile of the miss-rank scan

// One batch in flight through the pipeline: index results of its prepare
// (slots, sort) and its metadata; two of these are double-buffered so the
// index work of step k+1 overlaps the pool / fold+Adam of step k.
struct BatchCtx {
  int64_t cap_n = 0;          // capacity in positions
  uint32_t* slot = nullptr;   // [N] slot of position
  uint32_t* bag = nullptr;    // [N] bag of position
  uint32_t* skey = nullptr;   // [N] sorted slots
  uint32_t* sval = nullptr;   // [N] bags in sorted order
  uint8_t* miss = nullptr;    // [N]
  uint8_t* fresh = nullptr;   // [N] first occurrence of an unknown key
  int64_t* rank = nullptr;    // [N]
  uint32_t* fpos = nullptr;   // [N] position of the k-th fresh (new) key: admission walks K rows, not N
  int32_t* hslot = nullptr;   // [N] scratch-table index of a miss
  int64_t* tile_cnt = nullptr;  // [N / kRankTile + 2]
  HEntry* scratch = nullptr;  // [2*cap_n pow2 + 1]
  int64_t scratch_cap = 0;
  int64_t* dev = nullptr;     // [0] misses M, [1] new K, [2] unique U, [3] long runs
  LongRun* longs = nullptr;   // deferred long runs of the fold (hot ids)
  int64_t longs_cap = 0;
  MemberDev* members = nullptr;
  int64_t members_cap = 0;
  std::vector<MemberDev> members_host;
  void* sort_ws = nullptr;              // CUB temp storage of the index sort (persistent: no per-step
  size_t sort_ws_bytes = 0;             //  allocation on the index stream)
  MemberDev* members_pinned = nullptr;  // upload staging (ragged batches change it every step)
  cudaEvent_t members_ev = nullptr;     // the staging buffer's last upload
  // identity + metadata of the prepared batch
  const int64_t* ids = nullptr;
  const int64_t* bag_offs = nullptr;
  int64_t n = 0, G = 0, step = -1;
  int64_t tile_k = 0;  // mode 2: tile width (rows per bag)
  float pad = 0.f;
  int F = 0, mode = 0;
  bool any_seq = false;
  bool last_written = false;  // deferred last_step already flushed
  cudaEvent_t ev_ready = nullptr, ev_free = nullptr;
  cudaEvent_t ev_stats = nullptr;  // after a stats_async copy of dev (reuse of this buffer waits for it)
  bool stats_pending = false;
  bool ever_used = false;
  int64_t gen = 0;  // bumped when a buffer above is reallocated / the member table changes
  StepGraph g_prep, g_fwd, g_bwd;  // graph mode: captured device work of each phase
};

struct FusedCtx {
  cudaStream_t side = nullptr;  // index stream: probe, admission, bag-of, sort
  float* zrow = nullptr;        // D zeros: the gradient row of tile positions past k
  LongFoldPack pack;            // mega-run packing buffers of the long-run fold (backward only)
  int64_t pack_gen = 0;
  int64_t* lf_host = nullptr;   // pinned: long runs of a recent backward (async readback)
  cudaEvent_t lf_ev = nullptr;
  int64_t lf_last = 1;          // > 0: long runs seen recently (pack mega runs)
  int64_t lf_maxlen = 0;        // longest run of a recent backward (exclusive long-fold SMs)
  cudaEvent_t ev_in = nullptr, ev_side_last = nullptr;
  // hot-id batches: the long-run fold runs on its own stream concurrently
  // with the main fold kernel (forked after the runs are listed, joined
  // before the step ends)
  cudaStream_t lf_stream = nullptr;
  cudaEvent_t lf_fork = nullptr, lf_join = nullptr;
  BatchCtx b[2];
  int64_t prep_count = 0, pool_count = 0, bwd_count = 0;
  // per-table kernel variant overrides (-1: SKB_ADAM_VARIANT / SKB_POOL_VARIANT)
  // and the variants the last backward / pool actually ran (tests pin them)
  int adam_var = -1, pool_var = -1;
  int last_adam = -1, last_pool = -1;
  int64_t* iota = nullptr;  // 0, 1, 2, ...: bag offsets of one-id bags (owner side of the multi-GPU step)
  int64_t iota_cap = 0;
  bool tree = false;         // tolerance-mode long-run fold (set_fold_mode "tree")
  TreeWork tw;
  bool graphs = false;  // replay each phase's device work as a CUDA graph
  cudaStream_t cap = nullptr;  // capture stream of graph mode
  // optional per-kernel CUDA-event profiling: kProf phases x (begin, end) x cap steps
  int64_t prof_cap = 0;
  int64_t prof_n[5] = {0, 0, 0, 0, 0};
  std::vector<cudaEvent_t> prof_ev[5];
};

enum { P_PROBE = 0, P_MISS = 1, P_POOL = 2, P_SORT = 3, P_ADAM = 4, kProf = 5 };

static void prof_mark(FusedCtx* c, int phase, int edge, cudaStream_t s) {
  if (!c->prof_cap || c->prof_n[phase] >= c->prof_cap) return;
  SKB_CUDA(cudaEventRecord(c->prof_ev[phase][2 * c->prof_n[phase] + edge], s));
  if (edge == 1) c->prof_n[phase]++;
}

static void batch_free(BatchCtx& B) {
  cudaFree(B.slot);
  cudaFree(B.bag);
  cudaFree(B.skey);
  cudaFree(B.sval);
  cudaFree(B.miss);
  cudaFree(B.fresh);
  cudaFree(B.rank);
  cudaFree(B.fpos);
  cudaFree(B.hslot);
  cudaFree(B.tile_cnt);
  cudaFree(B.scratch);
  cudaFree(B.dev);
  cudaFree(B.members);
  cudaFree(B.sort_ws);
  if (B.members_pinned) cudaFreeHost(B.members_pinned);
  if (B.members_ev) cudaEventDestroy(B.members_ev);
  cudaFree(B.longs);
  if (B.ev_ready) cudaEventDestroy(B.ev_ready);
  if (B.ev_free) cudaEventDestroy(B.ev_free);
  if (B.ev_stats) cudaEventDestroy(B.ev_stats);
}

void fused_ctx_destroy(FusedCtx* c) {
  if (!c) return;
  if (c->side) cudaStreamSynchronize(c->side);
  for (auto& v : c->prof_ev)
    for (auto e : v) cudaEventDestroy(e);
  for (auto& B : c->b) batch_free(B);
  for (auto& B : c->b) {
    B.g_prep.reset();
    B.g_fwd.reset();
    B.g_bwd.reset();
  }
  if (c->side) cudaStreamDestroy(c->side);
  if (c->cap) cudaStreamDestroy(c->cap);
  cudaFree(c->zrow);
  cudaFree(c->iota);
  cudaFree(c->tw.chunk_off);
  cudaFree(c->tw.partial);
  cudaFree(c->pack.images);
  if (c->lf_host) cudaFreeHost(c->lf_host);
  if (c->lf_ev) cudaEventDestroy(c->lf_ev);
  cudaFree(c->pack.mlist);
  cudaFree(c->pack.moff);
  cudaFree(c->pack.morder);
  cudaFree(c->pack.mcount);
  cudaFree(c->pack.ready);
  cudaFree(c->pack.wctr);
  if (c->pack.pstream) cudaStreamDestroy(c->pack.pstream);
  if (c->pack.ev_fork) cudaEventDestroy(c->pack.ev_fork);
  if (c->pack.ev_join) cudaEventDestroy(c->pack.ev_join);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_side_last) cudaEventDestroy(c->ev_side_last);
  if (c->lf_stream) cudaStreamDestroy(c->lf_stream);
  if (c->lf_fork) cudaEventDestroy(c->lf_fork);
  if (c->lf_join) cudaEventDestroy(c->lf_join);
  delete c;
}

template <class T>
static void realloc_dev(T*& p, int64_t count, cudaStream_t s) {
  if (p) SKB_CUDA(cudaFreeAsync(p, s));
  SKB_CUDA(cudaMallocAsync(&p, sizeof(T) * (count > 0 ? count : 1), s));
}

static FusedCtx* ctx_get(Table* t) {
  if (!t->fused) {
    FusedCtx* c = new FusedCtx();
    // highest priority: index blocks take SM slots as soon as fold+Adam
    // blocks retire, so the prefetched index phase overlaps the optimizer
    int lo = 0, hi = 0;
    SKB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SKB_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
    SKB_CUDA(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
    SKB_CUDA(cudaEventCreateWithFlags(&c->ev_side_last, cudaEventDisableTiming));
    SKB_CUDA(cudaStreamCreateWithPriority(&c->lf_stream, cudaStreamNonBlocking, hi));
    SKB_CUDA(cudaEventCreateWithFlags(&c->lf_fork, cudaEventDisableTiming));
    SKB_CUDA(cudaEventCreateWithFlags(&c->lf_join, cudaEventDisableTiming));
    for (auto& B : c->b) {
      SKB_CUDA(cudaMalloc(&B.dev, sizeof(int64_t) * 4));
      SKB_CUDA(cudaMemset(B.dev, 0, sizeof(int64_t) * 4));
      SKB_CUDA(cudaEventCreateWithFlags(&B.ev_ready, cudaEventDisableTiming));
      SKB_CUDA(cudaEventCreateWithFlags(&B.ev_free, cudaEventDisableTiming));
    }
    if (const char* g = getenv("SKB_FUSED_GRAPHS")) c->graphs = atoi(g) != 0;
    SKB_CUDA(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
    SKB_CUDA(cudaMallocHost(&c->lf_host, 2 * sizeof(int64_t)));
    c->lf_host[0] = 1;
    c->lf_host[1] = 0;
    SKB_CUDA(cudaEventCreateWithFlags(&c->lf_ev, cudaEventDisableTiming));
    SKB_CUDA(cudaMalloc(&c->zrow, sizeof(float) * (t->dim + 4)));
    SKB_CUDA(cudaMemset(c->zrow, 0, sizeof(float) * (t->dim + 4)));
    t->fused = c;
  }
  return t->fused;
}

static void batch_reserve(BatchCtx& B, int64_t n, int64_t F, cudaStream_t s) {
  if (n > B.cap_n) {
    int64_t cap = n + n / 4;
    realloc_dev(B.slot, cap, s);
    realloc_dev(B.bag, cap, s);
    realloc_dev(B.skey, cap, s);
    realloc_dev(B.sval, cap, s);
    realloc_dev(B.miss, cap, s);
    realloc_dev(B.fresh, cap, s);
    realloc_dev(B.rank, cap, s);
    realloc_dev(B.fpos, cap, s);
    realloc_dev(B.hslot, cap, s);
    realloc_dev(B.tile_cnt, cap / kRankTile + 2, s);
    B.scratch_cap = next_pow2(2 * cap > 64 ? 2 * cap : 64);
    realloc_dev(B.scratch, B.scratch_cap + 1, s);
    B.longs_cap = cap / kLongRun + 1;
    realloc_dev(B.longs, B.longs_cap, s);
    B.cap_n = cap;
    B.gen++;
  }
  if (F + 1 > B.members_cap) {
    realloc_dev(B.members, F + 1, s);
    if (B.members_ev) SKB_CUDA(cudaEventSynchronize(B.members_ev));
    if (B.members_pinned) SKB_CUDA(cudaFreeHost(B.members_pinned));
    SKB_CUDA(cudaMallocHost(&B.members_pinned, sizeof(MemberDev) * (F + 1)));
    if (!B.members_ev) SKB_CUDA(cudaEventCreateWithFlags(&B.members_ev, cudaEventDisableTiming));
    B.members_cap = F + 1;
    B.members_host.clear();
    B.gen++;
  }
}

// member lookup over a (shared or global) member table
__device__ __forceinline__ int member_search_pos(const int64_t* __restrict__ pos, int F, int64_t i) {
  int lo = 0, hi = F;  // pos[lo] <= i < pos[lo+1]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pos[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// Stage member boundaries in shared memory when the table fits; returns the
// arrays to search (shared or a global fallback copy in `mt`).
struct MemberView {
  const int64_t* pos;  // F+1
  const int64_t* bag;  // F+1
  const uint64_t* salt;
  const int64_t* strat;
  int stride;          // element stride (1 in smem, 4 in the global AoS table)
};

__device__ __forceinline__ int64_t mv_pos(const MemberView& v, int f) { return v.pos[f * v.stride]; }
__device__ __forceinline__ int64_t mv_bag(const MemberView& v, int f) { return v.bag[f * v.stride]; }

__device__ __forceinline__ int mv_member_of_pos(const MemberView& v, int F, int64_t i) {
  int lo = 0, hi = F;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (mv_pos(v, mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int mv_member_of_bag(const MemberView& v, int F, int64_t g) {
  int lo = 0, hi = F;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (mv_bag(v, mid) <= g) lo = mid; else hi = mid;
  }
  return lo;
}

struct MemberSmem {
  int64_t pos[kSmemMembers + 1];
  int64_t bag[kSmemMembers + 1];
  uint64_t salt[kSmemMembers];
  int64_t strat[kSmemMembers];
};

__device__ __forceinline__ MemberView stage_members(MemberSmem* sm, const MemberDev* __restrict__ mt, int F) {
  if (F <= kSmemMembers) {
    for (int f = threadIdx.x; f <= F; f += blockDim.x) {
      MemberDev m = mt[f];
      sm->pos[f] = m.pos;
      sm->bag[f] = m.bag;
      if (f < F) {
        sm->salt[f] = m.salt;
        sm->strat[f] = m.strategy;
      }
    }
    __syncthreads();
    return MemberView{sm->pos, sm->bag, sm->salt, sm->strat, 1};
  }
  return MemberView{&mt[0].pos, &mt[0].bag, &mt[0].salt, &mt[0].strategy, 4};
}

__device__ __forceinline__ long long key_of(long long id, const MemberView& v, int F, int namespaced, int64_t i) {
  if (!namespaced) return id;
  return (long long)mix64((uint64_t)id ^ v.salt[mv_member_of_pos(v, F, i) * v.stride]);
}

__device__ __forceinline__ HEntry ldg_entry(const HEntry* p) {
  longlong2 v = __ldg(reinterpret_cast<const longlong2*>(p));
  return HEntry{v.x, v.y};
}

__device__ __forceinline__ long long idmap_find_ro(const HEntry* __restrict__ t, uint64_t mask, int64_t cap,
                                                   long long key) {
  if (key == kEmptyKey) return __ldg(&t[cap].val);
  uint64_t i = bucket_hash((uint64_t)key) & mask;
  while (true) {
    HEntry e = ldg_entry(t + i);
    if (e.key == key) return e.val;
    if (e.key == kEmptyKey) return -1;
    i = (i + 1) & mask;
  }
}

// K1
__global__ void __launch_bounds__(256) k_fused_probe(const int64_t* __restrict__ ids, int64_t n,
                                                     const MemberDev* __restrict__ mt, int F, int namespaced,
                                                     const HEntry* __restrict__ map, uint64_t mask, int64_t cap,
                                                     uint32_t* __restrict__ slot, uint8_t* __restrict__ miss,
                                                     int64_t* dev) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MemberView mv = stage_members(reinterpret_cast<MemberSmem*>(smem_raw), mt, F);
  int local = 0;
  // 4 positions per thread per pass: 4 independent probe chains in flight
  constexpr int R = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += R * stride) {
    long long key[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int64_t i = i0 + r * stride;
      key[r] = i < n ? key_of(__ldg(ids + i), mv, F, namespaced, i) : 0;
    }
    // first bucket of every chain issued before any chain is resolved
    uint64_t h[R];
    HEntry e[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      h[r] = key[r] == kEmptyKey ? (uint64_t)cap : (bucket_hash((uint64_t)key[r]) & mask);
      e[r] = ldg_entry(map + h[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int64_t i = i0 + r * stride;
      if (i < n) {
        long long s;
        if (key[r] == kEmptyKey) {
          s = e[r].val;  // side entry
        } else {
          while (e[r].key != key[r] && e[r].key != kEmptyKey) {
            h[r] = (h[r] + 1) & mask;
            e[r] = ldg_entry(map + h[r]);
          }
          s = e[r].key == key[r] ? e[r].val : -1;
        }
        slot[i] = s < 0 ? 0xFFFFFFFFu : (uint32_t)s;
        miss[i] = s < 0;
        local += s < 0;
      }
    }
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffff, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(reinterpret_cast<unsigned long long*>(&dev[0]), (unsigned long long)local);
}

__device__ __forceinline__ int64_t scratch_cap_for(int64_t M) { return next_pow2(2 * M > 64 ? 2 * M : 64); }

__global__ void k_fill_scratch(HEntry* t, const int64_t* dev) {
  if (dev[0] == 0) return;
  const int64_t cap = scratch_cap_for(dev[0]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cap; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<longlong2*>(t)[i] = make_longlong2(kEmptyKey, 0x7FFFFFFFFFFFFFFFll);
}

// K2: first-occurrence dedup among unknown keys
__global__ void __launch_bounds__(256) k_miss_insert(const int64_t* __restrict__ ids, int64_t n,
                                                     const MemberDev* __restrict__ mt, int F, int namespaced,
                                                     const uint8_t* __restrict__ miss, HEntry* t, const int64_t* dev,
                                                     int32_t* __restrict__ hslot) {
  if (dev[0] == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MemberView mv = stage_members(reinterpret_cast<MemberSmem*>(smem_raw), mt, F);
  const int64_t cap = scratch_cap_for(dev[0]);
  const uint64_t mask = (uint64_t)(cap - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!miss[i]) continue;
    long long key = key_of(ids[i], mv, F, namespaced, i);
    int64_t h;
    if (key == kEmptyKey) {
      h = cap;
      if (*reinterpret_cast<volatile long long*>(&t[h].val) > i) atomicMin(&t[h].val, (long long)i);
    } else {  // one 128-bit CAS claims the bucket with this position, or lowers it (none if already lower)
      h = (int64_t)insert_or_lower(t, bucket_hash((uint64_t)key) & mask, mask, key, (long long)i);
    }
    hslot[i] = (int32_t)h;
  }
}

// K3: fresh flags + per-tile fresh counts (tile = kRankTile positions, one block)
__global__ void __launch_bounds__(256) k_miss_fresh(int64_t n, const uint8_t* __restrict__ miss, const HEntry* t,
                                                    const int64_t* dev, const int32_t* __restrict__ hslot,
                                                    uint8_t* __restrict__ fresh, int64_t* __restrict__ tile_cnt) {
  if (dev[0] == 0) return;
  __shared__ int s_cnt;
  const int64_t ntiles = (n + kRankTile - 1) / kRankTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int local = 0;
    const int64_t b = tile * kRankTile, e = b + kRankTile < n ? b + kRankTile : n;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      uint8_t f = miss[i] && t[hslot[i]].val == i;
      fresh[i] = f;
      local += f;
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffff, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(&s_cnt, local);
    __syncthreads();
    if (threadIdx.x == 0) tile_cnt[tile] = s_cnt;
    __syncthreads();
  }
}

// K3b: exclusive scan of the tile counts in one block; K -> dev[1]
__global__ void __launch_bounds__(1024) k_scan_tiles(int64_t* tile_cnt, int64_t ntiles, int64_t* dev) {
  if (dev[0] == 0) return;
  __shared__ int64_t s_sum[32];
  __shared__ int64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < ntiles ? tile_cnt[i] : 0;
    // block inclusive scan
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffff, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_sum[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t s = lane < (int)(blockDim.x >> 5) ? s_sum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffff, s, o);
        if (lane >= o) s += y;
      }
      s_sum[lane] = s;
    }
    __syncthreads();
    int64_t incl = x + (w ? s_sum[w - 1] : 0) + s_carry;
    if (i < ntiles) tile_cnt[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) dev[1] = s_carry;
}

// K3c: rank of each fresh position = tile offset + rank within the tile
__global__ void __launch_bounds__(256) k_rank_fresh(int64_t n, const uint8_t* __restrict__ fresh,
                                                    const int64_t* __restrict__ tile_off, const int64_t* dev,
                                                    int64_t* __restrict__ rank, uint32_t* __restrict__ fpos) {
  if (dev[0] == 0) return;
  __shared__ int s_w[8];
  const int64_t ntiles = (n + kRankTile - 1) / kRankTile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int64_t carry = tile_off[tile];
    const int64_t b = tile * kRankTile, e = b + kRankTile < n ? b + kRankTile : n;
    for (int64_t base = b; base < e; base += blockDim.x) {
      int64_t i = base + threadIdx.x;
      bool f = i < e && fresh[i];
      unsigned bal = __ballot_sync(0xffffffff, f);
      if (lane == 0) s_w[w] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
      for (int k = 0; k < 8; ++k) {
        before += k < w ? s_w[k] : 0;
        total += s_w[k];
      }
      if (f) {
        const int64_t r = carry + before + __popc(bal & ((1u << lane) - 1));
        rank[i] = r;
        fpos[r] = (uint32_t)i;
      }
      carry += total;
      __syncthreads();
    }
  }
}

// K4: admission of the k-th fresh key (input order) — same slot rule as
// lookup_or_insert; the slot is published in the scratch entry for K5.
__global__ void __launch_bounds__(256) k_fused_admit(
    const int64_t* __restrict__ ids, int64_t n, const MemberDev* __restrict__ mt, int F, int namespaced,
    const uint32_t* __restrict__ fpos, const int32_t* __restrict__ hslot,
    HEntry* scratch, const int64_t* dev, const int64_t* __restrict__ counters, const int64_t* __restrict__ free_list,
    HEntry* map, uint64_t mask, int64_t cap, int64_t step, int D, uint64_t seed_mix, double scale,
    float* __restrict__ arena, int64_t* __restrict__ last_step, uint8_t* __restrict__ live,
    int64_t* __restrict__ slot_key, int64_t* __restrict__ ins_seq, int64_t arena_rows) {
  if (dev[0] == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MemberView mv = stage_members(reinterpret_cast<MemberSmem*>(smem_raw), mt, F);
  const int chunks = (D + 3) / 4;
  const int64_t total = dev[1] * chunks;  // K new keys (their positions compacted by k_rank_fresh)
  const int64_t A = counters[C_ALLOC], Fr = counters[C_FREE], seq = counters[C_SEQ];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / chunks;
    const int64_t i = fpos[k];
    const int ch = (int)(t - k * chunks);
    int64_t slot = assign_slot(k, Fr, A, free_list);
    if (slot >= arena_rows) __trap();  // host reservation bound violated: fail loudly
    long long key = key_of(ids[i], mv, F, namespaced, i);
    if (ch == 0) {
      idmap_insert(map, mask, cap, key, slot);
      last_step[slot] = step;
      live[slot] = 1;
      slot_key[slot] = key;
      ins_seq[slot] = seq + k;
      scratch[hslot[i]].val = slot;
    }
    uint64_t base = mix64((uint64_t)key ^ seed_mix);
    float* row = arena + slot * (int64_t)(3 * D);
    init_row_chunk(row, D, ch, base, scale);
  }
}

// K5
__global__ void k_miss_resolve(int64_t n, const uint8_t* __restrict__ miss, const HEntry* scratch,
                               const int32_t* __restrict__ hslot, const int64_t* dev, uint32_t* __restrict__ slot) {
  if (dev[0] == 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (miss[i]) slot[i] = (uint32_t)scratch[hslot[i]].val;
}

__global__ void k_fused_finish(int64_t* counters, int64_t* dev) {
  if (dev[0] == 0) return;
  int64_t K = dev[1], F = counters[C_FREE];
  int64_t take = K < F ? K : F;
  counters[C_FREE] = F - take;
  counters[C_ALLOC] += K - take;
  counters[C_ROWS] += K;
  counters[C_SEQ] += K;
}

// arena rows through a position->slot map (shared-memory tile or global)
struct ArenaSrc {
  const float* arena;
  const uint32_t* slot;  // indexed by position (already offset for smem tiles)
  int64_t stride;        // floats per row: 3*D in the table arena, D for plain rows
  int c;
  template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T load(int64_t p) const {
    return vload<VEC>(arena + (int64_t)slot[p] * stride + c);
  }
};

struct PoolSmem {
  MemberSmem m;
  int64_t off[kTileBags + 1];
  uint32_t slot[kTilePos];
};

// K6 (every member pools with `scatter`, the short-bag regime): warps own
// chunks of 32 bags; lane i loads bag i's offsets and first slot (coalesced),
// then sub-groups of L lanes gather R bags' rows at once.  The fold starts
// from +0 like np.add.at.  No member logic is needed on this path.
// one chunk of 32 bags (warp-cooperative), see k_fused_pool_scatter
template <int VEC, int R>
__device__ __forceinline__ void pool_chunk(const float* __restrict__ arena, const uint32_t* __restrict__ slot,
                                           int64_t g0, int nb, int64_t b, int64_t e, uint32_t s0, int lane, int mode,
                                           int D, int64_t D3, float* __restrict__ out) {
  using T = typename VecT<VEC>::T;
  const int rowv = D / VEC;
  const int L = rowv < 32 ? rowv : 32;
  const int P = 32 / L;
  const int sub = lane / L, sl = lane - sub * L;
  for (int base = 0; base < nb; base += R * P) {
    int bi[R];
    int64_t bb[R], ee[R];
    uint32_t ss[R];
    bool ok[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      bi[r] = base + r * P + sub;
      const int src = bi[r] < 32 ? bi[r] : 31;
      bb[r] = __shfl_sync(0xffffffffu, b, src);
      ee[r] = __shfl_sync(0xffffffffu, e, src);
      ss[r] = __shfl_sync(0xffffffffu, s0, src);
      ok[r] = sub < P && bi[r] < nb;
    }
    for (int c = sl * VEC; c < D; c += L * VEC) {
      T acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r] = vfill<VEC>(0.f);
        if (ok[r] && ee[r] > bb[r]) acc[r] = vadd<VEC>(acc[r], vload<VEC>(arena + (int64_t)ss[r] * D3 + c));
      }
      // the rest of every bag, kPoolBatch positions at a time: all R bags'
      // slot loads, then all their row loads, are in flight together before
      // the adds (which stay in position order: the fold is bit-exact)
      constexpr int kPoolBatch = R >= 4 ? 1 : 4 / R;  // R * kPoolBatch rows in flight per lane (no spills at MINB 4)
      int64_t pr[R];
      bool more = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        pr[r] = bb[r] + 1;
        more |= ok[r] && pr[r] < ee[r];
      }
      while (more) {
        uint32_t sl[R][kPoolBatch];
        T v[R][kPoolBatch];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int u = 0; u < kPoolBatch; ++u)
            sl[r][u] = (ok[r] && pr[r] + u < ee[r]) ? __ldg(slot + pr[r] + u) : 0xFFFFFFFFu;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int u = 0; u < kPoolBatch; ++u)
            if (sl[r][u] != 0xFFFFFFFFu) v[r][u] = vload<VEC>(arena + (int64_t)sl[r][u] * D3 + c);
        more = false;
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
          for (int u = 0; u < kPoolBatch; ++u)
            if (sl[r][u] != 0xFFFFFFFFu) acc[r] = vadd<VEC>(acc[r], v[r][u]);
          pr[r] += kPoolBatch;
          more |= ok[r] && pr[r] < ee[r];
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!ok[r]) continue;
        if (mode == 1 && ee[r] > bb[r]) acc[r] = vdiv<VEC>(acc[r], (float)(ee[r] - bb[r]));
        vstore<VEC>(out + (g0 + bi[r]) * D + c, acc[r]);
      }
    }
  }
}

// Wide rows (one or two rows per warp instruction, D >= 64): a sub-group
// owns a contiguous run of the chunk's bags, i.e. a contiguous range of
// positions, and streams it K positions at a time — K slot loads, then K row
// loads in flight, then the adds in position order, a bag's sum stored as
// soon as its last position is added.  Bit-exact (same fold from +0, same
// order); far more bytes in flight per warp than one bag at a time.
template <int VEC, int K>
__device__ __forceinline__ void pool_chunk_stream(const float* __restrict__ arena, const uint32_t* __restrict__ slot,
                                                  int64_t g0, int nb, int64_t b, int64_t e, int lane, int mode,
                                                  int D, int64_t D3, float* __restrict__ out, int64_t* s_e) {
  using T = typename VecT<VEC>::T;
  const int rowv = D / VEC;
  const int L = rowv < 32 ? rowv : 32;
  const int P = 32 / L;
  const int sub = lane / L, sl = lane - sub * L;
  const int per = (nb + P - 1) / P;
  const int q0 = sub * per < nb ? sub * per : nb, q1 = q0 + per < nb ? q0 + per : nb;
  __syncwarp();
  if (lane < nb) s_e[lane] = e;
  const int64_t bstart = __shfl_sync(0xffffffffu, b, q0 < 32 ? q0 : 31);
  __syncwarp();
  if (sub >= P || q0 >= q1) return;
  const int64_t pend = s_e[q1 - 1];
  for (int c = sl * VEC; c < D; c += L * VEC) {
    int q = q0;
    int64_t bq = bstart, eq = s_e[q];
    while (q < q1 && eq == bq) {  // leading empty bags
      vstore<VEC>(out + (g0 + q) * D + c, vfill<VEC>(0.f));
      ++q;
      eq = q < q1 ? s_e[q] : 0;
    }
    T acc = vfill<VEC>(0.f);
    for (int64_t p = bstart; p < pend; p += K) {
      uint32_t sv[K];
      T v[K];
#pragma unroll
      for (int u = 0; u < K; ++u) sv[u] = p + u < pend ? __ldg(slot + p + u) : 0u;
#pragma unroll
      for (int u = 0; u < K; ++u)
        if (p + u < pend) v[u] = vload<VEC>(arena + (int64_t)sv[u] * D3 + c);
#pragma unroll
      for (int u = 0; u < K; ++u) {
        if (p + u >= pend) continue;
        acc = vadd<VEC>(acc, v[u]);
        if (p + u + 1 == eq) {  // bag q complete
          vstore<VEC>(out + (g0 + q) * D + c, mode == 1 ? vdiv<VEC>(acc, (float)(eq - bq)) : acc);
          acc = vfill<VEC>(0.f);
          ++q;
          bq = eq;
          eq = q < q1 ? s_e[q] : 0;
          while (q < q1 && eq == bq) {  // empty bags after it
            vstore<VEC>(out + (g0 + q) * D + c, vfill<VEC>(0.f));
            ++q;
            eq = q < q1 ? s_e[q] : 0;
          }
        }
      }
    }
  }
}

template <int VEC, int R, int MINB>
__global__ void __launch_bounds__(256, MINB) k_fused_pool_scatter(const float* __restrict__ arena,
                                                                  const uint32_t* __restrict__ slot,
                                                                  const int64_t* __restrict__ bag_offs, int64_t G,
                                                                  int mode, int D, int64_t stride,
                                                                  float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (G + 31) / 32;
  for (int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += warps) {
    const int64_t g0 = ch * 32;
    const int nb = (int)(G - g0 < 32 ? G - g0 : 32);
    int64_t b = 0, e = 0;
    uint32_t s0 = 0;
    if (lane < nb) {
      b = __ldg(bag_offs + g0 + lane);
      e = __ldg(bag_offs + g0 + lane + 1);
      if (e > b) s0 = __ldg(slot + b);
    }
    pool_chunk<VEC, R>(arena, slot, g0, nb, b, e, s0, lane, mode, D, stride, out);
  }
}

// K6 for wide rows (VEC 4, 64 <= D <= 128): warps own chunks of 32 bags,
// sub-groups stream their bags' positions (pool_chunk_stream)
template <int K, int MINB>
__global__ void __launch_bounds__(256, MINB) k_fused_pool_stream(const float* __restrict__ arena,
                                                                 const uint32_t* __restrict__ slot,
                                                                 const int64_t* __restrict__ bag_offs, int64_t G,
                                                                 int mode, int D, int64_t stride,
                                                                 float* __restrict__ out) {
  __shared__ int64_t s_end[8][32];
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (G + 31) / 32;
  for (int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += warps) {
    const int64_t g0 = ch * 32;
    const int nb = (int)(G - g0 < 32 ? G - g0 : 32);
    int64_t b = 0, e = 0;
    if (lane < nb) {
      b = __ldg(bag_offs + g0 + lane);
      e = __ldg(bag_offs + g0 + lane + 1);
    }
    pool_chunk_stream<4, K>(arena, slot, g0, nb, b, e, lane, mode, D, stride, out, s_end[threadIdx.x >> 5]);
  }
}

// K6 staged variant (D % 4 == 0, D <= 128): a chunk whose 32 bags all hold
// exactly one id (the one-hot regime of C2) is a pure row gather — the
// warp's lanes issue 16-byte cp.async copies of all its rows into shared
// memory at once (no registers held while they fly: far more bytes in flight
// per SM than register-staged loads), then stream the chunk's contiguous
// output rows out.  +0.0f is added on the way out: np.add.at's fold from +0
// maps -0 to +0 (and x/1 == x for mean).  Other chunks take pool_chunk.
__global__ void __launch_bounds__(256) k_fused_pool_staged(const float* __restrict__ arena,
                                                           const uint32_t* __restrict__ slot,
                                                           const int64_t* __restrict__ bag_offs, int64_t G, int mode,
                                                           int D, int64_t stride, float* __restrict__ out) {
  extern __shared__ __align__(16) float pool_buf[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* buf = pool_buf + (int64_t)w * 32 * D;
  const int rowv = D >> 2;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (G + 31) / 32;
  for (int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += warps) {
    const int64_t g0 = ch * 32;
    const int nb = (int)(G - g0 < 32 ? G - g0 : 32);
    int64_t b = 0, e = 0;
    uint32_t s0 = 0;
    if (lane < nb) {
      b = __ldg(bag_offs + g0 + lane);
      e = __ldg(bag_offs + g0 + lane + 1);
      if (e > b) s0 = __ldg(slot + b);
    }
    if (__all_sync(0xffffffffu, lane >= nb || e - b == 1)) {
      for (int it = 0; it < rowv; ++it) {  // piece q = it*32 + lane of nb*rowv 16-byte pieces
        const int q = it * 32 + lane;
        const int r = q / rowv;
        const uint32_t sr = __shfl_sync(0xffffffffu, s0, r & 31);
        if (r < nb) {
          const int c = (q - r * rowv) * 4;
          cp_async16(buf + r * D + c, arena + (int64_t)sr * stride + c);
        }
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      float4* dst = reinterpret_cast<float4*>(out + g0 * D);
      const float4* src = reinterpret_cast<const float4*>(buf);
      for (int q = lane; q < nb * rowv; q += 32) {
        float4 v = src[q];
        v.x = __fadd_rn(v.x, 0.f);
        v.y = __fadd_rn(v.y, 0.f);
        v.z = __fadd_rn(v.z, 0.f);
        v.w = __fadd_rn(v.w, 0.f);
        __stcs(dst + q, v);
      }
      __syncwarp();
    } else {
      pool_chunk<4, 2>(arena, slot, g0, nb, b, e, s0, lane, mode, D, stride, out);
    }
  }
}

__global__ void k_iota_offs(int64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = i;
}

// bag of every position (sort payload for the backward), thread per bag
__global__ void k_bag_of(const int64_t* __restrict__ bag_offs, int64_t G, uint32_t* __restrict__ bag_of) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = __ldg(bag_offs + g), e = __ldg(bag_offs + g + 1);
    for (int64_t p = b; p < e; ++p) bag_of[p] = (uint32_t)g;
  }
}

// K6 (general: some member pools with the pairwise `sequential` strategy):
// tiles of kTileBags bags; lanes per row L = D / VEC (<= 32), groups of L
// lanes take bags round-robin.  Slots and bag offsets come from shared memory.
template <int VEC>
__global__ void __launch_bounds__(256) k_fused_pool_general(const float* __restrict__ arena, const uint32_t* __restrict__ slot,
                                                    const int64_t* __restrict__ bag_offs, int64_t G,
                                                    const MemberDev* __restrict__ mt, int F, int mode, int D,
                                                    int64_t stride, float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PoolSmem* sm = reinterpret_cast<PoolSmem*>(smem_raw);
  MemberView mv = stage_members(&sm->m, mt, F);
  const int rowv = D / VEC;
  const int L = rowv < 32 ? rowv : 32;
  const int groups = blockDim.x / L;
  const int grp = threadIdx.x / L, lane = threadIdx.x - grp * L;
  const int64_t ntiles = (G + kTileBags - 1) / kTileBags;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t g0 = tile * kTileBags;
    const int nb = (int)(G - g0 < kTileBags ? G - g0 : kTileBags);
    __syncthreads();
    for (int i = threadIdx.x; i <= nb; i += blockDim.x) sm->off[i] = __ldg(bag_offs + g0 + i);
    __syncthreads();
    const int64_t p0 = sm->off[0];
    const int64_t np = sm->off[nb] - p0;
    const bool staged = np <= kTilePos;
    if (staged)
      for (int i = threadIdx.x; i < np; i += blockDim.x) sm->slot[i] = __ldg(slot + p0 + i);
    __syncthreads();
    const uint32_t* sl = staged ? sm->slot - p0 : slot;
    if (grp >= groups) continue;
    for (int bi = grp; bi < nb; bi += groups) {
      const int64_t g = g0 + bi;
      const int64_t b = sm->off[bi], e = sm->off[bi + 1];
      const int f = F == 1 ? 0 : mv_member_of_bag(mv, F, g);
      const int strat = (int)mv.strat[f * mv.stride];
      const bool last = g == mv_bag(mv, f + 1) - 1;
      const int64_t nend = mv_pos(mv, f + 1);
      for (int c = lane * VEC; c < D; c += L * VEC) {
        ArenaSrc src{arena, sl, stride, c};
        typename VecT<VEC>::T acc = strat == 0 ? pool_sequential<VEC>(src, b, reduceat_end(b, e, last, nend))
                                               : pool_scatter<VEC>(src, b, e);
        if (mode == 1 && e > b) acc = vdiv<VEC>(acc, (float)(e - b));
        vstore<VEC>(out + g * D + c, acc);
      }
    }
  }
}

// adam1 over a vector of columns
template <int VEC>
__device__ __forceinline__ void adam_vec(typename VecT<VEC>::T& p, typename VecT<VEC>::T& m,
                                         typename VecT<VEC>::T& v, const typename VecT<VEC>::T& g, const AdamDev& a) {
  if constexpr (VEC == 4) {
    adam1(p.x, m.x, v.x, g.x, a);
    adam1(p.y, m.y, v.y, g.y, a);
    adam1(p.z, m.z, v.z, g.z, a);
    adam1(p.w, m.w, v.w, g.w, a);
  } else {
    adam1(p, m, v, g, a);
  }
}

// First position >= x whose sorted key differs from `key` (keys are sorted,
// so galloping + binary search: O(log run) dependent loads, not O(run)).
__device__ __forceinline__ int64_t run_end(const uint32_t* __restrict__ skey, int64_t n, int64_t x, uint32_t key) {
  if (x >= n || __ldg(skey + x) != key) return x;
  int64_t lo = x, step = 1;  // skey[lo] == key
  while (true) {
    const int64_t hi = lo + step;
    if (hi >= n || __ldg(skey + hi) != key) {
      int64_t a = lo, b = hi < n ? hi : n;  // skey[a] == key, b is past the run
      while (b - a > 1) {
        const int64_t mid = (a + b) >> 1;
        if (__ldg(skey + mid) == key) a = mid; else b = mid;
      }
      return b;
    }
    lo = hi;
    step <<= 1;
  }
}

// position of the k-th (0-based) set bit of x, or -1
__device__ __forceinline__ int nth_bit(unsigned x, int k) {
  unsigned r = __fns(x, 0, k + 1);
  return r == 0xFFFFFFFFu ? -1 : (int)r;
}

// gradient row of a sorted position: dpooled[g], or the all-zero row for
// positions outside their bag's tile (tile combiner, j >= k): folding +0 into
// a left fold from +0 never changes it, but the row is still touched
constexpr uint32_t kZeroRow = 0xFFFFFFFFu;
__device__ __forceinline__ const float* grad_row(const float* dp, const float* zrow, uint32_t g, int D) {
  return g == kZeroRow ? zrow : dp + (int64_t)g * D;
}

// tile combiner, index phase: gradient row of every position = its row of the
// bag's tile (g*k + j) for j < k, the zero row past k (segment_tile keeps only
// the first k rows, segments.py:94-116); one warp per bag
__global__ void k_tile_row_of(const int64_t* __restrict__ bag_offs, int64_t G, int64_t k, uint32_t* __restrict__ row_of) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < G; g += nw) {
    const int64_t b = __ldg(bag_offs + g), e = __ldg(bag_offs + g + 1);
    for (int64_t p = b + lane; p < e; p += 32) {
      const int64_t j = p - b;
      row_of[p] = j < k ? (uint32_t)(g * k + j) : kZeroRow;
    }
  }
}

// tile combiner, forward: out[g, j*D:(j+1)*D] = w[slot of position off[g]+j]
// for j < min(len, k), `pad` for len <= j < k (segment_tile, bit-exact copy).
template <int VEC>
__global__ void __launch_bounds__(256) k_fused_tile(const float* __restrict__ arena, const uint32_t* __restrict__ slot,
                                                    const int64_t* __restrict__ bag_offs, int64_t G, int64_t k, int D,
                                                    int64_t D3, float pad, float* __restrict__ out, int wpb) {
  // wpb warps own one bag's [k, D] output tile at a time: the bag's offsets are
  // read once, the tile is a contiguous run of k * D / VEC vectors walked
  // 32 lanes x U at a time (U loads in flight per lane), and the row / column
  // of an element come from 32-bit shifts (no 64-bit division per element)
  using V = typename VecT<VEC>::T;
  constexpr int U = 4;
  const int per_row = D / VEC;
  const bool pow2 = (per_row & (per_row - 1)) == 0;
  const int sh = __ffs(per_row) - 1;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t tile_v = k * per_row;  // vectors per bag tile
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < G * wpb; w += warps) {
    const int64_t g = w / wpb;
    const int part = (int)(w - g * wpb);
    const int64_t b = __ldg(bag_offs + g), len = __ldg(bag_offs + g + 1) - b;
    float* dst = out + g * k * D;
    for (int64_t q0 = lane + (int64_t)part * 32 * U; q0 < tile_v; q0 += (int64_t)32 * U * wpb) {
      V v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + 32 * u;
        v[u] = vfill<VEC>(pad);
        if (q < tile_v) {
          const int64_t j = pow2 ? (q >> sh) : q / per_row;
          if (j < len) {
            const int c = (int)(q - j * per_row) * VEC;
            v[u] = vload<VEC>(arena + (int64_t)__ldg(slot + b + j) * D3 + c);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + 32 * u;
        if (q < tile_v) vstore<VEC>(dst + q * VEC, v[u]);
      }
    }
  }
}

// K9: fold + Adam.  Warps own chunks of 32 sorted positions; a run head
// (first position of a slot) is found by ballot on skey[j] != skey[j-1], so
// no separate run-heads pass is needed.  Sub-groups of L lanes take 2 heads
// each per pass: both rows' w, m, v and first dpooled loads are in flight
// before any arithmetic.  A run continuing past its chunk is finished by the
// warp owning its head (the next chunk sees no head there).
constexpr int kFoldBatch = 2;  // gradient rows in flight per run in k_fused_adam's fold (same-box A/B: 1, 3, 4 slower)

template <int VEC, int R, int MINB, bool ADAM = true>
__global__ void __launch_bounds__(256, MINB) k_fused_adam(int64_t n, const uint32_t* __restrict__ skey,
                                                    const uint32_t* __restrict__ sval,
                                                    const int64_t* __restrict__ bag_offs,
                                                    const float* __restrict__ dpooled, int mode, int D, AdamDev a,
                                                    float* __restrict__ arena, int64_t* __restrict__ last_step,
                                                    int64_t step, int64_t* __restrict__ dev_unique,
                                                    LongRun* __restrict__ longs, int64_t* __restrict__ nlong,
                                                    int64_t longs_cap, const float* __restrict__ zrow = nullptr,
                                                    RowOut ro = RowOut{}) {
  using T = typename VecT<VEC>::T;
  __shared__ uint32_t s_bag[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int rowv = D / VEC;
  const int L = rowv < 32 ? rowv : 32;
  const int P = 32 / L;
  const int sub = lane / L, sl = lane - sub * L;
  const bool active_sub = sub < P;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (n + 31) / 32;
  const int64_t D3 = 3 * (int64_t)D;
  unsigned long long heads_seen = 0;
  for (int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += warps) {
    const int64_t j0 = ch * 32;
    const int64_t j = j0 + lane;
    const bool valid = j < n;
    const uint32_t k = valid ? __ldg(skey + j) : 0xFFFFFFFFu;
    const uint32_t kp = (valid && j > 0) ? __ldg(skey + j - 1) : 0xFFFFFFFFu;
    s_bag[wib][lane] = valid ? __ldg(sval + j) : 0u;
    __syncwarp();
    const unsigned hm = __ballot_sync(0xffffffffu, valid && (j == 0 || k != kp));
    heads_seen += __popc(hm);
    unsigned rem = hm;
    while (rem) {
      int h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = active_sub ? nth_bit(rem, sub + r * P) : -1;
      const int last = nth_bit(rem, R * P - 1);
      rem = last < 0 ? 0u : (last == 31 ? 0u : rem & (~0u << (last + 1)));
      uint32_t slot[R];
      int64_t e[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        slot[r] = __shfl_sync(0xffffffffu, k, h[r] < 0 ? 0 : h[r]);
        unsigned above = (h[r] < 0 || h[r] == 31) ? 0u : (hm & (~0u << (h[r] + 1)));
        e[r] = above ? j0 + __ffs(above) - 1 : j0 + 32;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (h[r] >= 0 && e[r] == j0 + 32) {  // run may continue into later chunks
          int64_t x = e[r];
          x = run_end(skey, n, x, slot[r]);
          e[r] = x < n ? x : n;
        }
        // hot ids: defer to the CTA-per-run long fold (VEC == 4 only)
        if (VEC == 4 && longs && h[r] >= 0 && e[r] - (j0 + h[r]) > kLongRun) {
          if (sl == 0) push_long_run(longs, nlong, longs_cap, slot[r], (uint32_t)(j0 + h[r]), (uint32_t)e[r]);
          h[r] = -1;
        }
      }
      for (int c = sl * VEC; c < D; c += L * VEC) {
        T p[R], m[R], v[R], acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (h[r] >= 0) {
            if constexpr (ADAM) {
              const float* row = arena + (int64_t)slot[r] * D3;
              p[r] = vload<VEC>(row + c);
              m[r] = vload<VEC>(row + D + c);
              v[r] = vload<VEC>(row + 2 * D + c);
            }
            const uint32_t g = s_bag[wib][h[r]];
            T x = vload<VEC>(grad_row(dpooled, zrow, g, D) + c);
            if (mode == 1) x = vdiv<VEC>(x, (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g)));
            acc[r] = vadd<VEC>(vfill<VEC>(0.f), x);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (h[r] < 0) continue;
          int64_t jj = j0 + h[r] + 1;
          // runs of up to kLongRun positions: kFoldBatch gradient rows in
          // flight per step of the chain (their loads do not depend on the
          // accumulator), added strictly in position order — the same FADD
          // sequence as one row at a time, so still bit-exact
          for (; jj + kFoldBatch <= e[r]; jj += kFoldBatch) {
            uint32_t g[kFoldBatch];
            T x[kFoldBatch];
#pragma unroll
            for (int q = 0; q < kFoldBatch; ++q)
              g[q] = jj + q < j0 + 32 ? s_bag[wib][jj + q - j0] : __ldg(sval + jj + q);
#pragma unroll
            for (int q = 0; q < kFoldBatch; ++q) x[q] = vload<VEC>(grad_row(dpooled, zrow, g[q], D) + c);
            if (mode == 1) {
#pragma unroll
              for (int q = 0; q < kFoldBatch; ++q)
                x[q] = vdiv<VEC>(x[q], (float)(__ldg(bag_offs + g[q] + 1) - __ldg(bag_offs + g[q])));
            }
#pragma unroll
            for (int q = 0; q < kFoldBatch; ++q) acc[r] = vadd<VEC>(acc[r], x[q]);
          }
          for (; jj < e[r]; ++jj) {
            const uint32_t g = jj < j0 + 32 ? s_bag[wib][jj - j0] : __ldg(sval + jj);
            T x = vload<VEC>(grad_row(dpooled, zrow, g, D) + c);
            if (mode == 1) x = vdiv<VEC>(x, (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g)));
            acc[r] = vadd<VEC>(acc[r], x);
          }
          if constexpr (ADAM) {
            adam_vec<VEC>(p[r], m[r], v[r], acc[r], a);
            float* row = arena + (int64_t)slot[r] * D3;
            vstore<VEC>(row + c, p[r]);
            vstore<VEC>(row + D + c, m[r]);
            vstore<VEC>(row + 2 * D + c, v[r]);
          } else {  // fold only: acc -> out[key] (arena is the [U, D] output, or ro's peer rows)
            vstore<VEC>(ro.row(arena, slot[r], D) + c, acc[r]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (ADAM && h[r] >= 0 && sl == 0 && step >= 0) last_step[slot[r]] = step;
    }
    __syncwarp();
  }
  if (lane == 0 && heads_seen) atomicAdd(reinterpret_cast<unsigned long long*>(dev_unique), heads_seen);
  if (!ADAM && ro.peers) __threadfence_system();  // peer stores before the stream's barrier write
}

// ---------------------------------------------------------------------------
// K9 (TMA variant): warp-specialized fold + Adam.  Warp 0 of each CTA is the
// producer: it scans the CTA's slice of sorted positions 32 at a time, finds
// run heads by ballot, and for each run issues two bulk async copies
// (cp.async.bulk, completion on an mbarrier): the row's contiguous 12*D-byte
// [w|m|v] span and the dpooled row of the run's first position, into a ring
// of kTmaStages shared-memory stages of kTmaRows rows.  Warps 1.. consume:
// Adam from shared memory, results stored straight to HBM, the stage handed
// back through an `empty` mbarrier.  Loads are issued by the TMA engine, so
// bytes in flight no longer scale with registers per thread.
// ---------------------------------------------------------------------------
constexpr int kTmaStages = 3;

struct TmaDesc {
  uint32_t slot, bag, jh, je;
};

template <int kTmaRows, int kTmaThreads, int MINB>
__global__ void __launch_bounds__(kTmaThreads, MINB) k_fused_adam_tma(int64_t n, const uint32_t* __restrict__ skey,
                                                                    const uint32_t* __restrict__ sval,
                                                                    const int64_t* __restrict__ bag_offs,
                                                                    const float* __restrict__ dpooled, int mode, int D,
                                                                    AdamDev a, float* __restrict__ arena,
                                                                    int64_t* __restrict__ last_step, int64_t step,
                                                                    int64_t* __restrict__ dev_unique,
                                                                    LongRun* __restrict__ longs,
                                                                    int64_t* __restrict__ nlong, int64_t longs_cap,
                                                                    const float* __restrict__ zrow) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int rowf = 3 * D;        // floats of [w|m|v]
  const int stage_f = kTmaRows * (rowf + D);
  float* rows = reinterpret_cast<float*>(smem_raw);  // [stage][kTmaRows][3D] then [stage][kTmaRows][D]
  float* dps = rows + kTmaStages * kTmaRows * rowf;
  TmaDesc* desc = reinterpret_cast<TmaDesc*>(dps + kTmaStages * kTmaRows * D);  // [stage][kTmaRows]
  int* count = reinterpret_cast<int*>(desc + kTmaStages * kTmaRows);           // [stage]
  uint64_t* full = reinterpret_cast<uint64_t*>(count + 4);                     // 16B aligned (count: 4 ints)
  uint64_t* empty = full + kTmaStages;
  (void)stage_f;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int consumers = (blockDim.x >> 5) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t jb = n * (int64_t)blockIdx.x / gridDim.x;
  const int64_t je = n * ((int64_t)blockIdx.x + 1) / gridDim.x;
  const uint32_t row_bytes = (uint32_t)rowf * 4u, dp_bytes = (uint32_t)D * 4u;
  const int64_t D3 = rowf;

  if (warp == 0) {
    // ---------------- producer ----------------
    int64_t jc = jb;          // next chunk start
    int64_t cbase = 0;        // current chunk base
    unsigned pend = 0, hm = 0;
    uint32_t ck = 0, cbag = 0;
    unsigned long long heads = 0;
    // metadata of chunk jc is loaded one chunk ahead (the producer is serial)
    auto load_chunk = [&](int64_t base, uint32_t& k, uint32_t& kp, uint32_t& bg) {
      const int64_t j = base + lane;
      const bool valid = j < je;
      k = valid ? __ldg(skey + j) : 0xFFFFFFFFu;
      kp = (valid && j > 0) ? __ldg(skey + j - 1) : 0xFFFFFFFFu;
      bg = valid ? __ldg(sval + j) : 0u;
    };
    uint32_t nk = 0, nkp = 0, nbg = 0;
    if (jc < je) load_chunk(jc, nk, nkp, nbg);
    for (int it = 0;; ++it) {
      const int s = it % kTmaStages;
      const uint32_t ph = (uint32_t)(it / kTmaStages) & 1u;
      mbar_wait(&empty[s], ph ^ 1u);
      int nrun = 0;
      while (nrun < kTmaRows) {
        if (!pend) {
          if (jc >= je) break;
          cbase = jc;
          const int64_t j = jc + lane;
          const bool valid = j < je;
          ck = nk;
          cbag = nbg;
          hm = __ballot_sync(0xffffffffu, valid && (j == 0 || nk != nkp));
          pend = hm;
          jc += 32;
          if (jc < je) load_chunk(jc, nk, nkp, nbg);
          heads += __popc(hm);
          continue;
        }
        // take up to (kTmaRows - nrun) of the pending heads, one per lane
        const int take = min(__popc(pend), kTmaRows - nrun);
        const int h = lane < take ? nth_bit(pend, lane) : -1;
        const uint32_t hk = __shfl_sync(0xffffffffu, ck, h < 0 ? 0 : h);
        const uint32_t hb = __shfl_sync(0xffffffffu, cbag, h < 0 ? 0 : h);
        // first key of the (prefetched) next chunk ends most runs without a scan
        const uint32_t next_first = __shfl_sync(0xffffffffu, nk, 0);
        const bool next_loaded = jc < je;  // jc already advanced past this chunk
        if (h >= 0) {
          unsigned above = (h == 31) ? 0u : (hm & (~0u << (h + 1)));
          int64_t e;
          if (above) {
            e = cbase + __ffs(above) - 1;
          } else if (next_loaded && next_first != hk) {
            e = cbase + 32;
          } else {  // last head of the chunk: the run may cross the chunk / CTA slice
            int64_t x = cbase + h + 1;
            x = run_end(skey, n, x, hk);
            e = x;
          }
          const int slot_i = nrun + lane;
          desc[s * kTmaRows + slot_i] = TmaDesc{hk, hb, (uint32_t)(cbase + h), (uint32_t)e};
          bulk_g2s(rows + ((int64_t)s * kTmaRows + slot_i) * rowf, arena + (int64_t)hk * D3, row_bytes, &full[s]);
          bulk_g2s(dps + ((int64_t)s * kTmaRows + slot_i) * D, grad_row(dpooled, zrow, hb, D), dp_bytes, &full[s]);
        }
        const int last = nth_bit(pend, take - 1);
        pend = (last == 31) ? 0u : pend & (~0u << (last + 1));
        nrun += take;
      }
      __syncwarp();
      if (lane == 0) {
        count[s] = nrun;
        mbar_arrive_expect_tx(&full[s], (uint32_t)nrun * (row_bytes + dp_bytes));
      }
      if (nrun == 0) break;  // sentinel stage: consumers exit
    }
    if (lane == 0 && heads) atomicAdd(reinterpret_cast<unsigned long long*>(dev_unique), heads);
    return;
  }

  // ---------------- consumers ----------------
  const int rowv = D / 4;
  const int L = rowv < 32 ? rowv : 32;
  const int P = 32 / L;
  const int sub = lane / L, sl = lane - sub * L;
  const int cw = warp - 1;  // consumer warp index
  const int groups = consumers * P;
  const int grp = cw * P + sub;
  for (int it = 0;; ++it) {
    const int s = it % kTmaStages;
    const uint32_t ph = (uint32_t)(it / kTmaStages) & 1u;
    mbar_wait(&full[s], ph);
    const int nr = count[s];
    if (nr == 0) break;
    if (sub < P) {
      for (int i = grp; i < nr; i += groups) {
        const TmaDesc d = desc[s * kTmaRows + i];
        if (d.je - d.jh > (uint32_t)kLongRun) {  // hot id: CTA-per-run long fold
          if (sl == 0) push_long_run(longs, nlong, longs_cap, d.slot, d.jh, d.je);
          continue;
        }
        const float* srow = rows + ((int64_t)s * kTmaRows + i) * rowf;
        const float* sdp = dps + ((int64_t)s * kTmaRows + i) * D;
        float* grow = arena + (int64_t)d.slot * D3;
        for (int c = sl * 4; c < D; c += L * 4) {
          float4 p = *reinterpret_cast<const float4*>(srow + c);
          float4 m = *reinterpret_cast<const float4*>(srow + D + c);
          float4 v = *reinterpret_cast<const float4*>(srow + 2 * D + c);
          float4 x = *reinterpret_cast<const float4*>(sdp + c);
          if (mode == 1) x = vdiv<4>(x, (float)(__ldg(bag_offs + d.bag + 1) - __ldg(bag_offs + d.bag)));
          float4 acc = add4(make_float4(0.f, 0.f, 0.f, 0.f), x);
          uint32_t jj = d.jh + 1;
          // two gradient rows in flight per step of the run, added in
          // position order (the same FADD sequence: bit-exact)
          for (; jj + 2 <= d.je; jj += 2) {
            const uint32_t g0 = __ldg(sval + jj), g1 = __ldg(sval + jj + 1);
            float4 y0 = ldg4(grad_row(dpooled, zrow, g0, D) + c);
            float4 y1 = ldg4(grad_row(dpooled, zrow, g1, D) + c);
            if (mode == 1) {
              y0 = vdiv<4>(y0, (float)(__ldg(bag_offs + g0 + 1) - __ldg(bag_offs + g0)));
              y1 = vdiv<4>(y1, (float)(__ldg(bag_offs + g1 + 1) - __ldg(bag_offs + g1)));
            }
            acc = add4(acc, y0);
            acc = add4(acc, y1);
          }
          for (; jj < d.je; ++jj) {
            const uint32_t g = __ldg(sval + jj);
            float4 y = ldg4(grad_row(dpooled, zrow, g, D) + c);
            if (mode == 1) y = vdiv<4>(y, (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g)));
            acc = add4(acc, y);
          }
          adam_vec<4>(p, m, v, acc, a);
          st4(grow + c, p);
          st4(grow + D + c, m);
          st4(grow + 2 * D + c, v);
        }
        if (sl == 0 && step >= 0) last_step[d.slot] = step;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

static size_t tma_smem_bytes(int D, int kTmaRows) {
  return (size_t)kTmaStages * kTmaRows * (4 * D) * sizeof(float) + kTmaStages * kTmaRows * sizeof(TmaDesc) +
         4 * sizeof(int) + 2 * kTmaStages * sizeof(uint64_t);
}

static int env_int(const char* name, int dflt);
template <int ROWS, int THREADS, int MINB, class... Args>
static void launch_adam_tma(int64_t n, int D, cudaStream_t s, Args... args) {
  auto* kern = k_fused_adam_tma<ROWS, THREADS, MINB>;
  note_param_kernel((const void*)kern, 16, 7, 10);
  const size_t sm = tma_smem_bytes(D, ROWS);
  static size_t sm_set = 0;
  if (sm_set < sm) {
    SKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    sm_set = sm;
  }
  // non-persistent: each CTA owns a fixed slice of sorted positions and
  // retires, so the high-priority index stream can take SM slots (pipeline)
  // slice: 1024 positions (measured best on C2), shrunk for small batches so
  // at least ~4 CTAs per SM share the work (a C1-size batch of 4096
  // positions on 4 CTAs took 130 us of serial ring latency)
  static const int64_t slice_env = env_int("SKB_TMA_SLICE", 0);
  int64_t per_cta = slice_env;
  if (per_cta == 0) {
    const int64_t want = (n + 4 * sm_count() - 1) / (4 * sm_count());
    per_cta = want < 64 ? 64 : (want > 1024 ? 1024 : want);
  }
  int64_t ctas = per_cta > 0 ? (n + per_cta - 1) / per_cta : 0;
  // (rounding the grid up to whole waves of 4 x 148 CTAs was measured slower
  // on C2: 0.69 vs 0.60 ms — the index stream's kernels share the SMs anyway)
  if (per_cta <= 0) {
    int per_sm = 0;
    SKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, sm));
    ctas = (int64_t)(per_sm > 0 ? per_sm : 1) * sm_count();
  }
  if (ctas < 1) ctas = 1;
  kern<<<(unsigned)ctas, THREADS, sm, s>>>(args...);
}

// load_stats of a prepared batch: one count per run head of the sorted slots
// (= per unique key), histogrammed by owner shard in shared memory
__global__ void __launch_bounds__(256) k_head_shard_counts(const uint32_t* __restrict__ skey, int64_t n,
                                                           const int64_t* __restrict__ slot_key, int S,
                                                           unsigned long long* counts) {
  __shared__ unsigned int hist[4096];
  for (int k = threadIdx.x; k < S; k += blockDim.x) hist[k] = 0u;
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = __ldg(skey + j);
    if (j == 0 || __ldg(skey + j - 1) != k)
      atomicAdd(&hist[S == 1 ? 0 : (int)(mix64((uint64_t)__ldg(slot_key + k)) % (uint64_t)S)], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < S; k += blockDim.x)
    if (hist[k]) atomicAdd(&counts[k], (unsigned long long)hist[k]);
}

// last_step of every position's slot (deferred forward bookkeeping)
__global__ void k_flush_last(const uint32_t* __restrict__ slot, int64_t n, int64_t step, int64_t* last_step) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    last_step[slot[i]] = step;
}

// K2..K5 as ONE cooperative launch: phases separated by grid-wide syncs, and
// the whole kernel returns at once when the device miss count is 0 (the warm
// steady state), so the miss path costs a single launch.
struct AdmitArgs {
  const int64_t* ids;
  int64_t n;
  const MemberDev* mt;
  int F, namespaced;
  const uint8_t* miss;
  HEntry* scratch;
  int32_t* hslot;
  uint8_t* fresh;
  int64_t* tile_cnt;
  int64_t* rank;
  uint32_t* fpos;
  int64_t* dev;
  int64_t* counters;
  const int64_t* free_list;
  HEntry* map;
  uint64_t mask;
  int64_t cap;
  int64_t step;
  int D;
  uint64_t seed_mix;
  double scale;
  float* arena;
  int64_t* last_step;
  uint8_t* live;
  int64_t* slot_key;
  int64_t* ins_seq;
  uint32_t* slot;
  int64_t arena_rows;
};

__global__ void __launch_bounds__(256) k_admission(AdmitArgs A) {
  if (A.dev[0] == 0) return;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t s_sum[32];
  __shared__ int64_t s_carry;
  __shared__ int s_cnt;
  __shared__ int s_w[8];
  const MemberView mv = stage_members(reinterpret_cast<MemberSmem*>(smem_raw), A.mt, A.F);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = A.n;
  const int64_t M = A.dev[0];
  const int64_t scap = scratch_cap_for(M);
  const uint64_t smask = (uint64_t)(scap - 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // 1. scratch table
  for (int64_t i = tid; i <= scap; i += nth)
    reinterpret_cast<longlong2*>(A.scratch)[i] = make_longlong2(kEmptyKey, 0x7FFFFFFFFFFFFFFFll);
  grid.sync();
  // 2. first-occurrence dedup among unknown keys
  for (int64_t i = tid; i < n; i += nth) {
    if (!A.miss[i]) continue;
    const long long key = key_of(A.ids[i], mv, A.F, A.namespaced, i);
    int64_t h;
    if (key == kEmptyKey) {
      h = scap;
    } else {
      h = (int64_t)(bucket_hash((uint64_t)key) & smask);
      while (true) {
        long long k = *reinterpret_cast<volatile long long*>(&A.scratch[h].key);
        if (k == key) break;
        if (k == kEmptyKey) {
          long long prev = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&A.scratch[h].key),
                                                (unsigned long long)kEmptyKey, (unsigned long long)key);
          if (prev == kEmptyKey || prev == key) break;
        }
        h = (int64_t)(((uint64_t)h + 1) & smask);
      }
    }
    if (*reinterpret_cast<volatile long long*>(&A.scratch[h].val) > i) atomicMin(&A.scratch[h].val, (long long)i);
    A.hslot[i] = (int32_t)h;
  }
  grid.sync();
  // 3. fresh flags + per-tile counts
  const int64_t ntiles = (n + kRankTile - 1) / kRankTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int local = 0;
    const int64_t b = tile * kRankTile, e = b + kRankTile < n ? b + kRankTile : n;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      uint8_t f = A.miss[i] && A.scratch[A.hslot[i]].val == i;
      A.fresh[i] = f;
      local += f;
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffff, local, o);
    if (lane == 0 && local) atomicAdd(&s_cnt, local);
    __syncthreads();
    if (threadIdx.x == 0) A.tile_cnt[tile] = s_cnt;
    __syncthreads();
  }
  grid.sync();
  // 4. exclusive scan of tile counts (block 0); K -> dev[1]
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < ntiles; base += blockDim.x) {
      const int64_t i = base + threadIdx.x;
      const int64_t v = i < ntiles ? A.tile_cnt[i] : 0;
      int64_t x = v;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffff, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_sum[w] = x;
      __syncthreads();
      if (w == 0) {
        int64_t t = lane < (int)(blockDim.x >> 5) ? s_sum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          int64_t y = __shfl_up_sync(0xffffffff, t, o);
          if (lane >= o) t += y;
        }
        s_sum[lane] = t;
      }
      __syncthreads();
      const int64_t incl = x + (w ? s_sum[w - 1] : 0) + s_carry;
      if (i < ntiles) A.tile_cnt[i] = incl - v;
      __syncthreads();
      if (threadIdx.x == blockDim.x - 1) s_carry = incl;
      __syncthreads();
    }
    if (threadIdx.x == 0) A.dev[1] = s_carry;
  }
  grid.sync();
  // 5. rank of each fresh position in input order
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int64_t carry = A.tile_cnt[tile];
    const int64_t b = tile * kRankTile, e = b + kRankTile < n ? b + kRankTile : n;
    for (int64_t base = b; base < e; base += blockDim.x) {
      const int64_t i = base + threadIdx.x;
      const bool f = i < e && A.fresh[i];
      const unsigned bal = __ballot_sync(0xffffffff, f);
      if (lane == 0) s_w[w] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
      for (int k = 0; k < 8; ++k) {
        before += k < w ? s_w[k] : 0;
        total += s_w[k];
      }
      if (f) {
        const int64_t r = carry + before + __popc(bal & ((1u << lane) - 1));
        A.rank[i] = r;
        A.fpos[r] = (uint32_t)i;
      }
      carry += total;
      __syncthreads();
    }
  }
  grid.sync();
  // 6. admission: slot rule of lookup_or_insert, init rows, publish slot
  {
    const int chunks = (A.D + 3) / 4;
    const int64_t total = A.dev[1] * chunks;  // K new keys, compacted in phase 5
    const int64_t Aa = A.counters[C_ALLOC], Fr = A.counters[C_FREE], seq = A.counters[C_SEQ];
    for (int64_t t = tid; t < total; t += nth) {
      const int64_t k = t / chunks;
      const int64_t i = A.fpos[k];
      const int ch = (int)(t - k * chunks);
      const int64_t slot = assign_slot(k, Fr, Aa, A.free_list);
      if (slot >= A.arena_rows) __trap();  // host reservation bound violated: fail loudly
      const long long key = key_of(A.ids[i], mv, A.F, A.namespaced, i);
      if (ch == 0) {
        idmap_insert(A.map, A.mask, A.cap, key, slot);
        A.last_step[slot] = A.step;
        A.live[slot] = 1;
        A.slot_key[slot] = key;
        A.ins_seq[slot] = seq + k;
        A.scratch[A.hslot[i]].val = slot;
      }
      const uint64_t base = mix64((uint64_t)key ^ A.seed_mix);
      float* row = A.arena + slot * (int64_t)(3 * A.D);
      init_row_chunk(row, A.D, ch, base, A.scale);
    }
  }
  grid.sync();
  // 7. every unknown position learns its slot; counters advance
  for (int64_t i = tid; i < n; i += nth)
    if (A.miss[i]) A.slot[i] = (uint32_t)A.scratch[A.hslot[i]].val;
  if (tid == 0) {
    const int64_t K = A.dev[1], F = A.counters[C_FREE];
    const int64_t take = K < F ? K : F;
    A.counters[C_FREE] = F - take;
    A.counters[C_ALLOC] += K - take;
    A.counters[C_ROWS] += K;
    A.counters[C_SEQ] += K;
  }
}

static int coop_grid(size_t smem) {
  static int blocks_per_sm = -1;
  if (blocks_per_sm < 0) {
    SKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_admission, 256, smem));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  return blocks_per_sm * sm_count();
}

// Pending-work barrier for every non-fused table op on stream s: index work
// must be complete, and pooled batches still awaiting their backward get
// their deferred last_step written (forward semantics of lookup_or_insert).
void fused_flush_pending(Table* t, cudaStream_t s) {
  FusedCtx* c = t->fused;
  if (!c) return;
  if (c->prep_count > 0) SKB_CUDA(cudaStreamWaitEvent(s, c->ev_side_last, 0));
  for (int64_t k = c->bwd_count; k < c->pool_count; ++k) {
    BatchCtx& B = c->b[k % 2];
    if (B.last_written || B.n == 0) continue;
    k_flush_last<<<grid_for(B.n, 256), 256, 0, s>>>(B.slot, B.n, B.step, t->last_step);
    SKB_LAUNCH_CHECK();
    B.last_written = true;
  }
}

void fused_wait_index(Table* t, cudaStream_t s) {
  FusedCtx* c = t->fused;
  if (c && c->prep_count > 0) SKB_CUDA(cudaStreamWaitEvent(s, c->ev_side_last, 0));
}

void fused_require_quiet(Table* t, bool allow_pooled, const char* op) {
  FusedCtx* c = t->fused;
  if (!c) return;
  if (c->prep_count > c->pool_count)
    raise(SKB_E_VALUE, 0, "%s while a prefetched fused batch is not pooled yet (prefetch admitted its ids): "
          "run its lookup_pool and pool_grad_adam first", op);
  if (!allow_pooled && c->pool_count > c->bwd_count)
    raise(SKB_E_VALUE, 0, "%s between a fused lookup_pool and its pool_grad_adam", op);
}

// kernel variant knobs for tuning sweeps (SKB_ADAM_VARIANT / SKB_POOL_VARIANT)
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
static int adam_variant() {
  static int v = env_int("SKB_ADAM_VARIANT", 0);
  return v;
}
static bool adam_tma_fits(int mode, int D, int64_t recent_long_runs) {
  // SKB_TMA_MEAN_MIN_D: narrowest row width whose mean batches also take the
  // TMA ring (0: mean batches always take the register kernel)
  static const int mean_min_d = env_int("SKB_TMA_MEAN_MIN_D", 0);
  // SKB_TMA_HOT=1: also for batches with recent long runs (the ring defers
  // them to the long fold like the register kernel)
  static const int hot = env_int("SKB_TMA_HOT", 0);
  const bool mode_ok = mode == 0 || (mode == 1 && mean_min_d > 0 && D >= mean_min_d);
  return mode_ok && D >= 48 && (hot || recent_long_runs == 0);
}
static int pool_variant() {
  static int v = env_int("SKB_POOL_VARIANT", 0);
  return v;
}

static size_t member_smem(int F) { return F <= kSmemMembers ? sizeof(MemberSmem) : 0; }


std::vector<ParamKernel>& param_kernels() {
  static std::vector<ParamKernel> v;
  return v;
}
void note_param_kernel(const void* func, int nargs, int ia, int is) {
  for (const ParamKernel& k : param_kernels())
    if (k.func == func) return;
  param_kernels().push_back(ParamKernel{func, nargs, ia, is});
}

// kernels of the step whose arguments carry the step / Adam scalars
// (argument positions are verified against the live values at capture)
static void register_param_kernels() {
  static bool done = false;
  if (done) return;
  done = true;
  note_param_kernel((const void*)k_fused_admit, 24, -1, 14);  // step is argument 14 (ids, n, mt, F, ns, fpos, hslot, ...)
  note_param_kernel((const void*)k_fused_adam<1, 1, 4>, 17, 7, 10);
  note_param_kernel((const void*)k_fused_adam<4, 2, 4>, 17, 7, 10);
  note_param_kernel((const void*)k_fused_adam<4, 1, 5>, 17, 7, 10);
  note_param_kernel((const void*)k_fused_adam<4, 1, 4>, 17, 7, 10);
  note_param_kernel((const void*)k_long_fold<true>, 22, 8, 11);  // (runs, nruns, cap, ridx, rows, D, bag_offs, mode, a, out, last_step, step, nst, zrow, packed, mlist, morder, mcount, ro, direct, ready, wctr)
}

// graph mode is off while per-phase event profiling is on (events cannot be
// recorded from inside a replayed graph)
static bool graph_mode(const FusedCtx* c) {
  if (!c->graphs || c->prof_cap != 0) return false;
  register_param_kernels();
  return true;
}

// Admission as a chain of ordinary launches that each return at once when
// the probe found no misses, or as ONE cooperative launch.  The cooperative
// kernel is capped at one CTA per SM so it co-resides with the previous
// step's fold+Adam: best when there is little or nothing to admit (C2 warm:
// 0.853 vs 0.876 ms/step, since eight launches on the index stream each
// queue behind the fold+Adam grid), but a growth regime (C3's zipf tail:
// ~400K new rows per step) runs 1.6x faster on the full-width phased grids.
// SKB_ADMIT_COOP: 1 (default) adaptive on the table's recent growth, 0
// always phased, 2 always cooperative.
constexpr int64_t kGrowthPhased = 65536;
static bool admit_coop(Table* t) {
  static int v = env_int("SKB_ADMIT_COOP", 1);
  if (v != 1) return v == 2;
  return table_recent_growth(t) < kGrowthPhased;
}

static void launch_admission_phased(const AdmitArgs& A, size_t msm, cudaStream_t x) {
  const int64_t n = A.n;
  const int64_t ntiles = (n + kRankTile - 1) / kRankTile;
  // the phased chain runs when a table is growing (its index phase then is
  // the step's critical path: C3): full occupancy for the latency-bound
  // insert / admit passes (SKB_ADMIT_WAVES, blocks per SM)
  static const int waves = env_int("SKB_ADMIT_WAVES", 8);
  const unsigned wide = grid_for(n, 256, waves);
  k_fill_scratch<<<wide, 256, 0, x>>>(A.scratch, A.dev);
  SKB_LAUNCH_CHECK();
  k_miss_insert<<<wide, 256, msm, x>>>(A.ids, n, A.mt, A.F, A.namespaced, A.miss, A.scratch, A.dev, A.hslot);
  SKB_LAUNCH_CHECK();
  const unsigned tiles = (unsigned)(ntiles < 4 * sm_count() ? (ntiles > 0 ? ntiles : 1) : 4 * sm_count());
  k_miss_fresh<<<tiles, 256, 0, x>>>(n, A.miss, A.scratch, A.dev, A.hslot, A.fresh, A.tile_cnt);
  SKB_LAUNCH_CHECK();
  k_scan_tiles<<<1, 1024, 0, x>>>(A.tile_cnt, ntiles, A.dev);
  SKB_LAUNCH_CHECK();
  k_rank_fresh<<<tiles, 256, 0, x>>>(n, A.fresh, A.tile_cnt, A.dev, A.rank, A.fpos);
  SKB_LAUNCH_CHECK();
  const int chunks = (A.D + 3) / 4;
  k_fused_admit<<<grid_for(n * chunks, 256, waves), 256, msm, x>>>(
      A.ids, n, A.mt, A.F, A.namespaced, A.fpos, A.hslot, A.scratch, A.dev, A.counters, A.free_list, A.map,
      A.mask, A.cap, A.step, A.D, A.seed_mix, A.scale, A.arena, A.last_step, A.live, A.slot_key, A.ins_seq,
      A.arena_rows);
  SKB_LAUNCH_CHECK();
  k_miss_resolve<<<wide, 256, 0, x>>>(n, A.miss, A.scratch, A.hslot, A.dev, A.slot);
  SKB_LAUNCH_CHECK();
  k_fused_finish<<<1, 1, 0, x>>>(A.counters, A.dev);
  SKB_LAUNCH_CHECK();
}

struct BatchArgs {
  const int64_t* ids;
  int64_t n;
  const int64_t* member_pos;
  const uint64_t* salts;
  int F;
  int namespaced;
  const int64_t* bag_offs;
  int64_t G;
  const int64_t* member_bag;
  const int32_t* strategy;
  int mode;
  int64_t step;
  int64_t tile_k = 0;  // mode 2 (tile combiner): rows kept per bag
  float pad = 0.f;     // mode 2: fill of a bag's rows past its length
};

// Index phase of one batch on the table's index stream: probe, admission,
// bag-of-position, stable sort.  Inputs are ordered after the caller's
// stream `s`; the batch buffer is reused only after its previous backward.
static void fused_prepare(Table* t, const BatchArgs& a, cudaStream_t s) {
  if (a.F < 1) raise(SKB_E_ARG, a.F, "need at least one member");
  if (a.member_pos[0] != 0 || a.member_pos[a.F] != a.n || a.member_bag[0] != 0 || a.member_bag[a.F] != a.G)
    raise(SKB_E_ARG, 0, "member ranges must cover [0, n) positions and [0, G) bags");
  if (a.n >= (1ll << 32) - 1 || a.G >= (1ll << 32) - 1) raise(SKB_E_UNSUPPORTED, a.n, "fused step: > 2^32 positions");
  FusedCtx* c = ctx_get(t);
  if (c->prep_count - c->bwd_count >= 2)
    raise(SKB_E_VALUE, 0, "fused pipeline full: two batches already in flight (run a backward first)");
  cudaStream_t x = c->side;
  BatchCtx& B = c->b[c->prep_count % 2];
  SKB_CUDA(cudaEventRecord(c->ev_in, s));
  SKB_CUDA(cudaStreamWaitEvent(x, c->ev_in, 0));
  if (B.ever_used) SKB_CUDA(cudaStreamWaitEvent(x, B.ev_free, 0));
  if (B.stats_pending) {  // a stats_async copy of this buffer's counters, possibly on another stream
    SKB_CUDA(cudaStreamWaitEvent(x, B.ev_stats, 0));
    B.stats_pending = false;
  }
  // growth moves the arena and side arrays: quiesce both streams before it and
  // finish the copies before any later main-stream kernel (e.g. the pending
  // fold+Adam of the previous step) can touch the new buffers (rare)
  // (VMM tables grow in place: rows never move and the IDMap rehash is
  // stream-ordered on this stream, the only one that reads the IDMap)
  const bool grow = !t->vmm && table_needs_growth(t, a.n);
  if (grow) {
    SKB_CUDA(cudaStreamSynchronize(s));
    SKB_CUDA(cudaStreamSynchronize(x));
  }
  table_reserve(t, a.n, x);
  if (grow) SKB_CUDA(cudaStreamSynchronize(x));
  if (t->arena_rows >= (1ll << 32) - 1) raise(SKB_E_UNSUPPORTED, t->arena_rows, "fused step: > 2^32 rows");
  batch_reserve(B, a.n, a.F, x);
  {  // persistent CUB workspace of the index sort (32 key bits: enough for any arena)
    const size_t need = sort_pairs_u32_bytes(B.cap_n > a.n ? B.cap_n : a.n, 32);
    if (need > B.sort_ws_bytes) {
      uint8_t* w = static_cast<uint8_t*>(B.sort_ws);
      realloc_dev(w, (int64_t)need, x);
      B.sort_ws = w;
      B.sort_ws_bytes = need;
      B.gen++;
    }
  }
  std::vector<MemberDev> mh(a.F + 1);
  bool any_seq = false;
  for (int f = 0; f <= a.F; ++f) {
    mh[f].pos = a.member_pos[f];
    mh[f].bag = a.member_bag[f];
    mh[f].salt = f < a.F ? a.salts[f] : 0;
    mh[f].strategy = f < a.F ? a.strategy[f] : 0;
    if (f < a.F) any_seq |= a.strategy[f] == 0;
  }
  if (B.members_host.size() != mh.size() || memcmp(B.members_host.data(), mh.data(), sizeof(MemberDev) * mh.size())) {
    // stream-ordered upload through pinned staging (no host sync): the side
    // stream already waited for this batch buffer's previous backward
    SKB_CUDA(cudaEventSynchronize(B.members_ev));  // the staging copy of the previous upload has run
    memcpy(B.members_pinned, mh.data(), sizeof(MemberDev) * mh.size());
    SKB_CUDA(cudaMemcpyAsync(B.members, B.members_pinned, sizeof(MemberDev) * mh.size(), cudaMemcpyHostToDevice, x));
    SKB_CUDA(cudaEventRecord(B.members_ev, x));
    B.members_host = mh;
  }
  const MemberDev* mt = B.members;
  const uint64_t mask = (uint64_t)(t->idmap_cap - 1);
  const int D = (int)t->dim;
  const int64_t n = a.n, G = a.G;
  const bool graph = graph_mode(c);
  auto work = [&](cudaStream_t x) {
  SKB_CUDA(cudaMemsetAsync(B.dev, 0, sizeof(int64_t) * 4, x));
  if (n > 0) {
    prof_mark(c, P_PROBE, 0, x);
    k_fused_probe<<<grid_for(n, 256), 256, member_smem(a.F), x>>>(a.ids, n, mt, a.F, a.namespaced, t->idmap, mask,
                                                                  t->idmap_cap, B.slot, B.miss, B.dev);
    SKB_LAUNCH_CHECK();
    prof_mark(c, P_PROBE, 1, x);
    prof_mark(c, P_MISS, 0, x);
    AdmitArgs A{a.ids, n, mt, a.F, a.namespaced, B.miss, B.scratch, B.hslot, B.fresh, B.tile_cnt, B.rank, B.fpos, B.dev,
                t->counters, t->free_list, t->idmap, mask, t->idmap_cap, a.step, D, t->seed_mix, t->init_scale,
                t->arena, t->last_step, t->live, t->slot_key, t->ins_seq, B.slot, t->arena_rows};
    const size_t csm = sizeof(MemberSmem);
    static const int graph_coop = env_int("SKB_GRAPH_COOP", 0);
    if ((!graph || graph_coop) && admit_coop(t)) {
      int cg_blocks = coop_grid(csm);
      if (cg_blocks > sm_count()) cg_blocks = sm_count();  // 1 per SM: co-resides with fold+Adam
      const int64_t want = (n + 255) / 256;
      if (want < cg_blocks) cg_blocks = (int)(want > 0 ? want : 1);
      void* kargs[] = {&A};
      SKB_CUDA(cudaLaunchCooperativeKernel((const void*)k_admission, dim3(cg_blocks), dim3(256), kargs, csm, x));
      SKB_LAUNCH_CHECK();
    } else {
      launch_admission_phased(A, member_smem(a.F), x);
    }
    prof_mark(c, P_MISS, 1, x);
    prof_mark(c, P_SORT, 0, x);
    if (a.mode == 2)  // tile: the gradient row of a position is its tile row (or the zero row past k)
      k_tile_row_of<<<grid_for((G > 0 ? G : 1) * 32, 256), 256, 0, x>>>(a.bag_offs, G, a.tile_k, B.bag);
    else
      k_bag_of<<<grid_for(G > 0 ? G : 1, 256), 256, 0, x>>>(a.bag_offs, G, B.bag);
    SKB_LAUNCH_CHECK();
    const int sbits = bits_for((uint64_t)(t->arena_rows - 1));
    sort_pairs_u32_ws(B.slot, B.skey, B.bag, B.sval, n, sbits, B.sort_ws, B.sort_ws_bytes, x);
    prof_mark(c, P_SORT, 1, x);
  }
  };
  if (graph) {
    GraphKey k;
    int64_t* v = k.v;
    v[0] = t->gen; v[1] = B.gen; v[2] = (int64_t)a.ids; v[3] = n; v[4] = (int64_t)a.bag_offs; v[5] = G;
    v[6] = a.F; v[7] = a.namespaced; v[8] = (int64_t)B.members; v[9] = t->arena_rows; v[10] = t->idmap_cap;
    B.g_prep.run(k, x, c->cap, a.step, nullptr, work);
  } else {
    work(x);
  }
  table_note_inserts(t, n, x);
  SKB_CUDA(cudaEventRecord(B.ev_ready, x));
  SKB_CUDA(cudaEventRecord(c->ev_side_last, x));
  B.ids = a.ids;
  B.bag_offs = a.bag_offs;
  B.n = n;
  B.G = G;
  B.F = a.F;
  B.mode = a.mode;
  B.tile_k = a.tile_k;
  B.pad = a.pad;
  B.step = a.step;
  B.any_seq = any_seq;
  B.last_written = false;
  B.ever_used = true;
  c->prep_count++;
}

// Pool phase on the caller's stream (uses the oldest prepared batch; prepares
// it here when the caller did not prefetch).
static void fused_forward(Table* t, const BatchArgs& a, float* pooled, cudaStream_t s) {
  FusedCtx* c = ctx_get(t);
  if (c->prep_count > c->pool_count) {
    BatchCtx& H = c->b[c->pool_count % 2];
    if (H.ids != a.ids || H.n != a.n || H.G != a.G || H.bag_offs != a.bag_offs || H.step != a.step ||
        H.mode != a.mode || H.tile_k != a.tile_k)
      raise(SKB_E_VALUE, 0, "fused forward does not match the prepared (prefetched) batch");
  } else {
    fused_prepare(t, a, s);
  }
  BatchCtx& B = c->b[c->pool_count % 2];
  SKB_CUDA(cudaStreamWaitEvent(s, B.ev_ready, 0));
  const int D = (int)t->dim;
  const int64_t G = B.G;
  auto work = [&](cudaStream_t s) {
  if (G > 0) {
    prof_mark(c, P_POOL, 0, s);
    const size_t psm = sizeof(PoolSmem);
    const int64_t ntiles = (G + kTileBags - 1) / kTileBags;
    const bool v4 = D % 4 == 0 && (uintptr_t)pooled % 16 == 0;
    if (B.mode == 2) {  // tile combiner: [G, k*D] rows, pad past each bag's length
      // warps per bag tile: enough warps to fill the GPU when bags are few
      const int64_t want = (int64_t)sm_count() * 64;
      const int wpb = (int)std::min<int64_t>(64, std::max<int64_t>(1, (want + G - 1) / G));
      if (v4)
        k_fused_tile<4><<<grid_for(G * wpb * 32, 256), 256, 0, s>>>(t->arena, B.slot, B.bag_offs, G, B.tile_k, D,
                                                                    3 * (int64_t)D, B.pad, pooled, wpb);
      else
        k_fused_tile<1><<<grid_for(G * wpb * 32, 256), 256, 0, s>>>(t->arena, B.slot, B.bag_offs, G, B.tile_k, D,
                                                                    3 * (int64_t)D, B.pad, pooled, wpb);
    } else if (!B.any_seq) {
      const unsigned grid = grid_for(((G + 31) / 32) * 32, 256, 8);
#define SKB_POOL_ARGS t->arena, B.slot, B.bag_offs, G, B.mode, D, 3 * (int64_t)D, pooled
      const int pv = c->pool_var >= 0 ? c->pool_var : pool_variant();
      const int pvar = !v4 ? -1 : (pv == 0 && D <= 128 && B.n == G ? 4 : pv);
      c->last_pool = pvar;
      if (!v4)
        k_fused_pool_scatter<1, 1, 4><<<grid, 256, 0, s>>>(SKB_POOL_ARGS);
      else
        // measured on B200 (C2, D=64): R=2 at 4 blocks/SM 0.162 ms; R=2/1 0.204;
        // R=1/4 0.236; R=4/2 0.235
        // staged one-hot gather only for one-hot batches (n == G): its shared
        // staging halves the resident warps of the general chunks (C5: mixed
        // bag lengths ran 0.75 ms/step slower through it)
        switch (pvar) {
          case 4: {
            const size_t sm = (size_t)8 * 32 * D * sizeof(float);
            static int attr_set = 0;
            if (sm > 48 * 1024 && attr_set < (int)sm) {
              SKB_CUDA(cudaFuncSetAttribute(k_fused_pool_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
              attr_set = (int)sm;
            }
            static const int bps_env = env_int("SKB_POOL_BPS", 0);
            // 128 KB of staging per SM: D=64 -> 2 blocks/SM (measured best on C2 — the
            // rest of the SM stays free for the index stream's overlapping sort)
            const int bps = bps_env > 0 ? bps_env : (int)std::max<size_t>(1, std::min<size_t>(8, (size_t)(128 * 1024) / sm));
            k_fused_pool_staged<<<grid_for(((G + 31) / 32) * 32, 256, bps), 256, sm, s>>>(SKB_POOL_ARGS);
            break;
          }
          case 1: k_fused_pool_scatter<4, 1, 4><<<grid, 256, 0, s>>>(SKB_POOL_ARGS); break;
          case 2: k_fused_pool_scatter<4, 2, 1><<<grid, 256, 0, s>>>(SKB_POOL_ARGS); break;
          case 3: k_fused_pool_scatter<4, 4, 2><<<grid, 256, 0, s>>>(SKB_POOL_ARGS); break;
          case 5: k_fused_pool_scatter<4, 2, 4><<<grid, 256, 0, s>>>(SKB_POOL_ARGS); break;
          default:
            // stream each sub-group's positions (C5: D=128 491 -> 345 us; and for
            // the narrow tables too: D=8/16/32 140/183/244 -> 127/140/177 us,
            // C5 6.20 -> 6.04-6.09 ms same-box)
            static const int stream_min_d = env_int("SKB_POOL_STREAM_MIN_D", 8);
            if (D >= stream_min_d && D <= 128) {
              c->last_pool = 6;
              k_fused_pool_stream<8, 3><<<grid, 256, 0, s>>>(SKB_POOL_ARGS);
            } else
              k_fused_pool_scatter<4, 2, 4><<<grid, 256, 0, s>>>(SKB_POOL_ARGS);
            break;
        }
#undef SKB_POOL_ARGS
    } else if (v4) {
      c->last_pool = 10;  // general (pairwise) pool
      k_fused_pool_general<4><<<grid_for(ntiles * 256, 256, 6), 256, psm, s>>>(t->arena, B.slot, B.bag_offs, G,
                                                                              B.members, B.F, B.mode, D,
                                                                              3 * (int64_t)D, pooled);
    } else {
      k_fused_pool_general<1><<<grid_for(ntiles * 256, 256, 6), 256, psm, s>>>(t->arena, B.slot, B.bag_offs, G,
                                                                              B.members, B.F, B.mode, D,
                                                                              3 * (int64_t)D, pooled);
    }
    SKB_LAUNCH_CHECK();
    prof_mark(c, P_POOL, 1, s);
  }
  };
  if (graph_mode(c) && G > 0) {
    GraphKey k;
    int64_t* v = k.v;
    v[0] = t->gen; v[1] = B.gen; v[2] = (int64_t)pooled; v[3] = B.n; v[4] = (int64_t)B.bag_offs; v[5] = G;
    v[6] = B.mode; v[7] = B.any_seq; v[8] = B.F; v[9] = (int64_t)B.members; v[10] = B.tile_k;
    memcpy(&v[11], &B.pad, sizeof(float));
    B.g_fwd.run(k, s, c->cap, B.step, nullptr, work);
  } else {
    work(s);
  }
  c->pool_count++;
}

// dpooled[g] / float32(len(g)) per bag (len 0 bags untouched: no positions)
__global__ void k_scale_bags(const float* __restrict__ dp, const int64_t* __restrict__ bag_offs, int64_t G, int D,
                             float* __restrict__ out) {
  const int per = D / 4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < G * per; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / per;
    const int c = (int)(t - g * per) * 4;
    const float l = (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g));
    float4 x = ldg4(dp + g * D + c);
    if (l > 0.f) x = make_float4(__fdiv_rn(x.x, l), __fdiv_rn(x.y, l), __fdiv_rn(x.z, l), __fdiv_rn(x.w, l));
    st4(out + g * D + c, x);
  }
}

// packing buffers for the batch's possible mega runs: plain cudaMalloc (grown
// rarely, synchronously) — taking them from the stream-ordered pool that the
// per-step scratch cycles through made step times bimodal (measured on C2)
static void pack_reserve(FusedCtx* c, int64_t rows, int64_t runs, int D, cudaStream_t s) {
  LongFoldPack& P = c->pack;
  const int64_t imgs = long_fold_pack_images(rows, D);
  const bool grow_img = imgs > P.cap_images, grow_runs = runs > P.cap_runs || !P.mcount;
  if (!grow_img && !grow_runs) return;
  SKB_CUDA(cudaStreamSynchronize(s));
  if (grow_img) {
    if (P.images) SKB_CUDA(cudaFree(P.images));
    SKB_CUDA(cudaMalloc(&P.images, sizeof(float) * imgs * long_fold_stage_f(D)));
    P.cap_images = imgs;
    // per (run, stage) pair ready flags (epochs), zero = never written
    if (P.ready) SKB_CUDA(cudaFree(P.ready));
    const int64_t pairs = imgs / long_fold_groups(D) + 1;
    SKB_CUDA(cudaMalloc(&P.ready, sizeof(uint32_t) * pairs));
    SKB_CUDA(cudaMemset(P.ready, 0, sizeof(uint32_t) * pairs));
  }
  if (!P.pstream) {  // the pack's own stream: it runs beside the long fold (eager steps)
    int lo = 0, hi = 0;
    SKB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SKB_CUDA(cudaStreamCreateWithPriority(&P.pstream, cudaStreamNonBlocking, hi));
    SKB_CUDA(cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming));
    SKB_CUDA(cudaEventCreateWithFlags(&P.ev_join, cudaEventDisableTiming));
  }
  if (grow_runs) {
    if (P.mlist) SKB_CUDA(cudaFree(P.mlist));
    if (P.moff) SKB_CUDA(cudaFree(P.moff));
    if (P.morder) SKB_CUDA(cudaFree(P.morder));
    if (!P.mcount) {
      SKB_CUDA(cudaMalloc(&P.mcount, sizeof(int64_t) * 4));
      SKB_CUDA(cudaMemset(P.mcount, 0, sizeof(int64_t) * 4));
      SKB_CUDA(cudaMalloc(&P.wctr, sizeof(unsigned long long)));
    }
    SKB_CUDA(cudaMalloc(&P.mlist, sizeof(uint32_t) * runs));
    SKB_CUDA(cudaMalloc(&P.moff, sizeof(uint32_t) * runs));
    SKB_CUDA(cudaMalloc(&P.morder, sizeof(uint32_t) * runs));
    P.cap_runs = runs;
  }
  c->pack_gen++;
}

static void tree_reserve(FusedCtx* c, int64_t n, int64_t runs_cap, int D, cudaStream_t s) {
  const int64_t need = tree_chunk_cap(n, runs_cap);
  if (need <= c->tw.chunk_cap) return;
  SKB_CUDA(cudaStreamSynchronize(s));
  cudaFree(c->tw.chunk_off);
  cudaFree(c->tw.partial);
  SKB_CUDA(cudaMalloc(&c->tw.chunk_off, sizeof(int64_t) * (runs_cap + 2)));
  SKB_CUDA(cudaMalloc(&c->tw.partial, sizeof(float) * need * D));
  c->tw.chunk_cap = need;
  c->pack_gen++;
}

// the long-run pass of a backward: exact (serial np.add.at chain per column)
// or, in tree mode, the two-level chunked reduction
static void long_pass(FusedCtx* c, BatchCtx& B, const float* dpooled, int D, int mode, const AdamDev& a, Table* t,
                      cudaStream_t st, bool deep, int budget = kLfSmemBudget) {
  if (c->tree)
    launch_long_fold_tree<true>(B.longs, B.dev + 3, B.longs_cap, B.sval, dpooled, D, B.bag_offs, mode, a, t->arena,
                                t->last_step, B.step, st, c->zrow, c->tw);
  else {
    // the pack runs beside the long fold (its own stream; the fold streams
    // the images already packed and gathers the rest) only when a hot chain
    // bounds the step — a recent longest run >= kLfExclusiveRun positions:
    // C4 4.12 -> 3.83 ms; with many short mega runs (C5) the early direct
    // gathers and the pack's high-priority blocks only slow the main fold
    // (6.74 -> 7.34 ms).  Graph capture keeps the pack on the capturing stream.
    LongFoldPack pk = c->pack;
    static const int stream_pack = env_int("SKB_LF_STREAM_PACK", -1);
    const bool hot = c->lf_maxlen >= kLfExclusiveRun;
    if (graph_mode(c) || stream_pack == 0 || (stream_pack < 0 && !hot)) pk.pstream = nullptr;
    launch_long_fold<true>(B.longs, B.dev + 3, B.longs_cap, B.sval, dpooled, D, B.bag_offs, mode, a, t->arena,
                           t->last_step, B.step, st, c->zrow, &pk, deep, budget, RowOut{},
                           c->lf_maxlen >= kLfExclusiveRun);
  }
}

static void fused_backward(Table* t, const float* dpooled, const skb_adam_t& sc, cudaStream_t s,
                           bool prescaled = false) {
  FusedCtx* c = t->fused;
  if (!c || c->bwd_count >= c->pool_count) raise(SKB_E_VALUE, 0, "fused backward without a preceding fused forward");
  BatchCtx& B = c->b[c->bwd_count % 2];
  const int64_t n = B.n;
  const int D = (int)t->dim;
  if (n > 0 && D % 4 == 0) {
    if (c->tree) tree_reserve(c, n, B.longs_cap, D, s);
    else pack_reserve(c, n, B.longs_cap, D, s);
  }
  // long runs seen by a recent backward (no sync: the last completed readback)
  if (cudaEventQuery(c->lf_ev) == cudaSuccess) {
    c->lf_last = c->lf_host[0];
    c->lf_maxlen = c->lf_host[1];
  }
  else cudaGetLastError();
  const bool deep = c->lf_last > 0;  // long runs recently: pack mega runs for TMA streaming
  const AdamDev a = to_dev(sc);
  const float* dpooled_in = dpooled;
  auto work = [&](cudaStream_t s) {
  const float* dpooled = dpooled_in;
  if (n > 0) {
    prof_mark(c, P_ADAM, 0, s);
    const int64_t chunks = (n + 31) / 32;
    const bool v4 = D % 4 == 0 && (uintptr_t)dpooled % 16 == 0;
    // long mean bags: scale each bag's gradient once (the same fp32 division
    // every position of the bag would do) and fold it as a sum
    // tile: per-position tile rows, folded as a sum; prescaled: the caller's
    // rows already are the per-position gradients
    int mode = (B.mode == 2 || prescaled) ? 0 : B.mode;
    Scratch scaled;
    static const int prescale_ratio = env_int("SKB_PRESCALE_RATIO", 8);
    if (mode == 1 && v4 && n >= prescale_ratio * B.G) {
      scaled = Scratch(sizeof(float) * B.G * D, s);
      k_scale_bags<<<grid_for(B.G * (D / 4), 256), 256, 0, s>>>(dpooled, B.bag_offs, B.G, D, scaled.as<float>());
      SKB_LAUNCH_CHECK();
      dpooled = scaled.as<float>();
      mode = 0;
    }
    // non-persistent grid (one chunk per warp): retiring blocks free SM slots
    // for the prefetched index phase of the next step
    static const int persist = env_int("SKB_ADAM_PERSIST", 0);
    const unsigned grid = persist ? grid_for(chunks * 32, 256, 8)
                                                         : (unsigned)((chunks + 7) / 8);
    // hot-id batches (eager mode): list the long runs now and fold them on
    // lf_stream while the main fold kernel handles the rest (it skips the
    // listed runs: longs_cap 0) — the hot chains no longer follow the main
    // fold, they run beside it
    static const int overlap_env = env_int("SKB_LF_OVERLAP", 1);
    const bool overlap = overlap_env && deep && v4 && !graph_mode(c);
    if (overlap) {
      k_list_long_runs<<<grid_for(n, 256), 256, 0, s>>>(B.skey, n, B.longs, B.dev + 3, B.longs_cap);
      SKB_LAUNCH_CHECK();
      SKB_CUDA(cudaEventRecord(c->lf_fork, s));
      SKB_CUDA(cudaStreamWaitEvent(c->lf_stream, c->lf_fork, 0));
      static const int budget_env = env_int("SKB_LF_BUDGET", 0);
      long_pass(c, B, dpooled, D, mode, a, t, c->lf_stream, deep, budget_env > 0 ? budget_env * 1024 : kLfSmemBudget);
      SKB_CUDA(cudaEventRecord(c->lf_join, c->lf_stream));
    }
    const int64_t lcap = overlap ? 0 : B.longs_cap;
#define SKB_ADAM_ARGS n, B.skey, B.sval, B.bag_offs, dpooled, mode, D, a, t->arena, t->last_step, B.step, B.dev + 2, \
                      (v4 ? B.longs : nullptr), B.dev + 3, lcap, (const float*)c->zrow
    if (!v4) {
      c->last_adam = -1;  // generic-D register kernel
      k_fused_adam<1, 1, 4><<<grid, 256, 0, s>>>(SKB_ADAM_ARGS);
    } else {
      // measured on B200 (C2, D=64): R=1 at 4 blocks/SM 0.59 ms; R=2/4 0.60;
      // R=2/3 0.70; R=1/6 (spills) 0.68; R=2/2 0.81 — occupancy beats ILP here
      // default: the TMA ring for singleton-heavy sum batches of wide rows
      // (C2: 0.855 vs 0.904 ms/step), the register kernel otherwise — mean
      // bags (per-position division), narrow rows (per-copy TMA cost) and
      // hot-id batches (extra gradient rows per run): C5's five tables 6.1 ->
      // 3.4 ms, C3 1.13 -> 0.91 ms, C4 7.99 -> 7.76 ms (B200)
      const int forced = c->adam_var >= 0 ? c->adam_var : adam_variant();
      // register kernel <4,1,4> with the 2-row fold batch (same-box A/B:
      // C4 3.07 -> 3.02, C5 6.25 -> 6.21 ms vs <4,1,5>; C1/C3 equal)
      const int var = forced ? forced : (adam_tma_fits(mode, D, c->lf_last) ? 0 : 3);
      c->last_adam = var;
      switch (var) {
        case 1: k_fused_adam<4, 2, 4><<<grid, 256, 0, s>>>(SKB_ADAM_ARGS); break;
        case 2: k_fused_adam<4, 1, 5><<<grid, 256, 0, s>>>(SKB_ADAM_ARGS); break;
        case 3: k_fused_adam<4, 1, 4><<<grid, 256, 0, s>>>(SKB_ADAM_ARGS); break;
        // TMA ring variants (rows per stage, threads, CTAs per SM); measured on
        // B200 C2: <16,192,4> 0.562 ms vs 0.602 for the register kernel
        case 4: launch_adam_tma<8, 128, 8>(n, D, s, SKB_ADAM_ARGS); break;
        case 5: launch_adam_tma<16, 256, 3>(n, D, s, SKB_ADAM_ARGS); break;
        case 6: launch_adam_tma<12, 160, 5>(n, D, s, SKB_ADAM_ARGS); break;
        case 7: launch_adam_tma<16, 192, 3>(n, D, s, SKB_ADAM_ARGS); break;
        case 8: launch_adam_tma<24, 192, 3>(n, D, s, SKB_ADAM_ARGS); break;
        default: launch_adam_tma<16, 192, 4>(n, D, s, SKB_ADAM_ARGS); break;
      }
    }
#undef SKB_ADAM_ARGS
    SKB_LAUNCH_CHECK();
    if (overlap)
      SKB_CUDA(cudaStreamWaitEvent(s, c->lf_join, 0));
    else if (v4)
      long_pass(c, B, dpooled, D, mode, a, t, s, deep);
    prof_mark(c, P_ADAM, 1, s);
  }
  };
  if (graph_mode(c) && n > 0) {
    GraphKey k;
    int64_t* v = k.v;
    v[0] = t->gen; v[1] = B.gen; v[2] = (int64_t)dpooled; v[3] = n; v[4] = (int64_t)B.bag_offs; v[5] = B.G;
    v[6] = B.mode + (prescaled ? 8 : 0); v[7] = B.tile_k; v[8] = c->pack_gen;
    v[9] = deep + (c->tree ? 2 : 0) + (c->lf_maxlen >= kLfExclusiveRun ? 4 : 0);  // deep also picks the fold kernel
    B.g_bwd.run(k, s, c->cap, B.step, &a, work);
  } else {
    work(s);
  }
  // sampled every 4th backward: a heuristic input, and small steps are launch-bound
  if (n > 0 && D % 4 == 0 && (c->bwd_count & 3) == 0 && cudaEventQuery(c->lf_ev) != cudaErrorNotReady) {
    SKB_CUDA(cudaMemcpyAsync(c->lf_host, B.dev + 3, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (c->pack.mcount)
      SKB_CUDA(cudaMemcpyAsync(c->lf_host + 1, c->pack.mcount + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SKB_CUDA(cudaEventRecord(c->lf_ev, s));
  }
  cudaGetLastError();
  B.last_written = true;
  SKB_CUDA(cudaEventRecord(B.ev_free, s));
  c->bwd_count++;
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_fused_prepare(skb_table_t h, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                      const uint64_t* salts_host, int32_t num_members, int32_t namespaced, const int64_t* bag_offs,
                      int64_t num_bags, const int64_t* member_bag_host, const int32_t* strategy_host, int32_t mode,
                      int64_t step, void* stream) {
  SKB_API_BEGIN
  BatchArgs a{ids, n, member_pos_host, salts_host, num_members, namespaced, bag_offs, num_bags, member_bag_host,
              strategy_host, mode, step};
  fused_prepare(table_from(h), a, as_stream(stream));
  SKB_API_END
}

// mode 2 checks shared by the tile entry points
static BatchArgs tile_args(BatchArgs a, int64_t k, float pad) {
  if (k < 0) raise(SKB_E_VALUE, k, "k must be >= 0");
  if (a.G * (k > 0 ? k : 1) >= (int64_t)kZeroRow) raise(SKB_E_UNSUPPORTED, a.G, "fused tile: G * k >= 2^32 - 1");
  a.mode = 2;
  a.tile_k = k;
  a.pad = pad;
  return a;
}

int skb_fused_prepare_tile(skb_table_t h, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                           const uint64_t* salts_host, int32_t num_members, int32_t namespaced,
                           const int64_t* bag_offs, int64_t num_bags, const int64_t* member_bag_host, int64_t k,
                           float pad, int64_t step, void* stream) {
  SKB_API_BEGIN
  std::vector<int32_t> strat(num_members > 0 ? num_members : 1, 1);
  BatchArgs a{ids, n, member_pos_host, salts_host, num_members, namespaced, bag_offs, num_bags, member_bag_host,
              strat.data(), 2, step};
  fused_prepare(table_from(h), tile_args(a, k, pad), as_stream(stream));
  SKB_API_END
}

int skb_fused_forward_tile(skb_table_t h, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                           const uint64_t* salts_host, int32_t num_members, int32_t namespaced,
                           const int64_t* bag_offs, int64_t num_bags, const int64_t* member_bag_host, int64_t k,
                           float pad, int64_t step, float* tiles_out, void* stream) {
  SKB_API_BEGIN
  std::vector<int32_t> strat(num_members > 0 ? num_members : 1, 1);
  BatchArgs a{ids, n, member_pos_host, salts_host, num_members, namespaced, bag_offs, num_bags, member_bag_host,
              strat.data(), 2, step};
  fused_forward(table_from(h), tile_args(a, k, pad), tiles_out, as_stream(stream));
  SKB_API_END
}

int skb_fused_forward(skb_table_t h, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                      const uint64_t* salts_host, int32_t num_members, int32_t namespaced, const int64_t* bag_offs,
                      int64_t num_bags, const int64_t* member_bag_host, const int32_t* strategy_host, int32_t mode,
                      int64_t step, float* pooled_out, void* stream) {
  SKB_API_BEGIN
  BatchArgs a{ids, n, member_pos_host, salts_host, num_members, namespaced, bag_offs, num_bags, member_bag_host,
              strategy_host, mode, step};
  fused_forward(table_from(h), a, pooled_out, as_stream(stream));
  SKB_API_END
}

int skb_fused_backward(skb_table_t h, const float* dpooled, const skb_adam_t* scalars_host, void* stream) {
  SKB_API_BEGIN
  fused_backward(table_from(h), dpooled, *scalars_host, as_stream(stream));
  SKB_API_END
}

int skb_fused_backward_ex(skb_table_t h, const float* dpooled, const skb_adam_t* scalars_host, int32_t flags,
                          void* stream) {
  SKB_API_BEGIN
  fused_backward(table_from(h), dpooled, *scalars_host, as_stream(stream), (flags & SKB_BWD_PRESCALED) != 0);
  SKB_API_END
}

int skb_fused_shard_counts(skb_table_t h, int64_t num_shards, int64_t* counts_out, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  FusedCtx* c = t->fused;
  if (num_shards < 1 || num_shards > 4096) raise(SKB_E_VALUE, num_shards, "num_shards must be in [1, 4096]");
  if (!c || c->prep_count == 0) raise(SKB_E_VALUE, 0, "no fused batch has been prepared on this table");
  cudaStream_t s = as_stream(stream);
  BatchCtx& B = c->b[(c->prep_count - 1) % 2];
  SKB_CUDA(cudaMemsetAsync(counts_out, 0, sizeof(int64_t) * num_shards, s));
  SKB_CUDA(cudaStreamWaitEvent(s, B.ev_ready, 0));
  if (B.n > 0)
    k_head_shard_counts<<<grid_for(B.n, 256), 256, 0, s>>>(B.skey, B.n, t->slot_key, (int)num_shards,
                                                          reinterpret_cast<unsigned long long*>(counts_out));
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_fused_set_fold_mode(skb_table_t h, int32_t mode) {
  SKB_API_BEGIN
  if (mode != 0 && mode != 1) raise(SKB_E_VALUE, mode, "fold mode must be 0 (exact) or 1 (tree)");
  FusedCtx* c = ctx_get(table_from(h));
  if (c->prep_count > c->bwd_count) raise(SKB_E_VALUE, 0, "set_fold_mode while a fused step is in flight");
  c->tree = mode == 1;
  SKB_API_END
}

int skb_fused_set_variants(skb_table_t h, int32_t adam_variant, int32_t pool_variant) {
  SKB_API_BEGIN
  if (adam_variant > 8 || pool_variant > 5) raise(SKB_E_VALUE, 0, "adam variant must be <= 8, pool variant <= 5");
  FusedCtx* c = ctx_get(table_from(h));
  c->adam_var = adam_variant;
  c->pool_var = pool_variant;
  SKB_API_END
}

int skb_fused_last_variants(skb_table_t h, int32_t* adam_host, int32_t* pool_host) {
  SKB_API_BEGIN
  FusedCtx* c = ctx_get(table_from(h));
  *adam_host = c->last_adam;
  *pool_host = c->last_pool;
  SKB_API_END
}

int skb_fused_set_graphs(skb_table_t h, int32_t enable) {
  SKB_API_BEGIN
  FusedCtx* c = ctx_get(table_from(h));
  if (enable) register_param_kernels();
  c->graphs = enable != 0;
  if (!c->graphs)
    for (auto& B : c->b) {
      B.g_prep.reset();
      B.g_fwd.reset();
      B.g_bwd.reset();
      B.g_prep.primed = B.g_fwd.primed = B.g_bwd.primed = false;
    }
  SKB_API_END
}

int skb_fused_profile(skb_table_t h, int64_t max_steps, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  FusedCtx* c = ctx_get(t);
  SKB_CUDA(cudaStreamSynchronize(as_stream(stream)));
  SKB_CUDA(cudaStreamSynchronize(c->side));
  for (auto& v : c->prof_ev) {
    for (auto e : v) cudaEventDestroy(e);
    v.clear();
  }
  for (int p = 0; p < kProf; ++p) {
    c->prof_n[p] = 0;
    c->prof_ev[p].resize(2 * (max_steps > 0 ? max_steps : 0));
    for (auto& e : c->prof_ev[p]) SKB_CUDA(cudaEventCreate(&e));
  }
  c->prof_cap = max_steps > 0 ? max_steps : 0;
  SKB_API_END
}

int skb_fused_profile_read(skb_table_t h, int32_t phase, float* ms_host, int64_t capacity, int64_t* n_host) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  if (phase < 0 || phase >= kProf) raise(SKB_E_ARG, phase, "phase must be in [0, 5)");
  FusedCtx* c = t->fused;
  int64_t n = c ? c->prof_n[phase] : 0;
  if (n > capacity) n = capacity;
  for (int64_t i = 0; i < n; ++i) {
    SKB_CUDA(cudaEventSynchronize(c->prof_ev[phase][2 * i + 1]));
    SKB_CUDA(cudaEventElapsedTime(&ms_host[i], c->prof_ev[phase][2 * i], c->prof_ev[phase][2 * i + 1]));
  }
  *n_host = n;
  SKB_API_END
}

int skb_fused_stats_async(skb_table_t h, int64_t* dst_pinned_host, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  FusedCtx* c = t->fused;
  if (!c || c->bwd_count == 0) raise(SKB_E_VALUE, 0, "no fused step has completed on this table");
  BatchCtx& B = c->b[(c->bwd_count - 1) % 2];
  cudaStream_t s = as_stream(stream);
  SKB_CUDA(cudaStreamWaitEvent(s, B.ev_free, 0));  // after that step's backward, whatever stream this is
  SKB_CUDA(cudaMemcpyAsync(dst_pinned_host, B.dev, sizeof(int64_t) * 4, cudaMemcpyDeviceToHost, s));
  if (!B.ev_stats) SKB_CUDA(cudaEventCreateWithFlags(&B.ev_stats, cudaEventDisableTiming));
  SKB_CUDA(cudaEventRecord(B.ev_stats, s));
  B.stats_pending = true;
  SKB_API_END
}

int skb_fused_last_unique(skb_table_t h, int64_t* n_unique_host, int64_t* n_new_host, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  FusedCtx* c = t->fused;
  if (!c || c->bwd_count == 0) raise(SKB_E_VALUE, 0, "no fused step has completed on this table");
  BatchCtx& B = c->b[(c->bwd_count - 1) % 2];
  int64_t v[4];
  cudaStream_t s = as_stream(stream);
  SKB_CUDA(cudaMemcpyAsync(v, B.dev, sizeof(v), cudaMemcpyDeviceToHost, s));
  SKB_CUDA(cudaStreamSynchronize(s));
  *n_unique_host = v[2];
  *n_new_host = v[1];
  SKB_API_END
}

}  // extern "C"

namespace skb {
// ---------------------------------------------------------------------------
// generic building blocks for the multi-GPU step (dist.cu, distributed.py):
// keys of every member in one launch, pooling from any row source through a
// per-position row index, and the ordered fold of pooled grads per index.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_keys_members(const int64_t* __restrict__ ids, int64_t n,
                                                      const MemberDev* __restrict__ mt, int F,
                                                      int64_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const MemberView mv = stage_members(reinterpret_cast<MemberSmem*>(smem_raw), mt, F);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = key_of(__ldg(ids + i), mv, F, 1, i);
}

void keys_of_members(const int64_t* ids, int64_t n, const MemberDev* mt, int F, int64_t* out, cudaStream_t s) {
  if (n <= 0) return;
  k_keys_members<<<grid_for(n, 256), 256, member_smem(F), s>>>(ids, n, mt, F, out);
  SKB_LAUNCH_CHECK();
}

void bag_of_positions(const int64_t* bag_offs, int64_t G, uint32_t* bag_of, cudaStream_t s) {
  k_bag_of<<<grid_for(G > 0 ? G : 1, 256), 256, 0, s>>>(bag_offs, G, bag_of);
  SKB_LAUNCH_CHECK();
}

void pool_by_index(const float* rows, int64_t stride, const uint32_t* idx, const int64_t* bag_offs, int64_t G,
                   const MemberDev* mt, int F, bool any_sequential, int mode, int D, float* out, cudaStream_t s) {
  if (G <= 0) return;
  const bool v4 = D % 4 == 0 && stride % 4 == 0 && (uintptr_t)out % 16 == 0 && (uintptr_t)rows % 16 == 0;
  if (!any_sequential) {
    const unsigned grid = grid_for(((G + 31) / 32) * 32, 256, 8);
    static const int stream_env = env_int("SKB_POOL_BY_INDEX_STREAM", 1);
    if (v4 && stream_env && D >= 64 && D <= 128)  // wide rows: stream positions (as the fused pool)
      k_fused_pool_stream<8, 3><<<grid, 256, 0, s>>>(rows, idx, bag_offs, G, mode, D, stride, out);
    else if (v4)
      k_fused_pool_scatter<4, 2, 4><<<grid, 256, 0, s>>>(rows, idx, bag_offs, G, mode, D, stride, out);
    else
      k_fused_pool_scatter<1, 1, 4><<<grid, 256, 0, s>>>(rows, idx, bag_offs, G, mode, D, stride, out);
  } else {
    const int64_t ntiles = (G + kTileBags - 1) / kTileBags;
    if (v4)
      k_fused_pool_general<4><<<grid_for(ntiles * 256, 256, 6), 256, sizeof(PoolSmem), s>>>(
          rows, idx, bag_offs, G, mt, F, mode, D, stride, out);
    else
      k_fused_pool_general<1><<<grid_for(ntiles * 256, 256, 6), 256, sizeof(PoolSmem), s>>>(
          rows, idx, bag_offs, G, mt, F, mode, D, stride, out);
  }
  SKB_LAUNCH_CHECK();
}

void fold_sorted(int64_t n, const uint32_t* skey, const uint32_t* sval, const int64_t* bag_offs,
                 const float* dpooled, int mode, int D, float* out, const FoldWork& w, cudaStream_t s,
                 const RowOut& ro) {
  SKB_CUDA(cudaMemsetAsync(w.cnt, 0, sizeof(int64_t) * 2, s));
  if (n <= 0) return;
  const int64_t chunks = (n + 31) / 32;
  AdamDev none{};
  // peer windows (ro) hold D-float rows at 16-byte aligned bases
  const bool v4 = D % 4 == 0 && (uintptr_t)dpooled % 16 == 0 && (uintptr_t)out % 16 == 0;
  if (v4) {
    static const int fold_r = env_int("SKB_FOLD_ONLY_R", 2);  // rows per sub-group in flight (fold-only kernel)
    if (fold_r == 2)
      k_fused_adam<4, 2, 4, false><<<(unsigned)((chunks + 7) / 8), 256, 0, s>>>(
          n, skey, sval, bag_offs, dpooled, mode, D, none, out, nullptr, -1, w.cnt, w.longs, w.cnt + 1, w.lcap,
          nullptr, ro);
    else
    k_fused_adam<4, 1, 4, false><<<(unsigned)((chunks + 7) / 8), 256, 0, s>>>(
        n, skey, sval, bag_offs, dpooled, mode, D, none, out, nullptr, -1, w.cnt, w.longs, w.cnt + 1, w.lcap,
        nullptr, ro);
    SKB_LAUNCH_CHECK();
    launch_long_fold<false>(w.longs, w.cnt + 1, w.lcap, sval, dpooled, D, bag_offs, mode, none, out, nullptr, -1, s,
                            nullptr, w.pack, true, kLfSmemBudget, ro);
  } else {
    k_fused_adam<1, 1, 4, false><<<(unsigned)((chunks + 7) / 8), 256, 0, s>>>(
        n, skey, sval, bag_offs, dpooled, mode, D, none, out, nullptr, -1, w.cnt, nullptr, nullptr, 0, nullptr, ro);
    SKB_LAUNCH_CHECK();
  }
}

// ---------------------------------------------------------------------------
// Owner side of the row-sharded step (distributed.py): the ids
// every rank sent this owner (rank-ordered, each rank's list in its own
// first-occurrence order) go through the fused index phase as a batch of
// one-id bags — probe, admission in global first-occurrence order, sort —
// and the "pool" of that batch is a gather of each position's row stored
// straight into the requesting rank's receive window (NVLink P2P stores).
// The matching backward is skb_fused_backward with the gradient window as
// dpooled: every slot folds its ranks' partial sums in rank order, then
// Adam, on the same TMA / register kernels as the single-GPU step.
// ---------------------------------------------------------------------------
static const int64_t* iota_offsets(FusedCtx* c, int64_t n, cudaStream_t s) {
  if (n + 1 > c->iota_cap) {
    if (c->iota) SKB_CUDA(cudaFreeAsync(c->iota, s));
    const int64_t cap = (n + 1) + (n + 1) / 4;
    SKB_CUDA(cudaMallocAsync(&c->iota, sizeof(int64_t) * cap, s));
    k_iota_offs<<<grid_for(cap, 256), 256, 0, s>>>(c->iota, cap);
    SKB_LAUNCH_CHECK();
    c->iota_cap = cap;
  }
  return c->iota;
}

static void fused_forward_send(Table* t, const int64_t* recv_ids, int64_t n, int64_t step, const int64_t* recv_pre,
                               int S, float* const* peers, const int64_t* dst_base, cudaStream_t s) {
  FusedCtx* c = ctx_get(t);
  if (c->prep_count > c->pool_count) raise(SKB_E_VALUE, 0, "forward_send: a prefetched batch is pending");
  const int64_t* bag_offs = iota_offsets(c, n, s);
  const int64_t mpos[2] = {0, n}, mbag[2] = {0, n};
  const uint64_t salt[1] = {0};
  const int32_t strat[1] = {1};
  BatchArgs a{recv_ids, n, mpos, salt, 1, 0, bag_offs, n, mbag, strat, 0, step};
  fused_prepare(t, a, s);
  BatchCtx& B = c->b[c->pool_count % 2];
  SKB_CUDA(cudaStreamWaitEvent(s, B.ev_ready, 0));
  p2p_send_slot_rows(t->arena, 3 * t->dim, B.slot, n, (int)t->dim, recv_pre, S, peers, dst_base, s);
  c->pool_count++;
}

}  // namespace skb

extern "C" {

int skb_keys_members(const int64_t* ids, int64_t n, const int64_t* members_dev, int32_t num_members, int64_t* out,
                     void* stream) {
  SKB_API_BEGIN
  skb::keys_of_members(ids, n, reinterpret_cast<const skb::MemberDev*>(members_dev), num_members, out,
                       skb::as_stream(stream));
  SKB_API_END
}

int skb_pool_indexed(const float* rows, int64_t row_stride, const uint32_t* idx, const int64_t* bag_offs,
                     int64_t num_bags, const int64_t* members_dev, int32_t num_members, int32_t any_sequential,
                     int32_t mode, int64_t dim, float* out, void* stream) {
  SKB_API_BEGIN
  skb::pool_by_index(rows, row_stride, idx, bag_offs, num_bags, reinterpret_cast<const skb::MemberDev*>(members_dev),
                     num_members, any_sequential != 0, mode, (int)dim, out, skb::as_stream(stream));
  SKB_API_END
}

int skb_fold_bags(const float* dpooled, int64_t dim, const uint32_t* idx, int64_t n, int64_t num_unique,
                  const int64_t* bag_offs, int64_t num_bags, int32_t mode, int64_t max_index, float* out,
                  void* stream) {
  SKB_API_BEGIN
  using namespace skb;
  cudaStream_t s = as_stream(stream);
  const int D = (int)dim;
  if (num_unique > 0) SKB_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * num_unique * D, s));
  if (n <= 0) return SKB_OK;
  Scratch bag(4 * n, s), skey(4 * n, s), sval(4 * n, s), cnt(16, s);
  const int64_t lcap = n / kLongRun + 1;
  Scratch longs(sizeof(LongRun) * lcap, s);
  bag_of_positions(bag_offs, num_bags, bag.as<uint32_t>(), s);
  sort_pairs_u32(idx, skey.as<uint32_t>(), bag.as<uint32_t>(), sval.as<uint32_t>(), n,
                 bits_for((uint64_t)(max_index > 0 ? max_index : 1)), s);
  const int64_t imgs = long_fold_pack_images(n, D);
  Scratch prow(D % 4 == 0 ? sizeof(float) * imgs * long_fold_stage_f(D) : 16, s), pl(sizeof(uint32_t) * lcap, s),
      po(sizeof(uint32_t) * lcap, s), pc(sizeof(int64_t) * 2, s);
  LongFoldPack pk{prow.as<float>(), imgs, pl.as<uint32_t>(), po.as<uint32_t>(), pc.as<int64_t>(), lcap};
  FoldWork w{longs.as<LongRun>(), lcap, cnt.as<int64_t>(), &pk};
  fold_sorted(n, skey.as<uint32_t>(), sval.as<uint32_t>(), bag_offs, dpooled, mode, D, out, w, s);
  SKB_API_END
}

int skb_fused_forward_send(skb_table_t h, const int64_t* recv_ids, int64_t n, int64_t step,
                           const int64_t* recv_prefix, int32_t num_ranks, float* const* peer_windows,
                           const int64_t* dst_base, void* stream) {
  SKB_API_BEGIN
  skb::fused_forward_send(skb::table_from(h), recv_ids, n, step, recv_prefix, num_ranks, peer_windows, dst_base,
                          skb::as_stream(stream));
  SKB_API_END
}

}  // extern "C"
