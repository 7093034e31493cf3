// fused.cu — the request-merged sparse step for one logical table on one GPU.
//
// Forward (replaces keys_for + unique_partition + lookup_or_insert + gather +
// restore + segment_reduce of train.py:130-176 for S = 1):
//   K1 probe   : per position — namespaced key (sharding.py:178), IDMap probe
//                -> slot (uint32) or miss; misses counted on device.
//   K2..K5 miss: only positions whose key is unknown do work: first-occurrence
//                dedup among misses (atomicMin scratch table sized from the
//                device miss count), exclusive scan -> rank, admission with the
//                reference's slot order, slot broadcast to duplicate misses.
//   K6 pool    : per (bag, 4 columns) — gather arena rows through the slots and
//                fold (scatter / pairwise, bit-exact), mean, write pooled;
//                records bag-of-position and last_step.
// Backward (replaces the per-row grad expansion train.py:181-186 +
// all_to_all_grad_update sharding.py:257-297):
//   K7 stable radix sort of (slot, bag) by slot, K8 run heads,
//   K9 fold + Adam: per (unique row, 4 columns) fold dpooled[bag] (/len) in
//                position order from +0 — the np.add.at order — then AdamW on
//                the AoS [w|m|v] row, one read + one write of 12*D bytes.
#include <cstring>
#include <vector>

#include "common.cuh"
#include "pool.cuh"
#include "table.cuh"

namespace skb {

struct MemberDev {
  int64_t pos;   // first position of member f (pos[F] = N)
  int64_t bag;   // first bag of member f (bag[F] = G)
  uint64_t salt;
  int64_t strategy;
};

struct FusedCtx {
  int64_t cap_n = 0;         // capacity in positions
  uint32_t* slot = nullptr;  // [N] slot of position
  uint32_t* bag = nullptr;   // [N] bag of position
  uint32_t* skey = nullptr;  // [N] sorted slots
  uint32_t* sval = nullptr;  // [N] bags in sorted order
  uint32_t* heads = nullptr; // [N] run heads
  uint8_t* miss = nullptr;   // [N]
  uint8_t* fresh = nullptr;  // [N] first occurrence of an unknown key
  int64_t* rank = nullptr;   // [N]
  int32_t* hslot = nullptr;  // [N] scratch-table index of a miss
  HEntry* scratch = nullptr; // [2*cap_n pow2 + 1]
  int64_t scratch_cap = 0;
  int64_t* dev = nullptr;    // [0] misses M, [1] new K, [2] unique U
  MemberDev* members = nullptr;
  int64_t members_cap = 0;
  std::vector<MemberDev> members_host;
  // last forward
  int64_t n = 0, G = 0, F = 0;
  int mode = 0;
  const int64_t* bag_offs = nullptr;
  bool have_fwd = false;
};

void fused_ctx_destroy(FusedCtx* c) {
  if (!c) return;
  cudaFree(c->slot);
  cudaFree(c->bag);
  cudaFree(c->skey);
  cudaFree(c->sval);
  cudaFree(c->heads);
  cudaFree(c->miss);
  cudaFree(c->fresh);
  cudaFree(c->rank);
  cudaFree(c->hslot);
  cudaFree(c->scratch);
  cudaFree(c->dev);
  cudaFree(c->members);
  delete c;
}

template <class T>
static void realloc_dev(T*& p, int64_t count, cudaStream_t s) {
  if (p) SKB_CUDA(cudaFreeAsync(p, s));
  SKB_CUDA(cudaMallocAsync(&p, sizeof(T) * (count > 0 ? count : 1), s));
}

static FusedCtx* ctx_for(Table* t, int64_t n, int64_t F, cudaStream_t s) {
  if (!t->fused) {
    t->fused = new FusedCtx();
    SKB_CUDA(cudaMalloc(&t->fused->dev, sizeof(int64_t) * 4));
  }
  FusedCtx* c = t->fused;
  if (n > c->cap_n) {
    int64_t cap = n + n / 4;
    realloc_dev(c->slot, cap, s);
    realloc_dev(c->bag, cap, s);
    realloc_dev(c->skey, cap, s);
    realloc_dev(c->sval, cap, s);
    realloc_dev(c->heads, cap, s);
    realloc_dev(c->miss, cap, s);
    realloc_dev(c->fresh, cap, s);
    realloc_dev(c->rank, cap, s);
    realloc_dev(c->hslot, cap, s);
    c->scratch_cap = next_pow2(2 * cap > 64 ? 2 * cap : 64);
    realloc_dev(c->scratch, c->scratch_cap + 1, s);
    c->cap_n = cap;
  }
  if (F + 1 > c->members_cap) {
    realloc_dev(c->members, F + 1, s);
    c->members_cap = F + 1;
    c->members_host.clear();
  }
  return c;
}

__device__ __forceinline__ int64_t member_of_pos(const MemberDev* __restrict__ mt, int64_t F, int64_t i) {
  int64_t lo = 0, hi = F;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (mt[mid].pos <= i) lo = mid; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t member_of_bag(const MemberDev* __restrict__ mt, int64_t F, int64_t g) {
  int64_t lo = 0, hi = F;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (mt[mid].bag <= g) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ long long key_at(const int64_t* __restrict__ ids, const MemberDev* __restrict__ mt,
                                            int64_t F, int namespaced, int64_t i) {
  long long id = ids[i];
  if (!namespaced) return id;
  return (long long)mix64((uint64_t)id ^ mt[member_of_pos(mt, F, i)].salt);
}

// K1
__global__ void k_fused_probe(const int64_t* __restrict__ ids, int64_t n, const MemberDev* __restrict__ mt,
                              int64_t F, int namespaced, const HEntry* __restrict__ map, uint64_t mask, int64_t cap,
                              uint32_t* __restrict__ slot, uint8_t* __restrict__ miss, int64_t* dev) {
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    long long s = idmap_find(map, mask, cap, key_at(ids, mt, F, namespaced, i));
    slot[i] = s < 0 ? 0xFFFFFFFFu : (uint32_t)s;
    miss[i] = s < 0;
    local += s < 0;
  }
  // warp-aggregated miss count
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffff, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(reinterpret_cast<unsigned long long*>(&dev[0]), (unsigned long long)local);
}

__device__ __forceinline__ int64_t scratch_cap_for(int64_t M) { return next_pow2(2 * M > 64 ? 2 * M : 64); }

__global__ void k_fill_scratch(HEntry* t, const int64_t* dev) {
  const int64_t cap = scratch_cap_for(dev[0]);
  if (dev[0] == 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cap; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<longlong2*>(t)[i] = make_longlong2(kEmptyKey, 0x7FFFFFFFFFFFFFFFll);
}

// K2: first-occurrence dedup among unknown keys
__global__ void k_miss_insert(const int64_t* __restrict__ ids, int64_t n, const MemberDev* __restrict__ mt, int64_t F,
                              int namespaced, const uint8_t* __restrict__ miss, HEntry* t, const int64_t* dev,
                              int32_t* __restrict__ hslot) {
  if (dev[0] == 0) return;
  const int64_t cap = scratch_cap_for(dev[0]);
  const uint64_t mask = (uint64_t)(cap - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!miss[i]) continue;
    long long key = key_at(ids, mt, F, namespaced, i);
    int64_t h;
    if (key == kEmptyKey) {
      h = cap;
    } else {
      h = (int64_t)(bucket_hash((uint64_t)key) & mask);
      while (true) {
        long long k = *reinterpret_cast<volatile long long*>(&t[h].key);
        if (k == key) break;
        if (k == kEmptyKey) {
          long long prev = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&t[h].key),
                                                (unsigned long long)kEmptyKey, (unsigned long long)key);
          if (prev == kEmptyKey || prev == key) break;
        }
        h = (int64_t)(((uint64_t)h + 1) & mask);
      }
    }
    if (*reinterpret_cast<volatile long long*>(&t[h].val) > i) atomicMin(&t[h].val, (long long)i);
    hslot[i] = (int32_t)h;
  }
}

// K3
__global__ void k_miss_fresh(int64_t n, const uint8_t* __restrict__ miss, const HEntry* t, const int64_t* dev,
                             const int32_t* __restrict__ hslot, uint8_t* __restrict__ fresh) {
  const bool any = dev[0] != 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    fresh[i] = any && miss[i] && t[hslot[i]].val == i;
}

// K4: admission of the k-th fresh key (input order) — same slot rule as
// lookup_or_insert; the slot is published in the scratch entry for K5.
__global__ void k_fused_admit(const int64_t* __restrict__ ids, int64_t n, const MemberDev* __restrict__ mt, int64_t F,
                              int namespaced, const uint8_t* __restrict__ fresh, const int64_t* __restrict__ rank,
                              const int32_t* __restrict__ hslot, HEntry* scratch, const int64_t* dev,
                              const int64_t* __restrict__ counters, const int64_t* __restrict__ free_list,
                              HEntry* map, uint64_t mask, int64_t cap, int64_t step, int D, uint64_t seed_mix,
                              double scale, float* __restrict__ arena, int64_t* __restrict__ last_step,
                              uint8_t* __restrict__ live, int64_t* __restrict__ slot_key,
                              int64_t* __restrict__ ins_seq) {
  if (dev[0] == 0) return;
  const int chunks = (D + 3) / 4;
  const int64_t total = n * chunks;
  const int64_t A = counters[C_ALLOC], Fr = counters[C_FREE], seq = counters[C_SEQ];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / chunks;
    if (!fresh[i]) continue;
    int ch = (int)(t - i * chunks);
    int64_t k = rank[i];
    int64_t slot = assign_slot(k, Fr, A, free_list);
    long long key = key_at(ids, mt, F, namespaced, i);
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
    for (int c = ch * 4; c < ch * 4 + 4 && c < D; ++c) {
      row[c] = init_value(base, c, scale);
      row[D + c] = 0.f;
      row[2 * D + c] = 0.f;
    }
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
  int64_t K = dev[1], F = counters[C_FREE];
  int64_t take = K < F ? K : F;
  counters[C_FREE] = F - take;
  counters[C_ALLOC] += K - take;
  counters[C_ROWS] += K;
  counters[C_SEQ] += K;
}

// arena rows through the position->slot map
struct ArenaSrc {
  const float* arena;
  const uint32_t* slot;
  int D;
  int c;
  template <int VEC> __device__ __forceinline__ typename VecT<VEC>::T load(int64_t p) const {
    return vload<VEC>(arena + (int64_t)slot[p] * (3 * D) + c);
  }
};

// K6
template <int VEC>
__global__ void __launch_bounds__(256) k_fused_pool(const float* __restrict__ arena, const uint32_t* __restrict__ slot,
                                                    const int64_t* __restrict__ bag_offs, int64_t G,
                                                    const MemberDev* __restrict__ mt, int64_t F, int mode, int D,
                                                    int64_t step, float* __restrict__ out, uint32_t* __restrict__ bag_of,
                                                    int64_t* __restrict__ last_step) {
  const int per_row = D / VEC;
  const int64_t total = G * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t g = t / per_row;
    int cc = (int)(t - g * per_row);
    int c = cc * VEC;
    int64_t b = bag_offs[g], e = bag_offs[g + 1];
    const int64_t f = F == 1 ? 0 : member_of_bag(mt, F, g);
    const int strat = (int)mt[f].strategy;
    ArenaSrc src{arena, slot, D, c};
    typename VecT<VEC>::T acc =
        strat == 0 ? pool_sequential<VEC>(src, b, reduceat_end(b, e, g == mt[f + 1].bag - 1, mt[f + 1].pos))
                   : pool_scatter<VEC>(src, b, e);
    if (mode == 1 && e > b) acc = vdiv<VEC>(acc, (float)(e - b));
    vstore<VEC>(out + g * D + c, acc);
    // bookkeeping spread over the row's lanes
    for (int64_t p = b + cc; p < e; p += per_row) {
      bag_of[p] = (uint32_t)g;
      last_step[slot[p]] = step;
    }
  }
}

// K9: ordered grad fold + Adam/AdamW per unique row
template <int VEC>
__global__ void __launch_bounds__(256) k_fused_adam(const uint32_t* __restrict__ heads, const int64_t* __restrict__ dev,
                                                    int64_t n, const uint32_t* __restrict__ skey,
                                                    const uint32_t* __restrict__ sval,
                                                    const int64_t* __restrict__ bag_offs,
                                                    const float* __restrict__ dpooled, int mode, int D, AdamDev a,
                                                    float* __restrict__ arena) {
  using T = typename VecT<VEC>::T;
  const int per_row = D / VEC;
  const int64_t U = dev[2];
  const int64_t total = U * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = t / per_row;
    int c = (int)(t - u * per_row) * VEC;
    int64_t b = heads[u];
    int64_t e = u + 1 < U ? (int64_t)heads[u + 1] : n;
    T acc = vfill<VEC>(0.f);
    for (int64_t j = b; j < e; ++j) {
      uint32_t g = sval[j];
      T x = vload<VEC>(dpooled + (int64_t)g * D + c);
      if (mode == 1) x = vdiv<VEC>(x, (float)(bag_offs[g + 1] - bag_offs[g]));
      acc = vadd<VEC>(acc, x);
    }
    float* row = arena + (int64_t)skey[b] * (3 * D);
    if constexpr (VEC == 4) {
      float4 p = *reinterpret_cast<float4*>(row + c), m = *reinterpret_cast<float4*>(row + D + c),
             v = *reinterpret_cast<float4*>(row + 2 * D + c);
      adam1(p.x, m.x, v.x, acc.x, a);
      adam1(p.y, m.y, v.y, acc.y, a);
      adam1(p.z, m.z, v.z, acc.z, a);
      adam1(p.w, m.w, v.w, acc.w, a);
      st4(row + c, p);
      st4(row + D + c, m);
      st4(row + 2 * D + c, v);
    } else {
      float p = row[c], m = row[D + c], v = row[2 * D + c];
      adam1(p, m, v, acc, a);
      row[c] = p;
      row[D + c] = m;
      row[2 * D + c] = v;
    }
  }
}

__global__ void k_copy_count(const int64_t* src, int64_t* dst) { *dst = *src; }

static void fused_forward(Table* t, const int64_t* ids, int64_t n, const int64_t* member_pos, const uint64_t* salts,
                          int F, int namespaced, const int64_t* bag_offs, int64_t G, const int64_t* member_bag,
                          const int32_t* strategy, int mode, int64_t step, float* pooled, cudaStream_t s) {
  if (F < 1) raise(SKB_E_ARG, F, "need at least one member");
  if (member_pos[0] != 0 || member_pos[F] != n || member_bag[0] != 0 || member_bag[F] != G)
    raise(SKB_E_ARG, 0, "member ranges must cover [0, n) positions and [0, G) bags");
  if (n >= (1ll << 32) - 1 || G >= (1ll << 32) - 1) raise(SKB_E_UNSUPPORTED, n, "fused step: > 2^32 positions");
  table_reserve(t, n, s);
  if (t->arena_rows >= (1ll << 32) - 1) raise(SKB_E_UNSUPPORTED, t->arena_rows, "fused step: > 2^32 rows");
  FusedCtx* c = ctx_for(t, n, F, s);
  // member table (re-uploaded only when it changes)
  std::vector<MemberDev> mh(F + 1);
  for (int f = 0; f <= F; ++f) {
    mh[f].pos = member_pos[f];
    mh[f].bag = member_bag[f];
    mh[f].salt = f < F ? salts[f] : 0;
    mh[f].strategy = f < F ? strategy[f] : 0;
  }
  if (c->members_host.size() != mh.size() || memcmp(c->members_host.data(), mh.data(), sizeof(MemberDev) * mh.size())) {
    SKB_CUDA(cudaMemcpyAsync(c->members, mh.data(), sizeof(MemberDev) * mh.size(), cudaMemcpyHostToDevice, s));
    SKB_CUDA(cudaStreamSynchronize(s));  // pageable source; rare (layout change)
    c->members_host = mh;
  }
  const MemberDev* mt = c->members;
  const uint64_t mask = (uint64_t)(t->idmap_cap - 1);
  const int D = (int)t->dim;
  SKB_CUDA(cudaMemsetAsync(c->dev, 0, sizeof(int64_t) * 4, s));
  if (n > 0) {
    k_fused_probe<<<grid_for(n, 256), 256, 0, s>>>(ids, n, mt, F, namespaced, t->idmap, mask, t->idmap_cap, c->slot,
                                                  c->miss, c->dev);
    SKB_LAUNCH_CHECK();
    // miss path: a handful of launches that exit at once when every key is known
    k_fill_scratch<<<grid_for(c->scratch_cap + 1, 256), 256, 0, s>>>(c->scratch, c->dev);
    SKB_LAUNCH_CHECK();
    k_miss_insert<<<grid_for(n, 256), 256, 0, s>>>(ids, n, mt, F, namespaced, c->miss, c->scratch, c->dev, c->hslot);
    SKB_LAUNCH_CHECK();
    k_miss_fresh<<<grid_for(n, 256), 256, 0, s>>>(n, c->miss, c->scratch, c->dev, c->hslot, c->fresh);
    SKB_LAUNCH_CHECK();
    scan_exclusive_u8_to_i64(c->fresh, c->rank, n, c->dev + 1, s);  // rank of fresh keys, K -> dev[1]
    const int chunks = (D + 3) / 4;
    k_fused_admit<<<grid_for(n * chunks, 256), 256, 0, s>>>(
        ids, n, mt, F, namespaced, c->fresh, c->rank, c->hslot, c->scratch, c->dev, t->counters, t->free_list,
        t->idmap, mask, t->idmap_cap, step, D, t->seed_mix, t->init_scale, t->arena, t->last_step, t->live,
        t->slot_key, t->ins_seq);
    SKB_LAUNCH_CHECK();
    k_miss_resolve<<<grid_for(n, 256), 256, 0, s>>>(n, c->miss, c->scratch, c->hslot, c->dev, c->slot);
    SKB_LAUNCH_CHECK();
    k_fused_finish<<<1, 1, 0, s>>>(t->counters, c->dev);
    SKB_LAUNCH_CHECK();
  }
  if (G > 0) {
    bool v4 = D % 4 == 0 && (uintptr_t)pooled % 16 == 0;
    if (v4)
      k_fused_pool<4><<<grid_for(G * (D / 4), 256), 256, 0, s>>>(t->arena, c->slot, bag_offs, G, mt, F, mode, D, step,
                                                                pooled, c->bag, t->last_step);
    else
      k_fused_pool<1><<<grid_for(G * D, 256), 256, 0, s>>>(t->arena, c->slot, bag_offs, G, mt, F, mode, D, step,
                                                          pooled, c->bag, t->last_step);
    SKB_LAUNCH_CHECK();
  }
  table_note_inserts(t, n, s);
  c->n = n;
  c->G = G;
  c->F = F;
  c->mode = mode;
  c->bag_offs = bag_offs;
  c->have_fwd = true;
}

static void fused_backward(Table* t, const float* dpooled, const skb_adam_t& sc, cudaStream_t s) {
  FusedCtx* c = t->fused;
  if (!c || !c->have_fwd) raise(SKB_E_VALUE, 0, "fused backward without a preceding fused forward");
  const int64_t n = c->n;
  const int D = (int)t->dim;
  if (n > 0) {
    sort_pairs_u32(c->slot, c->skey, c->bag, c->sval, n, bits_for((uint64_t)(t->arena_rows - 1)), s);
    select_run_heads_u32(c->skey, n, c->heads, c->dev + 2, s);
    AdamDev a = to_dev(sc);
    bool v4 = D % 4 == 0 && (uintptr_t)dpooled % 16 == 0;
    if (v4)
      k_fused_adam<4><<<grid_for(n * (D / 4), 256), 256, 0, s>>>(c->heads, c->dev, n, c->skey, c->sval, c->bag_offs,
                                                                dpooled, c->mode, D, a, t->arena);
    else
      k_fused_adam<1><<<grid_for(n * D, 256), 256, 0, s>>>(c->heads, c->dev, n, c->skey, c->sval, c->bag_offs, dpooled,
                                                          c->mode, D, a, t->arena);
    SKB_LAUNCH_CHECK();
  }
  c->have_fwd = false;
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_fused_forward(skb_table_t h, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                      const uint64_t* salts_host, int32_t num_members, int32_t namespaced, const int64_t* bag_offs,
                      int64_t num_bags, const int64_t* member_bag_host, const int32_t* strategy_host, int32_t mode,
                      int64_t step, float* pooled_out, void* stream) {
  SKB_API_BEGIN
  fused_forward(table_from(h), ids, n, member_pos_host, salts_host, num_members, namespaced, bag_offs, num_bags,
                member_bag_host, strategy_host, mode, step, pooled_out, as_stream(stream));
  SKB_API_END
}

int skb_fused_backward(skb_table_t h, const float* dpooled, const skb_adam_t* scalars_host, void* stream) {
  SKB_API_BEGIN
  fused_backward(table_from(h), dpooled, *scalars_host, as_stream(stream));
  SKB_API_END
}

int skb_fused_last_unique(skb_table_t h, int64_t* n_unique_host, int64_t* n_new_host, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  if (!t->fused) raise(SKB_E_VALUE, 0, "no fused step has run on this table");
  int64_t v[4];
  cudaStream_t s = as_stream(stream);
  SKB_CUDA(cudaMemcpyAsync(v, t->fused->dev, sizeof(v), cudaMemcpyDeviceToHost, s));
  SKB_CUDA(cudaStreamSynchronize(s));
  *n_unique_host = v[2];
  *n_new_host = v[1];
  SKB_API_END
}

}  // extern "C"
