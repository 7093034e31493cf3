// dist.cu — requester side of the fused row-sharded multi-GPU step
// (reference sharding.py:222-297, train.py:120-195).
//
// One process per GPU; rank r owns the rows with mix64(key) % S == r.  Per
// logical table and step, this rank as a REQUESTER:
//   prepare   keys of every member (namespaced, sharding.py:170-178) ->
//             first-occurrence dedup + stable owner split (the reference's
//             unique_partition order, sharding.py:74-100) -> per-position
//             index into the owner-concatenated unique list (gidx) ->
//             (gidx, bag) pairs sorted by gidx for the backward fold.  All
//             buffers persistent: no allocation and no host sync per step.
//   send_ids  unique ids of owner j stored straight into owner j's id window
//             at this rank's rank-ordered offset (NVLink P2P stores).
//   pool      pooled[g] from the rows the owners stored into this rank's row
//             window, through gidx (sum / mean, scatter or pairwise order).
//   fold_send per local unique id, the in-order fold of dpooled[bag] (/len)
//             — np.add.at order — stored by the fold kernels themselves
//             straight into its owner's gradient window at this rank's
//             rank-ordered offset (no staging buffer, no copy kernel).
// The owner side is the single-GPU fused step itself (fused.cu
// skb_fused_forward_send / skb_fused_backward).  The only host
// synchronisation of a step is the caller's read of the all-gathered count
// matrix, which sizes every transfer.
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fused.cuh"
#include "p2p.cuh"
#include "partition.cuh"

namespace skb {

struct DistCtx {
  int S = 1, D = 1;
  int device = 0;
  int64_t cap_n = 0;
  int64_t* keys = nullptr;     // [cap_n] namespaced keys
  int64_t* uniq = nullptr;     // [cap_n] unique keys, owner-concatenated
  int64_t* counts = nullptr;   // [S] per-owner unique counts (device)
  uint32_t* gidx = nullptr;    // [cap_n] position -> index into uniq
  uint32_t* bag = nullptr;     // [cap_n] bag of position
  uint32_t* skey = nullptr;    // [cap_n] gidx sorted
  uint32_t* sval = nullptr;    // [cap_n] bags in sorted order
  void* part_ws = nullptr;
  size_t part_ws_bytes = 0;
  void* sort_ws = nullptr;
  size_t sort_ws_bytes = 0;
  LongRun* longs = nullptr;
  int64_t lcap = 0;
  int64_t* cnt = nullptr;      // [2]
  LongFoldPack pack;
  MemberDev* members = nullptr;
  MemberDev* members_pinned = nullptr;
  int64_t members_cap = 0;
  cudaEvent_t members_ev = nullptr;
  std::vector<MemberDev> members_host;
  // the prepared batch
  const int64_t* bag_offs = nullptr;
  int64_t n = 0, G = 0;
  int F = 0;
  bool any_seq = false, prepared = false;
};

static DistCtx* dist_from(skb_dist_t h) {
  if (!h) raise(SKB_E_ARG, 0, "null dist handle");
  return reinterpret_cast<DistCtx*>(h);
}

template <class T>
static void grow_buf(T*& p, int64_t count) {
  if (p) SKB_CUDA(cudaFree(p));
  SKB_CUDA(cudaMalloc(&p, sizeof(T) * (count > 0 ? count : 1)));
}

// persistent buffers for n positions (plain cudaMalloc, grown rarely and
// synchronously: per-step stream-ordered allocations made step times bimodal
// on the single-GPU path)
static void dist_reserve(DistCtx* d, int64_t n, int F, cudaStream_t s) {
  if (n > d->cap_n) {
    SKB_CUDA(cudaStreamSynchronize(s));
    const int64_t cap = n + n / 4;
    grow_buf(d->keys, cap);
    grow_buf(d->uniq, cap);
    grow_buf(d->gidx, cap);
    grow_buf(d->bag, cap);
    grow_buf(d->skey, cap);
    grow_buf(d->sval, cap);
    d->lcap = cap / kLongRun + 1;
    grow_buf(d->longs, d->lcap);
    d->part_ws_bytes = unique_partition_ws_bytes(cap, d->S);
    uint8_t* w = static_cast<uint8_t*>(d->part_ws);
    grow_buf(w, (int64_t)d->part_ws_bytes);
    d->part_ws = w;
    d->sort_ws_bytes = sort_pairs_u32_bytes(cap, 32);
    w = static_cast<uint8_t*>(d->sort_ws);
    grow_buf(w, (int64_t)d->sort_ws_bytes);
    d->sort_ws = w;
    if (d->D % 4 == 0) {
      const int64_t imgs = long_fold_pack_images(cap, d->D);
      grow_buf(d->pack.images, imgs * long_fold_stage_f(d->D));
      d->pack.cap_images = imgs;
      grow_buf(d->pack.mlist, d->lcap);
      grow_buf(d->pack.moff, d->lcap);
      grow_buf(d->pack.morder, d->lcap);
      if (!d->pack.mcount) {
        SKB_CUDA(cudaMalloc(&d->pack.mcount, sizeof(int64_t) * 4));
        SKB_CUDA(cudaMemset(d->pack.mcount, 0, sizeof(int64_t) * 4));
      }
      d->pack.cap_runs = d->lcap;
    }
    d->cap_n = cap;
  }
  if (F + 1 > d->members_cap) {
    if (d->members_ev) SKB_CUDA(cudaEventSynchronize(d->members_ev));
    grow_buf(d->members, F + 1);
    if (d->members_pinned) SKB_CUDA(cudaFreeHost(d->members_pinned));
    SKB_CUDA(cudaMallocHost(&d->members_pinned, sizeof(MemberDev) * (F + 1)));
    if (!d->members_ev) SKB_CUDA(cudaEventCreateWithFlags(&d->members_ev, cudaEventDisableTiming));
    d->members_cap = F + 1;
    d->members_host.clear();
  }
}

static void dist_prepare(DistCtx* d, const int64_t* ids, int64_t n, const int64_t* member_pos,
                         const uint64_t* salts, int F, int namespaced, const int64_t* bag_offs, int64_t G,
                         const int64_t* member_bag, const int32_t* strategy, int64_t* counts_out, cudaStream_t s) {
  if (F < 1) raise(SKB_E_ARG, F, "need at least one member");
  if (member_pos[0] != 0 || member_pos[F] != n || member_bag[0] != 0 || member_bag[F] != G)
    raise(SKB_E_ARG, 0, "member ranges must cover [0, n) positions and [0, G) bags");
  if (n >= (1ll << 30)) raise(SKB_E_UNSUPPORTED, n, "dist step: >= 2^30 positions per rank");
  dist_reserve(d, n, F, s);
  std::vector<MemberDev> mh(F + 1);
  bool any_seq = false;
  for (int f = 0; f <= F; ++f) {
    mh[f].pos = member_pos[f];
    mh[f].bag = member_bag[f];
    mh[f].salt = f < F ? salts[f] : 0;
    mh[f].strategy = f < F ? strategy[f] : 1;
    if (f < F) any_seq |= strategy[f] == 0;
  }
  if (d->members_host.size() != mh.size() ||
      memcmp(d->members_host.data(), mh.data(), sizeof(MemberDev) * mh.size())) {
    SKB_CUDA(cudaEventSynchronize(d->members_ev));  // the staging buffer's previous upload has run
    memcpy(d->members_pinned, mh.data(), sizeof(MemberDev) * mh.size());
    SKB_CUDA(cudaMemcpyAsync(d->members, d->members_pinned, sizeof(MemberDev) * mh.size(), cudaMemcpyHostToDevice, s));
    SKB_CUDA(cudaEventRecord(d->members_ev, s));
    d->members_host = mh;
  }
  const int64_t* keys = ids;
  if (namespaced) {
    keys_of_members(ids, n, d->members, F, d->keys, s);
    keys = d->keys;
  }
  unique_partition_ws(keys, n, d->S, d->uniq, d->counts, d->gidx, d->part_ws, s);
  if (counts_out && counts_out != d->counts)
    SKB_CUDA(cudaMemcpyAsync(counts_out, d->counts, sizeof(int64_t) * d->S, cudaMemcpyDeviceToDevice, s));
  if (n > 0) {
    bag_of_positions(bag_offs, G, d->bag, s);
    sort_pairs_u32_ws(d->gidx, d->skey, d->bag, d->sval, n, bits_for((uint64_t)n), d->sort_ws, d->sort_ws_bytes, s);
  }
  d->bag_offs = bag_offs;
  d->n = n;
  d->G = G;
  d->F = F;
  d->any_seq = any_seq;
  d->prepared = true;
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_dist_create(int64_t dim, int32_t num_ranks, skb_dist_t* out_host) {
  SKB_API_BEGIN
  if (dim < 1) raise(SKB_E_VALUE, dim, "dim must be >= 1");
  if (num_ranks < 1 || num_ranks > 256) raise(SKB_E_VALUE, num_ranks, "num_ranks must be in [1, 256]");
  DistCtx* d = new DistCtx();
  d->S = num_ranks;
  d->D = (int)dim;
  SKB_CUDA(cudaGetDevice(&d->device));
  SKB_CUDA(cudaMalloc(&d->counts, sizeof(int64_t) * num_ranks));
  SKB_CUDA(cudaMalloc(&d->cnt, sizeof(int64_t) * 2));
  *out_host = reinterpret_cast<skb_dist_t>(d);
  SKB_API_END
}

int skb_dist_destroy(skb_dist_t h) {
  SKB_API_BEGIN
  DistCtx* d = dist_from(h);
  SKB_CUDA(cudaDeviceSynchronize());
  for (void* p : {(void*)d->keys, (void*)d->uniq, (void*)d->counts, (void*)d->gidx, (void*)d->bag, (void*)d->skey,
                  (void*)d->sval, d->part_ws, d->sort_ws, (void*)d->longs, (void*)d->cnt,
                  (void*)d->pack.images, (void*)d->pack.mlist, (void*)d->pack.moff, (void*)d->pack.morder,
                  (void*)d->pack.mcount, (void*)d->members})
    if (p) cudaFree(p);
  if (d->members_pinned) cudaFreeHost(d->members_pinned);
  if (d->members_ev) cudaEventDestroy(d->members_ev);
  delete d;
  SKB_API_END
}

int skb_dist_prepare(skb_dist_t h, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                     const uint64_t* salts_host, int32_t num_members, int32_t namespaced, const int64_t* bag_offs,
                     int64_t num_bags, const int64_t* member_bag_host, const int32_t* strategy_host,
                     int64_t* counts_out, void* stream) {
  SKB_API_BEGIN
  dist_prepare(dist_from(h), ids, n, member_pos_host, salts_host, num_members, namespaced, bag_offs, num_bags,
               member_bag_host, strategy_host, counts_out, as_stream(stream));
  SKB_API_END
}

int skb_dist_send_ids(skb_dist_t h, int64_t num_unique, const int64_t* seg_prefix, int64_t* const* peer_windows,
                      const int64_t* dst_base, void* stream) {
  SKB_API_BEGIN
  DistCtx* d = dist_from(h);
  if (!d->prepared) raise(SKB_E_VALUE, 0, "send_ids before prepare");
  if (num_unique < 0 || num_unique > d->n) raise(SKB_E_ARG, num_unique, "num_unique out of range");
  p2p_send_ids(d->uniq, num_unique, seg_prefix, d->S, peer_windows, dst_base, as_stream(stream));
  SKB_API_END
}

int skb_dist_pool(skb_dist_t h, const float* rows, int32_t mode, float* out, void* stream) {
  SKB_API_BEGIN
  DistCtx* d = dist_from(h);
  if (!d->prepared) raise(SKB_E_VALUE, 0, "pool before prepare");
  if (mode != 0 && mode != 1) raise(SKB_E_VALUE, mode, "mode must be sum (0) or mean (1)");
  pool_by_index(rows, d->D, d->gidx, d->bag_offs, d->G, d->members, d->F, d->any_seq, mode, d->D, out,
                as_stream(stream));
  SKB_API_END
}

int skb_dist_fold_send(skb_dist_t h, const float* dpooled, int32_t mode, int64_t num_unique,
                       const int64_t* seg_prefix, float* const* peer_windows, const int64_t* dst_base, void* stream) {
  SKB_API_BEGIN
  DistCtx* d = dist_from(h);
  cudaStream_t s = as_stream(stream);
  if (!d->prepared) raise(SKB_E_VALUE, 0, "fold_send before prepare");
  if (num_unique < 0 || num_unique > d->n) raise(SKB_E_ARG, num_unique, "num_unique out of range");
  FoldWork w{d->longs, d->lcap, d->cnt, d->D % 4 == 0 ? &d->pack : nullptr};
  // each folded row is stored straight into its owner's gradient window
  // (RowOut: segment of the unique index -> peer j, row base[j] + offset)
  fold_sorted(d->n, d->skey, d->sval, d->bag_offs, dpooled, mode, d->D, nullptr, w, s,
              RowOut{seg_prefix, d->S, peer_windows, dst_base});
  d->prepared = false;
  SKB_API_END
}

int skb_dist_buffers(skb_dist_t h, const int64_t** uniq_out, const int64_t** counts_out, const uint32_t** gidx_out) {
  SKB_API_BEGIN
  DistCtx* d = dist_from(h);
  if (uniq_out) *uniq_out = d->uniq;
  if (counts_out) *counts_out = d->counts;
  if (gidx_out) *gidx_out = d->gidx;
  SKB_API_END
}

}  // extern "C"
