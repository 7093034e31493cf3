// fused.cuh — building blocks of the fused step shared with the multi-GPU
// step (dist.cu): member table layout, bag-of-position, pooling through a
// per-position row index, the ordered per-key fold of pooled gradients.
#pragma once
#include "common.cuh"
#include "longfold.cuh"

namespace skb {

struct MemberDev {
  int64_t pos;   // first position of member f (pos[F] = N)
  int64_t bag;   // first bag of member f (bag[F] = G)
  uint64_t salt;
  int64_t strategy;
};

// namespaced key of every position (sharding.py:170-178), members in smem
void keys_of_members(const int64_t* ids, int64_t n, const MemberDev* mt, int F, int64_t* out, cudaStream_t s);

// bag index of every position from CSR offsets
void bag_of_positions(const int64_t* bag_offs, int64_t G, uint32_t* bag_of, cudaStream_t s);

// pooled[g] = fold over bag g's positions p of rows[idx[p] * stride ..] (sum /
// mean; `sequential` members fold in numpy's pairwise order)
void pool_by_index(const float* rows, int64_t stride, const uint32_t* idx, const int64_t* bag_offs, int64_t G,
                   const MemberDev* mt, int F, bool any_sequential, int mode, int D, float* out, cudaStream_t s);

// Work buffers of the ordered fold (hot keys deferred to the long-run fold).
struct FoldWork {
  LongRun* longs = nullptr;
  int64_t lcap = 0;              // n / kLongRun + 1
  int64_t* cnt = nullptr;        // device [2]: unique keys seen, long runs (zeroed by fold_sorted)
  const LongFoldPack* pack = nullptr;
};

// out[key] = left fold from +0 of dpooled[bag] (/ float32(len) for mean) over
// the (key, bag) pairs sorted stably by key — np.add.at order.  Only keys
// that occur are written.
void fold_sorted(int64_t n, const uint32_t* skey, const uint32_t* sval, const int64_t* bag_offs,
                 const float* dpooled, int mode, int D, float* out, const FoldWork& w, cudaStream_t s,
                 const RowOut& ro = RowOut{});

}  // namespace skb
