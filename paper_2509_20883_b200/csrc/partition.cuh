// partition.cuh — dedup / partition / fold building blocks shared across TUs.
#pragma once
#include "common.cuh"

namespace skb {

// First-occurrence dedup of ids[0:n) on a scratch open-addressing table.
struct DedupResult {
  int64_t cap = 0;   // power of two; entry `cap` is the side slot for kEmptyKey
  Scratch table;     // HEntry[cap+1]: {key, first position}
  Scratch hslot;     // int64[n]: table index of each position's key
  Scratch fpos;      // int64[n]: first-occurrence positions, ascending (U valid)
  Scratch d_u;       // int64: U (device)
};
void dedup_first_occurrence(const int64_t* ids, int64_t n, DedupResult& r, cudaStream_t s);
// table + hslot only (no compaction of first occurrences)
void dedup_insert(const int64_t* ids, int64_t n, DedupResult& r, cudaStream_t s);

// true when some id of ids[0:n) occurs twice (synchronizes)
bool has_duplicate(const int64_t* ids, int64_t n, cudaStream_t s);

void unique_partition(const int64_t* ids, int64_t n, int64_t S, int64_t* uniq, int64_t* counts,
                      int64_t* inv_shard, int64_t* inv_pos, cudaStream_t s);

// the split path with a caller-owned persistent workspace (no allocation),
// emitting each position's index into the owner-concatenated unique list
// (gidx) instead of (inv_shard, inv_pos); S <= 256, n < 2^30
size_t unique_partition_ws_bytes(int64_t n, int64_t S);
void unique_partition_ws(const int64_t* ids, int64_t n, int64_t S, int64_t* uniq, int64_t* counts, uint32_t* gidx,
                         void* ws, cudaStream_t s);

void grad_fold(const float* grads, int64_t n, int D, const int64_t* inverse, int64_t U, float* out,
               cudaStream_t s);

}  // namespace skb
