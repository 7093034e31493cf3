// partition.cuh — dedup / partition / fold building blocks shared across TUs.
#pragma once
#include "common.cuh"

namespace skb {

// 128-bit CAS on a whole {key, first position} entry (sm_90+ atom.cas.b128)
__device__ __forceinline__ void cas_entry(HEntry* p, long long ck, long long cv, long long nk, long long nv,
                                          long long& ok, long long& ov) {
  asm volatile("{\n\t.reg .b128 c, n, o;\n\t"
               "mov.b128 c, {%2, %3};\n\t"
               "mov.b128 n, {%4, %5};\n\t"
               "atom.global.cas.b128 o, [%6], c, n;\n\t"
               "mov.b128 {%0, %1}, o;\n\t}"
               : "=l"(ok), "=l"(ov)
               : "l"(ck), "l"(cv), "l"(nk), "l"(nv), "l"(p)
               : "memory");
}

// insert-or-lower: the bucket ends as {key, min position}.  The bucket is
// read first (L2, no atomic): a bucket already holding the key at an earlier
// position needs no atomic at all — hot keys (zipf) would otherwise serialise
// every occurrence on one address — and a foreign key moves on to the next
// bucket (keys are never removed).  Otherwise one 128-bit CAS claims an empty
// bucket or lowers a later position; a failed CAS re-examines the bucket
// with the value it returned.
__device__ __forceinline__ uint64_t insert_or_lower(HEntry* t, uint64_t slot, uint64_t mask, long long key,
                                                    long long i) {
  constexpr long long kMaxPos = 0x7FFFFFFFFFFFFFFFll;
  longlong2 e = __ldcg(reinterpret_cast<const longlong2*>(&t[slot]));
  while (true) {
    if (e.x == key) {
      if (e.y <= i) return slot;
    } else if (e.x != kEmptyKey) {
      slot = (slot + 1) & mask;
      e = __ldcg(reinterpret_cast<const longlong2*>(&t[slot]));
      continue;
    } else {
      e.y = kMaxPos;  // an empty bucket always holds {EMPTY, max}
    }
    long long ok, ov;
    cas_entry(&t[slot], e.x, e.y, key, i, ok, ov);
    if (ok == e.x && ov == e.y) return slot;
    e = make_longlong2(ok, ov);
  }
}


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
