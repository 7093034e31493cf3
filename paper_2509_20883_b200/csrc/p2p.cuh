// p2p.cuh — peer-memory stores of the row-sharded exchange (p2p.cu).
#pragma once
#include "common.cuh"

namespace skb {

// Row q of a received list (rank-ordered segments pre[j]..pre[j+1]) is the
// arena row of slot[q] (row stride `stride` floats, D columns); it is stored
// at peers[j] + (base[j] + q - pre[j]) * D — the requester's receive window.
void p2p_send_slot_rows(const float* arena, int64_t stride, const uint32_t* slot, int64_t nq, int D,
                        const int64_t* pre, int S, float* const* peers, const int64_t* base, cudaStream_t s);

// Rows [0, n) of a local [n, D] matrix split into segments pre[j]..pre[j+1],
// segment j stored at peers[j] + (base[j] + q - pre[j]) * D.
void p2p_send_segments(const float* rows, int64_t n, int D, const int64_t* pre, int S, float* const* peers,
                       const int64_t* base, cudaStream_t s);

// The same for int64 elements (id lists): one element per row.
void p2p_send_ids(const int64_t* ids, int64_t n, const int64_t* pre, int S, int64_t* const* peers,
                  const int64_t* base, cudaStream_t s);

}  // namespace skb
