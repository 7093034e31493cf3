// table.cuh — the GPU dynamic embedding table (EmbeddingTable embedding.py:151-308).
//
// HBM layout (one table):
//   idmap     HEntry[idmap_cap + 1]   open addressing, linear probing, load <= 0.5;
//                                     {int64 key, int64 slot}; entry idmap_cap is
//                                     the side slot for key == INT64_MIN (EMPTY).
//   arena     float32[arena_rows][3*D]  AoS row = [w | m | v]: Adam reads and
//                                     writes one contiguous 12*D-byte span; gather
//                                     reads the leading 4*D bytes.
//   last_step int64[arena_rows]        BlockStore last-touched step
//   live      uint8[arena_rows]        EmbeddingTable._live
//   slot_key  int64[arena_rows]        reverse map slot -> id (export / evict)
//   ins_seq   int64[arena_rows]        dict insertion sequence of the live entry
//                                     (evict appends stale slots in this order)
//   free_list int64[arena_rows]        LIFO free list (top = free_list[F-1])
//   counters  int64[4]                 {allocated, free_count, num_rows, seq}
// Slot numbers are exactly the reference's offsets.
#pragma once
#include <thread>

#include "common.cuh"
#include "vmm.cuh"

namespace skb {

enum { C_ALLOC = 0, C_FREE = 1, C_ROWS = 2, C_SEQ = 3, C_N = 4 };

// evict_threshold=None (eviction disabled); any other value, negative ones
// included, evicts with the reference's `step - last_step > threshold`
constexpr int64_t kNoEvict = (int64_t)0x8000000000000000ull;  // INT64_MIN

struct FusedCtx;  // fused.cu

struct Table {
  int64_t dim = 0, seed = 0, block_size = 0, evict_threshold = kNoEvict;
  int64_t gen = 0;  // bumped whenever a device array is reallocated (captured graphs bake pointers)
  int device = 0;
  double init_scale = 0.0;  // 1 / sqrt(dim), host double (embedding.py:34)
  uint64_t seed_mix = 0;    // mix64(u64(seed))

  float* arena = nullptr;
  int64_t arena_rows = 0;
  int64_t* last_step = nullptr;
  uint8_t* live = nullptr;
  int64_t* slot_key = nullptr;
  int64_t* ins_seq = nullptr;
  int64_t* free_list = nullptr;
  // copy-free growth: the six per-row arrays above live in reserved virtual
  // address ranges and grow by mapping more memory (vmm.cuh); rows never move
  bool vmm = false;
  int64_t rows_hint = 0;  // capacity_hint: VA reserved for this many rows up front
  VmmArray va[6];         // arena, last_step, live, slot_key, ins_seq, free_list
  std::thread va_prep;    // maps the next growth chunk of every array ahead of need

  HEntry* idmap = nullptr;
  int64_t idmap_cap = 0;

  int64_t* counters = nullptr;  // device int64[C_N]
  int64_t ensured_slots = 0;    // BlockStore.ensure_capacity high-water mark (host)

  // host-side upper bounds on device counters (async snapshot + pending adds)
  int64_t* snap_host = nullptr;  // pinned int64[C_N]
  cudaEvent_t snap_ev = nullptr;
  bool snap_pending = false;
  int64_t known[C_N] = {0, 0, 0, 0};
  int64_t pending_adds = 0;      // row admissions enqueued but not covered by `known`
  int64_t adds_after_snap = 0;   // ... of which enqueued after the in-flight snapshot
  int64_t recent_growth = 0;     // rows admitted between the last two harvested snapshots

  FusedCtx* fused = nullptr;

  // checked ops: persistent error flags (device, ~0 = clear; re-armed only
  // after an error), their pinned readback, and a zeroed slot bitmap for
  // scatter_update's distinctness test (cleared again by the op that set it)
  unsigned long long* dflags = nullptr;  // [4]
  int64_t* hflags = nullptr;             // pinned [4]
  uint32_t* bitmap = nullptr;
  int64_t bitmap_words = 0;

  int64_t row_stride() const { return 3 * dim; }
};

Table* table_from(skb_table_t h);

// Ensure room for n more insertions (arena + idmap), growing stream-ordered.
void table_reserve(Table* t, int64_t n, cudaStream_t s);
// Whether table_reserve(n) might have to grow (host bound check, no sync).
bool table_needs_growth(Table* t, int64_t n);
// After enqueueing an op that may insert up to n rows: update bounds, snapshot.
void table_note_inserts(Table* t, int64_t n, cudaStream_t s);
// Exact counters (synchronizes).
void table_refresh(Table* t, cudaStream_t s);
// Rows admitted between the two latest counter snapshots (no sync): tells a
// growth regime (cold tables, zipf tails) from the warm steady state.
int64_t table_recent_growth(Table* t);
// admission of duplicate-free ids (no duplicate check), offsets out
void table_admit(Table* t, const int64_t* ids, int64_t n, int64_t step, int64_t* offsets, cudaStream_t s);
void fused_ctx_destroy(FusedCtx* c);
// apply a fused forward's deferred last_step writes before any other table op
void fused_flush_pending(Table* t, cudaStream_t s);
// order stream s after the fused index stream's last work (counter reads)
void fused_wait_index(Table* t, cudaStream_t s);
// ValueError while a prefetched fused batch is not pooled yet (its ids are
// admitted already), or — allow_pooled false — while a fused step awaits its
// backward: `op` would change slots that batch still uses
void fused_require_quiet(Table* t, bool allow_pooled, const char* op);

// device helpers ------------------------------------------------------------
__device__ __forceinline__ long long idmap_find(const HEntry* t, uint64_t mask, int64_t cap, long long key) {
  if (key == kEmptyKey) return t[cap].val;
  uint64_t i = bucket_hash((uint64_t)key) & mask;
  while (true) {
    HEntry e = ld_entry(t + i);
    if (e.key == key) return e.val;
    if (e.key == kEmptyKey) return -1;
    i = (i + 1) & mask;
  }
}

__device__ __forceinline__ void idmap_insert(HEntry* t, uint64_t mask, int64_t cap, long long key, long long slot) {
  if (key == kEmptyKey) {
    t[cap].val = slot;
    return;
  }
  uint64_t i = bucket_hash((uint64_t)key) & mask;
  while (true) {
    long long prev = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&t[i].key),
                                          (unsigned long long)kEmptyKey, (unsigned long long)key);
    if (prev == kEmptyKey || prev == key) {
      t[i].val = slot;
      return;
    }
    i = (i + 1) & mask;
  }
}

// initial_rows element (embedding.py:24-36), bit-exact: one double rounding
// for the scale multiply and one float rounding.
__device__ __forceinline__ float init_value(uint64_t base, int c, double scale) {
  uint64_t u = mix64(base + (uint64_t)(c + 1) * kGolden);
  double u01 = __dmul_rn((double)(u >> 11), 0x1p-53);
  double x = __dsub_rn(__dmul_rn(2.0, u01), 1.0);
  return __double2float_rn(__dmul_rn(x, scale));
}

// chunk ch (columns 4ch..4ch+3) of a freshly admitted row: initial weights,
// zero Adam moments.  16-byte stores when D % 4 == 0 (arena rows are then
// 16-byte aligned: 3*D floats per row).
__device__ __forceinline__ void init_row_chunk(float* row, int D, int ch, uint64_t base, double scale) {
  const int c0 = ch * 4;
  if ((D & 3) == 0) {
    const float4 w = make_float4(init_value(base, c0, scale), init_value(base, c0 + 1, scale),
                                 init_value(base, c0 + 2, scale), init_value(base, c0 + 3, scale));
    *reinterpret_cast<float4*>(row + c0) = w;
    *reinterpret_cast<float4*>(row + D + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(row + 2 * D + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    for (int c = c0; c < c0 + 4 && c < D; ++c) {
      row[c] = init_value(base, c, scale);
      row[D + c] = 0.f;
      row[2 * D + c] = 0.f;
    }
  }
}

// slot assignment of the k-th new id given free count F, allocated A
// (free list LIFO first, then sequential growth; embedding.py:203-207)
__device__ __forceinline__ int64_t assign_slot(int64_t k, int64_t F, int64_t A, const int64_t* free_list) {
  return k < F ? free_list[F - 1 - k] : A + (k - F);
}

// Adam / AdamW on one float4 of a row, every op separately rounded
// (optim.py:77-83).
struct AdamDev {
  float lr, b1, b2, eps, omb1, omb2, bc1, bc2, lrwd;
  int decay;
};
__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, const AdamDev& a) {
  if (a.decay) p = __fsub_rn(p, __fmul_rn(a.lrwd, p));
  m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, g));
  v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(a.omb2, __fmul_rn(g, g)));
  float mh = __fdiv_rn(m, a.bc1);
  float vh = __fdiv_rn(v, a.bc2);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(a.lr, mh), __fadd_rn(__fsqrt_rn(vh), a.eps)));
}
inline AdamDev to_dev(const skb_adam_t& s) {
  return AdamDev{s.lr, s.beta1, s.beta2, s.eps, s.one_minus_beta1, s.one_minus_beta2, s.bc1, s.bc2, s.lr_wd,
                 (int)s.decoupled_decay};
}

}  // namespace skb
