// table.cu — GPU dynamic embedding table: admission / lookup with the
// reference's exact slot assignment, gather / scatter, eviction in dict
// insertion order, export / restore, BlockStore accessors, sparse Adam.
//
// Admission (embedding.py:185-223) runs as probe -> exclusive scan of the
// miss flags -> insert: the k-th unknown id (input order) gets
// free_list[F-1-k] if k < F else allocated + k - F, so offsets are identical
// to the reference's dict loop while every id is handled by its own thread.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "partition.cuh"
#include "rows.cuh"
#include "table.cuh"

namespace skb {

static std::atomic<int64_t> g_snap_waits{0}, g_refreshes{0}, g_growths{0};  // SKB_DEBUG_SYNC diagnostics

Table* table_from(skb_table_t h) {
  if (!h) raise(SKB_E_ARG, 0, "null table handle");
  return reinterpret_cast<Table*>(h);
}

// ---------------------------------------------------------------------------
// growth
// ---------------------------------------------------------------------------
template <class T>
static void grow_array(T*& p, int64_t old_n, int64_t new_n, cudaStream_t s) {
  T* q = nullptr;
  SKB_CUDA(cudaMallocAsync(&q, sizeof(T) * new_n, s));
  if (old_n) SKB_CUDA(cudaMemcpyAsync(q, p, sizeof(T) * old_n, cudaMemcpyDeviceToDevice, s));
  SKB_CUDA(cudaMemsetAsync(q + old_n, 0, sizeof(T) * (new_n - old_n), s));
  if (p) SKB_CUDA(cudaFreeAsync(p, s));
  p = q;
}

// VMM growth: map more memory behind the six per-row arrays (rows never
// move); VA is reserved for the capacity hint, else 8x the rows needed, and
// re-reserved (remap, no copy) only when outgrown
static void grow_arena_vmm(Table* t, int64_t new_rows, cudaStream_t s) {
  const int64_t res_rows = std::max<int64_t>(t->rows_hint + t->rows_hint / 4, 64 * new_rows);
  const size_t esz[6] = {sizeof(float) * (size_t)t->row_stride(), sizeof(int64_t), sizeof(uint8_t), sizeof(int64_t),
                         sizeof(int64_t), sizeof(int64_t)};
  if (t->va_prep.joinable()) t->va_prep.join();  // the chunks prepared ahead are adopted below
  bool moved = false;
  for (int i = 0; i < 6; ++i) {
    // VA is cheap: at least 16 GB per array (a re-reservation drains the device)
    const size_t res = std::max<size_t>(esz[i] * (size_t)res_rows, (size_t)16 << 30);
    moved |= vmm_grow(t->va[i], esz[i] * (size_t)new_rows, res, s);
  }
  t->arena = reinterpret_cast<float*>(t->va[0].base);
  t->last_step = reinterpret_cast<int64_t*>(t->va[1].base);
  t->live = reinterpret_cast<uint8_t*>(t->va[2].base);
  t->slot_key = reinterpret_cast<int64_t*>(t->va[3].base);
  t->ins_seq = reinterpret_cast<int64_t*>(t->va[4].base);
  t->free_list = reinterpret_cast<int64_t*>(t->va[5].base);
  // mapped sizes are granularity-rounded: every array holds at least this many rows
  int64_t rows = INT64_MAX;
  for (int i = 0; i < 6; ++i) rows = std::min<int64_t>(rows, (int64_t)(t->va[i].mapped / esz[i]));
  t->arena_rows = rows;
  if (moved) t->gen++;  // only a re-reservation changes pointers (captured graphs re-prime)
  // the next growth step (1/8 of the rows) is created and mapped now on a
  // helper thread: the ~0.3 ms per array of driver calls leave the host
  // thread that feeds the step (measured: growth steps 2-3 ms vs 0.7 steady)
  size_t free_b = 0, total_b = 0;
  SKB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  int64_t prep_bytes = 0;
  for (int i = 0; i < 6; ++i) prep_bytes += (int64_t)esz[i] * (rows / 4);
  // only with room to spare: a prepared chunk is memory held before it is needed
  static const int prep_env = getenv("SKB_VMM_PREPARE") ? atoi(getenv("SKB_VMM_PREPARE")) : 1;
  if (prep_env && rows >= 65536 && (int64_t)free_b > 2 * prep_bytes + (8ll << 30)) {
    const int64_t inc = rows / 4;  // the next geometric step
    const int dev = t->device;
    t->va_prep = std::thread([t, inc, dev, esz] {
      try {
        for (int i = 0; i < 6; ++i) vmm_prepare(t->va[i], esz[i] * (size_t)inc, dev);
      } catch (...) {  // growth retries synchronously (and raises there)
      }
    });
  }
}

static void grow_arena(Table* t, int64_t new_rows, cudaStream_t s) {
  if (new_rows <= t->arena_rows) return;
  g_growths++;
  if (t->vmm) {
    grow_arena_vmm(t, new_rows, s);
    return;
  }
  const int64_t old = t->arena_rows;
  grow_array(t->arena, old * t->row_stride(), new_rows * t->row_stride(), s);
  grow_array(t->last_step, old, new_rows, s);
  grow_array(t->live, old, new_rows, s);
  grow_array(t->slot_key, old, new_rows, s);
  grow_array(t->ins_seq, old, new_rows, s);
  grow_array(t->free_list, old, new_rows, s);
  t->arena_rows = new_rows;
  t->gen++;
}

__global__ void k_rehash(const HEntry* __restrict__ old, int64_t old_cap, HEntry* nt, uint64_t mask, int64_t cap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= old_cap; i += (int64_t)gridDim.x * blockDim.x) {
    HEntry e = old[i];
    if (i == old_cap) {
      nt[cap].val = e.val;  // side slot travels as-is
    } else if (e.key != kEmptyKey) {
      idmap_insert(nt, mask, cap, e.key, e.val);
    }
  }
}

static void rehash(Table* t, int64_t new_cap, cudaStream_t s) {
  HEntry* nt = nullptr;
  SKB_CUDA(cudaMallocAsync(&nt, sizeof(HEntry) * (new_cap + 1), s));
  ht_fill(nt, new_cap + 1, -1, s);
  if (t->idmap) {
    k_rehash<<<grid_for(t->idmap_cap + 1, 256), 256, 0, s>>>(t->idmap, t->idmap_cap, nt, (uint64_t)(new_cap - 1),
                                                             new_cap);
    SKB_LAUNCH_CHECK();
    SKB_CUDA(cudaFreeAsync(t->idmap, s));
  }
  t->idmap = nt;
  t->idmap_cap = new_cap;
  t->gen++;
}

void table_refresh(Table* t, cudaStream_t s) {
  g_refreshes++;
  // a prefetched batch's admission may still run on the fused index stream:
  // the counters are read after it (else num_rows / export would size from
  // stale counters and the next reserve would miss that batch's rows)
  fused_wait_index(t, s);
  SKB_CUDA(cudaMemcpyAsync(t->snap_host, t->counters, sizeof(int64_t) * C_N, cudaMemcpyDeviceToHost, s));
  SKB_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < C_N; ++i) t->known[i] = t->snap_host[i];
  t->pending_adds = 0;
  t->adds_after_snap = 0;
  t->snap_pending = false;
}

static void harvest_snapshot(Table* t) {
  if (!t->snap_pending) return;
  if (cudaEventQuery(t->snap_ev) != cudaSuccess) {
    cudaGetLastError();  // clear cudaErrorNotReady
    return;
  }
  t->recent_growth = t->snap_host[C_ROWS] - t->known[C_ROWS];
  for (int i = 0; i < C_N; ++i) t->known[i] = t->snap_host[i];
  t->snap_pending = false;
  // the snapshot covers every op enqueued before it; later ones stay pending
  t->pending_adds = t->adds_after_snap;
  t->adds_after_snap = 0;
}

int64_t table_recent_growth(Table* t) {
  harvest_snapshot(t);
  return t->recent_growth;
}

static bool bound_ok(const Table* t, int64_t n) {
  const int64_t ub_alloc = t->known[C_ALLOC] + t->pending_adds + n;
  const int64_t ub_rows = t->known[C_ROWS] + t->pending_adds + n;
  return ub_alloc <= t->arena_rows && ub_rows * 10 < t->idmap_cap * 9;  // never fill the probe table
}

// The no-sync bound counts every position of the steps enqueued since the
// last harvested snapshot as a possible new row.  When it fails, first wait
// for the in-flight snapshot only (a step or so behind the host, not a full
// drain of the queue) and re-check; only then does the caller refresh.
static bool bound_ok_after_snapshot(Table* t, int64_t n) {
  harvest_snapshot(t);
  if (bound_ok(t, n)) return true;
  if (!t->snap_pending) return false;
  g_snap_waits++;
  SKB_CUDA(cudaEventSynchronize(t->snap_ev));
  harvest_snapshot(t);
  return bound_ok(t, n);
}

bool table_needs_growth(Table* t, int64_t n) { return !bound_ok_after_snapshot(t, n); }

void table_reserve(Table* t, int64_t n, cudaStream_t s) {
  if (t->vmm) {
    // Copy-free growth needs no exact counters: when the no-sync upper bound
    // (every enqueued position a possible new row) passes the arena, map
    // more rows — geometrically (1/4 of the arena, or the bound + 1/8), so
    // a growing table maps O(log) chunks, each prepared ahead on a helper
    // thread.  One exception: a large mapping (> 256 MB) for a table that
    // is barely growing (its last snapshot interval admitted less than a
    // quarter of the pending positions: a warm table whose bound is all
    // hits) first waits for the in-flight snapshot — one index phase behind
    // the host, not a drain — and re-checks with its counts, so a host
    // running steps ahead never maps memory for rows that never come.
    // A host more than 8 steps ahead of its last snapshot waits for that
    // snapshot first (the device still has >= 8 steps queued, so this only
    // throttles the host): the bound then never outruns the rows by more
    // than 8 steps and a warm table settles on a fixed arena (C1: a host
    // 200 graph-replayed steps ahead grew the arena ten times, 56 -> 105 us/step).
    harvest_snapshot(t);
    if (t->snap_pending && t->pending_adds > 8 * n) {
      g_snap_waits++;
      SKB_CUDA(cudaEventSynchronize(t->snap_ev));
      harvest_snapshot(t);
    }
    int64_t ub = t->known[C_ALLOC] + t->pending_adds + n;
    if (ub > t->arena_rows) {
      const int64_t row_bytes = (int64_t)sizeof(float) * t->row_stride() + 4 * (int64_t)sizeof(int64_t) + 1;
      const int64_t target = std::max<int64_t>(ub + ub / 8, t->arena_rows + t->arena_rows / 4);
      const bool big = (target - t->arena_rows) * row_bytes > (256ll << 20);
      if (big && t->snap_pending && t->recent_growth * 4 < t->pending_adds) {
        g_snap_waits++;
        SKB_CUDA(cudaEventSynchronize(t->snap_ev));
        harvest_snapshot(t);
        ub = t->known[C_ALLOC] + t->pending_adds + n;
      }
      if (ub > t->arena_rows)
        grow_arena(t, std::max<int64_t>({ub + ub / 8, t->arena_rows + t->arena_rows / 4, (int64_t)1024}), s);
    }
  }
  if (bound_ok_after_snapshot(t, n)) return;
  table_refresh(t, s);
  int64_t need_alloc = t->known[C_ALLOC] + n;
  int64_t need_rows = t->known[C_ROWS] + n;
  if (need_alloc > t->arena_rows) {
    // copy-free (VMM) growth is cheap: 1/8 headroom keeps the mapped arena
    // within ~1.1x of the rows; the copying fallback grows 1.5x
    int64_t nr = t->arena_rows + (t->vmm ? t->arena_rows / 8 : t->arena_rows / 2);
    if (nr < need_alloc) nr = need_alloc;
    if (nr < 1024) nr = 1024;
    grow_arena(t, nr, s);
  }
  if (need_rows * 2 > t->idmap_cap) rehash(t, next_pow2(need_rows * 3), s);
}

void table_note_inserts(Table* t, int64_t n, cudaStream_t s) {
  // `known` stays the last HARVESTED snapshot until the in-flight one lands,
  // so every admission since then must stay in pending_adds (upper bound)
  t->pending_adds += n;
  if (t->snap_pending) {
    t->adds_after_snap += n;
  } else {
    SKB_CUDA(cudaMemcpyAsync(t->snap_host, t->counters, sizeof(int64_t) * C_N, cudaMemcpyDeviceToHost, s));
    SKB_CUDA(cudaEventRecord(t->snap_ev, s));
    t->snap_pending = true;
    t->adds_after_snap = 0;  // this op is covered by the new snapshot
  }
}

// ---------------------------------------------------------------------------
// admission
// ---------------------------------------------------------------------------
__global__ void k_probe(const int64_t* __restrict__ ids, int64_t n, const HEntry* __restrict__ map, uint64_t mask,
                        int64_t cap, int64_t step, int64_t* __restrict__ offsets, int32_t* __restrict__ miss,
                        int64_t* __restrict__ last_step) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    long long s = idmap_find(map, mask, cap, ids[i]);
    miss[i] = s < 0 ? 1 : 0;
    if (s >= 0) {
      offsets[i] = s;
      last_step[s] = step;
    }
  }
}

// One thread per (miss position, 4-column chunk): the slot formula needs no
// coordination, chunk 0 also publishes the key and the per-slot metadata.
__global__ void k_admit(const int64_t* __restrict__ ids, int64_t n, const int32_t* __restrict__ miss,
                        const int64_t* __restrict__ rank, const int64_t* __restrict__ counters,
                        const int64_t* __restrict__ free_list, HEntry* map, uint64_t mask, int64_t cap, int64_t step,
                        int D, uint64_t seed_mix, double scale, float* __restrict__ arena,
                        int64_t* __restrict__ last_step, uint8_t* __restrict__ live, int64_t* __restrict__ slot_key,
                        int64_t* __restrict__ ins_seq, int64_t* __restrict__ offsets) {
  const int chunks = (D + 3) / 4;
  const int64_t total = n * chunks;
  const int64_t A = counters[C_ALLOC], F = counters[C_FREE], seq = counters[C_SEQ];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / chunks;
    if (!miss[i]) continue;
    int ch = (int)(t - i * chunks);
    int64_t k = rank[i];
    int64_t slot = assign_slot(k, F, A, free_list);
    long long key = ids[i];
    if (ch == 0) {
      idmap_insert(map, mask, cap, key, slot);
      offsets[i] = slot;
      last_step[slot] = step;
      live[slot] = 1;
      slot_key[slot] = key;
      ins_seq[slot] = seq + k;
    }
    uint64_t base = mix64((uint64_t)key ^ seed_mix);
    float* row = arena + slot * (int64_t)(3 * D);
    init_row_chunk(row, D, ch, base, scale);
  }
}

__global__ void k_finish_admit(int64_t* counters, const int64_t* __restrict__ total_new) {
  int64_t K = *total_new, F = counters[C_FREE];
  int64_t take = K < F ? K : F;
  counters[C_FREE] = F - take;
  counters[C_ALLOC] += K - take;
  counters[C_ROWS] += K;
  counters[C_SEQ] += K;
}

static int64_t read_i64(const int64_t* dptr, cudaStream_t s) {
  int64_t v = 0;
  SKB_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SKB_CUDA(cudaStreamSynchronize(s));
  return v;
}

void table_admit(Table* t, const int64_t* ids, int64_t n, int64_t step, int64_t* offsets, cudaStream_t s) {
  fused_flush_pending(t, s);
  table_reserve(t, n, s);
  Scratch miss(sizeof(int32_t) * n, s), rank(sizeof(int64_t) * n, s), total(sizeof(int64_t), s);
  const uint64_t mask = (uint64_t)(t->idmap_cap - 1);
  k_probe<<<grid_for(n, 256), 256, 0, s>>>(ids, n, t->idmap, mask, t->idmap_cap, step, offsets, miss.as<int32_t>(),
                                          t->last_step);
  SKB_LAUNCH_CHECK();
  scan_exclusive_i32_to_i64(miss.as<int32_t>(), rank.as<int64_t>(), n, total.as<int64_t>(), s);
  const int chunks = (int)((t->dim + 3) / 4);
  k_admit<<<grid_for(n * chunks, 256), 256, 0, s>>>(ids, n, miss.as<int32_t>(), rank.as<int64_t>(), t->counters,
                                                   t->free_list, t->idmap, mask, t->idmap_cap, step, (int)t->dim,
                                                   t->seed_mix, t->init_scale, t->arena, t->last_step, t->live,
                                                   t->slot_key, t->ins_seq, offsets);
  SKB_LAUNCH_CHECK();
  k_finish_admit<<<1, 1, 0, s>>>(t->counters, total.as<int64_t>());
  SKB_LAUNCH_CHECK();
  table_note_inserts(t, n, s);
}

// ---------------------------------------------------------------------------
// gather / scatter with liveness checks (embedding.py:225-250)
// ---------------------------------------------------------------------------
__global__ void k_check_live(const int64_t* __restrict__ offs, int64_t n, const uint8_t* __restrict__ live,
                             int64_t limit, unsigned long long* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offs[i];
    if (o < 0 || o >= limit || !live[o]) atomicMin(flag, (unsigned long long)i);
  }
}

__global__ void k_check_range(const int64_t* __restrict__ offs, int64_t n, int64_t limit, unsigned long long* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offs[i];
    if (o < 0 || o >= limit) atomicMin(flag, (unsigned long long)i);
  }
}

static void check_live(Table* t, const int64_t* offs, int64_t n, const char* op, cudaStream_t s) {
  DevFlag f(s);
  k_check_live<<<grid_for(n, 256), 256, 0, s>>>(offs, n, t->live, t->arena_rows, f.ptr());
  SKB_LAUNCH_CHECK();
  int64_t bad = f.read();
  if (bad >= 0) {
    int64_t o = read_i64(offs + bad, s);
    raise(SKB_E_INDEX, o, "%s: offset %lld is not a live slot", op, (long long)o);
  }
}

static int64_t reported_capacity(Table* t) {
  int64_t hw = t->known[C_ALLOC] > t->ensured_slots ? t->known[C_ALLOC] : t->ensured_slots;
  return (hw + t->block_size - 1) / t->block_size * t->block_size;
}

// ---------------------------------------------------------------------------
// checked row ops without extra round trips.  Every check runs on the device
// against the table's persistent flags and is read back once (pinned, one
// synchronize); the store limit (BlockStore.capacity, embedding.py:83-85)
// is computed on the device from the allocation counter, so no counter
// refresh.  Check-then-write ops (scatter_update embedding.py:240-250,
// BlockStore.write embedding.py:113-115) are two back-to-back launches with
// no host round trip between them: the check kernel sets the flags, the
// write kernel reads them on the device and writes only if nothing was
// flagged — the table is untouched on error, as in the reference.
//   flags[0] duplicate (min index)   flags[1] not live / out of range
//   flags[2] out of range (scatter_update: duplicates then need the hash test)
// ---------------------------------------------------------------------------
constexpr unsigned long long kNoFlag = ~0ull;

__device__ __forceinline__ int64_t store_limit(const int64_t* counters, int64_t ensured, int64_t bs, int64_t rows) {
  const int64_t hw = counters[C_ALLOC] > ensured ? counters[C_ALLOC] : ensured;
  const int64_t cap = (hw + bs - 1) / bs * bs;
  return cap < rows ? cap : rows;
}

__global__ void k_check_range(const int64_t* __restrict__ offs, int64_t n, const int64_t* __restrict__ counters,
                              int64_t ensured, int64_t bs, int64_t rows, unsigned long long* flags) {
  const int64_t limit = store_limit(counters, ensured, bs, rows);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offs[i];
    if (o < 0 || o >= limit) atomicMin(&flags[1], (unsigned long long)i);
  }
}

// MODE 0: scatter_update (distinct + live), MODE 1: BlockStore.write (range),
// MODE 2: sparse_adam_step (distinct + range)
template <int MODE>
__global__ void __launch_bounds__(256) k_check_rows(const int64_t* __restrict__ offs, int64_t n,
                                                    const uint8_t* __restrict__ live,
                                                    const int64_t* __restrict__ counters, int64_t ensured,
                                                    int64_t bs, int64_t rows, uint32_t* bitmap,
                                                    unsigned long long* flags) {
  const int64_t limit = MODE != 0 ? store_limit(counters, ensured, bs, rows) : rows;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t o = offs[i];
    if (o < 0 || o >= limit) {
      atomicMin(&flags[1], (unsigned long long)i);
      if (MODE != 1) atomicMin(&flags[2], (unsigned long long)i);
      continue;
    }
    if (MODE != 1) {
      const uint32_t bit = 1u << (o & 31);
      if (atomicOr(&bitmap[o >> 5], bit) & bit) atomicMin(&flags[0], (unsigned long long)i);
    }
    if (MODE == 0 && !live[o]) atomicMin(&flags[1], (unsigned long long)i);
  }
}

// second launch of a check-then-write op: writes only if the check kernel
// flagged nothing (read on the device — no host round trip in between), and
// returns the distinctness bitmap to all-clear
template <int VEC, int MODE>
__global__ void __launch_bounds__(256) k_write_rows_if_clear(const int64_t* __restrict__ offs, int64_t n,
                                                             const float* __restrict__ src, int D, float* dst,
                                                             int64_t dstride, int64_t rows, uint32_t* bitmap,
                                                             const unsigned long long* flags) {
  const bool ok = __ldcg(&flags[0]) == kNoFlag && __ldcg(&flags[1]) == kNoFlag;
  using V = typename VecT<VEC>::T;
  constexpr int U = kRowsUnroll;
  const int per_row = D / VEC;
  const bool pow2 = (per_row & (per_row - 1)) == 0;
  const int sh = __ffs(per_row) - 1;
  const int64_t total = n * per_row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < total; base += stride * U) {
    int64_t r[U], row[U];
    int col[U];
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = base + u * stride;
      r[u] = -1;
      if (t < total) {
        row[u] = pow2 ? (t >> sh) : t / per_row;  // no 64-bit division for power-of-two row widths
        col[u] = (int)(t - row[u] * per_row) * VEC;
        r[u] = offs[row[u]];
        if (MODE == 0 && bitmap && col[u] == 0 && r[u] >= 0 && r[u] < rows) bitmap[r[u] >> 5] = 0u;
        if (ok) v[u] = vload<VEC>(src + row[u] * (int64_t)D + col[u]);
      }
    }
    if (ok) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r[u] >= 0) vstore<VEC>(dst + r[u] * dstride + col[u], v[u]);
    }
  }
}

// flags: the table's own (read back by the caller right after) or a
// caller-owned device array (deferred checks)
template <int VEC, int MODE>
static void launch_checked_scatter(Table* t, const int64_t* offs, int64_t n, const float* src, float* dst,
                                   cudaStream_t s, unsigned long long* flags = nullptr) {
  if (!flags) flags = t->dflags;
  k_check_rows<MODE><<<grid_for(n, 256), 256, 0, s>>>(offs, n, t->live, t->counters, t->ensured_slots,
                                                      t->block_size, t->arena_rows, t->bitmap, flags);
  SKB_LAUNCH_CHECK();
  const int D = (int)t->dim;
  // the distinctness bitmap back to all-clear: one memset when the whole
  // bitmap is smaller than the rows' scattered sector writes would be (1M
  // rows over a 1M-row table: 128 KB instead of 1M random 32-byte sector
  // writes inside the write kernel), per row otherwise (few rows, big table)
  const bool memset_clear = MODE == 0 && t->bitmap_words * (int64_t)sizeof(uint32_t) <= n * 32;
  k_write_rows_if_clear<VEC, MODE><<<grid_for((n * (D / VEC) + kRowsUnroll - 1) / kRowsUnroll, 256), 256, 0, s>>>(
      offs, n, src, D, dst, 3 * t->dim, t->arena_rows, memset_clear ? nullptr : t->bitmap, flags);
  SKB_LAUNCH_CHECK();
  if (memset_clear) SKB_CUDA(cudaMemsetAsync(t->bitmap, 0, sizeof(uint32_t) * t->bitmap_words, s));
}

// pinned readback of the persistent flags (synchronizes)
static const int64_t* flags_fetch(Table* t, cudaStream_t s) {
  SKB_CUDA(cudaMemcpyAsync(t->hflags, t->dflags, sizeof(int64_t) * 4, cudaMemcpyDeviceToHost, s));
  SKB_CUDA(cudaStreamSynchronize(s));
  return t->hflags;
}
static void flags_rearm(Table* t, cudaStream_t s) {
  SKB_CUDA(cudaMemsetAsync(t->dflags, 0xFF, sizeof(unsigned long long) * 4, s));
  SKB_CUDA(cudaStreamSynchronize(s));
}

static void ensure_bitmap(Table* t, cudaStream_t s) {
  const int64_t words = (t->arena_rows + 31) / 32 + 1;
  if (words <= t->bitmap_words) return;
  if (t->bitmap) SKB_CUDA(cudaFreeAsync(t->bitmap, s));
  SKB_CUDA(cudaMallocAsync(&t->bitmap, sizeof(uint32_t) * words, s));
  SKB_CUDA(cudaMemsetAsync(t->bitmap, 0, sizeof(uint32_t) * words, s));
  t->bitmap_words = words;
}

static void raise_range(Table* t, const int64_t* offs, int64_t bad, cudaStream_t s) {
  const int64_t o = read_i64(offs + bad, s);
  table_refresh(t, s);
  int64_t lim = reported_capacity(t);
  if (lim > t->arena_rows) lim = t->arena_rows;
  raise(SKB_E_INDEX, o, "offset %lld is outside the store capacity %lld", (long long)o, (long long)lim);
}

__global__ void k_clear_bits(const int64_t* __restrict__ offs, int64_t n, int64_t rows, uint32_t* bitmap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = offs[i];
    if (o >= 0 && o < rows) bitmap[o >> 5] = 0u;
  }
}

// sparse_adam_step preconditions (embedding.py sparse_adam_step): distinct
// offsets (ValueError) before the store range (IndexError) — two launches and
// one readback, distinctness on the slot bitmap instead of a hash table
static void check_adam_offsets(Table* t, const int64_t* offs, int64_t n, cudaStream_t s) {
  fused_flush_pending(t, s);
  ensure_bitmap(t, s);
  k_check_rows<2><<<grid_for(n, 256), 256, 0, s>>>(offs, n, t->live, t->counters, t->ensured_slots, t->block_size,
                                                  t->arena_rows, t->bitmap, t->dflags);
  SKB_LAUNCH_CHECK();
  if (t->bitmap_words * (int64_t)sizeof(uint32_t) <= n * 32)  // as launch_checked_scatter: memset when cheaper
    SKB_CUDA(cudaMemsetAsync(t->bitmap, 0, sizeof(uint32_t) * t->bitmap_words, s));
  else
    k_clear_bits<<<grid_for(n, 256), 256, 0, s>>>(offs, n, t->arena_rows, t->bitmap);
  SKB_LAUNCH_CHECK();
  const int64_t* f = flags_fetch(t, s);
  const unsigned long long f0 = (uint64_t)f[0], f1 = (uint64_t)f[1], f2 = (uint64_t)f[2];
  if (f0 == kNoFlag && f1 == kNoFlag) return;
  flags_rearm(t, s);
  const bool dup = f2 != kNoFlag ? has_duplicate(offs, n, s) : f0 != kNoFlag;
  if (dup) raise(SKB_E_VALUE, 0, "sparse_adam_step requires distinct offsets");
  raise_range(t, offs, (int64_t)f1, s);
}

static void check_range(Table* t, const int64_t* offs, int64_t n, cudaStream_t s) {
  fused_flush_pending(t, s);
  k_check_range<<<grid_for(n, 256), 256, 0, s>>>(offs, n, t->counters, t->ensured_slots, t->block_size,
                                                 t->arena_rows, t->dflags);
  SKB_LAUNCH_CHECK();
  const int64_t bad = flags_fetch(t, s)[1];
  if ((uint64_t)bad != kNoFlag) {
    flags_rearm(t, s);
    raise_range(t, offs, bad, s);
  }
}

// BlockStore.write of column `which` (range-checked, one launch)
static void checked_write(Table* t, const int64_t* offs, int64_t n, int which, const float* rows, cudaStream_t s) {
  fused_flush_pending(t, s);
  float* dst = t->arena + which * t->dim;
  const bool v4 = t->dim % 4 == 0 && (uintptr_t)rows % 16 == 0;
  if (v4) launch_checked_scatter<4, 1>(t, offs, n, rows, dst, s);
  else launch_checked_scatter<1, 1>(t, offs, n, rows, dst, s);
  const int64_t bad = flags_fetch(t, s)[1];
  if ((uint64_t)bad != kNoFlag) {
    flags_rearm(t, s);
    raise_range(t, offs, bad, s);
  }
}

// EmbeddingTable.scatter_update: distinct + live, then write (one launch)
static void checked_scatter_update(Table* t, const int64_t* offs, int64_t n, const float* rows, cudaStream_t s) {
  fused_require_quiet(t, true, "scatter_update");
  ensure_bitmap(t, s);
  const bool v4 = t->dim % 4 == 0 && (uintptr_t)rows % 16 == 0;
  if (v4) launch_checked_scatter<4, 0>(t, offs, n, rows, t->arena, s);
  else launch_checked_scatter<1, 0>(t, offs, n, rows, t->arena, s);
  const int64_t* f = flags_fetch(t, s);
  const unsigned long long f0 = (uint64_t)f[0], f1 = (uint64_t)f[1], f2 = (uint64_t)f[2];
  if (f0 == kNoFlag && f1 == kNoFlag) return;
  flags_rearm(t, s);
  // reference order: duplicates (ValueError) before liveness (IndexError); an
  // out-of-range offset can only duplicate another out-of-range one, so that
  // rare case re-checks distinctness with the hash path
  const bool dup = f2 != kNoFlag ? has_duplicate(offs, n, s) : f0 != kNoFlag;
  if (dup) raise(SKB_E_VALUE, 0, "scatter_update requires distinct offsets");
  const int64_t o = read_i64(offs + (int64_t)f1, s);
  raise(SKB_E_INDEX, o, "scatter_update: offset %lld is not a live slot", (long long)o);
}

// ---------------------------------------------------------------------------
// eviction (embedding.py:252-274)
// ---------------------------------------------------------------------------
// stale IDMap entries (embedding.py:262-264 iterates the dict, not the live
// flags: an id removed from the IDMap is never evicted, a put entry is)
__global__ void k_stale_entries(const HEntry* __restrict__ map, int64_t cap, const int64_t* __restrict__ last,
                                int64_t step, int64_t thr, uint8_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cap; i += (int64_t)gridDim.x * blockDim.x) {
    const HEntry e = map[i];
    const bool valid = i == cap ? e.val >= 0 : e.key != kEmptyKey;
    flags[i] = (valid && (step - last[e.val]) > thr) ? 1 : 0;
  }
}

__global__ void k_gather_i64(const int64_t* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                             int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

// one thread per (evicted slot, 4-column chunk): zero the Adam moments
// (16-byte stores when D % 4 == 0); chunk 0 returns the slot to the free list
__global__ void k_evict_apply(const int64_t* __restrict__ slots, int64_t E, int D, int64_t* counters,
                              int64_t* __restrict__ free_list, uint8_t* __restrict__ live,
                              int64_t* __restrict__ last, float* __restrict__ arena) {
  const int64_t F = counters[C_FREE];
  const int chunks = (D + 3) >> 2;
  const int64_t total = E * chunks;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / chunks;
    const int c0 = (int)(t - j * chunks) * 4;
    const int64_t s = slots[j];
    float* row = arena + s * (int64_t)(3 * D);
    if ((D & 3) == 0) {
      *reinterpret_cast<float4*>(row + D + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(row + 2 * D + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (int c = c0; c < c0 + 4 && c < D; ++c) {
        row[D + c] = 0.f;
        row[2 * D + c] = 0.f;
      }
    }
    if (c0 == 0) {
      free_list[F + j] = s;
      live[s] = 0;
      last[s] = 0;
    }
  }
}

__global__ void k_evict_counters(int64_t* counters, int64_t E) {
  counters[C_FREE] += E;
  counters[C_ROWS] -= E;
}

// keep every entry except the evicted ones (rebuild instead of tombstones)
__global__ void k_rebuild_drop(const HEntry* __restrict__ old, int64_t cap, const uint8_t* __restrict__ drop,
                               HEntry* nt) {
  const uint64_t mask = (uint64_t)(cap - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cap; i += (int64_t)gridDim.x * blockDim.x) {
    HEntry e = old[i];
    if (i == cap) {
      nt[cap].val = drop[i] ? -1 : e.val;
    } else if (e.key != kEmptyKey && !drop[i]) {
      idmap_insert(nt, mask, cap, e.key, e.val);
    }
  }
}

__global__ void k_entry_pairs(const HEntry* __restrict__ map, int64_t cap, const int64_t* __restrict__ idx, int64_t n,
                              const int64_t* __restrict__ ins_seq, int64_t* __restrict__ keys,
                              int64_t* __restrict__ slots, int64_t* __restrict__ seq);

int64_t table_evict(Table* t, int64_t step, cudaStream_t s) {
  fused_require_quiet(t, false, "evict");
  fused_flush_pending(t, s);
  if (t->evict_threshold == kNoEvict || t->arena_rows == 0) return 0;
  // stale IDMap entries, in dict insertion order (embedding.py:262-272)
  const int64_t cap = t->idmap_cap;
  Scratch flags(cap + 1, s), idx(sizeof(int64_t) * (cap + 1), s), cnt(sizeof(int64_t) * 2, s);
  k_stale_entries<<<grid_for(cap + 1, 256), 256, 0, s>>>(t->idmap, cap, t->last_step, step, t->evict_threshold,
                                                         flags.as<uint8_t>());
  SKB_LAUNCH_CHECK();
  select_flagged_index(flags.as<uint8_t>(), cap + 1, idx.as<int64_t>(), cnt.as<int64_t>(), s);
  // E and the insertion-sequence counter in one readback: every ins_seq is
  // below C_SEQ, so the order sort needs only bit_width(C_SEQ) key bits
  SKB_CUDA(cudaMemcpyAsync(cnt.as<int64_t>() + 1, t->counters + C_SEQ, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  int64_t* h = pinned_mailbox();
  SKB_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, s));
  SKB_CUDA(cudaStreamSynchronize(s));
  const int64_t E = h[0], seq_hi = h[1];
  if (E == 0) return 0;
  int bits = 1;
  while (bits < 64 && (seq_hi >> bits) != 0) ++bits;
  Scratch keys(sizeof(int64_t) * E, s), slots(sizeof(int64_t) * E, s), seq(sizeof(int64_t) * E, s),
      seq2(sizeof(int64_t) * E, s), slots2(sizeof(int64_t) * E, s);
  k_entry_pairs<<<grid_for(E, 256), 256, 0, s>>>(t->idmap, cap, idx.as<int64_t>(), E, t->ins_seq, keys.as<int64_t>(),
                                                slots.as<int64_t>(), seq.as<int64_t>());
  SKB_LAUNCH_CHECK();
  sort_pairs_i64(seq.as<int64_t>(), seq2.as<int64_t>(), slots.as<int64_t>(), slots2.as<int64_t>(), E, s, bits);
  k_evict_apply<<<grid_for(E * ((t->dim + 3) / 4), 256), 256, 0, s>>>(slots2.as<int64_t>(), E, (int)t->dim, t->counters,
                                                         t->free_list, t->live, t->last_step, t->arena);
  SKB_LAUNCH_CHECK();
  k_evict_counters<<<1, 1, 0, s>>>(t->counters, E);
  SKB_LAUNCH_CHECK();
  HEntry* nt = nullptr;
  SKB_CUDA(cudaMallocAsync(&nt, sizeof(HEntry) * (cap + 1), s));
  ht_fill(nt, cap + 1, -1, s);
  k_rebuild_drop<<<grid_for(cap + 1, 256), 256, 0, s>>>(t->idmap, cap, flags.as<uint8_t>(), nt);
  SKB_LAUNCH_CHECK();
  SKB_CUDA(cudaFreeAsync(t->idmap, s));
  t->idmap = nt;
  t->gen++;
  table_refresh(t, s);
  return E;
}

// ---------------------------------------------------------------------------
// export / restore (embedding.py:276-308)
// ---------------------------------------------------------------------------
struct IdxSlotArena {
  const int64_t* slots;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return slots[i]; }
};

__global__ void k_entry_flags(const HEntry* __restrict__ map, int64_t cap, uint8_t* __restrict__ flags);

// the IDMap's entries sorted by id (embedding.py:276-284 iterates the dict:
// a slot whose id was removed from the IDMap is not exported, even if live)
int64_t table_export(Table* t, int64_t* ids, float* w, float* m, float* v, int64_t* last, int64_t capacity,
                     cudaStream_t s) {
  fused_flush_pending(t, s);
  const int64_t cap = t->idmap_cap;
  Scratch flags(cap + 1, s), idx(sizeof(int64_t) * (cap + 1), s), cnt(sizeof(int64_t), s);
  k_entry_flags<<<grid_for(cap + 1, 256), 256, 0, s>>>(t->idmap, cap, flags.as<uint8_t>());
  SKB_LAUNCH_CHECK();
  select_flagged_index(flags.as<uint8_t>(), cap + 1, idx.as<int64_t>(), cnt.as<int64_t>(), s);
  int64_t n = read_i64(cnt.as<int64_t>(), s);
  if (n > capacity) raise(SKB_E_ARG, n, "export buffers hold %lld rows, table has %lld", (long long)capacity,
                          (long long)n);
  if (n == 0) return 0;
  Scratch keys(sizeof(int64_t) * n, s), slots(sizeof(int64_t) * n, s), seq(sizeof(int64_t) * n, s),
      slots2(sizeof(int64_t) * n, s);
  k_entry_pairs<<<grid_for(n, 256), 256, 0, s>>>(t->idmap, cap, idx.as<int64_t>(), n, t->ins_seq, keys.as<int64_t>(),
                                                slots.as<int64_t>(), seq.as<int64_t>());
  SKB_LAUNCH_CHECK();
  sort_pairs_i64(keys.as<int64_t>(), ids, slots.as<int64_t>(), slots2.as<int64_t>(), n, s);
  const int D = (int)t->dim;
  IdxSlotArena ix{slots2.as<int64_t>()};
  if (w) launch_rows_gather(ix, t->arena, 3 * D, w, D, n, D, s);
  if (m) launch_rows_gather(ix, t->arena + D, 3 * D, m, D, n, D, s);
  if (v) launch_rows_gather(ix, t->arena + 2 * D, 3 * D, v, D, n, D, s);
  if (last) {
    k_gather_i64<<<grid_for(n, 256), 256, 0, s>>>(t->last_step, slots2.as<int64_t>(), n, last);
    SKB_LAUNCH_CHECK();
  }
  return n;
}

__global__ void k_present_flag(const int64_t* __restrict__ ids, int64_t n, const HEntry* __restrict__ map,
                               uint64_t mask, int64_t cap, const HEntry* __restrict__ dt,
                               const int64_t* __restrict__ hslot, unsigned long long* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (idmap_find(map, mask, cap, ids[i]) >= 0 || dt[hslot[i]].val != i) atomicMin(flag, (unsigned long long)i);
}

__global__ void k_restore(const int64_t* __restrict__ ids, int64_t n, const int64_t* __restrict__ counters,
                          const int64_t* __restrict__ free_list, HEntry* map, uint64_t mask, int64_t cap,
                          const int64_t* __restrict__ last_in, int64_t* __restrict__ last_step,
                          uint8_t* __restrict__ live, int64_t* __restrict__ slot_key, int64_t* __restrict__ ins_seq,
                          int64_t* __restrict__ slots_out) {
  const int64_t A = counters[C_ALLOC], F = counters[C_FREE], seq = counters[C_SEQ];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t slot = assign_slot(i, F, A, free_list);
    idmap_insert(map, mask, cap, ids[i], slot);
    last_step[slot] = last_in[i];
    live[slot] = 1;
    slot_key[slot] = ids[i];
    ins_seq[slot] = seq + i;
    slots_out[i] = slot;
  }
}

__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }

__global__ void k_range_flag(const int64_t* __restrict__ v, int64_t n, int64_t hi, unsigned long long* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (v[i] < 0 || v[i] >= hi) atomicMin(flag, (unsigned long long)i);
}

void table_restore(Table* t, const int64_t* ids, int64_t n, const float* w, const float* m, const float* v,
                   const int64_t* last, cudaStream_t s) {
  fused_require_quiet(t, false, "restore_rows");
  fused_flush_pending(t, s);
  if (n == 0) return;
  {
    DedupResult r;
    dedup_insert(ids, n, r, s);
    DevFlag f(s);
    k_present_flag<<<grid_for(n, 256), 256, 0, s>>>(ids, n, t->idmap, (uint64_t)(t->idmap_cap - 1), t->idmap_cap,
                                                    r.table.as<HEntry>(), r.hslot.as<int64_t>(), f.ptr());
    SKB_LAUNCH_CHECK();
    int64_t bad = f.read();
    if (bad >= 0) {
      int64_t id = read_i64(ids + bad, s);
      raise(SKB_E_VALUE, id, "restore_rows: id %lld already present", (long long)id);
    }
  }
  table_reserve(t, n, s);
  Scratch slots(sizeof(int64_t) * n, s), total(sizeof(int64_t), s);
  k_restore<<<grid_for(n, 256), 256, 0, s>>>(ids, n, t->counters, t->free_list, t->idmap,
                                            (uint64_t)(t->idmap_cap - 1), t->idmap_cap, last, t->last_step, t->live,
                                            t->slot_key, t->ins_seq, slots.as<int64_t>());
  SKB_LAUNCH_CHECK();
  const int D = (int)t->dim;
  IdxSlotArena ix{slots.as<int64_t>()};
  launch_rows_scatter(ix, w, D, t->arena, 3 * D, n, D, s);
  launch_rows_scatter(ix, m, D, t->arena + D, 3 * D, n, D, s);
  launch_rows_scatter(ix, v, D, t->arena + 2 * D, 3 * D, n, D, s);
  k_set_i64<<<1, 1, 0, s>>>(total.as<int64_t>(), n);
  SKB_LAUNCH_CHECK();
  k_finish_admit<<<1, 1, 0, s>>>(t->counters, total.as<int64_t>());
  SKB_LAUNCH_CHECK();
  table_note_inserts(t, n, s);
}

// ---------------------------------------------------------------------------
// sparse Adam (optim.py:42-83)
// ---------------------------------------------------------------------------
template <int VEC>
__global__ void k_adam_rows(const int64_t* __restrict__ offs, int64_t n, const float* __restrict__ grads, int D,
                            AdamDev a, float* __restrict__ arena) {
  const int per_row = D / VEC;
  const int64_t total = n * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / per_row;
    int c = (int)(t - i * per_row) * VEC;
    float* row = arena + offs[i] * (int64_t)(3 * D);
    if constexpr (VEC == 4) {
      float4 p = *reinterpret_cast<float4*>(row + c), m = *reinterpret_cast<float4*>(row + D + c),
             v = *reinterpret_cast<float4*>(row + 2 * D + c), g = ldg4(grads + i * D + c);
      adam1(p.x, m.x, v.x, g.x, a);
      adam1(p.y, m.y, v.y, g.y, a);
      adam1(p.z, m.z, v.z, g.z, a);
      adam1(p.w, m.w, v.w, g.w, a);
      st4(row + c, p);
      st4(row + D + c, m);
      st4(row + 2 * D + c, v);
    } else {
      float p = row[c], m = row[D + c], v = row[2 * D + c];
      adam1(p, m, v, grads[i * D + c], a);
      row[c] = p;
      row[D + c] = m;
      row[2 * D + c] = v;
    }
  }
}

void table_adam(Table* t, const int64_t* offs, int64_t n, const float* grads, const skb_adam_t& sc, cudaStream_t s) {
  AdamDev a = to_dev(sc);
  const int D = (int)t->dim;
  if (D % 4 == 0 && (uintptr_t)grads % 16 == 0)
    k_adam_rows<4><<<grid_for(n * (D / 4), 256), 256, 0, s>>>(offs, n, grads, D, a, t->arena);
  else
    k_adam_rows<1><<<grid_for(n * D, 256), 256, 0, s>>>(offs, n, grads, D, a, t->arena);
  SKB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// misc accessors
// ---------------------------------------------------------------------------
__global__ void k_write_last(const int64_t* __restrict__ offs, int64_t n, const int64_t* __restrict__ vals,
                             int64_t scalar, int64_t* __restrict__ last) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    last[offs[i]] = vals ? vals[i] : scalar;
}

__global__ void k_clear_aux(const int64_t* __restrict__ offs, int64_t n, int D, float* __restrict__ arena,
                            int64_t* __restrict__ last) {
  const int64_t total = n * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / D;
    int c = (int)(t - i * D);
    float* row = arena + offs[i] * (int64_t)(3 * D);
    row[D + c] = 0.f;
    row[2 * D + c] = 0.f;
    if (c == 0) last[offs[i]] = 0;
  }
}

__global__ void k_idmap_get(const int64_t* __restrict__ ids, int64_t n, const HEntry* __restrict__ map, uint64_t mask,
                            int64_t cap, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = idmap_find(map, mask, cap, ids[i]);
}

// put: update in place or insert (dict semantics: a new key is appended)
__global__ void k_idmap_put(HEntry* map, uint64_t mask, int64_t cap, long long key, long long slot,
                            int64_t* counters, int64_t* ins_seq) {
  long long old = idmap_find(map, mask, cap, key);
  if (old >= 0) {
    if (key == kEmptyKey) {
      map[cap].val = slot;
    } else {
      uint64_t i = bucket_hash((uint64_t)key) & mask;
      while (map[i].key != key) i = (i + 1) & mask;
      map[i].val = slot;
    }
    ins_seq[slot] = ins_seq[old];
    return;
  }
  idmap_insert(map, mask, cap, key, slot);
  ins_seq[slot] = counters[C_SEQ]++;
  counters[C_ROWS] += 1;
}

// remove with backward-shift deletion (linear probing stays tombstone-free)
__global__ void k_idmap_remove(HEntry* map, uint64_t mask, int64_t cap, long long key, int64_t* counters,
                               int64_t* out_slot) {
  if (key == kEmptyKey) {
    *out_slot = map[cap].val;
    if (map[cap].val >= 0) counters[C_ROWS] -= 1;
    map[cap].val = -1;
    return;
  }
  uint64_t i = bucket_hash((uint64_t)key) & mask;
  while (true) {
    if (map[i].key == key) break;
    if (map[i].key == kEmptyKey) {
      *out_slot = -1;
      return;
    }
    i = (i + 1) & mask;
  }
  *out_slot = map[i].val;
  counters[C_ROWS] -= 1;
  map[i].key = kEmptyKey;
  map[i].val = -1;
  uint64_t j = i;
  while (true) {
    j = (j + 1) & mask;
    if (map[j].key == kEmptyKey) break;
    uint64_t h = bucket_hash((uint64_t)map[j].key) & mask;
    bool stays = (i <= j) ? (i < h && h <= j) : (i < h || h <= j);
    if (!stays) {
      map[i] = map[j];
      map[j].key = kEmptyKey;
      map[j].val = -1;
      i = j;
    }
  }
}

__global__ void k_entry_flags(const HEntry* __restrict__ map, int64_t cap, uint8_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cap; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == cap) ? (map[i].val >= 0) : (map[i].key != kEmptyKey);
}

__global__ void k_entry_pairs(const HEntry* __restrict__ map, int64_t cap, const int64_t* __restrict__ idx, int64_t n,
                              const int64_t* __restrict__ ins_seq, int64_t* __restrict__ keys,
                              int64_t* __restrict__ slots, int64_t* __restrict__ seq) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx[j];
    HEntry e = map[i];
    keys[j] = i == cap ? kEmptyKey : e.key;
    slots[j] = e.val;
    seq[j] = ins_seq[e.val];
  }
}

__global__ void k_permute2(const int64_t* __restrict__ order, int64_t n, const int64_t* __restrict__ a,
                           const int64_t* __restrict__ b, int64_t* __restrict__ ao, int64_t* __restrict__ bo) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    ao[j] = a[order[j]];
    bo[j] = b[order[j]];
  }
}

__global__ void k_iota64(int64_t* p, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) p[j] = j;
}

// one thread per (row, 4-column chunk): the row's hash base once, no 64-bit
// division per element, a 16-byte store when D % 4 == 0
template <bool V4>
__global__ void __launch_bounds__(256) k_initial_rows(const int64_t* __restrict__ ids, int64_t n, int D,
                                                      uint64_t seed_mix, double scale, float* __restrict__ out) {
  const int chunks = (D + 3) >> 2;
  const int64_t total = n * chunks;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / chunks;
    const int c0 = (int)(t - i * chunks) * 4;
    const uint64_t base = mix64((uint64_t)__ldg(ids + i) ^ seed_mix);
    float* row = out + i * D;
    if (V4) {
      float4 v = make_float4(init_value(base, c0, scale), init_value(base, c0 + 1, scale),
                             init_value(base, c0 + 2, scale), init_value(base, c0 + 3, scale));
      __stcs(reinterpret_cast<float4*>(row + c0), v);
    } else {
      for (int c = c0; c < c0 + 4 && c < D; ++c) row[c] = init_value(base, c, scale);
    }
  }
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_initial_rows(int64_t seed, const int64_t* ids, int64_t n, int64_t dim, float* out, void* stream) {
  SKB_API_BEGIN
  if (dim < 1) raise(SKB_E_VALUE, dim, "dim must be >= 1");
  if (n <= 0) return SKB_OK;
  const int64_t total = n * ((dim + 3) / 4);
  const double scale = 1.0 / std::sqrt((double)dim);
  if (dim % 4 == 0 && (uintptr_t)out % 16 == 0)
    k_initial_rows<true><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(ids, n, (int)dim, mix64((uint64_t)seed),
                                                                              scale, out);
  else
    k_initial_rows<false><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(ids, n, (int)dim,
                                                                               mix64((uint64_t)seed), scale, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_table_create(int64_t dim, int64_t seed, int64_t block_size, int64_t evict_threshold, int64_t capacity_hint,
                     skb_table_t* out_host) {
  SKB_API_BEGIN
  if (dim < 1 || block_size < 1) raise(SKB_E_VALUE, dim, "dim and block_size must be >= 1");
  Table* t = new Table();
  t->dim = dim;
  t->seed = seed;
  t->block_size = block_size;
  t->evict_threshold = evict_threshold;
  SKB_CUDA(cudaGetDevice(&t->device));
  t->init_scale = 1.0 / std::sqrt((double)dim);
  t->seed_mix = mix64((uint64_t)seed);
  cudaStream_t s = nullptr;
  SKB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  SKB_CUDA(cudaMallocHost(&t->snap_host, sizeof(int64_t) * C_N));
  SKB_CUDA(cudaEventCreateWithFlags(&t->snap_ev, cudaEventDisableTiming));
  SKB_CUDA(cudaMalloc(&t->counters, sizeof(int64_t) * C_N));
  SKB_CUDA(cudaMemsetAsync(t->counters, 0, sizeof(int64_t) * C_N, s));
  SKB_CUDA(cudaMalloc(&t->dflags, sizeof(unsigned long long) * 4));
  SKB_CUDA(cudaMemsetAsync(t->dflags, 0xFF, sizeof(unsigned long long) * 4, s));
  SKB_CUDA(cudaMallocHost(&t->hflags, sizeof(int64_t) * 4));
  int64_t rows = capacity_hint > 1024 ? capacity_hint : 1024;
  t->vmm = vmm_available();
  t->rows_hint = capacity_hint;
  // The hint's rows are mapped (VMM) or allocated now: creating physical
  // memory inside a step costs driver calls that can stall the process for
  // 20-200 ms when the driver scrubs reused memory (C3 growth runs); past the
  // hint the arena grows copy-free.  The IDMap is sized for the hint either
  // way (no rehash while growing to it).
  grow_arena(t, rows, s);
  rehash(t, next_pow2(rows * 2 > 2048 ? rows * 2 : 2048), s);
  SKB_CUDA(cudaStreamSynchronize(s));
  SKB_CUDA(cudaStreamDestroy(s));
  *out_host = reinterpret_cast<skb_table_t>(t);
  SKB_API_END
}

int skb_table_destroy(skb_table_t h) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  if (getenv("SKB_DEBUG_SYNC"))
    fprintf(stderr, "[skb] snapshot waits %lld, counter refreshes %lld, arena growths %lld (all tables so far)\n",
            (long long)g_snap_waits.load(), (long long)g_refreshes.load(), (long long)g_growths.load());
  SKB_CUDA(cudaDeviceSynchronize());
  if (t->va_prep.joinable()) t->va_prep.join();
  if (t->vmm) {
    for (auto& a : t->va) vmm_free(a);
  } else {
    cudaFree(t->arena);
    cudaFree(t->last_step);
    cudaFree(t->live);
    cudaFree(t->slot_key);
    cudaFree(t->ins_seq);
    cudaFree(t->free_list);
  }
  cudaFree(t->idmap);
  cudaFree(t->counters);
  cudaFree(t->dflags);
  cudaFree(t->bitmap);
  cudaFreeHost(t->hflags);
  cudaFreeHost(t->snap_host);
  cudaEventDestroy(t->snap_ev);
  if (t->fused) fused_ctx_destroy(t->fused);
  delete t;
  SKB_API_END
}

int skb_table_stats(skb_table_t h, int64_t* stats_host, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  table_refresh(t, as_stream(stream));
  stats_host[0] = t->known[C_ROWS];
  stats_host[1] = t->known[C_ALLOC];
  stats_host[2] = t->known[C_FREE];
  stats_host[3] = reported_capacity(t);
  stats_host[4] = t->arena_rows;
  stats_host[5] = t->idmap_cap;
  SKB_API_END
}

int skb_table_lookup_or_insert(skb_table_t h, const int64_t* ids, int64_t n, int64_t step, int64_t* offsets_out,
                               void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  if (has_duplicate(ids, n, s)) raise(SKB_E_VALUE, 0, "lookup_or_insert requires duplicate-free ids");
  table_admit(t, ids, n, step, offsets_out, s);
  SKB_API_END
}

int skb_table_admit_unique(skb_table_t h, const int64_t* ids, int64_t n, int64_t step, int64_t* offsets_out,
                           void* stream) {
  SKB_API_BEGIN
  if (n <= 0) return SKB_OK;
  table_admit(table_from(h), ids, n, step, offsets_out, as_stream(stream));
  SKB_API_END
}

int skb_table_gather_unchecked(skb_table_t h, const int64_t* offsets, int64_t n, float* rows_out, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  if (n <= 0) return SKB_OK;
  const int D = (int)t->dim;
  launch_rows_gather(IdxArray{offsets}, t->arena, 3 * D, rows_out, D, n, D, as_stream(stream));
  SKB_API_END
}

int skb_sparse_adam_step_unchecked(skb_table_t h, const int64_t* offsets, int64_t n, const float* grads,
                                   const skb_adam_t* scalars_host, void* stream) {
  SKB_API_BEGIN
  if (n <= 0) return SKB_OK;
  table_adam(table_from(h), offsets, n, grads, *scalars_host, as_stream(stream));
  SKB_API_END
}

int skb_table_gather(skb_table_t h, const int64_t* offsets, int64_t n, float* rows_out, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  const int D = (int)t->dim;
  launch_rows_gather_checked(IdxArray{offsets}, t->arena, 3 * D, rows_out, D, n, D, t->live, t->arena_rows,
                             t->dflags, s);
  const int64_t bad = flags_fetch(t, s)[0];
  if ((uint64_t)bad != kNoFlag) {
    flags_rearm(t, s);
    const int64_t o = read_i64(offsets + bad, s);
    raise(SKB_E_INDEX, o, "gather: offset %lld is not a live slot", (long long)o);
  }
  SKB_API_END
}

int skb_table_gather_deferred(skb_table_t h, const int64_t* offsets, int64_t n, float* rows_out, int64_t* flags_dev,
                              void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  if (!flags_dev) raise(SKB_E_ARG, 0, "gather_deferred: flags_dev is null");
  if (n <= 0) return SKB_OK;
  const int D = (int)t->dim;
  launch_rows_gather_checked(IdxArray{offsets}, t->arena, 3 * D, rows_out, D, n, D, t->live, t->arena_rows,
                             reinterpret_cast<unsigned long long*>(flags_dev), as_stream(stream));
  SKB_API_END
}

int skb_table_scatter_update_deferred(skb_table_t h, const int64_t* offsets, int64_t n, const float* rows,
                                      int64_t* flags_dev, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (!flags_dev) raise(SKB_E_ARG, 0, "scatter_update_deferred: flags_dev is null");
  if (n <= 0) return SKB_OK;
  fused_require_quiet(t, true, "scatter_update");
  ensure_bitmap(t, s);
  auto* f = reinterpret_cast<unsigned long long*>(flags_dev);
  const bool v4 = t->dim % 4 == 0 && (uintptr_t)rows % 16 == 0;
  if (v4) launch_checked_scatter<4, 0>(t, offsets, n, rows, t->arena, s, f);
  else launch_checked_scatter<1, 0>(t, offsets, n, rows, t->arena, s, f);
  SKB_API_END
}

int skb_table_scatter_update(skb_table_t h, const int64_t* offsets, int64_t n, const float* rows, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  checked_scatter_update(t, offsets, n, rows, s);
  SKB_API_END
}

int skb_table_evict(skb_table_t h, int64_t current_step, int64_t* n_evicted_host, void* stream) {
  SKB_API_BEGIN
  *n_evicted_host = table_evict(table_from(h), current_step, as_stream(stream));
  SKB_API_END
}

int skb_table_export(skb_table_t h, int64_t* ids, float* w, float* m, float* v, int64_t* last_step, int64_t capacity,
                     int64_t* n_out_host, void* stream) {
  SKB_API_BEGIN
  *n_out_host = table_export(table_from(h), ids, w, m, v, last_step, capacity, as_stream(stream));
  SKB_API_END
}

int skb_table_restore(skb_table_t h, const int64_t* ids, int64_t n, const float* w, const float* m, const float* v,
                      const int64_t* last_step, void* stream) {
  SKB_API_BEGIN
  table_restore(table_from(h), ids, n, w, m, v, last_step, as_stream(stream));
  SKB_API_END
}

int skb_table_read_rows(skb_table_t h, const int64_t* offsets, int64_t n, int32_t which, float* out, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (which < 0 || which > 2) raise(SKB_E_ARG, which, "which must be 0 (w), 1 (m) or 2 (v)");
  if (n <= 0) return SKB_OK;
  check_range(t, offsets, n, s);
  const int D = (int)t->dim;
  launch_rows_gather(IdxArray{offsets}, t->arena + which * D, 3 * D, out, D, n, D, s);
  SKB_API_END
}

int skb_table_write_rows(skb_table_t h, const int64_t* offsets, int64_t n, int32_t which, const float* rows,
                         void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (which < 0 || which > 2) raise(SKB_E_ARG, which, "which must be 0 (w), 1 (m) or 2 (v)");
  if (n <= 0) return SKB_OK;
  checked_write(t, offsets, n, which, rows, s);
  SKB_API_END
}

int skb_table_read_last_step(skb_table_t h, const int64_t* offsets, int64_t n, int64_t* out, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  check_range(t, offsets, n, s);
  k_gather_i64<<<grid_for(n, 256), 256, 0, s>>>(t->last_step, offsets, n, out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_table_write_last_step(skb_table_t h, const int64_t* offsets, int64_t n, const int64_t* vals, int64_t scalar,
                              void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  check_range(t, offsets, n, s);
  k_write_last<<<grid_for(n, 256), 256, 0, s>>>(offsets, n, vals, scalar, t->last_step);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_table_clear_aux(skb_table_t h, const int64_t* offsets, int64_t n, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  check_range(t, offsets, n, s);
  k_clear_aux<<<grid_for(n * t->dim, 256), 256, 0, s>>>(offsets, n, (int)t->dim, t->arena, t->last_step);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_table_ensure_capacity(skb_table_t h, int64_t slots, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (slots > t->ensured_slots) t->ensured_slots = slots;
  int64_t want = (slots + t->block_size - 1) / t->block_size * t->block_size;
  if (want > t->arena_rows) grow_arena(t, want, s);
  SKB_API_END
}

int skb_table_idmap_get(skb_table_t h, const int64_t* ids, int64_t n, int64_t* slots_out, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  k_idmap_get<<<grid_for(n, 256), 256, 0, s>>>(ids, n, t->idmap, (uint64_t)(t->idmap_cap - 1), t->idmap_cap,
                                              slots_out);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_table_idmap_put(skb_table_t h, int64_t id, int64_t slot, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (slot < 0) raise(SKB_E_VALUE, slot, "slot must be >= 0");
  fused_require_quiet(t, false, "IDMap.put");
  table_reserve(t, 1, s);
  if (slot >= t->arena_rows) grow_arena(t, slot + 1, s);
  k_idmap_put<<<1, 1, 0, s>>>(t->idmap, (uint64_t)(t->idmap_cap - 1), t->idmap_cap, id, slot, t->counters,
                              t->ins_seq);
  SKB_LAUNCH_CHECK();
  table_refresh(t, s);
  SKB_API_END
}

int skb_table_idmap_remove(skb_table_t h, int64_t id, int64_t* slot_out_host, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  fused_require_quiet(t, false, "IDMap.remove");
  fused_flush_pending(t, s);
  Scratch out(sizeof(int64_t), s);
  k_idmap_remove<<<1, 1, 0, s>>>(t->idmap, (uint64_t)(t->idmap_cap - 1), t->idmap_cap, id, t->counters,
                                 out.as<int64_t>());
  SKB_LAUNCH_CHECK();
  int64_t slot = read_i64(out.as<int64_t>(), s);
  table_refresh(t, s);
  if (slot < 0) raise(SKB_E_KEY, id, "%lld", (long long)id);
  *slot_out_host = slot;
  SKB_API_END
}

int skb_table_free_list(skb_table_t h, int64_t* out, int64_t capacity, int64_t* n_out_host, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  table_refresh(t, s);
  int64_t F = t->known[C_FREE];
  if (F > capacity) raise(SKB_E_ARG, F, "free list has %lld entries, buffer holds %lld", (long long)F,
                          (long long)capacity);
  if (F) SKB_CUDA(cudaMemcpyAsync(out, t->free_list, sizeof(int64_t) * F, cudaMemcpyDeviceToDevice, s));
  *n_out_host = F;
  SKB_API_END
}

int skb_table_set_free_list(skb_table_t h, const int64_t* slots, int64_t n, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n < 0) raise(SKB_E_VALUE, n, "free list length must be >= 0");
  fused_require_quiet(t, false, "free_list mutation");
  fused_flush_pending(t, s);
  if (n > 0) {
    DevFlag f(s);
    k_range_flag<<<grid_for(n, 256), 256, 0, s>>>(slots, n, t->arena_rows, f.ptr());
    SKB_LAUNCH_CHECK();
    const int64_t bad = f.read();
    if (bad >= 0) {
      const int64_t o = read_i64(slots + bad, s);
      raise(SKB_E_VALUE, o, "free_list: slot %lld is outside the store (%lld rows)", (long long)o,
            (long long)t->arena_rows);
    }
    SKB_CUDA(cudaMemcpyAsync(t->free_list, slots, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, s));
  }
  k_set_i64<<<1, 1, 0, s>>>(t->counters + C_FREE, n);
  SKB_LAUNCH_CHECK();
  table_refresh(t, s);
  SKB_API_END
}

int skb_table_items(skb_table_t h, int64_t* ids, int64_t* slots, int64_t capacity, int64_t* n_out_host,
                    void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  const int64_t cap = t->idmap_cap;
  Scratch flags(cap + 1, s), idx(sizeof(int64_t) * (cap + 1), s), cnt(sizeof(int64_t), s);
  k_entry_flags<<<grid_for(cap + 1, 256), 256, 0, s>>>(t->idmap, cap, flags.as<uint8_t>());
  SKB_LAUNCH_CHECK();
  select_flagged_index(flags.as<uint8_t>(), cap + 1, idx.as<int64_t>(), cnt.as<int64_t>(), s);
  int64_t n = read_i64(cnt.as<int64_t>(), s);
  if (n > capacity) raise(SKB_E_ARG, n, "items buffer too small");
  *n_out_host = n;
  if (n == 0) return SKB_OK;
  Scratch k(8 * n, s), sl(8 * n, s), sq(8 * n, s), sq2(8 * n, s), ord(8 * n, s), ord2(8 * n, s);
  k_entry_pairs<<<grid_for(n, 256), 256, 0, s>>>(t->idmap, cap, idx.as<int64_t>(), n, t->ins_seq, k.as<int64_t>(),
                                                sl.as<int64_t>(), sq.as<int64_t>());
  SKB_LAUNCH_CHECK();
  k_iota64<<<grid_for(n, 256), 256, 0, s>>>(ord.as<int64_t>(), n);
  SKB_LAUNCH_CHECK();
  sort_pairs_i64(sq.as<int64_t>(), sq2.as<int64_t>(), ord.as<int64_t>(), ord2.as<int64_t>(), n, s);
  k_permute2<<<grid_for(n, 256), 256, 0, s>>>(ord2.as<int64_t>(), n, k.as<int64_t>(), sl.as<int64_t>(), ids, slots);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_sparse_adam_step(skb_table_t h, const int64_t* offsets, int64_t n, const float* grads,
                         const skb_adam_t* scalars_host, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return SKB_OK;
  check_adam_offsets(t, offsets, n, s);
  table_adam(t, offsets, n, grads, *scalars_host, s);
  SKB_API_END
}

}  // extern "C"
