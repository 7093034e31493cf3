/*
 * sparsekit_b200.h — C ABI of libsparsekit_b200.so, the B200 (sm_100a) native
 * implementation of the RecIS dynamic-embedding hot path.
 *
 * The reference (`sparsekit`, /root/reference/pkg/src/sparsekit) is a Python
 * package with no FFI; each entry point below names the reference function it
 * replaces (file:line).  The Python package `paper_2509_20883_b200` binds these
 * with ctypes and keeps the reference's Python API on top.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    unless the parameter name ends in `_host`.  Sizes are int64_t.
 *  - `stream` is a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 *    work is stream-ordered.  Calls that must report a data-dependent error
 *    (ValueError / IndexError in the reference) synchronize `stream` once.
 *  - Return value: SKB_OK or an SKB_E_* status; skb_last_error() gives the
 *    thread-local message and skb_last_error_arg() the offending value (first
 *    bad offset, duplicate id, ...).  The Python layer maps SKB_E_VALUE ->
 *    ValueError, SKB_E_INDEX -> IndexError, SKB_E_KEY -> KeyError.
 *  - Floating point rows/state are float32; ids/offsets/steps are int64.
 *  - A table handle is single-writer: one stream at a time may mutate it
 *    (embedding.py:10-11).  Distinct handles may run concurrently.
 */
#ifndef SPARSEKIT_B200_H
#define SPARSEKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKB_OK 0
#define SKB_E_VALUE 1       /* reference raises ValueError  */
#define SKB_E_INDEX 2       /* reference raises IndexError  */
#define SKB_E_KEY 3         /* reference raises KeyError    */
#define SKB_E_CUDA 4        /* CUDA runtime failure          */
#define SKB_E_NOMEM 5       /* device allocation failure     */
#define SKB_E_ARG 6         /* bad argument at the C boundary */
#define SKB_E_UNSUPPORTED 7
#define SKB_E_IO 8          /* reference raises ColumnIOError */

typedef struct skb_table* skb_table_t;
typedef struct skb_dist* skb_dist_t;  /* requester context of the multi-GPU step (dist.cu) */

/* Host-computed float32 Adam scalars, exactly as optim.py:69-75 forms them
 * (bias corrections use Python double pow, then round to float32). */
typedef struct {
  float lr, beta1, beta2, eps;
  float one_minus_beta1, one_minus_beta2; /* float32(1) - float32(beta) */
  float bc1, bc2;                         /* float32(1 - beta**t)       */
  float lr_wd;                            /* float32(lr) * float32(wd)  */
  int32_t decoupled_decay;                /* variant == adamw and wd != 0 */
} skb_adam_t;

/* ---- library ---------------------------------------------------------- */
const char* skb_version(void);
const char* skb_last_error(void);
int64_t skb_last_error_arg(void);
int skb_device_sm_count(int device, int* out_host);
/* number of this library's kernel launches so far (process-wide) */
int64_t skb_launch_count(void);
/* stream-ordered copy between any two addresses (device, pinned host, IPC) */
int skb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* ---- L0 hashing: hashing.py:35-40, sharding.py:41-43, sharding.py:170-178 */
/* out[i] = int64(mix64(u64(ids[i])))                       hashing.py:35-40 */
int skb_mix64(const int64_t* ids, int64_t n, int64_t* out, void* stream);
/* out[i] = mix64(ids[i]) % S  (unsigned)        ShardPlan.shard_of sharding.py:41-43 */
int skb_shard_of(const int64_t* ids, int64_t n, int64_t num_shards, int64_t* out, void* stream);
/* out[i] = int64(mix64(u64(ids[i]) ^ salt))     LogicalTable.keys_for sharding.py:170-178 */
int skb_keys_for(const int64_t* ids, int64_t n, uint64_t salt, int64_t* out, void* stream);
/* FNV-1a 64 of one host byte string (member salts)           hashing.py:43-48 */
uint64_t skb_fnv1a64_host(const uint8_t* bytes_host, int64_t len);
/* out[i] = FNV-1a64(blob[offs[i]:offs[i+1]]) as int64   fnv1a64_batch hashing.py:51-71,
 * hash_feature features.py:30-38 */
int skb_fnv1a64_strings(const uint8_t* blob, const int64_t* str_offs, int64_t n, int64_t* out,
                        void* stream);
/* out[i] = FNV-1a64(LE8(x[i]) || LE8(y[i]))                fnv1a64_pairs hashing.py:74-86 */
int skb_fnv1a64_pairs(const int64_t* x, const int64_t* y, int64_t n, int64_t* out, void* stream);

/* ---- L3 dedup + owner partition: unique_partition sharding.py:74-100 ---- */
/* uniq_out[n]: per-shard unique ids in global first-occurrence order, shard 0
 * first, then shard 1, ...; shard_counts_out[S] (device) their counts;
 * inv_shard[n], inv_pos[n] the inverse routing index (PartitionResult). */
int skb_unique_partition(const int64_t* ids, int64_t n, int64_t num_shards, int64_t* uniq_out,
                         int64_t* shard_counts_out, int64_t* inv_shard, int64_t* inv_pos,
                         void* stream);
/* counts_out[S] (device): unique ids owned by each shard — load_stats
 * sharding.py:103-119 without materialising the partition */
int skb_shard_unique_counts(const int64_t* ids, int64_t n, int64_t num_shards, int64_t* counts_out,
                            void* stream);
/* out[i,:] = rows_cat[shard_base[inv_shard[i]] + inv_pos[i], :]
 *                                          PartitionResult.restore sharding.py:58-66 */
int skb_partition_restore(const float* rows_cat, int64_t dim, const int64_t* shard_base,
                          const int64_t* inv_shard, const int64_t* inv_pos, int64_t n, float* out,
                          void* stream);

/* ---- L2 dynamic embedding table: EmbeddingTable embedding.py:151-308 --- */
/* EmbeddingTable(name, dim, seed, block_size, evict_threshold) embedding.py:157-171;
 * evict_threshold < 0 means None.  capacity_hint pre-sizes the row arena. */
int skb_table_create(int64_t dim, int64_t seed, int64_t block_size, int64_t evict_threshold,
                     int64_t capacity_hint, skb_table_t* out_host);
/* initial_rows embedding.py:24-36: out[n, dim] float32, keyed by (seed, id, column) */
int skb_initial_rows(int64_t seed, const int64_t* ids, int64_t n, int64_t dim, float* out,
                     void* stream);
int skb_table_destroy(skb_table_t t);
/* stats_host[0..5] = {num_rows (len(idmap)), allocated, free_count,
 *   capacity (block-granular, BlockStore.capacity embedding.py:83-85),
 *   arena_rows (physical rows reserved), idmap_capacity}.  Synchronizes. */
int skb_table_stats(skb_table_t t, int64_t* stats_host, void* stream);
/* lookup_or_insert embedding.py:185-223: offsets_out[i] = slot of ids[i];
 * unknown ids are admitted in input order (free list LIFO, then sequential),
 * initialised with initial_rows (embedding.py:24-36), zero m/v; last_step of
 * every returned slot = step.  Duplicate ids -> SKB_E_VALUE. */
int skb_table_lookup_or_insert(skb_table_t t, const int64_t* ids, int64_t n, int64_t step,
                               int64_t* offsets_out, void* stream);
/* Trusted variant for callers whose ids are unique by construction
 * (unique_partition output, all_to_all_lookup sharding.py:248-251): no
 * duplicate check, no synchronization. */
int skb_table_admit_unique(skb_table_t t, const int64_t* ids, int64_t n, int64_t step,
                           int64_t* offsets_out, void* stream);
/* Trusted gather / Adam for offsets produced by admission on the same stream
 * (all_to_all_lookup / all_to_all_grad_update inner steps): no checks, no sync. */
int skb_table_gather_unchecked(skb_table_t t, const int64_t* offsets, int64_t n, float* rows_out,
                               void* stream);
int skb_sparse_adam_step_unchecked(skb_table_t t, const int64_t* offsets, int64_t n,
                                   const float* grads, const skb_adam_t* scalars_host, void* stream);
/* gather embedding.py:233-238 (liveness checked -> SKB_E_INDEX, arg = first bad offset) */
int skb_table_gather(skb_table_t t, const int64_t* offsets, int64_t n, float* rows_out,
                     void* stream);
/* scatter_update embedding.py:240-250 (distinct -> SKB_E_VALUE, live -> SKB_E_INDEX) */
int skb_table_scatter_update(skb_table_t t, const int64_t* offsets, int64_t n, const float* rows,
                             void* stream);
/* The same two checked operators with the check recorded on the device
 * instead of read back (deferred_checks(), no synchronization): flags_dev is
 * a caller-owned int64[4] preset to -1 (all ones); the first failing input
 * index is atomically lowered into it — gather: [0] = not a live slot;
 * scatter_update: [0] = duplicate, [1] = not live / out of range, [2] = an
 * out-of-range offset (distinctness then re-checked by the caller).  The
 * scatter writes nothing unless every check passed (read on the device). */
int skb_table_gather_deferred(skb_table_t t, const int64_t* offsets, int64_t n, float* rows_out,
                              int64_t* flags_dev, void* stream);
int skb_table_scatter_update_deferred(skb_table_t t, const int64_t* offsets, int64_t n, const float* rows,
                                      int64_t* flags_dev, void* stream);
/* evict embedding.py:252-274: stale slots join the free list in insertion order */
int skb_table_evict(skb_table_t t, int64_t current_step, int64_t* n_evicted_host, void* stream);
/* export_rows embedding.py:276-284 into caller buffers of >= num_rows entries,
 * rows sorted by id; n_out_host receives the row count. */
int skb_table_export(skb_table_t t, int64_t* ids, float* w, float* m, float* v, int64_t* last_step,
                     int64_t capacity, int64_t* n_out_host, void* stream);
/* restore_rows embedding.py:286-308 (id already present -> SKB_E_VALUE, arg = id) */
int skb_table_restore(skb_table_t t, const int64_t* ids, int64_t n, const float* w, const float* m,
                      const float* v, const int64_t* last_step, void* stream);
/* BlockStore row/state access by slot (no liveness check), which: 0=w,1=m,2=v
 *   read / read_state embedding.py:113-126, write / write_state embedding.py:117-131 */
int skb_table_read_rows(skb_table_t t, const int64_t* offsets, int64_t n, int32_t which, float* out,
                        void* stream);
int skb_table_write_rows(skb_table_t t, const int64_t* offsets, int64_t n, int32_t which,
                         const float* rows, void* stream);
/* read_last_step / write_last_step embedding.py:133-140 (vals == NULL -> scalar) */
int skb_table_read_last_step(skb_table_t t, const int64_t* offsets, int64_t n, int64_t* out,
                             void* stream);
int skb_table_write_last_step(skb_table_t t, const int64_t* offsets, int64_t n,
                              const int64_t* vals, int64_t scalar, void* stream);
/* clear_aux embedding.py:142-148 */
int skb_table_clear_aux(skb_table_t t, const int64_t* offsets, int64_t n, void* stream);
/* BlockStore.ensure_capacity embedding.py:87-92 (block-granular) */
int skb_table_ensure_capacity(skb_table_t t, int64_t slots, void* stream);
/* IDMap embedding.py:39-61: get (slot or -1), put, remove (-> SKB_E_KEY), free list */
int skb_table_idmap_get(skb_table_t t, const int64_t* ids, int64_t n, int64_t* slots_out,
                        void* stream);
int skb_table_idmap_put(skb_table_t t, int64_t id, int64_t slot, void* stream);
int skb_table_idmap_remove(skb_table_t t, int64_t id, int64_t* slot_out_host, void* stream);
/* free_list copy (bottom .. top), n_out_host <= capacity */
int skb_table_free_list(skb_table_t t, int64_t* out, int64_t capacity, int64_t* n_out_host,
                        void* stream);
/* IDMap.free_list mutation (embedding.py:46: a plain mutable list): replace the
 * free list with slots[0..n) (bottom .. top, device int64); every slot must be
 * in [0, arena rows) -> SKB_E_VALUE otherwise */
int skb_table_set_free_list(skb_table_t t, const int64_t* slots, int64_t n, void* stream);
/* items(): (id, slot) pairs in dict insertion order */
int skb_table_items(skb_table_t t, int64_t* ids, int64_t* slots, int64_t capacity,
                    int64_t* n_out_host, void* stream);

/* ---- L2 sparse optimizer: sparse_adam_step optim.py:42-83 --------------- */
/* distinct offsets (else SKB_E_VALUE); grads [n, dim]; one lazy Adam/AdamW step */
int skb_sparse_adam_step(skb_table_t t, const int64_t* offsets, int64_t n, const float* grads,
                         const skb_adam_t* scalars_host, void* stream);

/* ---- L2 ragged pooling: segments.py:61-116 ------------------------------ */
/* strategy: 0 = sequential (np.add.reduceat: first + numpy pairwise),
 *           1 = scatter (np.add.at left fold from +0); mode: 0 = sum, 1 = mean.
 * offsets must be valid (see skb_validate_offsets).          segment_reduce */
int skb_segment_reduce(const float* rows, int64_t n, int64_t dim, const int64_t* offsets,
                       int64_t num_segments, int32_t mode, int32_t strategy, float* out,
                       void* stream);
/* segment_tile segments.py:94-116 -> out [num_segments, k*dim] */
int skb_segment_tile(const float* rows, int64_t n, int64_t dim, const int64_t* offsets,
                     int64_t num_segments, int64_t k, float pad, float* out, void* stream);
/* Other row dtypes (the reference's output dtype follows its input,
 * segments.py:51-58, 103-116).  float64: the same fold orders in double.
 * int64 (any integer input widened): wrapping sum, order-free.  tile_x64: a
 * bit copy of 8-byte elements (float64 or int64) with the pad as raw bits. */
int skb_segment_reduce_f64(const double* rows, int64_t n, int64_t dim, const int64_t* offsets,
                           int64_t num_segments, int32_t mode, int32_t strategy, double* out,
                           void* stream);
int skb_segment_sum_i64(const int64_t* rows, int64_t n, int64_t dim, const int64_t* offsets,
                        int64_t num_segments, int64_t* out, void* stream);
int skb_segment_tile_x64(const void* rows, int64_t n, int64_t dim, const int64_t* offsets,
                         int64_t num_segments, int64_t k, uint64_t pad_bits, void* out, void* stream);
/* _check_segments segments.py:25-33 / _check_offsets ragged.py:32-42 on device:
 * SKB_E_VALUE if offsets[0] != 0, decreasing, or offsets[len-1] != n_expected */
int skb_validate_offsets(const int64_t* offsets, int64_t len, int64_t n_expected, void* stream);
/* np.add.at(g, inverse, grads) left fold by unique index (sharding.py:283-290) */
int skb_grad_fold(const float* grads, int64_t n, int64_t dim, const int64_t* inverse,
                  int64_t num_unique, float* out, void* stream);

/* ---- fused step (request-merged logical table; SURVEY §8b additions) ----
 * Forward = keys_for + unique/admission (lookup_or_insert order) + gather +
 * pooling of every bag, one logical table, one call.  The per-position grads
 * of the reference pipeline (train.py:181-186) are dpooled[bag] (sum) or
 * dpooled[bag] / float32(len) (mean); backward folds them per unique row in
 * input order and applies Adam/AdamW — bit-identical to
 * all_to_all_lookup + segment_reduce + all_to_all_grad_update on S = 1.
 *   ids[N]           raw feature ids, members concatenated (train.py:137-140)
 *   member_pos[F+1]  (host) position range of each member
 *   salts[F]         (host) fnv1a64(member) salts (namespaced) — ignored if !namespaced
 *   bag_offs[G+1]    (device) bag offsets over positions (members' bags concatenated)
 *   member_bag[F+1]  (host) bag range of each member
 *   mode             0 sum / 1 mean; strategy per member: 0 sequential / 1 scatter */
int skb_fused_forward(skb_table_t t, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                      const uint64_t* salts_host, int32_t num_members, int32_t namespaced,
                      const int64_t* bag_offs, int64_t num_bags, const int64_t* member_bag_host,
                      const int32_t* strategy_host, int32_t mode, int64_t step, float* pooled_out,
                      void* stream);
/* Index phase only (probe, admission, sort) of a batch, enqueued on the
 * table's internal index stream after `stream`'s pending work: prefetching
 * batch k+1 before the backward of batch k overlaps its index work with the
 * fold+Adam of step k (at most two batches in flight).  The following
 * skb_fused_forward with the same arguments pools it.  Table edits that would
 * move the prefetched batch's slots (evict, restore, IDMap put / remove /
 * free list, scatter_update) fail with SKB_E_VALUE until it is pooled. */
int skb_fused_prepare(skb_table_t t, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                      const uint64_t* salts_host, int32_t num_members, int32_t namespaced,
                      const int64_t* bag_offs, int64_t num_bags, const int64_t* member_bag_host,
                      const int32_t* strategy_host, int32_t mode, int64_t step, void* stream);
/* Tile combiner (segment_tile, segments.py:94-116) on the fused path: the
 * forward writes tiles_out[G, k*dim] (the first min(len, k) rows of each bag,
 * `pad` after them); skb_fused_backward then takes dtiles [G, k*dim] and
 * folds each position's tile row (zero past k) in position order before
 * SparseAdam/AdamW — identical to segment_tile + the per-position gradient
 * expansion + all_to_all_grad_update.  Same prefetch rules as above. */
int skb_fused_prepare_tile(skb_table_t t, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                           const uint64_t* salts_host, int32_t num_members, int32_t namespaced,
                           const int64_t* bag_offs, int64_t num_bags, const int64_t* member_bag_host, int64_t k,
                           float pad, int64_t step, void* stream);
int skb_fused_forward_tile(skb_table_t t, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                           const uint64_t* salts_host, int32_t num_members, int32_t namespaced,
                           const int64_t* bag_offs, int64_t num_bags, const int64_t* member_bag_host, int64_t k,
                           float pad, int64_t step, float* tiles_out, void* stream);
/* Backward of the oldest pooled, not yet backwarded fused batch. */
int skb_fused_backward(skb_table_t t, const float* dpooled, const skb_adam_t* scalars_host,
                       void* stream);
/* flags bit 0 (SKB_BWD_PRESCALED): dpooled already holds the per-position
 * gradient of each bag (e.g. train.py:181-186's float32(dpooled64 / len)),
 * folded as given even for mean bags — bit-exact with the reference's float64
 * per-row expansion. */
#define SKB_BWD_PRESCALED 1
int skb_fused_backward_ex(skb_table_t t, const float* dpooled, const skb_adam_t* scalars_host,
                          int32_t flags, void* stream);
/* load_stats (sharding.py:103-119) of the last prepared fused batch for a
 * plan of num_shards shards: per-shard counts of its unique keys (device
 * int64[num_shards], zeroed here; stream-ordered, no sync) — what train.py
 * computes every step (train.py:223-228), from the step's own sorted keys. */
int skb_fused_shard_counts(skb_table_t t, int64_t num_shards, int64_t* counts_out, void* stream);
/* Per-kernel CUDA-event timing of the fused step on its own stream:
 * skb_fused_profile arms max_steps records per phase (0 disables); phases
 * 0 probe, 1 miss path, 2 pool, 3 sort + run heads, 4 grad fold + Adam.
 * skb_fused_profile_read returns the recorded durations in milliseconds. */
int skb_fused_profile(skb_table_t t, int64_t max_steps, void* stream);
int skb_fused_profile_read(skb_table_t t, int32_t phase, float* ms_host, int64_t capacity,
                           int64_t* n_host);
/* Stream-ordered copy of the last completed fused step's counters
 * {misses, new rows, unique rows, 0} into pinned host memory (no sync).  Any
 * stream: the copy waits for that step's backward, and the next reuse of the
 * step's buffers waits for the copy (so a side stream keeps it off the
 * compute stream). */
int skb_fused_stats_async(skb_table_t t, int64_t* dst_pinned_host, void* stream);
/* Number of unique rows the last fused forward touched (synchronizes). */
int skb_fused_last_unique(skb_table_t t, int64_t* n_unique_host, int64_t* n_new_host, void* stream);

/* ---- building blocks of the multi-GPU step (distributed.py) ------------
 * members_dev: int64[F+1][4] = {first position, first bag, salt, strategy}
 * per member (strategy 0 sequential / 1 scatter); last row = {N, G, 0, 0}. */
/* out[i] = namespaced key of ids[i] for its member (keys_for, sharding.py:170-178) */
int skb_keys_members(const int64_t* ids, int64_t n, const int64_t* members_dev, int32_t num_members,
                     int64_t* out, void* stream);
/* pooled[g] = fold over positions p of bag g of rows[idx[p] * row_stride ...]
 * (segment_reduce semantics per member strategy, segments.py:61-91) */
int skb_pool_indexed(const float* rows, int64_t row_stride, const uint32_t* idx, const int64_t* bag_offs,
                     int64_t num_bags, const int64_t* members_dev, int32_t num_members,
                     int32_t any_sequential, int32_t mode, int64_t dim, float* out, void* stream);
/* out[u] = in-position-order fold from +0 of dpooled[bag(p)] (/len for mean)
 * over positions p with idx[p] == u  (np.add.at, sharding.py:283-290) */
int skb_fold_bags(const float* dpooled, int64_t dim, const uint32_t* idx, int64_t n, int64_t num_unique,
                  const int64_t* bag_offs, int64_t num_bags, int32_t mode, int64_t max_index, float* out,
                  void* stream);

/* ---- feature engine: features.py ---------------------------------------- */
/* bucketize / fused_bucketize features.py:41-53,165-177: columns concatenated,
 * col_offs[C+1], edges_cat with edge_offs[C+1]; NaN -> SKB_E_VALUE */
int skb_bucketize_multi(const float* values, const int64_t* col_offs, int64_t num_cols,
                        const float* edges_cat, const int64_t* edge_offs, int64_t* out,
                        int64_t n_total, void* stream);
/* Same, without the synchronous NaN check: the lowest index of a NaN input is
 * atomicMin-ed into *nan_flag (device, caller-initialised to ~0) for the
 * caller to read at its next synchronisation point (deferred ValueError). */
int skb_bucketize_multi_async(const float* values, const int64_t* col_offs, int64_t num_cols, const float* edges_cat,
                              const int64_t* edge_offs, int64_t* out, int64_t n_total, unsigned long long* nan_flag,
                              void* stream);
/* mod_transform / fused_mod features.py:56-62,180-189 (moduli > 0 checked on host) */
int skb_mod_multi(const int64_t* values, const int64_t* col_offs, int64_t num_cols,
                  const int64_t* moduli, int64_t* out, int64_t n_total, void* stream);
/* The same multi-column ops over a device table of per-column input
 * pointers (col_ptrs[c] holds col_offs[c+1] - col_offs[c] values): no
 * concatenation copy before the launch; the output stays concatenated.
 * nan_flag (optional device word, caller sets ~0): deferred NaN check. */
int skb_bucketize_cols(const float* const* col_ptrs, const int64_t* col_offs, int64_t num_cols,
                       const float* edges_cat, const int64_t* edge_offs, int64_t* out, int64_t n_total,
                       unsigned long long* nan_flag, void* stream);
int skb_mod_cols(const int64_t* const* col_ptrs, const int64_t* col_offs, int64_t num_cols,
                 const int64_t* moduli, int64_t* out, int64_t n_total, void* stream);
/* PackedBatch for the fused step: members' ids concatenated into ids_out[N]
 * and their bag offsets shifted by each member's first position into
 * bag_offs_out[G+1], in one launch (device tables of per-member pointers and
 * the member_pos / member_bag prefix arrays). */
int skb_pack_members(const int64_t* const* ids_ptrs, const int64_t* const* offs_ptrs, const int64_t* member_pos,
                     const int64_t* member_bag, int64_t num_members, int64_t n_total, int64_t num_bags,
                     int64_t* ids_out, int64_t* bag_offs_out, void* stream);
/* cross features.py:65-89: out_offs[rows+1] computed here; out sized by caller
 * from out_offs[rows] (use skb_cross_offsets first). */
int skb_cross_offsets(const int64_t* a_offs, const int64_t* b_offs, int64_t rows,
                      int64_t* out_offs, void* stream);
int skb_cross(const int64_t* a_vals, const int64_t* a_offs, const int64_t* b_vals,
              const int64_t* b_offs, int64_t rows, const int64_t* out_offs, int64_t total, int64_t* out,
              int64_t* size_flag, void* stream);
/* cross over many column pairs (features.cross_many) in two launches.
 * descs_dev: device array of npairs 80-byte descriptors
 *   { a_vals, a_offs, b_vals, b_offs, rows, out_offs[rows+1], total, out_base,
 *     size_flag (optional, caller sets -1), pad }  (all 8-byte fields);
 * skb_cross_offsets_many fills every pair's out_offs (and size_flag, as
 * skb_cross does); skb_cross_many writes every pair's products to
 * out[out_base .. out_base + total) (total = sum of the pairs' totals, <= 1024
 * pairs per launch). */
int skb_cross_offsets_many(const void* descs_dev, int64_t npairs, void* stream);
int skb_cross_many(const void* descs_dev, int64_t npairs, int64_t total, int64_t* out, void* stream);
/* size_flag (optional device int64, caller sets -1): set to the true product
 * count when `total` (a caller-supplied size, features.cross_many(sizes=))
 * differs from out_offs[rows]; positions past the true count are zeroed and
 * never read past the inputs */
/* RaggedTensor.truncate ragged.py:139-163: new offsets + element gather index */
int skb_ragged_truncate(const int64_t* offs, int64_t rows, int64_t max_len, int32_t tail,
                        int64_t* new_offs, int64_t* src_index, void* stream);

/* out[i] = src[idx[i]] for elements of elem_bytes (1, 4 or 8) — ragged value
 * selection (truncate ragged.py:139-163, row_ranges ragged.py:18-29) */
int skb_gather_elems(const void* src, int64_t elem_bytes, const int64_t* idx, int64_t n, void* out,
                     void* stream);
/* RaggedTensor.pad_to_dense ragged.py:165-188: dense [rows, max_len, width]
 * elements of elem_bytes*width bytes, pad pattern pad_host (elem_bytes bytes),
 * mask [rows, max_len] uint8.  Row longer than max_len -> SKB_E_VALUE. */
int skb_ragged_pad_dense(const void* values, int64_t elem_bytes, int64_t width, const int64_t* offs,
                         int64_t rows, int64_t max_len, const void* pad_host, void* out,
                         uint8_t* mask, void* stream);

/* Graph mode for the fused step: each phase's device work
 * (index phase / pool / fold+Adam) is captured as a CUDA graph on its second
 * call with an unchanged signature (buffers, sizes, table arrays) and replayed
 * with the step and Adam scalars patched in; growth re-primes.  Results are
 * identical to eager mode.  Default off (SKB_FUSED_GRAPHS=1 turns it on). */
/* Kernel variant of the fused step, per table (tuning sweeps and tests):
 * adam 0 = auto (TMA ring <16,192,4> for sum batches of D >= 48 without
 * recent long runs, else the register kernel), 1-3 register shapes, 4-8 TMA
 * ring shapes; pool 0 = auto (staged one-hot gather when n == G, else the
 * position-streaming kernel for 64 <= D <= 128), 1-5 forced register shapes
 * / staged; -1 = the SKB_ADAM_VARIANT / SKB_POOL_VARIANT environment default.
 * last_variants: what the last backward / pool ran (adam 0 = TMA default,
 * -1 = generic-D kernel; pool -1 generic-D, 6 streaming, 10 pairwise general). */
/* Fold mode of the fused backward's long runs (ids with > 32 positions in a
 * batch): 0 exact (default) — np.add.at's serial left fold, bit-exact with
 * sharding.py:283-290; 1 tree (opt-in tolerance mode) — chunks of 256
 * positions folded in parallel, then the chunk sums in order; error per
 * column <= (256 + len/256) * 2^-24 * sum|g| (SURVEY §7.3-5's normwise
 * bound).  Runs of <= 32 positions are exact in both modes. */
int skb_fused_set_fold_mode(skb_table_t t, int32_t mode);
int skb_fused_set_variants(skb_table_t t, int32_t adam_variant, int32_t pool_variant);
int skb_fused_last_variants(skb_table_t t, int32_t* adam_host, int32_t* pool_host);
int skb_fused_set_graphs(skb_table_t t, int32_t enable);

/* ---- checkpoint boundary (checkpoint.py:192-313) ------------------------ */
/* Stable ascending (signed) argsort of int64 keys: sorted_keys[i] =
 * keys[perm[i]] — the global key order of save_sharded (checkpoint.py:212-214,
 * np.argsort(ids, kind="stable")). */
int skb_argsort_i64(const int64_t* keys, int64_t n, int64_t* sorted_keys, int64_t* perm, void* stream);
/* Row moves of row_bytes (multiple of 4) bytes: gather out[i] = src[idx[i]]
 * (save: rows into key order), scatter out[idx[i]] = src[i] (load_sharded
 * re-routing rows to target shards, checkpoint.py:300-311). */
int skb_gather_rows(const void* src, int64_t row_bytes, const int64_t* idx, int64_t n, void* out, void* stream);
int skb_scatter_rows(const void* src, int64_t row_bytes, const int64_t* idx, int64_t n, void* out, void* stream);
/* dest[i] = shard_base[inv_shard[i]] + inv_pos[i]: position of input i in the
 * shard-grouped (stable) order of a unique_partition result */
int skb_partition_dest(const int64_t* shard_base, const int64_t* inv_shard, const int64_t* inv_pos, int64_t n,
                       int64_t* dest, void* stream);

/* ---- input side: columnar batch reader (columnio.py:328-409) ----------- */
typedef struct skb_reader_s* skb_reader_t;
/* chunks: [nchunks][5] int64 {path index, absolute byte offset, byte length,
 * rows, chunk index within its file} — this shard's chunks in global order
 * (the plan of columnio.py:306-325).  Columns in schema order: dtype 0 f32,
 * 1 i64, 2 bytes; ragged; selected (unselected columns are never decoded).
 * Batches of batch_rows rows (the last may be short) concatenate rows across
 * chunk boundaries; `threads` decoder threads, up to prefetch_depth batches
 * assembled ahead; pinned != 0: batch buffers are page-locked for `device`.
 * Decode / truncation errors -> SKB_E_IO with the reference's message. */
int skb_reader_open(const char* const* paths, int64_t npaths, const int64_t* chunks, int64_t nchunks,
                    const char* const* col_names, const int32_t* col_dtype, const int32_t* col_ragged,
                    const int32_t* col_selected, int64_t ncols, int64_t batch_rows, int64_t prefetch_depth,
                    int32_t threads, int32_t pinned, int32_t device, skb_reader_t* out);
/* advance to the next batch (blocks); *rows = 0 at the end.  The previous
 * batch's buffers are recycled. */
int skb_reader_next(skb_reader_t r, int64_t* rows);
/* selected column j of the current batch: row_offsets [rows+1] (int64),
 * values (n_values elements; for bytes columns the blob of blob_bytes bytes
 * with str_offsets [n_values+1]) — host pointers valid until the next call */
int skb_reader_column(skb_reader_t r, int64_t j, const int64_t** row_offsets, const void** values,
                      int64_t* n_values, const int64_t** str_offsets, int64_t* blob_bytes);
int skb_reader_close(skb_reader_t r);

/* ---- peer-memory transport of the row-sharded exchange ----
 * Replaces distributed.py's rows / grads all_to_all_v: the producing kernel
 * stores every row straight into the consuming rank's window (CUDA IPC
 * memory; NVLink P2P stores between GPUs).  Handles are 64-byte
 * cudaIpcMemHandle_t blobs, exchanged by the caller (all_gather). */
int skb_ipc_alloc(int64_t bytes, void** ptr_out, void* handle_out);
int skb_ipc_open(const void* handle, void** ptr_out);
int skb_ipc_close(void* ptr);
int skb_ipc_free(void* ptr);
/* owner side of the lookup: for the q-th id received (requester j = segment
 * of q in recv_prefix[0..R]), w row of slot slots_u[inv[q]] -> window_j at row
 * dst_base[j] + q - recv_prefix[j].  Device arrays: slots_u, inv,
 * recv_prefix, peer_windows (float*[R]), dst_base. */
int skb_p2p_send_rows(skb_table_t t, const int64_t* slots_u, const int64_t* inv, int64_t nrecv,
                      const int64_t* recv_prefix, int32_t num_ranks, float* const* peer_windows,
                      const int64_t* dst_base, void* stream);
/* requester side of the update: row i of rows[n, dim] (owner s = segment of i
 * in seg_prefix) -> window_s at row dst_base[s] + i - seg_prefix[s]. */
int skb_p2p_send_grads(const float* rows, int64_t dim, int64_t n, const int64_t* seg_prefix, int32_t num_ranks,
                       float* const* peer_windows, const int64_t* dst_base, void* stream);
/* Stream-ordered barrier over peer memory (no kernel, no host round trip, no
 * NCCL): epoch written into slot `rank` of every peer's int64[num_ranks] flag
 * window (cuStreamWriteValue64, behind a memory barrier), then the stream
 * waits until every slot of this rank's window reached `epoch`
 * (cuStreamWaitValue64).  flag_ptrs_host[j] = rank j's flag window as mapped
 * here.  memops_supported reports whether the driver exposes the ops. */
int skb_p2p_memops_supported(int32_t* supported_host);
int skb_p2p_barrier(const int64_t* flag_ptrs_host, int32_t num_ranks, int32_t rank, int64_t epoch,
                    void* stream);
/* counts[num_ranks] -> row `rank` of every peer's num_ranks x num_ranks count
 * matrix window (the all-gather of the multi-GPU step's per-owner counts). */
int skb_p2p_put_counts(const int64_t* counts, int32_t num_ranks, int32_t rank, int64_t* const* peer_windows,
                       void* stream);

/* ---- fused row-sharded multi-GPU step (replaces the exchange of
 * sharding.py:222-297 as driven by train.py:120-195).  One process per GPU.
 * Requester context: persistent buffers, no per-step allocation; every
 * transfer is a P2P store by the producing kernel into the consumer's IPC
 * window.  Per step (S ranks, this rank r):
 *   skb_dist_prepare      keys + unique_partition (reference order) + sort; counts[S] on device
 *   (caller)              all-gather counts -> C[q][j] on the host (the step's one sync)
 *   skb_dist_send_ids     uniq segment j -> owner j's id window at sum_{q<r} C[q][j]
 *   skb_fused_forward_send (owner) fused index phase of the received ids + row
 *                         gather stored into each requester q's row window
 *   skb_dist_pool         pooled[G, D] from this rank's row window
 *   skb_dist_fold_send    per-unique ordered fold of dpooled -> owner grad windows
 *   skb_fused_backward    (owner) rank-ordered fold of the grad window + Adam
 * Window layouts: id / grad window of owner j = every rank's segment for j,
 * rank-ordered; row window of requester q = q's unique list (owner order). */
int skb_dist_create(int64_t dim, int32_t num_ranks, skb_dist_t* out_host);
int skb_dist_destroy(skb_dist_t d);
int skb_dist_prepare(skb_dist_t d, const int64_t* ids, int64_t n, const int64_t* member_pos_host,
                     const uint64_t* salts_host, int32_t num_members, int32_t namespaced,
                     const int64_t* bag_offs, int64_t num_bags, const int64_t* member_bag_host,
                     const int32_t* strategy_host, int64_t* counts_out, void* stream);
int skb_dist_send_ids(skb_dist_t d, int64_t num_unique, const int64_t* seg_prefix,
                      int64_t* const* peer_windows, const int64_t* dst_base, void* stream);
int skb_dist_pool(skb_dist_t d, const float* rows, int32_t mode, float* out, void* stream);
int skb_dist_fold_send(skb_dist_t d, const float* dpooled, int32_t mode, int64_t num_unique,
                       const int64_t* seg_prefix, float* const* peer_windows, const int64_t* dst_base,
                       void* stream);
/* device pointers of the prepared batch (tests / diagnostics) */
int skb_dist_buffers(skb_dist_t d, const int64_t** uniq_out, const int64_t** counts_out,
                     const uint32_t** gidx_out);
/* owner side: the received ids (n, rank-ordered segments recv_prefix[0..S])
 * as a batch of one-id bags through the fused index phase (admission in the
 * rank-ordered first-occurrence order), then row q -> requester j's window
 * at dst_base[j] + q - recv_prefix[j].  skb_fused_backward with the grad
 * window as dpooled completes the step. */
int skb_fused_forward_send(skb_table_t t, const int64_t* recv_ids, int64_t n, int64_t step,
                           const int64_t* recv_prefix, int32_t num_ranks, float* const* peer_windows,
                           const int64_t* dst_base, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEKIT_B200_H */
