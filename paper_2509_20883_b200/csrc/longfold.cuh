// longfold.cuh — bit-exact in-order fold of LONG runs (hot zipf ids).
//
// The reference pre-aggregates a row's gradients with np.add.at, a strict
// left fold in input order (sharding.py:289).  For a hot id with ~10^6
// positions that chain is inherently serial in fp32; what must not be serial
// is the memory traffic.  Runs longer than kLongRun are deferred by the main
// fold kernels into a device list; here one CTA owns one long run at a time:
// producer warps stream the run's gradient rows through a shared-memory ring
// while consumer warps fold them in position order (details at k_long_fold).
// Cost ~ one FADD latency per position instead of one DRAM round trip.
#pragma once
#include <cstdlib>

#include "common.cuh"
#include "table.cuh"
#include "tma.cuh"

namespace skb {

constexpr int kLongRun = 32;  // runs longer than this are deferred
constexpr uint32_t kNoPack = 0xFFFFFFFFu;  // LongRun.pad: not packed
constexpr int64_t kMegaRunMin = 2048;      // smallest run ever packed for TMA streaming
// runs at least this long are packed: 8192 positions, or 2048 for mean bags
// (their unpacked producers divide row by row, ~4x slower than the 16-byte
// copies of sum bags); SKB_LF_MEGA overrides (>= kMegaRunMin)
inline int64_t mega_run_threshold(int mode) {
  static const int64_t v = getenv("SKB_LF_MEGA") ? atoll(getenv("SKB_LF_MEGA")) : 0;
  if (v > 0) return v < kMegaRunMin ? kMegaRunMin : v;
  return mode == 1 ? 2048 : 8192;
}

struct LongRun {
  uint32_t key, jh, je, pad;
};

// cap == 0: the runs were listed up front (k_list_long_runs) — skip, do not push
__device__ __forceinline__ void push_long_run(LongRun* list, int64_t* count, int64_t cap, uint32_t key, uint32_t jh,
                                              uint32_t je) {
  if (cap <= 0) return;
  unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(count), 1ull);
  if ((int64_t)i < cap) list[i] = LongRun{key, jh, je, 0};
}

// Up-front listing of the long runs of a sorted key array (so the long fold
// can start concurrently with the main fold kernel, which then skips them):
// a head j (j == 0 or key change) starts a run longer than kLongRun iff
// skey[j + kLongRun] still holds its key; its end is a binary search.
static __global__ void k_list_long_runs(const uint32_t* __restrict__ skey, int64_t n, LongRun* list, int64_t* count,
                                        int64_t cap) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = __ldg(skey + j);
    if (j > 0 && __ldg(skey + j - 1) == k) continue;
    if (j + kLongRun >= n || __ldg(skey + j + kLongRun) != k) continue;
    int64_t lo = j + kLongRun, hi = n;  // skey[lo] == k; first index > lo with a different key
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(skey + mid) == k) lo = mid; else hi = mid;
    }
    unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(count), 1ull);
    if ((int64_t)i < cap) list[i] = LongRun{k, (uint32_t)j, (uint32_t)hi, 0};
  }
}

// One CTA folds one long run at a time (runs strided over CTAs).  A stage
// holds TP consecutive positions of the run.  Consumer warps 0..NC-1 own
// the columns (one per lane, kLfCols per lane above 32*kLfMaxNC) and fold a
// stage's rows in position order from +0; the remaining NPW warps produce:
//  - ordinary runs: producer warp pw owns the stages it = pw (mod NPW),
//    loads the stage's row indices once, then 16-byte cp.async copies of the
//    gradient rows (row-major stage), each lane signalling `full` when ITS
//    copies land (cp.async.mbarrier.arrive.noinc).  One SM's outstanding-
//    request budget caps this at ~25 GB/s.
//  - mega runs (>= mega_run_threshold(mode) positions, the hottest ids): k_pack_rows has
//    already laid the run out as stage IMAGES — each stage transposed to
//    column-major with a padded column stride PS = TP + 4 — so a stage is
//    ONE TMA bulk copy, and a consumer lane reads four positions of its
//    column with one conflict-free LDS.128: the serial chain, not the load
//    path, sets the pace (~4 cycles per position).
// rows: gradient source rows (dpooled [G, D] or per-position grads [N, D]);
// ridx[j]: row of sorted position j (0xFFFFFFFF: the zero row `zrow`);
// mode 1 (mean): divide by len(bag ridx[j]).
// ADAM: update arena row `key` (and last_step); else write out[key * D].
constexpr int kLfStages = 12;
constexpr int kLfStageBytes = 32768;
constexpr int kLfMaxTP = 512;   // rows per stage cap (small dims)
constexpr int kLfMaxPW = 8;     // producer warps (index buffers)
constexpr int kLfPad = 4;       // column padding of a packed stage image
constexpr int kLfSmemBudget = 192 * 1024;  // ring + index buffers; leaves room for co-resident index-stream CTAs

// rows per stage: kLfStageBytes of rows, a multiple of 4 (16-byte columns in
// a packed image), at most kLfMaxTP (small dims)
__host__ __device__ inline int long_fold_tp(int D) {
  const int tp = (kLfStageBytes / (4 * D)) & ~3;
  return tp < 4 ? 4 : (tp > kLfMaxTP ? kLfMaxTP : tp);
}
// floats of one stage slot: a row-major stage (TP*D) or a packed image
__host__ __device__ inline int64_t long_fold_stage_f(int D) { return (int64_t)D * (long_fold_tp(D) + kLfPad); }
// Column groups of a packed (mega) run: kLfGW columns each, one work unit
// (one CTA, one serial chain per column) per group — the hottest id's rows
// are folded by ceil(D / kLfGW) CTAs in parallel, each streaming only its
// columns (a 32-column group left the C4 hot run bound by one SM's stream).
constexpr int kLfGW = 8;
// a run this long (positions) keeps its column-group CTAs busy for >~0.5 ms:
// the long fold then runs as the step's critical path (launch_long_fold `hot_chain`)
constexpr int64_t kLfExclusiveRun = 200000;
__host__ __device__ inline int long_fold_groups(int D) { return (D + kLfGW - 1) / kLfGW; }
// packed image of one column group (min(kLfGW, D) columns): the whole slot,
// column-major with stride PS = TPI + kLfPad; TPI a multiple of 32 so PS is
// 4 (mod 32) and eight lanes' LDS.128 of their columns hit distinct banks
__host__ __device__ inline int long_fold_img_w(int D) { return D < kLfGW ? D : kLfGW; }
__host__ __device__ inline int long_fold_tpi(int D) {
  const int64_t t = ((long_fold_stage_f(D) / long_fold_img_w(D) - kLfPad) / 32) * 32;
  return (int)(t < 32 ? 32 : t);
}
// positions per direct column-group stage ([TPG][kLfGW] floats, row-major):
// as many as the slot holds, a multiple of 32, at most the index buffer
__host__ __device__ inline int long_fold_tpg(int D) {
  const int64_t t = (long_fold_stage_f(D) / kLfGW) & ~31ll;
  return (int)(t > kLfMaxTP ? kLfMaxTP : (t < 32 ? 32 : t));
}
constexpr int kLfMaxNC = 16;  // consumer warps
constexpr int kLfCols = 4;    // columns per consumer lane: dims up to 32 * kLfMaxNC * kLfCols = 2048
__host__ __device__ inline int long_fold_consumers(int D) {
  const int nc = (D + 31) / 32;
  return nc < kLfMaxNC ? nc : kLfMaxNC;
}
// ring depth that fits the shared-memory budget
inline int long_fold_stages(int D, int budget = kLfSmemBudget) {
  const int64_t fixed = (int64_t)kLfMaxPW * kLfMaxTP * 4 + 2 * kLfStages * 8;
  int64_t st = (budget - fixed) / (long_fold_stage_f(D) * 4);
  return (int)(st > kLfStages ? kLfStages : (st < 2 ? 2 : st));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float4 vdiv4(float4 x, float l) {
  return make_float4(__fdiv_rn(x.x, l), __fdiv_rn(x.y, l), __fdiv_rn(x.z, l), __fdiv_rn(x.w, l));
}

// work unit wu -> (run, column group, packed?); false: nothing to do
__device__ __forceinline__ bool long_fold_unit(int64_t wu, int64_t MU, int NCG, const LongRun* __restrict__ runs,
                                               const uint32_t* __restrict__ mlist,
                                               const uint32_t* __restrict__ morder, bool grouped,
                                               LongRun& run, int& cg, bool& img) {
  if (wu < MU) {  // column group of a mega run; unfitted mega runs come back as ordinary units
    const int64_t m = wu / NCG;
    cg = (int)(wu - m * NCG);
    run = runs[__ldg(mlist + __ldg(morder + m))];
    img = run.pad != kNoPack;
    return img;
  }
  run = runs[wu - MU];
  cg = 0;
  img = false;
  return !(grouped && run.pad != kNoPack);  // grouped runs were covered by their groups
}

// SKB_LF_MIX_TEST=1 (tests only): with streamed packs, treat every odd stage
// as not yet packed, so one run mixes TMA image stages and gathered stages
// deterministically
__device__ int g_lf_mix_test = 0;

template <bool ADAM>
__global__ void k_long_fold(const LongRun* __restrict__ runs, const int64_t* __restrict__ nruns, int64_t cap,
                            const uint32_t* __restrict__ ridx, const float* __restrict__ rows, int D,
                            const int64_t* __restrict__ bag_offs, int mode, AdamDev a, float* __restrict__ out,
                            int64_t* __restrict__ last_step, int64_t step, int nst,
                            const float* __restrict__ zrow, const float* __restrict__ packed,
                            const uint32_t* __restrict__ mlist, const uint32_t* __restrict__ morder,
                            const int64_t* __restrict__ mcount, RowOut ro = RowOut{}, bool direct = false,
                            const uint32_t* __restrict__ ready = nullptr, unsigned long long* wctr = nullptr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // stage layout (packed mode with ready flags): 0 = column-major image
  // (TMA), 1 = row-major [positions][kLfGW] gathered directly because the
  // pack had not reached that image yet
  __shared__ int s_lay[kLfStages];
  // dynamic unit scheduling (wctr): the k-th unit this CTA folds is fetched
  // once, by the first producer warp, from the launch's counter and handed
  // to every warp through a small ring — units are taken in walking order
  // (the head id's column groups first), so the CTA that holds the longest
  // chain takes nothing after it and short runs spread over the others
  constexpr int kUnitRing = 64;
  __shared__ long long s_wu[kUnitRing];
  __shared__ int s_wseq[kUnitRing];
  const int TP = long_fold_tp(D);                // positions per row-major stage
  const int TPI = long_fold_tpi(D);              // positions per packed column-group image
  const int PS = TPI + kLfPad;                   // column stride of a packed image
  const int64_t stage_f = long_fold_stage_f(D);  // floats per stage slot
  float* buf = reinterpret_cast<float*>(smem_raw);
  uint32_t* idx = reinterpret_cast<uint32_t*>(buf + (int64_t)nst * stage_f);  // [kLfMaxPW][kLfMaxTP]
  uint64_t* full = reinterpret_cast<uint64_t*>(idx + kLfMaxPW * kLfMaxTP);
  uint64_t* empty = full + kLfStages;
  const int NC = long_fold_consumers(D);
  const int NCG = long_fold_groups(D);  // column groups: work units of a packed run
  const int64_t R = *nruns < cap ? *nruns : cap;
  // work units: first every packed (mega) run's column groups, longest run
  // first (morder), so the hottest ids' chains start in the first wave on
  // distinct SMs; then one unit per ordinary run.  Producers and consumers
  // walk the same sequence.
  // direct: mega runs are column-group units too, but their producers gather
  // the group's columns straight from the gradient rows (no packed images)
  const bool grouped = packed != nullptr || direct;
  const uint32_t epoch = ready ? (uint32_t)mcount[3] : 0u;
  const int TPG = long_fold_tpg(D);  // positions per direct group stage ([TPG][kLfGW] row-major)
  const int64_t MU = grouped ? (mcount[0] < R ? mcount[0] : R) * NCG : 0;
  const int64_t units = MU + R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 32);  // the owning producer warp's lanes
      mbar_init(&empty[s], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < kUnitRing; i += blockDim.x) s_wseq[i] = -1;
  __syncthreads();
  // the unit of this CTA's k-th walk step (the same sequence in every warp);
  // >= units ends the walk.  The fetcher skips units without work, so every
  // ring entry holds at least one stage: no warp can fall a ring lap behind
  // (the others trail the fetcher by at most the ring's nst stages)
  auto unit_at = [&](int k) -> int64_t {
    if (!wctr) return (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
    const int slot = k & (kUnitRing - 1);
    if (warp == NC && lane == 0) {
      long long u;
      while (true) {
        u = (long long)atomicAdd(wctr, 1ull);
        if (u >= units) break;
        int cg_;
        LongRun r_;
        bool im_;
        if (long_fold_unit(u, MU, NCG, runs, mlist, morder, grouped, r_, cg_, im_)) break;
      }
      s_wu[slot] = u;
      __threadfence_block();
      *reinterpret_cast<volatile int*>(&s_wseq[slot]) = k;
    }
    while (*reinterpret_cast<volatile int*>(&s_wseq[slot]) != k) {
    }
    __threadfence_block();
    return (int64_t)*reinterpret_cast<volatile long long*>(&s_wu[slot]);
  };
  uint32_t it = 0;  // stage sequence number, identical in producers and consumers
  if (warp >= NC) {  // ---------------- producers: warp pw fills stages it = pw (mod NPW) ----------------
    const int pw = warp - NC, NPW = (int)(blockDim.x >> 5) - NC;
    const int cpr = D / 4;  // 16-byte chunks per row
    for (int uk = 0;; ++uk) {
      const int64_t wu = unit_at(uk);
      if (wu >= units) break;
      int cg;
      LongRun run;
      bool img;
      if (!long_fold_unit(wu, MU, NCG, runs, mlist, morder, grouped, run, cg, img)) continue;
      const int ncol = D - kLfGW * cg < kLfGW ? D - kLfGW * cg : kLfGW;
      const int step_p = img ? (packed ? TPI : TPG) : TP;
      const int64_t nimg = img ? ((int64_t)run.je - run.jh + TPI - 1) / TPI : 0;  // images per column group
      for (int64_t p0 = run.jh; p0 < run.je; p0 += step_p, ++it) {
        if ((int)(it % (uint32_t)NPW) != pw) continue;
        const int s = (int)(it % (uint32_t)nst);
        const uint32_t ph = (it / (uint32_t)nst) & 1u;
        const int np = (int)((int64_t)run.je - p0 < step_p ? (int64_t)run.je - p0 : step_p);
        float* dst = buf + s * stage_f;
        if (img && !packed) {  // direct group stage: [TPG][kLfGW] of this group's columns
          const int cpg = ncol >> 2;  // 16-byte chunks per position (D % 4 == 0)
          uint32_t* ix = idx + pw * kLfMaxTP;
          {
            uint32_t gi[kLfMaxTP / 32];  // all index loads in flight before the stores
#pragma unroll
            for (int k = 0; k < kLfMaxTP / 32; ++k) gi[k] = k * 32 + lane < np ? __ldg(ridx + p0 + k * 32 + lane) : 0u;
#pragma unroll
            for (int k = 0; k < kLfMaxTP / 32; ++k)
              if (k * 32 + lane < np) ix[k * 32 + lane] = gi[k];
          }
          __syncwarp();
          mbar_wait(&empty[s], ph ^ 1u);
          const int items = np * cpg;
          const int col0 = kLfGW * cg;
          if (mode == 1) {
            for (int b = lane; b < items; b += 4 * 32) {
              float4 x[4];
              float l[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int i = b + k * 32;
                if (i < items) {
                  const int row = i / cpg, ch = i - row * cpg;
                  const uint32_t gg = ix[row];
                  x[k] = ldg4((gg == 0xFFFFFFFFu ? zrow : rows + (int64_t)gg * D) + col0 + ch * 4);
                  l[k] = (float)(__ldg(bag_offs + gg + 1) - __ldg(bag_offs + gg));
                }
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int i = b + k * 32;
                if (i < items) {
                  const int row = i / cpg, ch = i - row * cpg;
                  st4(dst + row * kLfGW + ch * 4, vdiv4(x[k], l[k]));
                }
              }
            }
            mbar_arrive(&full[s]);
          } else {
            for (int i = lane; i < items; i += 32) {
              const int row = i / cpg, ch = i - row * cpg;
              const uint32_t gg = ix[row];
              cp_async16(dst + row * kLfGW + ch * 4, (gg == 0xFFFFFFFFu ? zrow : rows + (int64_t)gg * D) + col0 + ch * 4);
            }
            cp_async_arrive_noinc(&full[s]);
          }
          __syncwarp();  // ix is rewritten by this warp's next stage
          continue;
        }
        int gather = 0;  // packed mode: the pack has not written this image yet -> gather directly
        if (img && ready) {
          if (lane == 0) {
            uint32_t f;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];"
                         : "=r"(f) : "l"(ready + run.pad / NCG + (p0 - run.jh) / TPI) : "memory");
            gather = f != epoch || (g_lf_mix_test && (((p0 - run.jh) / TPI) & 1));
            if (!gather) asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads after the acquire
          }
          gather = __shfl_sync(0xffffffffu, gather, 0);
        }
        if (img && gather) {  // row-major [np][kLfGW] of this group's columns, 16-byte cp.async
          const int cpg = ncol >> 2;
          const int col0 = kLfGW * cg;
          const int RS = long_fold_img_w(D);  // row stride: TPI rows of the group's columns fit the slot
          uint32_t* ix = idx + pw * kLfMaxTP;
          mbar_wait(&empty[s], ph ^ 1u);
          if (lane == 0) s_lay[s] = 1;
          for (int h0 = 0; h0 < np; h0 += kLfMaxTP) {  // index buffer holds kLfMaxTP positions
            const int nh = np - h0 < kLfMaxTP ? np - h0 : kLfMaxTP;
            __syncwarp();
            {
              uint32_t gi[kLfMaxTP / 32];
#pragma unroll
              for (int k = 0; k < kLfMaxTP / 32; ++k)
                gi[k] = k * 32 + lane < nh ? __ldg(ridx + p0 + h0 + k * 32 + lane) : 0u;
#pragma unroll
              for (int k = 0; k < kLfMaxTP / 32; ++k)
                if (k * 32 + lane < nh) ix[k * 32 + lane] = gi[k];
            }
            __syncwarp();
            const int items = nh * cpg;
            if (mode == 1) {
              for (int i = lane; i < items; i += 32) {
                const int row = i / cpg, ch = i - row * cpg;
                const uint32_t gg = ix[row];
                const float4 x = ldg4((gg == 0xFFFFFFFFu ? zrow : rows + (int64_t)gg * D) + col0 + ch * 4);
                const float l = (float)(__ldg(bag_offs + gg + 1) - __ldg(bag_offs + gg));
                st4(dst + (h0 + row) * RS + ch * 4, vdiv4(x, l));
              }
            } else {
              for (int i = lane; i < items; i += 32) {
                const int row = i / cpg, ch = i - row * cpg;
                const uint32_t gg = ix[row];
                cp_async16(dst + (h0 + row) * RS + ch * 4,
                           (gg == 0xFFFFFFFFu ? zrow : rows + (int64_t)gg * D) + col0 + ch * 4);
              }
            }
          }
          if (mode == 1) mbar_arrive(&full[s]); else cp_async_arrive_noinc(&full[s]);
          __syncwarp();
          continue;
        }
        if (img) {  // one bulk copy: this column group's image of TPI positions
          const uint32_t bytes = (uint32_t)ncol * (uint32_t)PS * 4u;
          mbar_wait(&empty[s], ph ^ 1u);
          if (lane == 0) s_lay[s] = 0;
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[s], bytes);
            const int64_t im = (int64_t)run.pad + (int64_t)cg * nimg + (p0 - run.jh) / TPI;
            bulk_g2s(dst, packed + im * stage_f, bytes, &full[s]);
          } else {
            mbar_arrive(&full[s]);
          }
          __syncwarp();
          continue;
        }
        const int items = np * cpr;
        // the stage's row indices: one coalesced batch of loads per lane, staged in
        // the warp's index buffer (a single memory latency per stage)
        uint32_t gi[kLfMaxTP / 32];
#pragma unroll
        for (int k = 0; k < kLfMaxTP / 32; ++k) {
          const int row = k * 32 + lane;
          gi[k] = row < np ? __ldg(ridx + p0 + row) : 0u;
        }
        uint32_t* ix = idx + pw * kLfMaxTP;
#pragma unroll
        for (int k = 0; k < kLfMaxTP / 32; ++k) {
          const int row = k * 32 + lane;
          if (row < np) ix[row] = gi[k];
        }
        __syncwarp();                   // ix visible to the whole warp
        mbar_wait(&empty[s], ph ^ 1u);  // the stage is free again
        if (mode == 1) {
          // mean bags: the producer divides by the bag length (x / len, exactly
          // the reference's per-position grad) so the fold chain stays one FADD
          for (int b = lane; b < items; b += 4 * 32) {
            float4 x[4];
            float l[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int i = b + k * 32;
              if (i < items) {
                const int row = i / cpr, ch = i - row * cpr;
                const uint32_t gg = ix[row];
                x[k] = ldg4((gg == 0xFFFFFFFFu ? zrow : rows + (int64_t)gg * D) + ch * 4);
                l[k] = (float)(__ldg(bag_offs + gg + 1) - __ldg(bag_offs + gg));
              }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int i = b + k * 32;
              if (i < items) {
                const int row = i / cpr, ch = i - row * cpr;
                st4(dst + (int64_t)row * D + ch * 4, make_float4(__fdiv_rn(x[k].x, l[k]), __fdiv_rn(x[k].y, l[k]),
                                                                 __fdiv_rn(x[k].z, l[k]), __fdiv_rn(x[k].w, l[k])));
              }
            }
          }
          mbar_arrive(&full[s]);  // release of this lane's stores
        } else {
          for (int i = lane; i < items; i += 32) {
            const int row = i / cpr, ch = i - row * cpr;
            const uint32_t gg = ix[row];  // 0xFFFFFFFF: the zero row (tile positions past k)
            cp_async16(dst + (int64_t)row * D + ch * 4, (gg == 0xFFFFFFFFu ? zrow : rows + (int64_t)gg * D) + ch * 4);
          }
          cp_async_arrive_noinc(&full[s]);  // fires when this lane's copies have landed
        }
        __syncwarp();  // ix is rewritten by this warp's next stage
      }
    }
    return;
  }
  // ---------------- consumers: warp w owns columns 32 w + lane (+ 32 NC, ...) ----------------
  // one column per lane: a position costs each warp one FADD on the chain.
  // A packed (mega) run is split into column groups of kLfGW: each unit (run,
  // group) streams only its columns, so the hottest id's rows are read by
  // ceil(D/32) CTAs in parallel — each with its own serial chain per column
  const int c0 = warp * 32 + lane;
  const int cstep = 32 * NC;
  for (int uk = 0;; ++uk) {
    const int64_t wu = unit_at(uk);
    if (wu >= units) break;
    int cg;
    LongRun run;
    bool img;
    if (!long_fold_unit(wu, MU, NCG, runs, mlist, morder, grouped, run, cg, img)) continue;
    const int ncol = D - kLfGW * cg < kLfGW ? D - kLfGW * cg : kLfGW;
    const int step_p = img ? (packed ? TPI : TPG) : TP;
    float acc[kLfCols];
#pragma unroll
    for (int q = 0; q < kLfCols; ++q) acc[q] = 0.f;
    for (int64_t p0 = run.jh; p0 < run.je; p0 += step_p, ++it) {
      const int s = (int)(it % (uint32_t)nst);
      const uint32_t ph = (it / (uint32_t)nst) & 1u;
      const int np = (int)((int64_t)run.je - p0 < step_p ? (int64_t)run.je - p0 : step_p);
      mbar_wait(&full[s], ph);
      if (img && (!packed || s_lay[s] == 1)) {  // direct group stage: lane c folds column c, one position per LDS
        if (warp == 0 && lane < ncol) {
          const float* src = buf + s * stage_f + lane;
          const int rs = packed ? long_fold_img_w(D) : kLfGW;  // mixed stages: img_w-wide rows
#pragma unroll 16
          for (int p = 0; p < np; ++p) acc[0] = __fadd_rn(acc[0], src[p * rs]);
        }
      } else if (img) {  // column-major image slice: four positions per 16-byte load,
                  // the next 16 positions' loads issued before this 16's adds
        if (warp == 0 && lane < ncol) {
          const float* col = buf + s * stage_f + (int64_t)lane * PS;
          const float4* c4 = reinterpret_cast<const float4*>(col);
          // two 16-position groups of loads in flight: every LDS.128 has a
          // full 32-FADD iteration (~128 cycles) to land before its adds
          const int n32 = np & ~31;
          auto fold4 = [&](const float4& v) {
            acc[0] = __fadd_rn(acc[0], v.x);
            acc[0] = __fadd_rn(acc[0], v.y);
            acc[0] = __fadd_rn(acc[0], v.z);
            acc[0] = __fadd_rn(acc[0], v.w);
          };
          if (n32) {
            float4 a[4], b[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              a[k] = c4[k];
              b[k] = c4[4 + k];
            }
            for (int p = 32; p < n32; p += 32) {
              float4 c[4], d[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) c[k] = c4[(p >> 2) + k];
#pragma unroll
              for (int k = 0; k < 4; ++k) fold4(a[k]);
#pragma unroll
              for (int k = 0; k < 4; ++k) d[k] = c4[(p >> 2) + 4 + k];
#pragma unroll
              for (int k = 0; k < 4; ++k) fold4(b[k]);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                a[k] = c[k];
                b[k] = d[k];
              }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) fold4(a[k]);
#pragma unroll
            for (int k = 0; k < 4; ++k) fold4(b[k]);
          }
          for (int p = n32; p < np; ++p) acc[0] = __fadd_rn(acc[0], col[p]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < kLfCols; ++q) {
          const int c = c0 + q * cstep;
          if (c >= D) continue;
          const float* src = buf + s * stage_f + c;
#pragma unroll 16
          for (int p = 0; p < np; ++p) acc[q] = __fadd_rn(acc[q], src[(int64_t)p * D]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // results: packed unit -> its column group (warp 0); unpacked -> all columns
#pragma unroll
    for (int q = 0; q < kLfCols; ++q) {
      int c;
      if (img) {
        if (q > 0 || warp != 0 || lane >= ncol) continue;
        c = kLfGW * cg + lane;
      } else {
        c = c0 + q * cstep;
        if (c >= D) continue;
      }
      if constexpr (ADAM) {
        float* row = out + (int64_t)run.key * (3 * D);
        float p = row[c], m = row[D + c], v = row[2 * D + c];
        adam1(p, m, v, acc[q], a);
        row[c] = p;
        row[D + c] = m;
        row[2 * D + c] = v;
        if (c == 0 && step >= 0) last_step[run.key] = step;
      } else {
        ro.row(out, run.key, D)[c] = acc[q];
      }
    }
  }
  if (!ADAM && ro.peers) __threadfence_system();  // peer stores before the stream's barrier write
}

// ---------------------------------------------------------------------------
// Mega-run packing: the whole grid gathers the gradient rows of the runs of
// at least mega_run_threshold(mode) positions into stage images (see k_long_fold), so the
// CTA folding such a run streams it with one bulk copy per stage.
struct LongFoldPack {
  float* images = nullptr;    // [cap_images][stage slot]: per (mega run, column group, TPI positions)
  int64_t cap_images = 0;
  uint32_t* mlist = nullptr;  // [cap_runs] run index of each mega run
  uint32_t* moff = nullptr;   // [cap_runs] first image of each mega run (ascending; kNoPack if it did not fit)
  int64_t* mcount = nullptr;  // [4] mega runs, images in use, longest run (positions), ready epoch
  int64_t cap_runs = 0;
  uint32_t* morder = nullptr; // [cap_runs] mega-list indices, longest run first
  uint32_t* ready = nullptr;  // [cap_images / groups + 1] per (run, stage) pair: the epoch once its images are written
  unsigned long long* wctr = nullptr;  // work-unit counter of one long-fold launch (dynamic unit scheduling)
  cudaStream_t pstream = nullptr;  // pack stream (eager steps): the pack runs beside the long fold
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

// one block: the mega runs (>= `mega` positions) in list order -> mlist;
// their longest-first order -> morder (rank by length, ties by list
// position; beyond kSortMax mega runs: list order); stage images assigned in
// morder order (so the hottest run's images come first and are packed first)
// -> moff / run.pad (kNoPack past capacity); mcount = {mega runs, images in
// use, longest run, epoch}: the epoch (bumped here) tags this pack's
// per-pair ready flags
static __global__ void __launch_bounds__(1024) k_pack_plan(LongRun* runs, const int64_t* __restrict__ nruns,
                                                           int64_t cap, int TPI, int NCG, int64_t mega,
                                                           int64_t cap_images,
                                                           uint32_t* __restrict__ mlist, uint32_t* __restrict__ moff,
                                                           int64_t* __restrict__ mcount, uint32_t* __restrict__ morder) {
  constexpr int kSortMax = 2048;
  __shared__ uint32_t s_len[kSortMax];
  __shared__ int64_t s_c[32];
  __shared__ int64_t s_cc;
  __shared__ unsigned long long s_maxlen;  // longest run: mcount[2] (the host's hint for exclusive SMs)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int64_t R = *nruns < cap ? *nruns : cap;
  if (threadIdx.x == 0) {
    s_cc = 0;
    s_maxlen = 0;
  }
  __syncthreads();
  for (int64_t b0 = 0; b0 < R; b0 += blockDim.x) {  // compaction of the mega runs, list order
    const int64_t r = b0 + threadIdx.x;
    int64_t len = 0;
    if (r < R) len = (int64_t)runs[r].je - runs[r].jh;
    if (len > 0) atomicMax(&s_maxlen, (unsigned long long)len);
    const int64_t f = (r < R && len >= mega) ? 1 : 0;
    int64_t ic = f;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t yc = __shfl_up_sync(0xffffffffu, ic, o);
      if (lane >= o) ic += yc;
    }
    if (lane == 31) s_c[w] = ic;
    __syncthreads();
    int64_t bc = s_cc, tc = 0;
    for (int q = 0; q < W; ++q) {
      if (q < w) bc += s_c[q];
      tc += s_c[q];
    }
    if (r < R) {
      runs[r].pad = kNoPack;
      if (f) mlist[bc + ic - f] = (uint32_t)r;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_cc += tc;
    __syncthreads();
  }
  const int64_t M = s_cc;
  if (M <= kSortMax) {
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      const LongRun ri = runs[mlist[i]];
      s_len[i] = ri.je - ri.jh;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      const uint32_t li = s_len[i];
      int64_t rank = 0;
      for (int64_t j = 0; j < M; ++j) {
        const uint32_t lj = s_len[j];
        rank += (lj > li || (lj == li && j < i)) ? 1 : 0;
      }
      morder[rank] = (uint32_t)i;
    }
  } else {
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) morder[i] = (uint32_t)i;
  }
  __threadfence_block();
  __syncthreads();
  // image offsets in morder order: exclusive scan of NCG * stages; a run fits
  // while the running total stays within capacity (a prefix of morder)
  __shared__ int64_t s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < M; b0 += blockDim.x) {
    const int64_t rk = b0 + threadIdx.x;
    int64_t l = 0, mi = 0;
    if (rk < M) {
      mi = morder[rk];
      const LongRun ri = runs[mlist[mi]];
      l = NCG * (((int64_t)ri.je - ri.jh + TPI - 1) / TPI);
    }
    int64_t il = l;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, il, o);
      if (lane >= o) il += y;
    }
    if (lane == 31) s_c[w] = il;
    __syncthreads();
    int64_t bl = s_base, tl = 0;
    for (int q = 0; q < W; ++q) {
      if (q < w) bl += s_c[q];
      tl += s_c[q];
    }
    if (rk < M) {
      const int64_t xl = bl + il - l;
      const bool fits = xl + l <= cap_images;
      moff[mi] = fits ? (uint32_t)xl : kNoPack;
      runs[mlist[mi]].pad = fits ? (uint32_t)xl : kNoPack;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += tl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    mcount[0] = M;
    mcount[1] = s_base <= cap_images ? s_base : 0;  // images in use (past capacity: the fitted prefix, below)
    mcount[2] = (int64_t)s_maxlen;
    mcount[3] += 1;  // epoch of this pack's ready flags
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_base > cap_images) {  // the fitted prefix ends before the first unfitted rank
    int64_t used = 0;
    for (int64_t rk = 0; rk < M; ++rk) {
      const uint32_t o = moff[morder[rk]];
      if (o == kNoPack) break;
      const LongRun ri = runs[mlist[morder[rk]]];
      used = (int64_t)o + NCG * (((int64_t)ri.je - ri.jh + TPI - 1) / TPI);
    }
    mcount[1] = used;
  }
}

// one block per (mega run, stage k): the stage's TPI gradient rows are
// gathered kPackSub positions at a time into shared memory by 16-byte
// cp.async (double-buffered: sub-chunk i+1 in flight while sub-chunk i is
// written out; zero row past a tile's k), then written out as contiguous
// column segments of all the run's column-group images at once (/ len for
// mean bags) — every gradient byte is read once, every image byte written
// once, and a block always has a sub-chunk of loads outstanding.
// positions per sub-chunk: 64 for D >= 64 (128 at D=64 was slower in C4,
// 630 vs 537 us); narrow rows take more per sub-chunk (4096 / D, up to 512:
// a D=8 block otherwise walks its 512-position stage in 8 serial rounds)
inline int pack_sub(int D) {
  const int cap = 4096 / D > 64 ? (4096 / D > 512 ? 512 : 4096 / D) : 64;
  const int sp = 9000 / (D + 4) > cap ? cap : 9000 / (D + 4);
  return sp < 4 ? 4 : sp & ~3;
}
inline size_t pack_smem(int D) { return (size_t)2 * pack_sub(D) * ((D + 4) * sizeof(float) + sizeof(uint32_t)); }
static __global__ void __launch_bounds__(256, 5) k_pack_rows(const LongRun* __restrict__ runs,
                                                          const uint32_t* __restrict__ mlist,
                                                          const uint32_t* __restrict__ moff,
                                                          const int64_t* __restrict__ mcount,
                                                          const uint32_t* __restrict__ ridx,
                                                          const float* __restrict__ rows,
                                                          const float* __restrict__ zrow, int D,
                                                          const int64_t* __restrict__ bag_offs, int mode, int SP,
                                                          float* __restrict__ images,
                                                          const uint32_t* __restrict__ morder,
                                                          uint32_t* __restrict__ ready) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int RS = D + 4;  // tile row stride (floats): 16-byte rows; LDS.128 of 8 consecutive rows hit distinct banks
  float* tile = reinterpret_cast<float*>(smem_raw);                   // [2][SP][RS]
  uint32_t* tgi = reinterpret_cast<uint32_t*>(tile + 2 * SP * RS);    // [2][SP] source row of each position
  const int TPI = long_fold_tpi(D), PS = TPI + kLfPad;
  const int64_t stage_f = long_fold_stage_f(D);
  const int NCG = long_fold_groups(D);
  const int64_t nm = mcount[0], npair = mcount[1] / NCG;  // (run, stage) pairs of the fitted runs
  const uint32_t epoch = (uint32_t)mcount[3];
  const int cpr = D >> 2;
  // pairs in image order = morder order: the longest run's stages first, so
  // a long fold streaming concurrently finds them ready soonest
  for (int64_t q = blockIdx.x; q < npair; q += gridDim.x) {
    int64_t lo = 0, hi = nm;  // rank owning pair q (moff[morder[.]] / NCG ascending; unfitted: kNoPack suffix)
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)__ldg(moff + __ldg(morder + mid)) / NCG <= q) lo = mid; else hi = mid;
    }
    const uint32_t mi = __ldg(morder + lo);
    const LongRun run = runs[__ldg(mlist + mi)];
    const int64_t per_group = ((int64_t)run.je - run.jh + TPI - 1) / TPI;
    const int64_t k = q - (int64_t)__ldg(moff + mi) / NCG;
    const int64_t img0 = (int64_t)__ldg(moff + mi) + k;  // image of group g: img0 + g * per_group
    const int64_t j0 = (int64_t)run.jh + k * TPI;
    const int np = (int)((int64_t)run.je - j0 < TPI ? (int64_t)run.je - j0 : TPI);
    const int nsub = (np + SP - 1) / SP;
    __syncthreads();  // the previous pair's last sub-chunk has been written out
    auto issue = [&](int i) {  // cp.async of sub-chunk i into buffer i & 1
      const int p0 = i * SP, sp = np - p0 < SP ? np - p0 : SP;
      float* tb = tile + (i & 1) * SP * RS;
      uint32_t* gb = tgi + (i & 1) * SP;
      const int items = sp * cpr;
      for (int t0 = threadIdx.x; t0 < items; t0 += 4 * blockDim.x) {
        uint32_t gi[4];  // the four index loads in flight together
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u * blockDim.x;
          gi[u] = t < items ? __ldg(ridx + j0 + p0 + t / cpr) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u * blockDim.x;
          if (t >= items) continue;
          const int p = t / cpr, c4 = t - p * cpr;
          if (c4 == 0) gb[p] = gi[u];
          cp_async16(tb + p * RS + c4 * 4, (gi[u] == 0xFFFFFFFFu ? zrow : rows + (int64_t)gi[u] * D) + c4 * 4);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    for (int i = 0; i < nsub; ++i) {
      if (i + 1 < nsub) {
        issue(i + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();  // sub-chunk i landed for every thread
      const int p0 = i * SP, sp = np - p0 < SP ? np - p0 : SP;
      const float* tb = tile + (i & 1) * SP * RS;
      const uint32_t* gb = tgi + (i & 1) * SP;
      // thread (position p, 4-column chunk c4): one LDS.128, four column
      // stores — consecutive lanes take consecutive positions of one chunk,
      // so each store instruction writes contiguous floats of one column
      for (int t = threadIdx.x; t < sp * cpr; t += blockDim.x) {
        const int c4 = t / sp, p = t - c4 * sp;
        float4 x = *reinterpret_cast<const float4*>(tb + p * RS + c4 * 4);
        if (mode == 1) {
          const uint32_t gi = gb[p];
          x = vdiv4(x, (float)(__ldg(bag_offs + gi + 1) - __ldg(bag_offs + gi)));
        }
        const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = c4 * 4 + e, g = c / kLfGW, cl = c - g * kLfGW;
          images[(img0 + (int64_t)g * per_group) * stage_f + (int64_t)cl * PS + p0 + p] = xv[e];
        }
      }
      __syncthreads();  // buffer i & 1 is refilled by issue(i + 2)
    }
    if (ready && threadIdx.x == 0) {  // every group's image of pair q written (the barrier above)
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + q), "r"(epoch) : "memory");
    }
  }
}

inline size_t long_fold_smem(int D, int nst) {
  return (size_t)nst * long_fold_stage_f(D) * sizeof(float) + (size_t)kLfMaxPW * kLfMaxTP * sizeof(uint32_t) +
         2 * kLfStages * sizeof(uint64_t);
}

// Launch the long-run pass (CTAs exit at once when the list is empty); with
// `pack`, mega runs are first gathered into stage images (plan + pack).
// Requires D % 4 == 0 and 16-byte aligned rows (the callers' vector path).
template <bool ADAM>
inline void launch_long_fold(LongRun* runs, const int64_t* nruns, int64_t cap, const uint32_t* ridx,
                             const float* rows, int D, const int64_t* bag_offs, int mode, AdamDev a, float* out,
                             int64_t* last_step, int64_t step, cudaStream_t s, const float* zrow = nullptr,
                             const LongFoldPack* pack = nullptr, bool expect_mega = true,
                             int smem_budget = kLfSmemBudget, const RowOut& ro = RowOut{}, bool hot_chain = false) {
  if (D > 32 * kLfMaxNC * kLfCols) raise(SKB_E_UNSUPPORTED, D, "long-run fold: dim > %d", 32 * kLfMaxNC * kLfCols);
  const int nc = long_fold_consumers(D);
  static const int env_pw = getenv("SKB_LF_PW") ? atoi(getenv("SKB_LF_PW")) : 0;
  static const int env_st = getenv("SKB_LF_STAGES") ? atoi(getenv("SKB_LF_STAGES")) : kLfStages;
  int npw = env_pw > 0 && env_pw <= kLfMaxPW ? env_pw : (nc > 4 ? 4 : 8 - nc);  // >= 4 producer warps
  int nst = env_st >= 2 && env_st <= kLfStages ? env_st : kLfStages;
  if (nst > long_fold_stages(D, smem_budget)) nst = long_fold_stages(D, smem_budget);
  if (npw > nst) npw = nst;  // a producer warp must never get a full ring lap ahead (parity waits)
  const int threads = 32 * (nc + npw);
  size_t sm = long_fold_smem(D, nst);
  // hot_chain (the caller saw a run >= kLfExclusiveRun positions recently:
  // the chain bounds the step):
  //  - the kernel asks for the maximum shared-memory carveout: an SM keeps
  //    the carveout of the blocks it holds, and the maximum leaves room for
  //    pack / index blocks beside a long-fold CTA (C4 3.26 -> 3.08 ms; on C5,
  //    without a hot chain, it cost 1%: off there);
  //  - SKB_LF_EXCLUSIVE=1 additionally claims a whole SM per CTA (no
  //    co-resident blocks on a chain's SM; measured neutral to slightly worse
  //    once units are scheduled dynamically, so off by default); 2 claims it
  //    for every launch (tests).
  static const int env_excl = getenv("SKB_LF_EXCLUSIVE") ? atoi(getenv("SKB_LF_EXCLUSIVE")) : 0;
  if ((env_excl == 1 && hot_chain) || env_excl > 1) {
    int dev = 0, optin = 0;
    SKB_CUDA(cudaGetDevice(&dev));
    SKB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    SKB_CUDA(cudaFuncGetAttributes(&fa, k_long_fold<ADAM>));
    if ((size_t)optin - fa.sharedSizeBytes > sm) sm = (size_t)optin - fa.sharedSizeBytes;  // + static smem = the SM's all
  }
  static size_t set = 0;  // attribute raised to the largest size launched so far
  if (set < sm) {
    SKB_CUDA(cudaFuncSetAttribute(k_long_fold<ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    set = sm;
  }
  {
    static const int env_carve = getenv("SKB_LF_CARVEOUT") ? atoi(getenv("SKB_LF_CARVEOUT")) : -2;
    const int want = env_carve != -2 ? env_carve : (hot_chain ? 100 : -1);
    static int cur = -1;  // cudaSharedmemCarveoutDefault
    if (want != cur) {
      SKB_CUDA(cudaFuncSetAttribute(k_long_fold<ADAM>, cudaFuncAttributePreferredSharedMemoryCarveout, want));
      cur = want;
    }
  }
  const float* packed = nullptr;
  const uint32_t* ready_flags = nullptr;
  bool direct = false;
  // mega runs as column-group units: by default packed into stage images
  // first (one TMA bulk copy per stage); SKB_LF_PACK=0: their producers
  // gather the group's columns straight from the gradient rows instead (no
  // pack pass, but a group CTA's random 32-byte gathers fall behind the
  // chain: C4 5.25 vs 4.45 ms/step measured)
  static const bool env_pack = getenv("SKB_LF_PACK") ? atoi(getenv("SKB_LF_PACK")) != 0 : true;
  // expect_mega: the caller saw long runs recently (else the planning
  // launches are skipped; mega runs then take the one-CTA path, same result)
  if (!env_pack && expect_mega && pack && pack->mlist && pack->cap_runs >= cap) {
    k_pack_plan<<<1, 1024, 0, s>>>(runs, nruns, cap, long_fold_tpg(D), long_fold_groups(D), mega_run_threshold(mode),
                                   INT64_MAX / 4, pack->mlist, pack->moff, pack->mcount, pack->morder);
    SKB_LAUNCH_CHECK();
    direct = true;
  } else if (env_pack && expect_mega && pack && pack->images && pack->cap_runs >= cap) {
    const int TPI = long_fold_tpi(D);
    k_pack_plan<<<1, 1024, 0, s>>>(runs, nruns, cap, TPI, long_fold_groups(D), mega_run_threshold(mode),
                                   pack->cap_images, pack->mlist, pack->moff, pack->mcount, pack->morder);
    SKB_LAUNCH_CHECK();
    const int sp = pack_sub(D);
    const size_t psm = pack_smem(D);
    static size_t pset = 0;
    if (pset < psm && psm > 48 * 1024) {
      SKB_CUDA(cudaFuncSetAttribute(k_pack_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
      pset = psm;
    }
    // with a pack stream (eager steps) the pack runs beside the long fold:
    // the fold streams every image the pack has already flagged and gathers
    // the others itself, so the hottest chain starts at once instead of
    // after the whole pack (C4: 0.54 ms off the critical path)
    const bool fork = pack->pstream && pack->ready;
    static bool mix_set = false;
    if (fork && !mix_set) {
      const int mix = getenv("SKB_LF_MIX_TEST") ? atoi(getenv("SKB_LF_MIX_TEST")) : 0;
      SKB_CUDA(cudaMemcpyToSymbol(g_lf_mix_test, &mix, sizeof(int)));
      mix_set = true;
    }
    cudaStream_t ps = s;
    if (fork) {
      SKB_CUDA(cudaEventRecord(pack->ev_fork, s));
      SKB_CUDA(cudaStreamWaitEvent(pack->pstream, pack->ev_fork, 0));
      ps = pack->pstream;
    }
    k_pack_rows<<<grid_for(pack->cap_images / long_fold_groups(D) * 256 + 256, 256, 4), 256, psm, ps>>>(
        runs, pack->mlist, pack->moff, pack->mcount, ridx, rows, zrow, D, bag_offs, mode, sp, pack->images,
        pack->morder, pack->ready);
    SKB_LAUNCH_CHECK();
    packed = pack->images;
    ready_flags = fork ? pack->ready : nullptr;
  }
  static const int64_t env_grid = getenv("SKB_LF_GRID") ? atoll(getenv("SKB_LF_GRID")) : 0;
  const int64_t gmax = env_grid > 0 ? env_grid : (int64_t)sm_count();
  int64_t grid = cap < gmax ? cap : gmax;
  if (grid < 1) grid = 1;
  if (pack && pack->wctr) SKB_CUDA(cudaMemsetAsync(pack->wctr, 0, sizeof(unsigned long long), s));
  k_long_fold<ADAM><<<(unsigned)grid, threads, sm, s>>>(runs, nruns, cap, ridx, rows, D, bag_offs, mode, a, out,
                                                        last_step, step, nst, zrow, packed,
                                                        (packed || direct) ? pack->mlist : nullptr,
                                                        (packed || direct) ? pack->morder : nullptr,
                                                        (packed || direct) ? pack->mcount : nullptr, ro, direct,
                                                        ready_flags, pack ? pack->wctr : nullptr);
  SKB_LAUNCH_CHECK();
  if (ready_flags) {  // later work on s (and the next pack plan) follows the pack
    SKB_CUDA(cudaEventRecord(pack->ev_join, pack->pstream));
    SKB_CUDA(cudaStreamWaitEvent(s, pack->ev_join, 0));
  }
}

// stage images needed to pack up to `rows` positions of mega runs
inline int64_t long_fold_pack_images(int64_t rows, int D) {
  const int64_t ng = long_fold_groups(D), tpi = long_fold_tpi(D);
  return ng * (rows / tpi + rows / kMegaRunMin + 1);
}

// ---------------------------------------------------------------------------
// Tolerance mode ("tree" fold, opt-in per table): a long run's gradients are
// summed as chunks of kTreeChunk positions folded in parallel, then the
// chunk partials folded in chunk order — a two-level reduction instead of
// np.add.at's serial chain, so a hot id costs memory bandwidth, not one FADD
// latency per position.  Error: |sum - exact| <= (kTreeChunk + n/kTreeChunk)
// * 2^-24 * sum|x| per column (the serial fold's bound is n * 2^-24 * sum|x|),
// the normwise tolerance SURVEY §7.3-5 allows; rows, slots and every run of
// <= kLongRun positions stay bit-exact.
// ---------------------------------------------------------------------------
constexpr int kTreeChunk = 256;

struct TreeWork {
  int64_t* chunk_off = nullptr;  // [cap + 1] first chunk of each run; [cap + ... ] total at [nruns]
  float* partial = nullptr;      // [chunk_cap, D]
  int64_t chunk_cap = 0;
};

inline int64_t tree_chunk_cap(int64_t n, int64_t runs_cap) { return n / kTreeChunk + runs_cap + 1; }

// exclusive scan of the runs' chunk counts (one block; total at chunk_off[R])
static __global__ void __launch_bounds__(1024) k_tree_plan(const LongRun* __restrict__ runs,
                                                           const int64_t* __restrict__ nruns, int64_t cap,
                                                           int64_t* __restrict__ chunk_off) {
  __shared__ int64_t warp_sum[32];
  __shared__ int64_t carry;
  const int64_t R = *nruns < cap ? *nruns : cap;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < R; b0 += blockDim.x) {
    const int64_t r = b0 + threadIdx.x;
    int64_t c = 0;
    if (r < R) c = ((int64_t)runs[r].je - runs[r].jh + kTreeChunk - 1) / kTreeChunk;
    int64_t inc = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) warp_sum[w] = inc;
    __syncthreads();
    int64_t base = carry;
    for (int q = 0; q < w; ++q) base += warp_sum[q];
    if (r < R) chunk_off[r] = base + inc - c;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = base + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) chunk_off[R] = carry;
}

// one warp per (chunk, 128-column slice): fold the chunk's positions with four
// interleaved accumulators (positions p, p+1, p+2, p+3 mod 4), then combine
template <bool MEAN>
static __global__ void __launch_bounds__(256) k_tree_partial(const LongRun* __restrict__ runs,
                                                             const int64_t* __restrict__ nruns, int64_t cap,
                                                             const int64_t* __restrict__ chunk_off,
                                                             const uint32_t* __restrict__ ridx,
                                                             const float* __restrict__ rows, int D,
                                                             const int64_t* __restrict__ bag_offs,
                                                             const float* __restrict__ zrow,
                                                             float* __restrict__ partial, int64_t chunk_cap) {
  const int64_t R = *nruns < cap ? *nruns : cap;
  const int64_t total = chunk_off[R] < chunk_cap ? chunk_off[R] : chunk_cap;
  const int slices = (D + 127) / 128;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wu = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; wu < total * slices; wu += nw) {
    const int64_t ch = wu / slices;
    const int c = (int)(wu - ch * slices) * 128 + lane * 4;
    int64_t lo = 0, hi = R;  // run r with chunk_off[r] <= ch < chunk_off[r + 1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(chunk_off + mid) <= ch) lo = mid; else hi = mid;
    }
    const LongRun run = runs[lo];
    const int64_t p0 = run.jh + (ch - __ldg(chunk_off + lo)) * kTreeChunk;
    const int64_t p1 = p0 + kTreeChunk < (int64_t)run.je ? p0 + kTreeChunk : (int64_t)run.je;
    if (c >= D) continue;
    float4 acc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = p0;
    for (; p + 4 <= p1; p += 4) {
      float4 x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t g = __ldg(ridx + p + k);
        x[k] = ldg4((g == 0xFFFFFFFFu ? zrow : rows + (int64_t)g * D) + c);
        if (MEAN) x[k] = vdiv4(x[k], (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g)));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = add4(acc[k], x[k]);
    }
    for (; p < p1; ++p) {
      const uint32_t g = __ldg(ridx + p);
      float4 x = ldg4((g == 0xFFFFFFFFu ? zrow : rows + (int64_t)g * D) + c);
      if (MEAN) x = vdiv4(x, (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g)));
      acc[0] = add4(acc[0], x);
    }
    st4(partial + ch * D + c, add4(add4(acc[0], acc[1]), add4(acc[2], acc[3])));
  }
}

// one warp per (run, 128-column slice): fold the run's chunk partials in chunk
// order, then Adam (ADAM) or write out[key]
template <bool ADAM>
static __global__ void __launch_bounds__(256) k_tree_final(const LongRun* __restrict__ runs,
                                                           const int64_t* __restrict__ nruns, int64_t cap,
                                                           const int64_t* __restrict__ chunk_off,
                                                           const float* __restrict__ partial, int64_t chunk_cap,
                                                           int D, AdamDev a, float* __restrict__ out,
                                                           int64_t* __restrict__ last_step, int64_t step) {
  const int64_t R = *nruns < cap ? *nruns : cap;
  const int slices = (D + 127) / 128;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wu = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; wu < R * slices; wu += nw) {
    const int64_t r = wu / slices;
    const int c = (int)(wu - r * slices) * 128 + lane * 4;
    const LongRun run = runs[r];
    if (c < D) {
      const int64_t cb = __ldg(chunk_off + r), ce = __ldg(chunk_off + r + 1) < chunk_cap ? __ldg(chunk_off + r + 1)
                                                                                       : chunk_cap;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t ch = cb; ch < ce; ++ch) acc = add4(acc, ldg4(partial + ch * D + c));
      if constexpr (ADAM) {
        float* row = out + (int64_t)run.key * (3 * D);
        float4 p = ldg4(row + c), m = ldg4(row + D + c), v = ldg4(row + 2 * D + c);
        adam1(p.x, m.x, v.x, acc.x, a);
        adam1(p.y, m.y, v.y, acc.y, a);
        adam1(p.z, m.z, v.z, acc.z, a);
        adam1(p.w, m.w, v.w, acc.w, a);
        st4(row + c, p);
        st4(row + D + c, m);
        st4(row + 2 * D + c, v);
      } else {
        st4(out + (int64_t)run.key * D + c, acc);
      }
    }
    if (ADAM && lane == 0 && wu % slices == 0 && step >= 0) last_step[run.key] = step;
  }
}

// Tolerance-mode long-run pass (D % 4 == 0): plan, chunk partials, final fold.
template <bool ADAM>
inline void launch_long_fold_tree(LongRun* runs, const int64_t* nruns, int64_t cap, const uint32_t* ridx,
                                  const float* rows, int D, const int64_t* bag_offs, int mode, AdamDev a, float* out,
                                  int64_t* last_step, int64_t step, cudaStream_t s, const float* zrow,
                                  const TreeWork& w) {
  k_tree_plan<<<1, 1024, 0, s>>>(runs, nruns, cap, w.chunk_off);
  SKB_LAUNCH_CHECK();
  const int slices = (D + 127) / 128;
  const unsigned grid = grid_for(w.chunk_cap * slices * 32, 256, 8);
  if (mode == 1)
    k_tree_partial<true><<<grid, 256, 0, s>>>(runs, nruns, cap, w.chunk_off, ridx, rows, D, bag_offs, zrow, w.partial,
                                              w.chunk_cap);
  else
    k_tree_partial<false><<<grid, 256, 0, s>>>(runs, nruns, cap, w.chunk_off, ridx, rows, D, bag_offs, zrow,
                                               w.partial, w.chunk_cap);
  SKB_LAUNCH_CHECK();
  k_tree_final<ADAM><<<grid_for((cap + 1) * slices * 32, 256, 4), 256, 0, s>>>(
      runs, nruns, cap, w.chunk_off, w.partial, w.chunk_cap, D, a, out, last_step, step);
  SKB_LAUNCH_CHECK();
}

}  // namespace skb
