// longfold.cuh — bit-exact in-order fold of LONG runs (hot zipf ids).
//
// The reference pre-aggregates a row's gradients with np.add.at, a strict
// left fold in input order (sharding.py:289).  For a hot id with ~10^6
// positions that chain is inherently serial in fp32; what must not be serial
// is the memory traffic.  Runs longer than kLongRun are deferred by the main
// fold kernels into a device list; here one CTA owns one long run at a time:
// a producer warp streams the run's gradient rows through a TMA ring while
// consumer warps fold them in position order (details at k_long_fold).
// Cost ~ one FADD latency per position instead of one DRAM round trip.
#pragma once
#include <cstdlib>

#include "common.cuh"
#include "table.cuh"
#include "tma.cuh"

namespace skb {

constexpr int kLongRun = 32;  // runs longer than this are deferred

struct LongRun {
  uint32_t key, jh, je, pad;
};

__device__ __forceinline__ void push_long_run(LongRun* list, int64_t* count, int64_t cap, uint32_t key, uint32_t jh,
                                              uint32_t je) {
  unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(count), 1ull);
  if ((int64_t)i < cap) list[i] = LongRun{key, jh, je, 0};
}

// One CTA folds one long run at a time (runs strided over CTAs).  Consumer
// warps 0..NC-1 each own 32 columns (one per lane) and fold a stage's
// rows in position order from +0; the remaining NPW warps are producers
// filling a kLfStages-deep shared-memory ring of kLfStageBytes stages with
// 16-byte cp.async copies of the run's gradient rows.  Producer warp pw owns
// the stages it = pw (mod NPW), so NPW stages are being addressed (row index
// loads) and copied at once; each lane signals the stage's `full` mbarrier
// when ITS copies land (cp.async.mbarrier.arrive.noinc).  ~kLfStages x 16 KB
// stay in flight per CTA and the single serial FADD chain is fed at ~one
// row per add latency.  (Small per-row TMA bulk
// copies were measured slower: per-copy issue cost; the earlier
// double-buffered version was bound by one DRAM round trip per tile.)
// rows: gradient source rows (dpooled [G, D] or per-position grads [N, D]);
// ridx[j]: row of sorted position j; mode 1 (mean): divide by len(bag ridx[j]).
// ADAM: update arena row `key` (and last_step); else write out[key * D].
constexpr int kLfStages = 12;
constexpr int kLfStageBytes = 16384;
constexpr int kLfMaxTP = 256;   // rows per stage cap (small dims)
constexpr int kLfMaxPW = 8;     // producer warps (index buffers)

// rows per stage: kLfStageBytes of rows, at most kLfMaxTP (small dims)
__host__ __device__ inline int long_fold_tp(int D) {
  const int tp = kLfStageBytes / (4 * D);
  return tp < 1 ? 1 : (tp > kLfMaxTP ? kLfMaxTP : tp);
}
constexpr int kLfMaxNC = 16;  // consumer warps
constexpr int kLfCols = 4;    // columns per consumer lane: dims up to 32 * kLfMaxNC * kLfCols = 2048
__host__ __device__ inline int long_fold_consumers(int D) {
  const int nc = (D + 31) / 32;
  return nc < kLfMaxNC ? nc : kLfMaxNC;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <bool ADAM>
__global__ void k_long_fold(const LongRun* __restrict__ runs, const int64_t* __restrict__ nruns, int64_t cap,
                            const uint32_t* __restrict__ ridx, const float* __restrict__ rows, int D,
                            const int64_t* __restrict__ bag_offs, int mode, AdamDev a, float* __restrict__ out,
                            int64_t* __restrict__ last_step, int64_t step, int nst,
                            const float* __restrict__ zrow) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int TP = long_fold_tp(D);
  const int64_t stage_f = (int64_t)TP * D;  // floats per stage
  float* buf = reinterpret_cast<float*>(smem_raw);
  uint32_t* idx = reinterpret_cast<uint32_t*>(buf + kLfStages * stage_f);  // [kLfMaxPW][kLfMaxTP]
  uint64_t* full = reinterpret_cast<uint64_t*>(idx + kLfMaxPW * kLfMaxTP);
  uint64_t* empty = full + kLfStages;
  const int NC = long_fold_consumers(D);
  const int64_t R = *nruns < cap ? *nruns : cap;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLfStages; ++s) {
      mbar_init(&full[s], 32);  // the owning producer warp's lanes
      mbar_init(&empty[s], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t it = 0;  // stage sequence number, identical in producers and consumers
  if (warp >= NC) {  // ---------------- producers: warp pw fills stages it = pw (mod NPW) ----------------
    const int pw = warp - NC, NPW = (int)(blockDim.x >> 5) - NC;
    const int cpr = D / 4;  // 16-byte chunks per row
    for (int64_t r = blockIdx.x; r < R; r += gridDim.x) {
      const LongRun run = runs[r];
      for (int64_t p0 = run.jh; p0 < run.je; p0 += TP, ++it) {
        if ((int)(it % (uint32_t)NPW) != pw) continue;
        const int s = (int)(it % (uint32_t)nst);
        const uint32_t ph = (it / (uint32_t)nst) & 1u;
        const int np = (int)((int64_t)run.je - p0 < TP ? (int64_t)run.je - p0 : TP);
        const int items = np * cpr;
        float* dst = buf + s * stage_f;
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
        __syncwarp();                          // ix is rewritten by this warp's next stage
      }
    }
    return;
  }
  // ---------------- consumers: warp w owns columns 32 w + lane (+ 32 NC, ...) ----------------
  // one column per lane: a row costs each warp one LDS + one FADD (the fp32
  // chain's 4-cycle latency), not four FADDs on one fma pipe; dims above
  // 32 * kLfMaxNC give a lane up to kLfCols columns
  const int c0 = warp * 32 + lane;
  const int cstep = 32 * NC;
  for (int64_t r = blockIdx.x; r < R; r += gridDim.x) {
    const LongRun run = runs[r];
    float acc[kLfCols];
#pragma unroll
    for (int q = 0; q < kLfCols; ++q) acc[q] = 0.f;
    for (int64_t p0 = run.jh; p0 < run.je; p0 += TP, ++it) {
      const int s = (int)(it % (uint32_t)nst);
      const uint32_t ph = (it / (uint32_t)nst) & 1u;
      const int np = (int)((int64_t)run.je - p0 < TP ? (int64_t)run.je - p0 : TP);
      mbar_wait(&full[s], ph);
#pragma unroll
      for (int q = 0; q < kLfCols; ++q) {
        const int c = c0 + q * cstep;
        if (c < D) {
          const float* src = buf + s * stage_f + c;
#pragma unroll 16
          for (int p = 0; p < np; ++p) acc[q] = __fadd_rn(acc[q], src[(int64_t)p * D]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int q = 0; q < kLfCols; ++q) {
      const int c = c0 + q * cstep;
      if (c >= D) continue;
      if constexpr (ADAM) {
        float* row = out + (int64_t)run.key * (3 * D);
        float p = row[c], m = row[D + c], v = row[2 * D + c];
        adam1(p, m, v, acc[q], a);
        row[c] = p;
        row[D + c] = m;
        row[2 * D + c] = v;
        if (c == 0 && step >= 0) last_step[run.key] = step;
      } else {
        out[(int64_t)run.key * D + c] = acc[q];
      }
    }
  }
}

inline size_t long_fold_smem(int D) {
  const int TP = long_fold_tp(D);
  return (size_t)kLfStages * TP * D * sizeof(float) + (size_t)kLfMaxPW * kLfMaxTP * sizeof(uint32_t) +
         2 * kLfStages * sizeof(uint64_t);
}

// Launch the long-run pass (CTAs exit at once when the list is empty).
// Requires D % 4 == 0 and 16-byte aligned rows (the callers' vector path).
template <bool ADAM>
inline void launch_long_fold(const LongRun* runs, const int64_t* nruns, int64_t cap, const uint32_t* ridx,
                             const float* rows, int D, const int64_t* bag_offs, int mode, AdamDev a, float* out,
                             int64_t* last_step, int64_t step, cudaStream_t s, const float* zrow = nullptr) {
  if (D > 32 * kLfMaxNC * kLfCols) raise(SKB_E_UNSUPPORTED, D, "long-run fold: dim > %d", 32 * kLfMaxNC * kLfCols);
  const size_t sm = long_fold_smem(D);
  static size_t set = 0;
  if (set < sm) {
    SKB_CUDA(cudaFuncSetAttribute(k_long_fold<ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    set = sm;
  }
  const int nc = long_fold_consumers(D);
  static const int env_pw = getenv("SKB_LF_PW") ? atoi(getenv("SKB_LF_PW")) : 0;
  static const int env_st = getenv("SKB_LF_STAGES") ? atoi(getenv("SKB_LF_STAGES")) : kLfStages;
  const int npw = env_pw > 0 && env_pw <= kLfMaxPW ? env_pw : (nc > 4 ? 4 : 8 - nc);  // >= 4 producer warps
  const int threads = 32 * (nc + npw);
  int nst = env_st >= 2 && env_st <= kLfStages ? env_st : kLfStages;
  if (nst < npw) nst = npw;  // a producer warp must never get a full ring lap ahead (parity waits)
  int64_t grid = cap < (int64_t)sm_count() ? cap : (int64_t)sm_count();
  if (grid < 1) grid = 1;
  k_long_fold<ADAM><<<(unsigned)grid, threads, sm, s>>>(runs, nruns, cap, ridx, rows, D, bag_offs, mode, a, out,
                                                        last_step, step, nst, zrow);
  SKB_LAUNCH_CHECK();
}

}  // namespace skb
