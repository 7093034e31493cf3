// longfold.cuh — bit-exact in-order fold of LONG runs (hot zipf ids).
//
// The reference pre-aggregates a row's gradients with np.add.at, a strict
// left fold in input order (sharding.py:289).  For a hot id with ~10^6
// positions that chain is inherently serial in fp32; what must not be serial
// is the memory traffic.  Runs longer than kLongRun are deferred by the main
// fold kernels into a device list; here one CTA owns one long run: warps
// 1..7 stage the run's gradient rows tile by tile into shared memory with
// cp.async (double buffered), while warp 0 folds the previous tile from
// shared memory in position order and finally applies Adam (or writes the
// folded row).  Cost ~ one FADD latency per position instead of one DRAM
// round trip.
#pragma once
#include "common.cuh"
#include "table.cuh"

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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// rows: gradient source rows (dpooled [G, D] or per-position grads [N, D]);
// ridx[j]: row of sorted position j; mean: divide by len(bag ridx[j]).
// ADAM: update arena row `key` (and last_step); else write out[key * D].
template <bool ADAM>
__global__ void __launch_bounds__(256) k_long_fold(const LongRun* __restrict__ runs, const int64_t* __restrict__ nruns,
                                                   int64_t cap, const uint32_t* __restrict__ ridx,
                                                   const float* __restrict__ rows, int D,
                                                   const int64_t* __restrict__ bag_offs, int mode, AdamDev a,
                                                   float* __restrict__ out, int64_t* __restrict__ last_step,
                                                   int64_t step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TP = 16384 / D;  // positions per tile: 64 KB of rows per buffer
  float* buf = reinterpret_cast<float*>(smem_raw);                    // [2][TP][D]
  float* lenb = buf + 2 * (int64_t)TP * D;                             // [2][TP] 1/len helpers (lengths)
  const int64_t R = *nruns < cap ? *nruns : cap;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = D / 4;  // 16-byte chunks per row
  for (int64_t r = blockIdx.x; r < R; r += gridDim.x) {
    const LongRun run = runs[r];
    const int64_t jb = run.jh, je = run.je;
    const int64_t ntile = (je - jb + TP - 1) / TP;
    // stage tile t into buffer t & 1 (warps 1..7, or all warps for tile 0)
    auto stage = [&](int64_t t, int tid0, int nthr) {
      const int64_t p0 = jb + t * TP;
      const int np = (int)(je - p0 < TP ? je - p0 : TP);
      float* dst = buf + (int64_t)(t & 1) * TP * D;
      float* ld = lenb + (int64_t)(t & 1) * TP;
      (void)ld;
      if (mode == 1) {  // mean: the staging warps divide, the folding warp only adds
        for (int i = threadIdx.x - tid0; i < np * chunks; i += nthr) {
          const int p = i / chunks, ch = i - p * chunks;
          const uint32_t g = __ldg(ridx + p0 + p);
          const float l = (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g));
          float4 x = ldg4(rows + (int64_t)g * D + ch * 4);
          x = make_float4(__fdiv_rn(x.x, l), __fdiv_rn(x.y, l), __fdiv_rn(x.z, l), __fdiv_rn(x.w, l));
          st4(dst + (int64_t)p * D + ch * 4, x);
        }
      } else {
        for (int i = threadIdx.x - tid0; i < np * chunks; i += nthr) {
          const int p = i / chunks, ch = i - p * chunks;
          const uint32_t g = __ldg(ridx + p0 + p);
          cp_async16(dst + (int64_t)p * D + ch * 4, rows + (int64_t)g * D + ch * 4);
        }
      }
      cp_async_commit();
    };
    stage(0, 0, blockDim.x);
    cp_async_wait_all();
    __syncthreads();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t t = 0; t < ntile; ++t) {
      if (warp > 0 && t + 1 < ntile) stage(t + 1, 32, blockDim.x - 32);
      if (warp == 0 && lane < chunks) {
        const int64_t p0 = jb + t * TP;
        const int np = (int)(je - p0 < TP ? je - p0 : TP);
        const float* src = buf + (int64_t)(t & 1) * TP * D + lane * 4;
        const float* ld = lenb + (int64_t)(t & 1) * TP;
        (void)ld;
#pragma unroll 8
        for (int p = 0; p < np; ++p) acc = add4(acc, *reinterpret_cast<const float4*>(src + (int64_t)p * D));
      }
      if (warp > 0) cp_async_wait_all();
      __syncthreads();
    }
    if (warp == 0 && lane < chunks) {
      const int c = lane * 4;
      if constexpr (ADAM) {
        float* row = out + (int64_t)run.key * (3 * D);
        float4 p = *reinterpret_cast<float4*>(row + c), m = *reinterpret_cast<float4*>(row + D + c),
               v = *reinterpret_cast<float4*>(row + 2 * D + c);
        adam1(p.x, m.x, v.x, acc.x, a);
        adam1(p.y, m.y, v.y, acc.y, a);
        adam1(p.z, m.z, v.z, acc.z, a);
        adam1(p.w, m.w, v.w, acc.w, a);
        st4(row + c, p);
        st4(row + D + c, m);
        st4(row + 2 * D + c, v);
        if (lane == 0 && step >= 0) last_step[run.key] = step;
      } else {
        st4(out + (int64_t)run.key * D + c, acc);
      }
    }
    // D > 128 needs more lanes than warp 0 has: handled by a second pass of
    // column groups (lanes cover 128 columns per pass)
    for (int cbase = 128; cbase < D; cbase += 128) {
      __syncthreads();
      // recompute for columns [cbase, cbase + 128) by re-streaming the run
      // (rare: only dims > 128), same order, same arithmetic
      float4 acc2 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (warp == 0 && cbase + lane * 4 < D) {
        for (int64_t j = jb; j < je; ++j) {
          const uint32_t g = __ldg(ridx + j);
          float4 x = ldg4(rows + (int64_t)g * D + cbase + lane * 4);
          if (mode == 1) {
            const float l = (float)(__ldg(bag_offs + g + 1) - __ldg(bag_offs + g));
            x = make_float4(__fdiv_rn(x.x, l), __fdiv_rn(x.y, l), __fdiv_rn(x.z, l), __fdiv_rn(x.w, l));
          }
          acc2 = add4(acc2, x);
        }
        const int c = cbase + lane * 4;
        if constexpr (ADAM) {
          float* row = out + (int64_t)run.key * (3 * D);
          float4 p = *reinterpret_cast<float4*>(row + c), m = *reinterpret_cast<float4*>(row + D + c),
                 v = *reinterpret_cast<float4*>(row + 2 * D + c);
          adam1(p.x, m.x, v.x, acc2.x, a);
          adam1(p.y, m.y, v.y, acc2.y, a);
          adam1(p.z, m.z, v.z, acc2.z, a);
          adam1(p.w, m.w, v.w, acc2.w, a);
          st4(row + c, p);
          st4(row + D + c, m);
          st4(row + 2 * D + c, v);
        } else {
          st4(out + (int64_t)run.key * D + c, acc2);
        }
      }
    }
    __syncthreads();
  }
}

inline size_t long_fold_smem(int D) {
  const int TP = 16384 / D;
  return (size_t)2 * TP * D * sizeof(float) + (size_t)2 * TP * sizeof(float);
}

// Launch the long-run pass (CTAs exit at once when the list is empty).
template <bool ADAM>
inline void launch_long_fold(const LongRun* runs, const int64_t* nruns, int64_t cap, const uint32_t* ridx,
                             const float* rows, int D, const int64_t* bag_offs, int mode, AdamDev a, float* out,
                             int64_t* last_step, int64_t step, cudaStream_t s) {
  const size_t sm = long_fold_smem(D);
  static size_t set = 0;
  if (set < sm) {
    SKB_CUDA(cudaFuncSetAttribute(k_long_fold<ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    set = sm;
  }
  int64_t grid = cap < 2 * (int64_t)sm_count() ? cap : 2 * (int64_t)sm_count();
  if (grid < 1) grid = 1;
  k_long_fold<ADAM><<<(unsigned)grid, 256, sm, s>>>(runs, nruns, cap, ridx, rows, D, bag_offs, mode, a, out,
                                                    last_step, step);
  SKB_LAUNCH_CHECK();
}

}  // namespace skb
