// p2p.cu — peer-memory transport of the row-sharded exchange.
//
// The NCCL exchange moves rows and gradients through staging buffers:
// owner gather -> send buffer -> all_to_all_v -> requester buffer.  Here the
// producing kernel writes each row straight into the consuming rank's
// window (CUDA IPC memory of the peer, NVLink/NVSwitch P2P stores between
// GPUs; the same code on one GPU when ranks share it):
//   skb_p2p_send_rows   owner: row of every id it received from rank j,
//                       gathered from its arena and stored at
//                       window_j[base_j + i]   (rows back to requesters)
//   skb_p2p_send_grads  requester: folded gradient of every local unique id
//                       stored at window_owner[base_owner + i]
// Both end with a system-scope fence; the caller orders the peers' reads
// after the writes with a stream-ordered barrier (an NCCL all-reduce of one
// element) or a host barrier.
#include <cstring>
#include <mutex>

#include <cuda.h>

#include "common.cuh"
#include "p2p.cuh"
#include "pool.cuh"
#include "table.cuh"

namespace skb {

// out row q (q-th id received, rank-ordered segments pre[j]..pre[j+1]) ->
// peer window j at row base[j] + (q - pre[j]); source row = src[idx[q]] with
// row stride sstride (arena rows through the slot list, or plain rows)
template <int VEC>
__global__ void __launch_bounds__(256) k_p2p_scatter(const float* __restrict__ src, int64_t sstride,
                                                     const int64_t* __restrict__ slot_of_u,
                                                     const int64_t* __restrict__ idx, int64_t nq, int D,
                                                     const int64_t* __restrict__ pre, int S,
                                                     float* const* __restrict__ peers,
                                                     const int64_t* __restrict__ base) {
  using V = typename VecT<VEC>::T;
  constexpr int U = 4;
  const int per = D / VEC;
  const int64_t total = nq * per;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b0 < total; b0 += stride * U) {
    V v[U];
    float* dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = b0 + u * stride;
      dst[u] = nullptr;
      if (t < total) {
        const int64_t q = t / per;
        const int c = (int)(t - q * per) * VEC;
        int64_t r = idx ? __ldg(idx + q) : q;
        if (slot_of_u) r = __ldg(slot_of_u + r);
        v[u] = vload<VEC>(src + r * sstride + c);
        const int j = seg_of(pre, S, q);
        dst[u] = peers[j] + (__ldg(base + j) + (q - __ldg(pre + j))) * D + c;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u]) vstore<VEC>(dst[u], v[u]);
  }
  __threadfence_system();
}

template <class... A>
static void launch_p2p(int64_t nq, int D, bool v4, cudaStream_t s, A... args) {
  if (nq <= 0) return;
  if (v4)
    k_p2p_scatter<4><<<grid_for((nq * (D / 4) + 3) / 4, 256), 256, 0, s>>>(args...);
  else
    k_p2p_scatter<1><<<grid_for((nq * D + 3) / 4, 256), 256, 0, s>>>(args...);
  SKB_LAUNCH_CHECK();
}

// arena rows through a uint32 slot per received position (owner side of the
// fused multi-GPU step): 16-byte loads from HBM, 16-byte stores over NVLink
template <int VEC>
__global__ void __launch_bounds__(256) k_p2p_slot_rows(const float* __restrict__ arena, int64_t stride,
                                                       const uint32_t* __restrict__ slot, int64_t nq, int D,
                                                       const int64_t* __restrict__ pre, int S,
                                                       float* const* __restrict__ peers,
                                                       const int64_t* __restrict__ base) {
  using V = typename VecT<VEC>::T;
  constexpr int U = 4;
  const int per = D / VEC;
  const int64_t total = nq * per;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b0 < total; b0 += gs * U) {
    V v[U];
    float* dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = b0 + u * gs;
      dst[u] = nullptr;
      if (t < total) {
        const int64_t q = t / per;
        const int c = (int)(t - q * per) * VEC;
        v[u] = vload<VEC>(arena + (int64_t)__ldg(slot + q) * stride + c);
        const int j = seg_of(pre, S, q);
        dst[u] = peers[j] + (__ldg(base + j) + (q - __ldg(pre + j))) * D + c;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u]) vstore<VEC>(dst[u], v[u]);
  }
  __threadfence_system();
}

__global__ void __launch_bounds__(256) k_p2p_ids(const int64_t* __restrict__ ids, int64_t n,
                                                 const int64_t* __restrict__ pre, int S, int64_t* const* __restrict__ peers,
                                                 const int64_t* __restrict__ base) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int j = seg_of(pre, S, q);
    peers[j][__ldg(base + j) + (q - __ldg(pre + j))] = __ldg(ids + q);
  }
  __threadfence_system();
}

// count row of this rank stored into row `me` of every peer's count matrix
__global__ void k_p2p_counts(const int64_t* __restrict__ counts, int S, int me, int64_t* const* __restrict__ peers) {
  for (int t = threadIdx.x; t < S * S; t += blockDim.x) {
    const int j = t / S, k = t - j * S;
    peers[j][(int64_t)me * S + k] = __ldg(counts + k);
  }
  __threadfence_system();
}

// ---------------------------------------------------------------------------
// Stream-ordered barrier over peer memory: each rank writes the epoch into
// its slot of every peer's flag word array (a stream memory operation: the
// write follows all prior work of the stream, behind a memory barrier, so
// that work's peer stores are visible first), then the stream waits until
// every peer's slot in its own array reached the epoch.  No kernel spins, no
// host round trip, no NCCL; works between GPUs (NVLink) and between
// processes sharing one GPU.
// ---------------------------------------------------------------------------
typedef CUresult (*PfnWaitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PfnWriteValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
static PfnWaitValue64 g_wait64 = nullptr;
static PfnWriteValue64 g_write64 = nullptr;

static bool memops_init() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = cudaDriverEntryPointSymbolNotFound;
    void* f1 = nullptr;
    void* f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f1, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue64", &f2, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
      g_wait64 = reinterpret_cast<PfnWaitValue64>(f1);
      g_write64 = reinterpret_cast<PfnWriteValue64>(f2);
    }
    cudaGetLastError();
  });
  return g_wait64 && g_write64;
}

void p2p_send_slot_rows(const float* arena, int64_t stride, const uint32_t* slot, int64_t nq, int D,
                        const int64_t* pre, int S, float* const* peers, const int64_t* base, cudaStream_t s) {
  if (nq <= 0) return;
  if (D % 4 == 0)
    k_p2p_slot_rows<4><<<grid_for((nq * (D / 4) + 3) / 4, 256), 256, 0, s>>>(arena, stride, slot, nq, D, pre, S,
                                                                            peers, base);
  else
    k_p2p_slot_rows<1><<<grid_for((nq * D + 3) / 4, 256), 256, 0, s>>>(arena, stride, slot, nq, D, pre, S, peers,
                                                                      base);
  SKB_LAUNCH_CHECK();
}

void p2p_send_segments(const float* rows, int64_t n, int D, const int64_t* pre, int S, float* const* peers,
                       const int64_t* base, cudaStream_t s) {
  launch_p2p(n, D, D % 4 == 0 && (uintptr_t)rows % 16 == 0, s, rows, (int64_t)D, (const int64_t*)nullptr,
             (const int64_t*)nullptr, n, D, pre, S, peers, base);
}

void p2p_send_ids(const int64_t* ids, int64_t n, const int64_t* pre, int S, int64_t* const* peers,
                  const int64_t* base, cudaStream_t s) {
  if (n <= 0) return;
  k_p2p_ids<<<grid_for(n, 256), 256, 0, s>>>(ids, n, pre, S, peers, base);
  SKB_LAUNCH_CHECK();
}

}  // namespace skb

using namespace skb;

extern "C" {

int skb_ipc_alloc(int64_t bytes, void** ptr_out, void* handle_out) {
  SKB_API_BEGIN
  void* p = nullptr;
  SKB_CUDA(cudaMalloc(&p, bytes > 0 ? bytes : 16));
  SKB_CUDA(cudaMemset(p, 0, bytes > 0 ? bytes : 16));  // flag words start at epoch 0
  cudaIpcMemHandle_t h;
  SKB_CUDA(cudaIpcGetMemHandle(&h, p));
  memcpy(handle_out, &h, sizeof h);
  *ptr_out = p;
  SKB_API_END
}

int skb_ipc_open(const void* handle, void** ptr_out) {
  SKB_API_BEGIN
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  SKB_CUDA(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  SKB_API_END
}

int skb_ipc_close(void* ptr) {
  SKB_API_BEGIN
  SKB_CUDA(cudaIpcCloseMemHandle(ptr));
  SKB_API_END
}

int skb_ipc_free(void* ptr) {
  SKB_API_BEGIN
  SKB_CUDA(cudaFree(ptr));
  SKB_API_END
}

int skb_p2p_send_rows(skb_table_t h, const int64_t* slots_u, const int64_t* inv, int64_t nrecv,
                      const int64_t* recv_prefix, int32_t num_ranks, float* const* peer_windows,
                      const int64_t* dst_base, void* stream) {
  SKB_API_BEGIN
  Table* t = table_from(h);
  const int D = (int)t->dim;
  const bool v4 = D % 4 == 0;
  launch_p2p(nrecv, D, v4, as_stream(stream), (const float*)t->arena, (int64_t)3 * D, slots_u, inv, nrecv, D,
             recv_prefix, (int)num_ranks, peer_windows, dst_base);
  SKB_API_END
}

int skb_p2p_memops_supported(int32_t* supported_host) {
  SKB_API_BEGIN
  *supported_host = memops_init() ? 1 : 0;
  SKB_API_END
}

int skb_p2p_barrier(const int64_t* flag_ptrs_host, int32_t num_ranks, int32_t rank, int64_t epoch, void* stream) {
  SKB_API_BEGIN
  if (!memops_init()) raise(SKB_E_UNSUPPORTED, 0, "stream memory operations unavailable");
  if (rank < 0 || rank >= num_ranks) raise(SKB_E_ARG, rank, "rank out of range");
  CUstream s = reinterpret_cast<CUstream>(as_stream(stream));
  for (int j = 0; j < num_ranks; ++j) {
    if (j == rank) continue;
    const CUresult r = g_write64(s, (CUdeviceptr)(flag_ptrs_host[j] + 8 * (int64_t)rank), (cuuint64_t)epoch, 0);
    if (r != CUDA_SUCCESS) raise(SKB_E_CUDA, r, "cuStreamWriteValue64 failed (%d)", (int)r);
  }
  for (int j = 0; j < num_ranks; ++j) {
    if (j == rank) continue;
    const CUresult r = g_wait64(s, (CUdeviceptr)(flag_ptrs_host[rank] + 8 * (int64_t)j), (cuuint64_t)epoch,
                                CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) raise(SKB_E_CUDA, r, "cuStreamWaitValue64 failed (%d)", (int)r);
  }
  SKB_API_END
}

int skb_p2p_put_counts(const int64_t* counts, int32_t num_ranks, int32_t rank, int64_t* const* peer_windows,
                       void* stream) {
  SKB_API_BEGIN
  k_p2p_counts<<<1, 256, 0, as_stream(stream)>>>(counts, num_ranks, rank, peer_windows);
  SKB_LAUNCH_CHECK();
  SKB_API_END
}

int skb_p2p_send_grads(const float* rows, int64_t dim, int64_t n, const int64_t* seg_prefix, int32_t num_ranks,
                       float* const* peer_windows, const int64_t* dst_base, void* stream) {
  SKB_API_BEGIN
  const int D = (int)dim;
  const bool v4 = D % 4 == 0 && (uintptr_t)rows % 16 == 0;
  launch_p2p(n, D, v4, as_stream(stream), rows, (int64_t)D, (const int64_t*)nullptr, (const int64_t*)nullptr, n,
             D, seg_prefix, (int)num_ranks, peer_windows, dst_base);
  SKB_API_END
}

}  // extern "C"
