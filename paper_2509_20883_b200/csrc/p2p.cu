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

#include "common.cuh"
#include "pool.cuh"
#include "table.cuh"

namespace skb {

// segment of x in the ascending prefix array pre[0..S] (pre[S] = total)
__device__ __forceinline__ int seg_of(const int64_t* __restrict__ pre, int S, int64_t x) {
  int lo = 0, hi = S;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(pre + mid) <= x) lo = mid; else hi = mid;
  }
  return lo;
}

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

}  // namespace skb

using namespace skb;

extern "C" {

int skb_ipc_alloc(int64_t bytes, void** ptr_out, void* handle_out) {
  SKB_API_BEGIN
  void* p = nullptr;
  SKB_CUDA(cudaMalloc(&p, bytes > 0 ? bytes : 16));
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
