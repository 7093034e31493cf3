// graph.cuh — CUDA-graph replay of the fused step's device work.
//
// Each phase of the fused step (index phase on the table's index stream, pool
// and fold+Adam on the caller's stream) is a fixed sequence of launches once
// the batch layout, buffers and table arrays are fixed.  In graph mode the
// first call with a new signature captures the phase (single-stream capture,
// so the cross-stream events stay outside the graph), later calls replay it
// with one cudaGraphLaunch.  The only per-step kernel arguments — the global
// step and the host-computed Adam scalars — are patched into the captured
// kernel nodes before each launch (cudaGraphExecKernelNodeSetParams); every
// other argument is a pointer or size covered by the signature key.  The
// host keeps all bookkeeping (pipeline counters, reservation bound, counter
// snapshots) exactly as in eager mode.
#pragma once
#include <cstring>
#include <vector>

#include "common.cuh"
#include "table.cuh"  // AdamDev

namespace skb {

// A kernel whose launch arguments include the step and/or the Adam scalars:
// nargs = number of kernel parameters, ia / is = index of the AdamDev / the
// int64 step argument (-1 = absent).
struct ParamKernel {
  const void* func;
  int nargs, ia, is;
};

std::vector<ParamKernel>& param_kernels();
void note_param_kernel(const void* func, int nargs, int ia, int is);

struct GraphKey {
  static constexpr int kN = 16;
  int64_t v[kN];
  GraphKey() { memset(v, 0, sizeof v); }
  bool operator==(const GraphKey& o) const { return memcmp(v, o.v, sizeof v) == 0; }
};

struct StepGraph {
  struct Patch {
    cudaGraphNode_t node;
    cudaKernelNodeParams base;  // func, dims, smem; kernelParams from the captured node
    std::vector<void*> args;
    int ia, is;
  };
  bool valid = false;
  GraphKey key;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<Patch> patches;

  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    patches.clear();
    valid = false;
  }
  ~StepGraph() { reset(); }

  // First call with a new signature: run work(st) eagerly (first launches
  // set kernel attributes, allocate pools; growth steps never get captured).
  // Second call with the same signature: capture work(st) and launch the
  // graph.  Later calls: patch the step / Adam arguments and launch.
  // `cap`: a private non-default stream to capture on (the caller's stream
  // may be the legacy default stream, which cannot be captured); the graph
  // is then launched on `st`.
  template <class Work>
  void run(const GraphKey& k, cudaStream_t st, cudaStream_t cap, int64_t step, const AdamDev* a, Work&& work) {
    if (!primed || !(key == k)) {
      reset();
      key = k;
      primed = true;
      work(st);
      return;
    }
    if (!valid) {
      capture(cap, step, a, work);
      valid = true;
    } else {
      patch(step, a);
    }
    SKB_CUDA(cudaGraphLaunch(exec, st));
  }

  bool primed = false;

 private:
  template <class Work>
  void capture(cudaStream_t st, int64_t step, const AdamDev* a, Work& work) {
    SKB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      work(st);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      throw;
    }
    SKB_CUDA(cudaStreamEndCapture(st, &graph));
    collect(step, a);
    SKB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  }

  void collect(int64_t step, const AdamDev* a) {
    size_t num = 0;
    SKB_CUDA(cudaGraphGetNodes(graph, nullptr, &num));
    std::vector<cudaGraphNode_t> nodes(num);
    if (num) SKB_CUDA(cudaGraphGetNodes(graph, nodes.data(), &num));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      SKB_CUDA(cudaGraphNodeGetType(nd, &ty));
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams p;
      SKB_CUDA(cudaGraphKernelNodeGetParams(nd, &p));
      for (const ParamKernel& pk : param_kernels()) {
        if (pk.func != p.func) continue;
        Patch pt{nd, p, std::vector<void*>(p.kernelParams, p.kernelParams + pk.nargs), pk.ia, pk.is};
        // the captured values must be the ones this call passed (guards the
        // argument indices against signature drift)
        if (pt.is >= 0 && *static_cast<const int64_t*>(pt.args[pt.is]) != step)
          raise(SKB_E_UNSUPPORTED, pt.is, "graph capture: step argument index mismatch");
        if (pt.ia >= 0 && (!a || memcmp(pt.args[pt.ia], a, sizeof(AdamDev)) != 0))
          raise(SKB_E_UNSUPPORTED, pt.ia, "graph capture: Adam argument index mismatch");
        patches.push_back(std::move(pt));
      }
    }
  }

  void patch(int64_t step, const AdamDev* a) {
    for (Patch& pt : patches) {
      std::vector<void*> args = pt.args;
      int64_t st = step;
      AdamDev av{};
      if (pt.is >= 0) args[pt.is] = &st;
      if (pt.ia >= 0) {
        av = *a;
        args[pt.ia] = &av;
      }
      cudaKernelNodeParams p = pt.base;
      p.kernelParams = args.data();
      p.extra = nullptr;
      SKB_CUDA(cudaGraphExecKernelNodeSetParams(exec, pt.node, &p));
    }
  }
};

}  // namespace skb
