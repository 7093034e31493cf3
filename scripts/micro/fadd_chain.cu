// Dependent FADD chain latency on this GPU (cycles per add): one warp, one
// chain per lane, operands from registers and from shared memory (LDS.128
// four positions at a time, as the long-run fold consumes its stage images).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_reg(float* out, int n, float x0) {
  float acc = 0.f, a = x0, b = x0 * 0.5f, c = x0 * 0.25f, d = x0 * 0.125f;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 4) {
    acc = __fadd_rn(acc, a);
    acc = __fadd_rn(acc, b);
    acc = __fadd_rn(acc, c);
    acc = __fadd_rn(acc, d);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) printf("reg chain: %.3f cycles/add\n", (double)(t1 - t0) / n);
  out[threadIdx.x] = acc;
}

__global__ void chain_lds(float* out, int n) {
  __shared__ __align__(16) float buf[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = 1e-3f * (i & 31);
  __syncthreads();
  const float4* c4 = reinterpret_cast<const float4*>(buf) + threadIdx.x * 4;
  float acc = 0.f;
  long long t0 = clock64();
  for (int rep = 0; rep < n / 1024; ++rep) {
#pragma unroll 4
    for (int p = 0; p < 1024; p += 16) {
      float4 x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k] = c4[((p >> 2) + k) & 1023 & ~7];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc = __fadd_rn(acc, x[k].x);
        acc = __fadd_rn(acc, x[k].y);
        acc = __fadd_rn(acc, x[k].z);
        acc = __fadd_rn(acc, x[k].w);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) printf("lds chain: %.3f cycles/add\n", (double)(t1 - t0) / n);
  out[threadIdx.x] = acc;
}

int main() {
  float* o;
  cudaMalloc(&o, 1024 * sizeof(float));
  chain_reg<<<1, 32>>>(o, 1 << 22, 1e-3f);
  chain_reg<<<1, 8>>>(o, 1 << 22, 1e-3f);
  chain_lds<<<1, 32>>>(o, 1 << 22);
  chain_lds<<<1, 8>>>(o, 1 << 22);
  cudaDeviceSynchronize();
  return 0;
}
