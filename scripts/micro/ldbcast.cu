// Microbenchmark (round-2 K2 investigation): cost of warp-uniform record
// fetches -- LDS.128 / LDS.64 broadcast vs LDG.128 (L1 hit) broadcast.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/ldbcast scripts/micro/ldbcast.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const float4* __restrict__ g, float* out, int iters) {
  __shared__ float4 s[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) s[i] = g[i];
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = 0;
  for (int it = 0; it < iters; ++it) {
    float4 v;
    if (MODE == 0) v = s[idx];                                   // LDS.128 uniform
    else if (MODE == 1) { const float2* s2 = reinterpret_cast<const float2*>(s); float2 a = s2[2 * idx]; v = make_float4(a.x, a.y, 0, 0); }  // LDS.64 uniform
    else if (MODE == 2) v = __ldg(g + idx);                      // LDG.128 uniform (L1 hit)
    else v = s[idx + (threadIdx.x & 1)];                          // LDS.128, two addresses
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    idx = (idx + 1 + __float_as_int(v.x) * 0) & 255;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

int main() {
  float4* g; float* out;
  cudaMalloc(&g, 512 * 16); cudaMemset(g, 0, 512 * 16);
  cudaMalloc(&out, 148 * 8 * 512 * 4);
  const int iters = 4096;
  for (int m = 0; m < 4; ++m) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) k<0><<<148 * 4, 512>>>(g, out, iters);
      if (m == 1) k<1><<<148 * 4, 512>>>(g, out, iters);
      if (m == 2) k<2><<<148 * 4, 512>>>(g, out, iters);
      if (m == 3) k<3><<<148 * 4, 512>>>(g, out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double warp_loads = 148.0 * 4 * 16 * iters;
    printf("mode %d: %.3f ms, %.2f warp-loads per SM-cycle\n", m, ms, warp_loads / (ms * 1e-3 * 1.965e9 * 148));
  }
  return 0;
}
