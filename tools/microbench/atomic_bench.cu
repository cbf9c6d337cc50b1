// Same-address returning atomicAdd throughput (one lane per warp), as used by
// per-warp output reservations.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void hammer(unsigned long long* ctr, int iters, int spread, unsigned long long* sink) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned long long acc = 0;
  for (int i = 0; i < iters; i++) {
    unsigned long long v = 0;
    if ((threadIdx.x & 31) == 0) v = atomicAdd(ctr + 32 * (warp % spread), 1ull);
    acc += __shfl_sync(0xffffffffu, v, 0);
  }
  if (acc == 42) *sink = acc;
}

int main() {
  unsigned long long *ctr, *sink;
  cudaMalloc(&ctr, 32 * 64 * 8 * 64);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int spread : {1, 4, 16, 64}) {
    for (int blocks : {148, 592}) {
      const int iters = 16;
      hammer<<<blocks, 256>>>(ctr, iters, spread, sink);
      cudaEventRecord(a);
      hammer<<<blocks, 256>>>(ctr, iters, spread, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double n = (double)blocks * 8 * iters;
      printf("spread %2d blocks %3d: %.0f atomics in %.1f us = %.2f ns/atomic (%.2f ns per address)\n",
             spread, blocks, n, ms * 1e3, ms * 1e6 / n, ms * 1e6 / n * spread);
    }
  }
  return 0;
}
