// Microbenchmark: CTA dispatch cost.  A near-empty kernel (each CTA writes
// one word) over grids of 148..5248 CTAs, 256 threads, with and without
// 74 KB of dynamic shared memory; event-timed, minus the 1-CTA launch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(int* out) {
  __shared__ int sm[1];
  if (threadIdx.x == 0) { sm[0] = blockIdx.x; out[blockIdx.x] = sm[0]; }
}

int main() {
  int* out;
  cudaMalloc(&out, 1 << 20);
  cudaFuncSetAttribute(tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int smem : {0, 74 * 1024}) {
    for (int grid : {1, 148, 328, 656, 1312, 2624, 5248}) {
      float best = 1e9;
      for (int r = 0; r < 20; ++r) {
        cudaEventRecord(e0);
        tiny<<<grid, 256, smem>>>(out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      // 10 back-to-back launches in a graph-free stream
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) tiny<<<grid, 256, smem>>>(out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms10;
      cudaEventElapsedTime(&ms10, e0, e1);
      if (cudaGetLastError() != cudaSuccess) printf("error\n");
      printf("smem %6d grid %5d: single %7.2f us, per launch in a row of 10: %7.2f us\n", smem, grid,
             best * 1e3, ms10 * 1e2);
    }
  }
  return 0;
}
