// Microbenchmark: latency of the block-level top-C' selection used by the
// scan's last cosine CTA (block_top_slots, ctkv_decode_dev.cuh) over C=2048
// group-max cosines, one CTA of 256 threads, timed with globaltimer inside.
#include <cstdio>
#include <cstdint>
#include "../../paper_2512_15550_b200/csrc/ctkv_decode_dev.cuh"

using namespace ctkv;

__global__ void bench(const double* vals, int C, int cp, int32_t* out, unsigned long long* t) {
  __shared__ double cv[128];
  __shared__ int ci[128];
  unsigned long long t0, t1, t2, c0, c1, c2;
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  c0 = clock64();
  block_top_slots(vals, C, cp, out, cv, ci);
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  c1 = clock64();
  block_top_slots(vals, C, cp, out, cv, ci);
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
  c2 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = c1 - c0; t[3] = c2 - c1; }
}

int main() {
  const int C = 2048;
  double* v;
  int32_t* out;
  unsigned long long* t;
  cudaMalloc(&v, C * 8);
  cudaMalloc(&out, 64);
  cudaMalloc(&t, 32);
  double h[C];
  for (int i = 0; i < C; ++i) h[i] = 0.5 + 1e-4 * ((i * 7919) % 2048);
  cudaMemcpy(v, h, C * 8, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) {
    bench<<<1, 256>>>(v, C, 4, out, t);
    unsigned long long ht[4];
    cudaMemcpy(ht, t, 32, cudaMemcpyDeviceToHost);
    int ho[4];
    cudaMemcpy(ho, out, 16, cudaMemcpyDeviceToHost);
    printf("cycles %llu %llu | block_top_slots: first %.2f us, second %.2f us; top %d %d %d %d (%s)\n", ht[2], ht[3], ht[0] / 1e3, ht[1] / 1e3,
           ho[0], ho[1], ho[2], ho[3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
