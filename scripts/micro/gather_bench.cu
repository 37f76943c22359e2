// Microbenchmark: 128 CTAs x 512 threads, each CTA gathers NR random 256-byte
// rows from a large array (the rerank K-row gather pattern).  Variants:
//  0: row per thread (16 x 16B loads per row)
//  1: 8 lanes per row, 2 passes in flight
//  2: 8 lanes per row, all passes in flight (up to 6)
//  3: TMA bulk copies of every row into smem (one mbarrier), then read
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int V>
__global__ void __launch_bounds__(512, 1) gather(const uint4* __restrict__ base, const int* __restrict__ ids,
                                                 int nr, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar;
  const int* my = ids + blockIdx.x * nr;
  float acc = 0.f;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (V == 0) {
    for (int t = tid; t < nr; t += 512) {
      const uint4* r = base + (int64_t)my[t] * 16;
      uint4 x[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = __ldg(r + k);
#pragma unroll
      for (int k = 0; k < 16; ++k) acc += __uint_as_float(x[k].x) + __uint_as_float(x[k].w);
    }
  } else if (V == 1 || V == 2) {
    constexpr int UN = V == 1 ? 2 : 6;
    const int sub = lane & 7, rw = lane >> 3;
    for (int b0 = warp * 4; b0 < nr; b0 += 64 * UN) {
      uint4 x[UN][2];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int t = b0 + u * 64 + rw;
        if (t < nr) {
          const uint4* r = base + (int64_t)my[t] * 16;
          x[u][0] = __ldg(r + sub);
          x[u][1] = __ldg(r + 8 + sub);
        } else {
          x[u][0] = x[u][1] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) acc += __uint_as_float(x[u][0].x) + __uint_as_float(x[u][1].w);
    }
  } else if (V == 4) {
    // cp.async (LDGSTS) 16 B per lane into smem, 16 lanes per row, all in flight
    for (int i = tid; i < nr * 16; i += 512) {
      const int t = i >> 4, c = i & 15;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(smem + t * 256 + c * 16)),
                   "l"(base + (int64_t)my[t] * 16 + c) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int t = tid; t < nr; t += 512) acc += reinterpret_cast<float*>(smem + t * 256)[lane];
  } else {
    // TMA bulk copy of every row (nr * 256 B must fit smem)
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(nr * 256));
    }
    __syncthreads();
    for (int t = tid; t < nr; t += 512)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                   ::"r"(sa(smem + t * 256)), "l"(base + (int64_t)my[t] * 16), "r"(sa(&bar)) : "memory");
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@P bra D;\nbra W;\nD:\n}" ::"r"(sa(&bar)));
    for (int t = tid; t < nr; t += 512) acc += reinterpret_cast<float*>(smem + t * 256)[lane];
  }
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t rows = 64LL * 98304;   // a layer's K rows, 1.6 GB
  uint4* base;
  cudaMalloc(&base, rows * 256);
  cudaMemset(base, 1, rows * 256);
  const int ctas = argc > 1 ? atoi(argv[1]) : 128, nr = argc > 2 ? atoi(argv[2]) : 750;
  int* ids;
  cudaMalloc(&ids, ctas * nr * sizeof(int));
  int* h = new int[ctas * nr];
  uint64_t s = 12345;
  for (int i = 0; i < ctas * nr; ++i) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    const int unit = (i / nr) / 2;
    h[i] = unit * 98304 + (int)((s >> 33) % 97152) + 128;
  }
  cudaMemcpy(ids, h, ctas * nr * sizeof(int), cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 4);
  // L2 flush buffer
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(gather<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int v = 0; v < 5; ++v) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(flush, rep, 256 << 20);
      cudaEventRecord(e0);
      if (v == 0) gather<0><<<ctas, 512>>>(base, ids, nr, out);
      if (v == 1) gather<1><<<ctas, 512>>>(base, ids, nr, out);
      if (v == 2) gather<2><<<ctas, 512>>>(base, ids, nr, out);
      if (v == 3) gather<3><<<ctas, 512, nr * 256>>>(base, ids, nr, out);
      if (v == 4) gather<4><<<ctas, 512, nr * 256>>>(base, ids, nr, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("variant %d: %.2f us  (%.0f GB/s)  err=%s\n", v, best * 1e3,
           ctas * (double)nr * 256 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  // empty-kernel launch cost reference
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    gather<1><<<ctas, 512>>>(base, ids, 0, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("empty kernel: %.2f us\n", best * 1e3);
  return 0;
}
