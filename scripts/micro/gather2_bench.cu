// Microbenchmark: random 256-byte row gathers (the chain's rerank K-row
// pattern), timed INSIDE the kernel (globaltimer, first CTA start -> last CTA
// end) so launch overhead does not hide the gather.  Each CTA (256 threads)
// gathers NR random rows of one unit's 96K-row region.  Variants:
//   0: registers, 8 lanes x 32 B per row, 8 passes of 4 rows per warp in flight
//   1: cp.async 16 B (LDGSTS) into shared memory, every row in flight
//   2: TMA bulk copy per row (cp.async.bulk, 256 B) into shared memory
//   3: TMA tile::gather4 (4 rows per instruction) into shared memory
// usage: gather2_bench [ctas] [rows per cta]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_t0, g_t1;

template <int V>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ base, const int* __restrict__ ids, int nr,
                                              const __grid_constant__ CUtensorMap map, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) atomicMin(&g_t0, (unsigned long long)gtime());
  const int* my = ids + blockIdx.x * nr;
  float acc = 0.f;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (V == 0) {
    constexpr int UN = 8;
    const int sub = lane & 7, rw = lane >> 3;
    for (int b0 = warp * 4; b0 < nr; b0 += 32 * UN) {
      uint4 x[UN][2];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int t = b0 + u * 32 + rw;
        if (t < nr) {
          const uint4* r = base + (int64_t)my[t] * 16;
          asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x[u][0].x), "=r"(x[u][0].y), "=r"(x[u][0].z), "=r"(x[u][0].w) : "l"(r + sub));
          asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x[u][1].x), "=r"(x[u][1].y), "=r"(x[u][1].z), "=r"(x[u][1].w) : "l"(r + 8 + sub));
        } else {
          x[u][0] = x[u][1] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) acc += __uint_as_float(x[u][0].x) + __uint_as_float(x[u][1].w);
    }
  } else if (V == 1) {
    for (int i = tid; i < nr * 16; i += 256) {
      const int t = i >> 4, c = i & 15;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(smem + t * 256 + c * 16)),
                   "l"(base + (int64_t)my[t] * 16 + c) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int t = tid; t < nr; t += 256) acc += reinterpret_cast<float*>(smem + t * 256)[lane];
  } else {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(nr * 256));
    }
    __syncthreads();
    if (V == 2) {
      for (int t = tid; t < nr; t += 256)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                     ::"r"(sa(smem + t * 256)), "l"(base + (int64_t)my[t] * 16), "r"(sa(&bar)) : "memory");
    } else {
      for (int t = 4 * tid; t < nr; t += 4 * 256) {
        const int r0 = my[t], r1 = my[t + 1], r2 = my[t + 2], r3 = my[t + 3];
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
            ::"r"(sa(smem + t * 256)), "l"(&map), "r"(sa(&bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
            : "memory");
      }
    }
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@P bra D;\nbra W;\nD:\n}" ::"r"(sa(&bar)));
    for (int t = tid; t < nr; t += 256) acc += reinterpret_cast<float*>(smem + t * 256)[lane];
  }
  if (acc == 12345.f) out[0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t1, (unsigned long long)gtime());
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int64_t rows = 64LL * 98304;   // a layer's K rows, 1.6 GB
  uint4* base;
  cudaMalloc(&base, rows * 256);
  cudaMemset(base, 1, rows * 256);
  const int ctas = argc > 1 ? atoi(argv[1]) : 32, nr = argc > 2 ? atoi(argv[2]) : 376;
  int* ids;
  cudaMalloc(&ids, ctas * nr * sizeof(int));
  int* h = new int[ctas * nr];
  uint64_t s = 12345;
  for (int i = 0; i < ctas * nr; ++i) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    const int unit = (i / nr) / 4;
    h[i] = unit * 98304 + (int)((s >> 33) % 97152) + 128;
  }
  cudaMemcpy(ids, h, ctas * nr * sizeof(int), cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 4);
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {128, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = reinterpret_cast<EncodeTiledFn>(fp)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides,
                                                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) printf("tensor map encode failed: %d\n", (int)cr);
  const size_t sm = (size_t)nr * 256;
  cudaFuncSetAttribute(gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gather<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[4] = {"regs 8x4 rows", "cp.async 16B", "bulk per row", "tma gather4"};
  for (int v = 0; v < 4; ++v) {
    if (v > 0 && sm > 200 * 1024) continue;
    double best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemset(flush, rep, 256 << 20);
      unsigned long long big = ~0ull, zero = 0;
      cudaMemcpyToSymbol(g_t0, &big, 8);
      cudaMemcpyToSymbol(g_t1, &zero, 8);
      if (v == 0) gather<0><<<ctas, 256, 0>>>(base, ids, nr, map, out);
      if (v == 1) gather<1><<<ctas, 256, sm>>>(base, ids, nr, map, out);
      if (v == 2) gather<2><<<ctas, 256, sm>>>(base, ids, nr, map, out);
      if (v == 3) gather<3><<<ctas, 256, sm>>>(base, ids, nr, map, out);
      cudaDeviceSynchronize();
      unsigned long long t0, t1;
      cudaMemcpyFromSymbol(&t0, g_t0, 8);
      cudaMemcpyFromSymbol(&t1, g_t1, 8);
      const double us = (t1 - t0) / 1e3;
      if (rep > 0 && us < best) best = us;
    }
    printf("ctas %4d rows %4d  %-16s %7.2f us  %6.1f GB/s per CTA  %7.0f GB/s total  %s\n", ctas, nr, names[v],
           best, nr * 256.0 / (best * 1e3), ctas * (double)nr * 256 / (best * 1e3),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
