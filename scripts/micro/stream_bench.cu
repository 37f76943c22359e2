// Microbenchmark: streaming read bandwidth of a 174 MB buffer (one decode
// layer's centroid + static bytes at cfg2) with the scan kernels' access
// patterns, no compute.  Variants:
//   tma S B  : persistent, 1 CTA/SM, S stages of B KB, TMA bulk copies of
//              16 KB pieces, a consumer warp group releases each stage
//   ldg T    : grid-stride LDG.128 (ld.global.nc.L1::no_allocate), T threads/CTA
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@P bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}

constexpr int kMaxStages = 8;

__global__ void __launch_bounds__(288, 1) tma_stream(const char* base, int64_t ntask, int stage_bytes,
                                                     int stages, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    for (int s = 0; s < stages; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 8); }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < ntask; t += gridDim.x, ++k) {
        const int s = k % stages;
        bar_wait(&empty[s], ((k / stages) & 1) ^ 1);
        bar_expect(&full[s], stage_bytes);
        for (int off = 0; off < stage_bytes; off += 16384)
          bulk(smem + (size_t)s * stage_bytes + off, base + t * stage_bytes + off, 16384, &full[s]);
      }
    }
  } else {
    float acc = 0.f;
    int k = 0;
    for (int64_t t = blockIdx.x; t < ntask; t += gridDim.x, ++k) {
      const int s = k % stages;
      bar_wait(&full[s], (k / stages) & 1);
      const float* f = reinterpret_cast<const float*>(smem + (size_t)s * stage_bytes);
      acc += f[(threadIdx.x - 32) * 4];
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[s]);
    }
    if (acc == 1234.5f) out[0] = acc;
  }
}

__global__ void ldg_stream(const uint4* base, int64_t n, float* out) {
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(base + i));
    acc += __uint_as_float(r.x);
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t bytes = (argc > 1 ? atoll(argv[1]) : 174LL) << 20;
  char* base;
  cudaMalloc(&base, bytes + (64 << 20));
  cudaMemset(base, 0, bytes);
  float* out;
  cudaMalloc(&out, 4);
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  auto timeit = [&](auto launch, const char* name) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemset(flush, rep, 256 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-28s %8.2f us  %7.0f GB/s  %s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  const int cfg[][2] = {{3, 64}, {4, 48}, {6, 32}, {2, 96}, {8, 16}, {12, 16}};
  for (auto& c : cfg) {
    const int st = c[0], kb = c[1] * 1024;
    if (st > kMaxStages) continue;
    char name[64];
    snprintf(name, sizeof name, "tma %d x %d KB", st, c[1]);
    const int64_t nt = bytes / kb;
    timeit([&] { tma_stream<<<sms, 288, st * kb>>>(base, nt, kb, st, out); }, name);
  }
  for (int t : {256, 512}) {
    for (int per : {1, 2, 4}) {
      char name[64];
      snprintf(name, sizeof name, "ldg %d thr x %d ctas/sm", t, per);
      timeit([&] { ldg_stream<<<sms * per, t>>>(reinterpret_cast<const uint4*>(base), bytes / 16, out); }, name);
    }
  }
  return 0;
}
