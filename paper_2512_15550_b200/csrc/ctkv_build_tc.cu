// Tensor-core prefill index build (Alg. 1, ck/index.py:59-99) for bf16 stores.
//
// Grouped scores S[c, j] = max_h (q_{h,c} . k_j) / sqrt(d) are a GEMM with
// M = offloaded keys, N = gs heads x CB centroids (= 256), K = d.  Keys are
// the A operand (TMA, 128B swizzle, 128 rows per tile), the centroid rows of
// one work item the resident B operand, accumulators live in TMEM (two
// 256-column buffers so the epilogue of tile i overlaps the MMAs of tile
// i+1).  Warp roles: 0 = TMA producer, 1 = MMA issuer (+TMEM owner),
// 2..9 = epilogue (tcgen05.ld -> group max -> scale -> filter/store).
//
// Top-rho per row without materialising the 6.4 GB/layer score matrix:
//   1. sample pass  -- the same GEMM against every S-th key, scores stored;
//   2. threshold    -- per row the k_s-th largest sample score, with k_s
//                      chosen so the full row has ~rho + 6 sigma candidates
//                      above it with overwhelming probability;
//   3. filter pass  -- the full GEMM; the epilogue keeps (score, key) pairs
//                      >= threshold in a per-row buffer (the CTA owns its
//                      rows, so counters are shared-memory atomics);
//   4. select       -- per row, sort the <= cap candidates by (score desc,
//                      key asc) and write the first rho ids -- exact top-rho
//                      of the tensor-core scores whenever rho <= count <= cap;
//   5. fallback     -- rows outside [rho, cap] (rare) are recomputed in full
//                      and radix-selected, so the result is exact always.
#include <cuda.h>

#include <cfloat>
#include <cmath>
#include <cstdio>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_internal.h"

namespace ctkv {

int topk_launch(const float* v, int64_t rows, int64_t n, int64_t ld, int k, int32_t* out,
                int64_t out_ld, int32_t add, cudaStream_t st, int64_t rows_per_group,
                int64_t group_stride, const int32_t* row_map);

namespace tc {

constexpr int kBM = 128;          // keys per tile (UMMA M)
constexpr int kBN = 256;          // gs * CB centroid-head rows (UMMA N)
constexpr int kStages = 4;        // A pipeline depth
constexpr int kThreads = 320;     // 10 warps
constexpr int kEpiWarps = 8;
constexpr int kAtomBytes = kBM * 128;  // one 128-row x 64-element bf16 swizzle atom

enum Mode : int { kStore = 0, kFilter = 1 };

// ---- PTX wrappers ---------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// K-major, 128B-swizzled operand: rows 128 B apart, 8-row core groups 1 KB apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// bf16 x bf16 -> f32, A and B K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);

struct Params {
  int U, C, CB, gs, h, g;  // units, centroids, centroids per item, group size
  int64_t n;               // keys per unit (columns of S)
  int64_t key_row0;        // first key row of unit 0 in the A map
  int64_t key_unit_rows;   // rows between units in the A map
  int n_cblocks;           // C / CB
  int items;               // U * n_cblocks
  float scale;
  int mode;
  // store mode
  float* out;              // [U][C][n]
  // filter mode
  const float* thresh;     // [U*C]
  int32_t* counts;         // [U*C]
  uint64_t* cand;          // [U*C][cap]
  int cap;
};

template <int KATOMS>
__global__ void __launch_bounds__(kThreads, 1)
    scores_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1 KB alignment for the 128B swizzle atoms
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sbase = smem_raw + (base - raw);
  constexpr uint32_t kABytes = KATOMS * kAtomBytes;         // one A stage
  constexpr uint32_t kBAtom = kBN * 128;                    // 32 KB per K atom
  constexpr uint32_t kBBytes = KATOMS * kBAtom;
  const uint32_t sA = base;
  const uint32_t sB = sA + kStages * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + kStages * kABytes + kBBytes);
  // barrier slots
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (kStages + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * kStages + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * kStages + 2 + a); };
  const uint32_t bfull = bar0 + 8u * (2 * kStages + 4);
  const uint32_t bempty = bar0 + 8u * (2 * kStages + 5);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 6);
  float* s_thr = reinterpret_cast<float*>(tmem_slot + 4);    // [CB]
  int* s_cnt = reinterpret_cast<int*>(s_thr + 256);          // [CB]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (p.n + kBM - 1) / kBM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), kEpiWarps);
    }
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&mapA);
    prefetch_map(&mapB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, item_phase = 0;
      for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
        const int u = it / p.n_cblocks, cb = it % p.n_cblocks;
        const int bi = u / p.g, gi = u % p.g;
        // B: centroid rows (head j, centroids cb*CB ..) of this unit, all K atoms
        mbar_wait(bempty, item_phase ^ 1);
        mbar_expect_tx(bfull, kBBytes);
        for (int ka = 0; ka < KATOMS; ++ka)
          for (int j = 0; j < p.gs; ++j) {
            const int32_t row = ((bi * p.h + gi * p.gs + j) * p.C) + cb * p.CB;
            tma_load_2d(sB + ka * kBAtom + j * p.CB * 128, &mapB, bfull, ka * 64, row);
          }
        item_phase ^= 1;
        const int64_t row0 = p.key_row0 + (int64_t)u * p.key_unit_rows;
        for (int64_t t = 0; t < ntiles; ++t) {
          mbar_wait(empty(stage), phase ^ 1);
          mbar_expect_tx(full(stage), kABytes);
          for (int ka = 0; ka < KATOMS; ++ka)
            tma_load_2d(sA + stage * kABytes + ka * kAtomBytes, &mapA, full(stage), ka * 64,
                        (int32_t)(row0 + t * kBM));
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0, item_phase = 0;
      for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
        mbar_wait(bfull, item_phase);
        item_phase ^= 1;
        tc_fence_after();
        for (int64_t t = 0; t < ntiles; ++t) {
          mbar_wait(tempty(acc), acc_phase ^ 1);
          mbar_wait(full(stage), phase);
          tc_fence_after();
          const uint32_t d_tmem = tmem + acc * kBN;
#pragma unroll
          for (int ka = 0; ka < KATOMS; ++ka) {
            const uint64_t ad = sw128_desc(sA + stage * kABytes + ka * kAtomBytes);
            const uint64_t bd = sw128_desc(sB + ka * kBAtom);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)  // 4 x K=16 per 64-element atom (32 B steps)
              mma_bf16(d_tmem, ad + 2 * ks, bd + 2 * ks, kIdesc, (ka | ks) != 0);
          }
          mma_commit(empty(stage));       // smem slot reusable once these MMAs retire
          mma_commit(tfull(acc));         // accumulator ready for the epilogue
          if (++stage == kStages) { stage = 0; phase ^= 1; }
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        mma_commit(bempty);               // B reusable after the item's last MMA
      }
    }
  } else {
    // ===================== epilogue (8 warps) =====================
    const int ew = warp - 2;               // 0..7
    const int quad = warp & 3;             // TMEM lane quadrant this warp may touch
    const int half = ew >> 2;              // which half of the CB centroids
    const int hcb = p.CB / 2;              // centroids per epilogue warp
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
      const int u = it / p.n_cblocks, cb = it % p.n_cblocks;
      const int64_t rowbase = (int64_t)u * p.C + (int64_t)cb * p.CB;
      if (p.mode == kFilter) {
        named_bar(1, kEpiWarps * 32);      // previous item's counters are flushed
        for (int i = threadIdx.x - 64; i < p.CB; i += kEpiWarps * 32) {
          s_thr[i] = p.thresh[rowbase + i];
          s_cnt[i] = 0;
        }
        named_bar(1, kEpiWarps * 32);
      }
      for (int64_t t = 0; t < ntiles; ++t) {
        mbar_wait(tfull(acc), acc_phase);
        tc_fence_after();
        const int64_t key = t * kBM + quad * 32 + lane;
        const bool valid = key < p.n;
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + acc * kBN;
        for (int c0 = half * hcb; c0 < (half + 1) * hcb; c0 += 16) {
          float m[16], v[16];
          tmem_ld16(tbase + c0, m);
          for (int j = 1; j < p.gs; ++j) {
            tmem_ld16(tbase + j * p.CB + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) m[i] = fmaxf(m[i], v[i]);
          }
          tmem_ld_wait();
          if (p.mode == kStore) {
            if (valid) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                p.out[(rowbase + c0 + i) * p.n + key] = m[i] * p.scale;
            }
          } else if (valid) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float s = m[i] * p.scale;
              if (s >= s_thr[c0 + i]) {
                const int pos = atomicAdd(&s_cnt[c0 + i], 1);
                if (pos < p.cap)
                  p.cand[(rowbase + c0 + i) * p.cap + pos] =
                      ((uint64_t)(~okey32(s)) << 32) | (uint32_t)key;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (p.mode == kFilter) {
        named_bar(1, kEpiWarps * 32);
        for (int i = threadIdx.x - 64; i < p.CB; i += kEpiWarps * 32) p.counts[rowbase + i] = s_cnt[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// every S-th offloaded key of every unit, compacted: dst[u][i] = keys[u][off + i*S]
__global__ void gather_sample_kernel(const uint4* __restrict__ keys, uint4* __restrict__ dst,
                                     int64_t cap, int64_t off, int64_t stride, int64_t ns,
                                     int vec_per_row, int U) {
  const int64_t total = (int64_t)U * ns * vec_per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i % vec_per_row;
    const int64_t r = (i / vec_per_row) % ns;
    const int64_t u = i / (vec_per_row * ns);
    dst[i] = keys[((u * cap) + off + r * stride) * vec_per_row + v];
  }
}

// per row: k-th largest of n sample scores (row resident in smem)
__global__ void __launch_bounds__(256) kth_value_kernel(const float* __restrict__ S, int64_t n,
                                                        int k, float* __restrict__ thr) {
  extern __shared__ uint32_t keys_s[];
  __shared__ int hist[2048];
  __shared__ int s_bin, s_above;
  const float* row = S + (int64_t)blockIdx.x * n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) keys_s[i] = okey32(row[i]);
  uint32_t prefix = 0;
  int above = 0;
  const int shifts[3] = {21, 10, 0}, widths[3] = {11, 11, 10};
  for (int pass = 0; pass < 3; ++pass) {
    const int sh = shifts[pass], nb = 1 << widths[pass], hsh = sh + widths[pass];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t key = keys_s[i];
      if (pass == 0 || (key >> hsh) == (prefix >> hsh)) atomicAdd(&hist[(key >> sh) & (nb - 1)], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // lane L owns the L-th block of bins from the top
      const int lane = threadIdx.x, per = nb / 32, hi = nb - lane * per, want = k - above;
      int sum = 0;
      for (int b = hi - 1; b >= hi - per; --b) sum += hist[b];
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - sum;
      const unsigned bal = __ballot_sync(0xffffffffu, incl >= want && excl < want);
      if (lane == __ffs(bal) - 1) {
        int run = excl;
        for (int b = hi - 1; b >= hi - per; --b) {
          if (run + hist[b] >= want) { s_bin = b; s_above = run; break; }
          run += hist[b];
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)s_bin << sh;
    above += s_above;
  }
  if (threadIdx.x == 0) thr[blockIdx.x] = okey32_inv(prefix);
}

// per row: exact top-rho of the candidates in (score desc, key asc) order, or
// flag the row for the fallback.  O(n) counting sort instead of a comparison
// sort: linear bins over [min, max] of the candidates' score keys, bin
// offsets by a block scan, then each candidate's exact rank inside its
// (small) bin; ranks < rho are written straight to the list.
constexpr int kSelT = 256, kSelBins = 2048;
__global__ void __launch_bounds__(kSelT) select_kernel(const uint64_t* __restrict__ cand,
                                                       const int32_t* __restrict__ counts, int cap,
                                                       int rho, int C, int32_t* __restrict__ lists,
                                                       int32_t add, int32_t* fail_n,
                                                       int32_t* fail_rows) {
  extern __shared__ uint64_t ck[];                            // [cap] candidates
  int* binned = reinterpret_cast<int*>(ck + cap);             // [cap] indices grouped by bin
  __shared__ int hist[kSelBins], cur[kSelBins];
  __shared__ uint32_t s_mm[2 * kSelT / 32];
  __shared__ int s_ws[kSelT / 32 + 1];
  const int64_t row = blockIdx.x;
  const int cnt = counts[row];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (cnt < rho || cnt > cap) {
    if (tid == 0) fail_rows[atomicAdd(fail_n, 1)] = (int32_t)row;
    return;
  }
  const uint64_t* src = cand + row * cap;
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int i = tid; i < cnt; i += kSelT) {
    const uint64_t k = __ldg(src + i);
    ck[i] = k;
    mn = min(mn, (uint32_t)(k >> 32));
    mx = max(mx, (uint32_t)(k >> 32));
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) { s_mm[warp] = mn; s_mm[kSelT / 32 + warp] = mx; }
  for (int b = tid; b < kSelBins; b += kSelT) hist[b] = 0;
  __syncthreads();
  mn = 0xffffffffu;
  mx = 0u;
  for (int w = 0; w < kSelT / 32; ++w) { mn = min(mn, s_mm[w]); mx = max(mx, s_mm[kSelT / 32 + w]); }
  const float fscale = (float)kSelBins / ((float)(mx - mn) + 1.0f);
  auto bin_of = [&](uint64_t k) {
    return min(kSelBins - 1, (int)((float)((uint32_t)(k >> 32) - mn) * fscale));
  };
  for (int i = tid; i < cnt; i += kSelT) atomicAdd(&hist[bin_of(ck[i])], 1);
  __syncthreads();
  // exclusive scan of the bins: thread t owns bins [8t, 8t+8)
  {
    constexpr int BPT = kSelBins / kSelT;
    int loc = 0;
#pragma unroll
    for (int x = 0; x < BPT; ++x) loc += hist[tid * BPT + x];
    int incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_ws[warp] = incl;
    __syncthreads();
    int wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += s_ws[w];
    int run = wpre + incl - loc;
#pragma unroll
    for (int x = 0; x < BPT; ++x) {
      cur[tid * BPT + x] = run;
      run += hist[tid * BPT + x];
    }
  }
  __syncthreads();
  for (int i = tid; i < cnt; i += kSelT) binned[atomicAdd(&cur[bin_of(ck[i])], 1)] = i;
  __syncthreads();
  int32_t* dst = lists + row * rho;
  for (int i = tid; i < cnt; i += kSelT) {
    const uint64_t k = ck[i];
    const int b = bin_of(k);
    const int e = cur[b], s0 = e - hist[b];
    if (s0 >= rho) continue;                    // the whole bin ranks below the list
    int r = s0;
    for (int x = s0; x < e; ++x) r += ck[binned[x]] < k;
    if (r < rho) dst[r] = (int32_t)(k & 0xffffffffu) + add;
  }
}

// full-row scores for fallback rows: one CTA per (row, 256-key block)
__global__ void __launch_bounds__(256) row_scores_kernel(const __nv_bfloat16* __restrict__ cent,
                                                         const __nv_bfloat16* __restrict__ keys,
                                                         const int32_t* __restrict__ rows, int C,
                                                         int gs, int h, int g, int d, int64_t cap,
                                                         int64_t off, int64_t n, float scale,
                                                         float* __restrict__ out) {
  __shared__ float qs[16 * 256];
  const int r = rows[blockIdx.y];
  const int u = r / C, c = r % C;
  const int bi = u / g, gi = u % g;
  for (int i = threadIdx.x; i < gs * d; i += blockDim.x) {
    const int j = i / d, e = i % d;
    qs[i] = __bfloat162float(cent[(((int64_t)bi * h + gi * gs + j) * C + c) * d + e]);
  }
  __syncthreads();
  const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= n) return;
  const __nv_bfloat16* kr = keys + ((int64_t)u * cap + off + key) * d;
  float m = -INFINITY;
  for (int j = 0; j < gs; ++j) {
    float a = 0.f;
    for (int e = 0; e < d; ++e) a = fmaf(qs[j * d + e], __bfloat162float(kr[e]), a);
    m = fmaxf(m, a);
  }
  out[(int64_t)blockIdx.y * n + key] = m * scale;
}

// ---- host -----------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 2-D bf16 map over `rows` rows of `d` elements, box = {64, box_rows}, 128B swizzle
static bool make_map(CUtensorMap* map, const void* ptr, int64_t rows, int d, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static size_t smem_bytes(int katoms) {
  return 1024 + (size_t)kStages * katoms * kAtomBytes + (size_t)katoms * kBN * 128 + 8 * 16 + 16 +
         256 * 4 * 2;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, int katoms,
                       cudaStream_t st) {
  const size_t sm = smem_bytes(katoms);
  const int grid = std::min(p.items, num_sms());
  if (katoms == 2) {
    cudaFuncSetAttribute(scores_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    scores_tc_kernel<2><<<grid, kThreads, sm, st>>>(ma, mb, p);
  } else if (katoms == 1) {
    cudaFuncSetAttribute(scores_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    scores_tc_kernel<1><<<grid, kThreads, sm, st>>>(ma, mb, p);
  } else {
    return CTKV_ESHAPE;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

struct Plan {
  int S;        // sample stride
  int64_t ns;   // sampled keys per unit
  int ks;       // sample rank giving the threshold
  int cap;      // candidate slots per row
  int CB;
};

static Plan make_plan(const BuildParams& p) {
  Plan pl;
  pl.S = 16;
  pl.ns = (p.n_off + pl.S - 1) / pl.S;
  const double mean = (double)p.rho / pl.S;
  pl.ks = (int)std::ceil(mean + 6.0 * std::sqrt(mean)) + 1;
  if (pl.ks > pl.ns) pl.ks = (int)pl.ns;
  const int64_t expect = (int64_t)pl.ks * pl.S;
  // candidates above the sample threshold: ~expect +- S*sqrt(ks); 8 sigma of
  // headroom (rows beyond it take the exact fallback)
  const int64_t head = (int64_t)std::ceil(8.0 * pl.S * std::sqrt((double)pl.ks));
  pl.cap = (int)std::min<int64_t>(((std::max<int64_t>(expect + head, p.rho + 1024) + 255) / 256) * 256,
                                  1 << 14);
  pl.CB = kBN / p.gs;
  return pl;
}

}  // namespace tc

// does the tensor-core build apply to this problem?
bool build_tc_supported(const BuildParams& p, int dtype) {
  if (dtype != CTKV_BF16) return false;
  if (p.d != 128 && p.d != 64) return false;
  if (p.gs != 1 && p.gs != 2 && p.gs != 4 && p.gs != 8 && p.gs != 16) return false;
  const int CB = tc::kBN / p.gs;
  if (p.C % CB != 0) return false;
  if (p.n_off < 4096 || p.rho < 1) return false;
  return true;
}

size_t build_tc_workspace_bytes(const BuildParams& p) {
  const tc::Plan pl = tc::make_plan(p);
  const int64_t U = (int64_t)p.b * p.g;
  size_t b = 0;
  auto a256 = [](size_t x) { return (x + 255) & ~size_t(255); };
  b += a256((size_t)U * pl.ns * p.d * 2);               // sample keys
  b += a256((size_t)U * p.C * pl.ns * 4);               // sample scores
  b += a256((size_t)U * p.C * 4) * 2;                   // thresholds + counts
  b += a256((size_t)U * p.C * pl.cap * 8);              // candidates
  b += a256((size_t)U * p.C * 4 + 16);                  // fail list
  return b;
}

int build_tc(const BuildParams& p, int /*dtype*/, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace tc;
  const Plan pl = make_plan(p);
  const int U = p.b * p.g;
  if (build_tc_workspace_bytes(p) > ws_bytes) return CTKV_EWORKSPACE;
  auto a256 = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* w = static_cast<char*>(ws);
  __nv_bfloat16* skeys = reinterpret_cast<__nv_bfloat16*>(w);
  w += a256((size_t)U * pl.ns * p.d * 2);
  float* sscore = reinterpret_cast<float*>(w);
  w += a256((size_t)U * p.C * pl.ns * 4);
  float* thr = reinterpret_cast<float*>(w);
  w += a256((size_t)U * p.C * 4);
  int32_t* counts = reinterpret_cast<int32_t*>(w);
  w += a256((size_t)U * p.C * 4);
  uint64_t* cand = reinterpret_cast<uint64_t*>(w);
  w += a256((size_t)U * p.C * pl.cap * 8);
  int32_t* fail_n = reinterpret_cast<int32_t*>(w);
  int32_t* fail_rows = fail_n + 4;
  const int katoms = p.d / 64;
  const float scale = (float)(1.0 / std::sqrt((double)p.d));

  // 1. sample keys
  {
    const int vpr = p.d * 2 / 16;
    const int64_t total = (int64_t)U * pl.ns * vpr;
    gather_sample_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
        static_cast<const uint4*>(p.keys), reinterpret_cast<uint4*>(skeys), p.cap, p.off_begin, pl.S,
        pl.ns, vpr, U);
  }
  CUtensorMap mapS, mapK, mapC;
  if (!make_map(&mapS, skeys, (int64_t)U * pl.ns, p.d, kBM) ||
      !make_map(&mapK, p.keys, (int64_t)U * p.cap, p.d, kBM) ||
      !make_map(&mapC, p.cent, (int64_t)p.b * p.h * p.C, p.d, pl.CB))
    return CTKV_ECUDA;
  Params gp{};
  gp.U = U;
  gp.C = p.C;
  gp.CB = pl.CB;
  gp.gs = p.gs;
  gp.h = p.h;
  gp.g = p.g;
  gp.n_cblocks = p.C / pl.CB;
  gp.items = U * gp.n_cblocks;
  gp.scale = scale;
  // 2. sample pass (store) + thresholds
  gp.n = pl.ns;
  gp.key_row0 = 0;
  gp.key_unit_rows = pl.ns;
  gp.mode = kStore;
  gp.out = sscore;
  if (int rc = launch_gemm(mapS, mapC, gp, katoms, st)) return rc;
  const size_t kth_smem = (size_t)pl.ns * 4;
  if (kth_smem > 200 * 1024) return CTKV_ECONFIG;
  cudaFuncSetAttribute(kth_value_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kth_smem);
  kth_value_kernel<<<(unsigned)(U * p.C), 256, kth_smem, st>>>(sscore, pl.ns, pl.ks, thr);
  // 3. filter pass over all keys
  gp.n = p.n_off;
  gp.key_row0 = p.off_begin;
  gp.key_unit_rows = p.cap;
  gp.mode = kFilter;
  gp.thresh = thr;
  gp.counts = counts;
  gp.cand = cand;
  gp.cap = pl.cap;
  if (int rc = launch_gemm(mapK, mapC, gp, katoms, st)) return rc;
  // 4. select
  cudaMemsetAsync(fail_n, 0, sizeof(int32_t), st);
  const size_t sel_smem = (size_t)pl.cap * 12;
  cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem);
  select_kernel<<<(unsigned)(U * p.C), kSelT, sel_smem, st>>>(cand, counts, pl.cap, p.rho, p.C,
                                                            p.lists, (int32_t)p.off_begin, fail_n,
                                                            fail_rows);
  // 5. exact fallback for rows outside [rho, cap] (host reads the count once)
  int32_t nf = 0;
  cudaMemcpyAsync(&nf, fail_n, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return CTKV_ECUDA;
  if (nf > 0) {
    if (p.flags) {
      const int32_t bit = kFlagBuildFallback;
      // OR the info bit in (tiny kernel-free path: read-modify-write on stream order)
      int32_t cur = 0;
      cudaMemcpy(&cur, p.flags, 4, cudaMemcpyDeviceToHost);
      cur |= bit;
      cudaMemcpy(p.flags, &cur, 4, cudaMemcpyHostToDevice);
    }
    // reuse the sample-score buffer as scratch, in chunks of rows
    const int64_t chunk = std::max<int64_t>(1, ((int64_t)U * p.C * pl.ns) / p.n_off);
    for (int64_t r0 = 0; r0 < nf; r0 += chunk) {
      const int64_t nr = std::min<int64_t>(chunk, nf - r0);
      dim3 grid((unsigned)((p.n_off + 255) / 256), (unsigned)nr);
      row_scores_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(p.cent),
                                              static_cast<const __nv_bfloat16*>(p.keys),
                                              fail_rows + r0, p.C, p.gs, p.h, p.g, p.d, p.cap,
                                              p.off_begin, p.n_off, scale, sscore);
      if (int rc = topk_launch(sscore, nr, p.n_off, p.n_off, p.rho, p.lists, p.rho,
                               (int32_t)p.off_begin, st, -1, 0, fail_rows + r0))
        return rc;
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

}  // namespace ctkv
