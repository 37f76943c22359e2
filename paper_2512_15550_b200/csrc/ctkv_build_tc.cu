// Tensor-core prefill index build (Alg. 1, ck/index.py:59-99) for bf16 stores.
//
// Grouped scores S[c, j] = max_h (q_{h,c} . k_j) / sqrt(d) are a GEMM with
// M = offloaded keys, N = gs heads x CB centroids (= 256), K = d.  Keys are
// the A operand (TMA, 128B swizzle, 128 rows per tile), the centroid rows of
// one work item the resident B operand, accumulators live in TMEM (two
// 256-column buffers so the epilogue of tile i overlaps the MMAs of tile
// i+1).  Warp roles: 0 = TMA producer, 1 = MMA issuer (+TMEM owner),
// 2..17 = epilogue: 4 warps per TMEM lane quadrant, each owning CB/4
// centroids x gs heads = 64 accumulator columns, read with one batch of
// tcgen05.ld and a single wait, group max + scale in registers.
// A work item is (unit, centroid block, key split); small problems split the
// keys so every SM has work; each (row, key split) owns a candidate segment
// whose counter lives in shared memory for the item (no global atomics).
//
// Top-rho per row without materialising the 6.4 GB/layer score matrix:
//   1. sample pass  -- the same GEMM against every S-th key; the epilogue
//                      stores only the top 16 bits of each score's
//                      order-preserving key (2 B per sampled score);
//   2. threshold    -- per row the lower edge of the histogram bin holding
//                      the k_s-th largest sample key (warp per row), with
//                      k_s chosen so the full row has ~rho + 6 sigma
//                      candidates above it with overwhelming probability;
//   3. filter pass  -- the full GEMM; the epilogue keeps (score, key) pairs
//                      >= threshold in a per-row buffer;
//   4. select       -- per row, order the <= cap candidates by (score desc,
//                      key asc) and write the first rho ids -- exact top-rho
//                      of the tensor-core scores whenever rho <= count <= cap;
//   5. fallback     -- rows outside [rho, cap] (rare) are recomputed in full
//                      and radix-selected by a fixed-grid kernel that reads
//                      the failure count on the device (no host sync; the
//                      whole build is stream-ordered and graph-capturable).
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
constexpr int kEpiWarps = 16;     // 4 per TMEM lane quadrant
constexpr int kThreads = 64 + 32 * kEpiWarps;   // producer + MMA + epilogue
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
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float* v) {
  uint32_t r[2];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(taddr));
  v[0] = __uint_as_float(r[0]);
  v[1] = __uint_as_float(r[1]);
}
__device__ __forceinline__ void tmem_ld1(uint32_t taddr, float* v) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  v[0] = __uint_as_float(r);
}
// NC consecutive accumulator columns of this warp's 32 TMEM lanes (no wait)
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* v) {
  if constexpr (NC >= 16) {
#pragma unroll
    for (int i = 0; i < NC / 16; ++i) tmem_ld16(taddr + 16 * i, v + 16 * i);
  } else if constexpr (NC == 8) {
    tmem_ld8(taddr, v);
  } else if constexpr (NC == 4) {
    tmem_ld4(taddr, v);
  } else if constexpr (NC == 2) {
    tmem_ld2(taddr, v);
  } else {
    static_assert(NC == 1, "column count");
    tmem_ld1(taddr, v);
  }
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// predicated (branch-free) shared-memory slot reservation: old value of
// *addr, incremented, when `pred`; `otherwise` when not
__device__ __forceinline__ int atom_inc_if(bool pred, uint32_t addr, int otherwise) {
  int r = otherwise;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "@p atom.shared.add.u32 %0, [%1], 1;\n\t}"
      : "+r"(r)
      : "r"(addr), "r"((int)pred)
      : "memory");
  return r;
}
__device__ __forceinline__ void st_global_if(bool pred, uint64_t* ptr, uint64_t v) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "@p st.global.u64 [%0], %1;\n\t}" ::"l"(ptr),
      "l"(v), "r"((int)pred)
      : "memory");
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
  int ksplit;              // key splits per (unit, centroid block)
  int64_t tiles_per_split;
  // store mode (sample pass)
  uint16_t* out16;         // [U][C][n] top 16 bits of the score keys
  // filter mode
  const float* thresh;     // [U*C]
  int32_t* counts;         // [U*C][ksplit] candidates per (row, key split)
  uint64_t* cand;          // [U*C][ksplit][cap]
  int cap;
};

template <int KATOMS, int GS>
__global__ void __launch_bounds__(kThreads, 1)
    scores_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     Params p) {
  constexpr int CB = kBN / GS;     // centroids per item
  constexpr int NC = CB / 4;       // centroids per epilogue warp (64 / GS)
  constexpr int WV = 32 / GS < 16 ? 32 / GS : 16;
  constexpr int W = NC < WV ? NC : WV;            // centroids per register chunk (<= 32 values)
  constexpr int NCH = NC / W;                     // chunks per tile
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
  float* s_thr = reinterpret_cast<float*>(tmem_slot + 4);    // [kEpiWarps][NC]
  int* s_cnt = reinterpret_cast<int*>(s_thr + kEpiWarps * 64); // [CB] candidates per row (item)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (p.n + kBM - 1) / kBM;
  // item = ((u * ksplit + ks) * n_cblocks + cb): CTAs running side by side
  // share a unit's key range (L2 reuse of the A tiles)
  auto decode = [&](int it, int& u, int& cb, int& ks, int64_t& t0, int64_t& t1) {
    cb = it % p.n_cblocks;
    const int r = it / p.n_cblocks;
    u = r / p.ksplit;
    ks = r % p.ksplit;
    t0 = (int64_t)ks * p.tiles_per_split;
    t1 = t0 + p.tiles_per_split < ntiles ? t0 + p.tiles_per_split : ntiles;
  };

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
        int u, cb, ks;
        int64_t t0, t1;
        decode(it, u, cb, ks, t0, t1);
        const int bi = u / p.g, gi = u % p.g;
        // B: centroid rows (head j, centroids cb*CB ..) of this unit, all K atoms
        mbar_wait(bempty, item_phase ^ 1);
        mbar_expect_tx(bfull, kBBytes);
        for (int ka = 0; ka < KATOMS; ++ka)
          for (int j = 0; j < GS; ++j) {
            const int32_t row = ((bi * p.h + gi * GS + j) * p.C) + cb * CB;
            tma_load_2d(sB + ka * kBAtom + j * CB * 128, &mapB, bfull, ka * 64, row);
          }
        item_phase ^= 1;
        const int64_t row0 = p.key_row0 + (int64_t)u * p.key_unit_rows;
        for (int64_t t = t0; t < t1; ++t) {
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
        int u, cb, ks;
        int64_t t0, t1;
        decode(it, u, cb, ks, t0, t1);
        mbar_wait(bfull, item_phase);
        item_phase ^= 1;
        tc_fence_after();
        for (int64_t t = t0; t < t1; ++t) {
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
    // ===================== epilogue (16 warps) =====================
    // warp ew = warp - 2 reads TMEM lanes 32*(warp % 4) (the quadrant its
    // hardware warp slot may touch) and centroids [part*NC, part*NC + NC)
    const int ew = warp - 2;
    const int quad = warp & 3;
    const int part = ew >> 2;
    const int etid = threadIdx.x - 64;
    constexpr int kEpiT = 32 * kEpiWarps;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
      int u, cb, ks;
      int64_t t0, t1;
      decode(it, u, cb, ks, t0, t1);
      const int64_t rowbase = (int64_t)u * p.C + (int64_t)cb * CB + part * NC;
      // this warp's NC row thresholds (its private smem slice: no cross-warp sync)
      float* thr = s_thr + ew * NC;
      int* cnt = s_cnt + part * NC;
      if (p.mode == kFilter) {
        __syncwarp();
        for (int c = lane; c < NC; c += 32) thr[c] = __ldg(p.thresh + rowbase + c);
        for (int i = etid; i < CB; i += kEpiT) s_cnt[i] = 0;
        named_bar(1, kEpiT);
      }
      for (int64_t t = t0; t < t1; ++t) {
        mbar_wait(tfull(acc), acc_phase);
        tc_fence_after();
        const int64_t key = t * kBM + quad * 32 + lane;
        const bool valid = key < p.n;
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + acc * kBN + part * NC;
        // column chunks of W centroids x GS heads (<= 64 live values: for
        // GS >= 4 all of the warp's columns in one batch and one wait); the
        // accumulator goes back to the MMA warp once the last chunk is in
        // registers, before the chunk's group max / filter
#pragma unroll 1
        for (int ch = 0; ch < NCH; ++ch) {
          float v[GS][W];
#pragma unroll
          for (int j = 0; j < GS; ++j) tmem_ld_cols<W>(tbase + j * CB + ch * W, v[j]);
          tmem_ld_wait();
          if (ch == NCH - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty(acc));
          }
#pragma unroll
          for (int c = 0; c < W; ++c) {
            float m = v[0][c];
#pragma unroll
            for (int j = 1; j < GS; ++j) m = fmaxf(m, v[j][c]);
            v[0][c] = m * p.scale;
          }
          const int64_t row0 = rowbase + ch * W;
          if (p.mode == kStore) {
            if (valid) {
#pragma unroll
              for (int c = 0; c < W; ++c)
                p.out16[(row0 + c) * p.n + key] = (uint16_t)(okey32(v[0][c]) >> 16);
            }
          } else {
            // hits are rare (~2 % of scores): each lane reserves its own
            // slots with shared-memory atomics on the row counters (no
            // ballots, no shuffles; same-row lanes are merged by the atomic unit)
            unsigned hits = 0u;
#pragma unroll
            for (int c = 0; c < W; c += 2) {
              const float2 t = *reinterpret_cast<const float2*>(thr + ch * W + c);
              hits |= (unsigned)(v[0][c] >= t.x) << c;
              hits |= (unsigned)(v[0][c + 1] >= t.y) << (c + 1);
            }
            if (!valid) hits = 0u;
            if (__any_sync(0xffffffffu, hits != 0u)) {
              // all of this lane's reservations first (independent, in
              // flight together), then the stores
              uint64_t* dst = p.cand + (row0 * p.ksplit + ks) * p.cap;
              const int rstride = p.ksplit * p.cap;
              const uint32_t cnt_s = smem_u32(cnt + ch * W);
              int pos[W];
#pragma unroll
              for (int c = 0; c < W; ++c) pos[c] = atom_inc_if((hits >> c) & 1u, cnt_s + 4 * c, p.cap);
#pragma unroll
              for (int c = 0; c < W; ++c)
                st_global_if(pos[c] < p.cap, dst + (uint32_t)(c * rstride + pos[c]),
                             ((uint64_t)(~okey32(v[0][c])) << 32) | (uint32_t)key);
            }
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (p.mode == kFilter) {
        named_bar(1, kEpiT);   // every warp's hits of this item are counted
        const int64_t r0 = (int64_t)u * p.C + (int64_t)cb * CB;
        for (int i = etid; i < CB; i += kEpiT) p.counts[(r0 + i) * p.ksplit + ks] = s_cnt[i];
        named_bar(1, kEpiT);   // before the next item resets the counters
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

// per row: a threshold with at least k of the row's n 16-bit sample keys at
// or above it -- the lower edge of the histogram bin holding the k-th
// largest key.  One warp per row: min/max of the keys, then a 1024-bin
// histogram over [min, max] (power-of-two bin width, so spread-out bins and
// little atomic contention), then a top-down prefix over the bins.  Any
// such threshold is valid (the filter pass keeps every score at or above
// it); a narrower bin only means fewer surplus candidates.
constexpr int kKthWarps = 8, kKthBins = 1024;

// f(key) for every 16-bit key of a row, the aligned middle with 16-byte
// loads (8 keys each, several in flight per lane), head and tail scalar
template <typename F>
__device__ __forceinline__ void row_keys16(const uint16_t* r, int64_t n, int lane, F&& f) {
  int64_t head = (int64_t)(((16u - (reinterpret_cast<uintptr_t>(r) & 15u)) & 15u) >> 1);
  if (head > n) head = n;
  if (lane < head) f((uint32_t)__ldg(r + lane));
  const uint4* v = reinterpret_cast<const uint4*>(r + head);
  const int64_t nv = (n - head) >> 3;
#pragma unroll 2
  for (int64_t i = lane; i < nv; i += 32) {
    const uint4 w = __ldg(v + i);
    f(w.x & 0xffffu); f(w.x >> 16); f(w.y & 0xffffu); f(w.y >> 16);
    f(w.z & 0xffffu); f(w.z >> 16); f(w.w & 0xffffu); f(w.w >> 16);
  }
  for (int64_t i = head + nv * 8 + lane; i < n; i += 32) f((uint32_t)__ldg(r + i));
}
__global__ void __launch_bounds__(32 * kKthWarps) kth_value_kernel(const uint16_t* __restrict__ S,
                                                                  int64_t n, int64_t rows, int k,
                                                                  float* __restrict__ thr) {
  __shared__ int hist_all[kKthWarps][kKthBins];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kKthWarps + warp;
  if (row >= rows) return;
  int* hist = hist_all[warp];
  const uint16_t* r = S + row * n;
  uint32_t mn = 0xffffu, mx = 0u;
  row_keys16(r, n, lane, [&](uint32_t x) {
    mn = min(mn, x);
    mx = max(mx, x);
  });
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  int sh = 0;
  while (((mx - mn) >> sh) >= (uint32_t)kKthBins) ++sh;
  for (int b = lane; b < kKthBins; b += 32) hist[b] = 0;
  __syncwarp();
  row_keys16(r, n, lane, [&](uint32_t x) { atomicAdd(&hist[(x - mn) >> sh], 1); });
  __syncwarp();
  // lane L owns bins [kKthBins - 32(L+1), kKthBins - 32L): counts from the top
  constexpr int per = kKthBins / 32;
  const int hi = kKthBins - lane * per;
  int sum = 0;
  for (int b = hi - 1; b >= hi - per; --b) sum += hist[b];
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int want = min(k, (int)n);
  unsigned bal = __ballot_sync(0xffffffffu, incl >= want && incl - sum < want);
  const int owner = __ffs(bal) - 1;
  int bin = 0, above = 0;
  if (lane == owner) {
    int run = incl - sum;
    bin = hi - per;
    for (int b = hi - 1; b >= hi - per; --b) {
      if (run + hist[b] >= want) { bin = b; break; }
      run += hist[b];
    }
    above = run;   // keys in bins above `bin`
  }
  bin = __shfl_sync(0xffffffffu, bin, owner);
  above = __shfl_sync(0xffffffffu, above, owner);
  uint32_t key = mn + ((uint32_t)bin << sh);
  if (sh > 0) {
    // refine inside the bin (2^sh <= 64 distinct keys): exact k-th largest
    __syncwarp();
    for (int b = lane; b < 64; b += 32) hist[b] = 0;
    __syncwarp();
    const uint32_t lo = key, wid = 1u << sh;
    row_keys16(r, n, lane, [&](uint32_t x) {
      x -= lo;
      if (x < wid) atomicAdd(&hist[x], 1);
    });
    __syncwarp();
    // lane L owns sub-bins 2L, 2L+1 counted from the top (63 - 2L, 62 - 2L)
    const int b0 = 63 - 2 * lane, b1 = 62 - 2 * lane;
    const int c0 = b0 < (int)wid ? hist[b0] : 0, c1 = b1 < (int)wid ? hist[b1] : 0;
    int inc2 = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc2, o);
      if (lane >= o) inc2 += y;
    }
    const int ex2 = above + inc2 - c0 - c1;
    bal = __ballot_sync(0xffffffffu, ex2 + c0 + c1 >= want && ex2 < want);
    const int o2 = __ffs(bal) - 1;
    const int sub = ex2 + c0 >= want ? b0 : b1;
    key = lo + (uint32_t)__shfl_sync(0xffffffffu, sub, o2);
  }
  if (lane == 0) thr[row] = okey32_inv(key << 16);
}

// per row: exact top-rho of the candidates in (score desc, key asc) order, or
// flag the row for the fallback.  O(n) counting sort instead of a comparison
// sort: linear bins over [min, max] of the candidates' score keys, bin
// offsets by a block scan, then each candidate's exact rank inside its
// (small) bin; ranks < rho are written straight to the list.
constexpr int kSelT = 256, kSelBins = 2048;
__global__ void __launch_bounds__(kSelT) select_kernel(const uint64_t* __restrict__ cand,
                                                       const int32_t* __restrict__ counts, int nsplit,
                                                       int cap,
                                                       int rho, int C, int32_t* __restrict__ lists,
                                                       int32_t add, int32_t* fail_n,
                                                       int32_t* fail_rows) {
  extern __shared__ uint64_t ck[];                            // [cap] candidates
  uint16_t* binned = reinterpret_cast<uint16_t*>(ck + cap);  // [cap] indices grouped by bin
  // bin counts, then (in place) exclusive starts, then after the scatter
  // each bin's end: bin b spans [end[b-1], end[b])
  __shared__ int hist[kSelBins];
  __shared__ uint32_t s_mm[2 * kSelT / 32];
  __shared__ int s_ws[kSelT / 32 + 1];
  const int64_t row = blockIdx.x;
  int cnt = 0;
  for (int s = 0; s < nsplit; ++s) cnt += __ldg(counts + row * nsplit + s);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (cnt < rho || cnt > cap) {
    if (tid == 0) fail_rows[atomicAdd(fail_n, 1)] = (int32_t)row;
    return;
  }
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int s = 0, at = 0; s < nsplit; ++s) {
    const int n_s = __ldg(counts + row * nsplit + s);
    // 16-byte loads (two candidates each, segments are 16-byte aligned),
    // several in flight per thread
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(cand + (row * nsplit + s) * cap);
#pragma unroll 4
    for (int i = tid; 2 * i < n_s; i += kSelT) {
      const ulonglong2 w = __ldg(src + i);
      ck[at + 2 * i] = w.x;
      mn = min(mn, (uint32_t)(w.x >> 32));
      mx = max(mx, (uint32_t)(w.x >> 32));
      if (2 * i + 1 < n_s) {
        ck[at + 2 * i + 1] = w.y;
        mn = min(mn, (uint32_t)(w.y >> 32));
        mx = max(mx, (uint32_t)(w.y >> 32));
      }
    }
    at += n_s;
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
      const int c = hist[tid * BPT + x];
      hist[tid * BPT + x] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int i = tid; i < cnt; i += kSelT) binned[atomicAdd(&hist[bin_of(ck[i])], 1)] = (uint16_t)i;
  __syncthreads();
  int32_t* dst = lists + row * rho;
  for (int i = tid; i < cnt; i += kSelT) {
    const uint64_t k = ck[i];
    const int b = bin_of(k);
    const int e = hist[b], s0 = b > 0 ? hist[b - 1] : 0;
    if (s0 >= rho) continue;                    // the whole bin ranks below the list
    int r = s0;
    for (int x = s0; x < e; ++x) r += ck[binned[x]] < k;
    if (r < rho) dst[r] = (int32_t)(k & 0xffffffffu) + add;
  }
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
         sizeof(float) * kEpiWarps * 64 + sizeof(int) * kBN;
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

template <int KATOMS, int GS>
static int launch_gemm_t(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p,
                         cudaStream_t st) {
  const size_t sm = smem_bytes(KATOMS);
  const int grid = std::min(p.items, num_sms());
  auto k = scores_tc_kernel<KATOMS, GS>;
  if (int rc = set_max_smem_k(k, sm)) return rc;
  k<<<grid, kThreads, sm, st>>>(ma, mb, p);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

template <int KATOMS>
static int launch_gemm_k(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p,
                         cudaStream_t st) {
  switch (p.gs) {
    case 1: return launch_gemm_t<KATOMS, 1>(ma, mb, p, st);
    case 2: return launch_gemm_t<KATOMS, 2>(ma, mb, p, st);
    case 4: return launch_gemm_t<KATOMS, 4>(ma, mb, p, st);
    case 8: return launch_gemm_t<KATOMS, 8>(ma, mb, p, st);
    case 16: return launch_gemm_t<KATOMS, 16>(ma, mb, p, st);
  }
  return CTKV_ESHAPE;
}

// work items: (unit, centroid block, key split); split the keys until every
// SM has ~8 items (load balance at small batch x C), keeping >= 16 tiles each
static int key_splits(int64_t n, int U, int n_cblocks, int64_t* tiles_per_split) {
  const int64_t ntiles = (n + kBM - 1) / kBM;
  const int base = U * n_cblocks;
  int ks = (8 * num_sms() + base - 1) / base;
  ks = (int)std::max<int64_t>(1, std::min<int64_t>(ks, ntiles / 16));
  const int64_t tps = (ntiles + ks - 1) / ks;
  if (tiles_per_split) *tiles_per_split = tps;
  return (int)((ntiles + tps - 1) / tps);
}

static void set_items(Params& gp) {
  gp.ksplit = key_splits(gp.n, gp.U, gp.n_cblocks, &gp.tiles_per_split);
  gp.items = gp.U * gp.n_cblocks * gp.ksplit;
}

static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, Params p, int katoms,
                       cudaStream_t st) {
  set_items(p);
  if (katoms == 2) return launch_gemm_k<2>(ma, mb, p, st);
  if (katoms == 1) return launch_gemm_k<1>(ma, mb, p, st);
  return CTKV_ESHAPE;
}

struct Plan {
  int S;        // sample stride
  int64_t ns;   // sampled keys per unit
  int ks;       // sample rank giving the threshold
  int cap;      // candidate slots per row (and per key split of a row)
  int CB;
  int fsplit;   // key splits of the filter pass
};

static Plan make_plan(const BuildParams& p) {
  Plan pl;
  pl.S = 16;
  pl.ns = (p.n_off + pl.S - 1) / pl.S;
  const double mean = (double)p.rho / pl.S;
  pl.ks = (int)std::ceil(mean + 6.0 * std::sqrt(mean)) + 1;
  if (pl.ks > pl.ns) pl.ks = (int)pl.ns;
  const int64_t expect = (int64_t)pl.ks * pl.S;
  // candidates above the sample threshold: ~expect +- S*sqrt(ks) (plus the
  // 16-bit bin the threshold is widened to); 8 sigma of headroom (rows beyond
  // it take the exact fallback)
  const int64_t head = (int64_t)std::ceil(8.0 * pl.S * std::sqrt((double)pl.ks));
  pl.cap = (int)std::min<int64_t>(((std::max<int64_t>(expect + head, p.rho + 1024) + 255) / 256) * 256,
                                  1 << 14);
  pl.CB = kBN / p.gs;
  pl.fsplit = key_splits(p.n_off, p.b * p.g, p.C / pl.CB, nullptr);
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

namespace {
struct TcWs {
  __nv_bfloat16* skeys;
  uint16_t* skey16;
  float* thr;
  int32_t* counts;
  uint64_t* cand;
  int32_t* fail_n;
  int32_t* fail_rows;
  float* scratch;      // fallback rows (aliases the sample keys + scores)
  int scratch_rows;
  size_t bytes;
};

TcWs carve_tc(const BuildParams& p, void* base) {
  const tc::Plan pl = tc::make_plan(p);
  const int64_t U = (int64_t)p.b * p.g;
  auto a256 = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  auto take = [&](size_t b) {
    char* q = base ? static_cast<char*>(base) + off : nullptr;
    off += a256(b);
    return q;
  };
  TcWs w;
  const size_t sk = (size_t)U * pl.ns * p.d * 2, ss = (size_t)U * p.C * pl.ns * 2;
  // the fallback scratch reuses the sample region (dead after the thresholds)
  const size_t fb_min = (size_t)8 * p.n_off * 4;
  const size_t shared = std::max(a256(sk) + a256(ss), fb_min);
  char* sh = take(shared);
  w.skeys = reinterpret_cast<__nv_bfloat16*>(sh);
  w.skey16 = reinterpret_cast<uint16_t*>(sh ? sh + a256(sk) : nullptr);
  w.scratch = reinterpret_cast<float*>(sh);
  w.scratch_rows = (int)std::min<int64_t>(148, (int64_t)(shared / ((size_t)p.n_off * 4)));
  w.thr = reinterpret_cast<float*>(take((size_t)U * p.C * 4));
  // each (row, key split) owns a whole cap-slot segment: a split never
  // overflows before the row does (top scores may cluster in one split)
  w.counts = reinterpret_cast<int32_t*>(take((size_t)U * p.C * pl.fsplit * 4));
  w.cand = reinterpret_cast<uint64_t*>(take((size_t)U * p.C * pl.fsplit * pl.cap * 8));
  w.fail_n = reinterpret_cast<int32_t*>(take((size_t)U * p.C * 4 + 16));
  w.fail_rows = w.fail_n ? w.fail_n + 4 : nullptr;
  w.bytes = off;
  return w;
}
}  // namespace

size_t build_tc_workspace_bytes(const BuildParams& p) { return carve_tc(p, nullptr).bytes; }

int build_tc(const BuildParams& p, int /*dtype*/, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace tc;
  const Plan pl = make_plan(p);
  const int U = p.b * p.g;
  const TcWs w = carve_tc(p, ws);
  if (w.bytes > ws_bytes) return CTKV_EWORKSPACE;
  const int katoms = p.d / 64;
  const float scale = (float)(1.0 / std::sqrt((double)p.d));

  // 1. sample keys
  {
    const int vpr = p.d * 2 / 16;
    const int64_t total = (int64_t)U * pl.ns * vpr;
    gather_sample_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
        static_cast<const uint4*>(p.keys), reinterpret_cast<uint4*>(w.skeys), p.cap, p.off_begin,
        pl.S, pl.ns, vpr, U);
  }
  CUtensorMap mapS, mapK, mapC;
  if (!make_map(&mapS, w.skeys, (int64_t)U * pl.ns, p.d, kBM) ||
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
  gp.scale = scale;
  // 2. sample pass (16-bit score keys) + thresholds
  gp.n = pl.ns;
  gp.key_row0 = 0;
  gp.key_unit_rows = pl.ns;
  gp.mode = kStore;
  gp.out16 = w.skey16;
  if (int rc = launch_gemm(mapS, mapC, gp, katoms, st)) return rc;
  const int64_t nrows = (int64_t)U * p.C;
  kth_value_kernel<<<(unsigned)((nrows + kKthWarps - 1) / kKthWarps), 32 * kKthWarps, 0, st>>>(
      w.skey16, pl.ns, nrows, pl.ks, w.thr);
  // 3. filter pass over all keys (every (row, split) count is written by its item)
  gp.n = p.n_off;
  gp.key_row0 = p.off_begin;
  gp.key_unit_rows = p.cap;
  gp.mode = kFilter;
  gp.thresh = w.thr;
  gp.counts = w.counts;
  gp.cand = w.cand;
  gp.cap = pl.cap;
  if (int rc = launch_gemm(mapK, mapC, gp, katoms, st)) return rc;
  // 4. select
  cudaMemsetAsync(w.fail_n, 0, sizeof(int32_t), st);
  const size_t sel_smem = (size_t)pl.cap * 10;
  if (int rc = set_max_smem_k(select_kernel, sel_smem)) return rc;
  select_kernel<<<(unsigned)(U * p.C), kSelT, sel_smem, st>>>(w.cand, w.counts, pl.fsplit, pl.cap, p.rho, p.C,
                                                            p.lists, (int32_t)p.off_begin, w.fail_n,
                                                            w.fail_rows);
  // 5. exact fallback for rows outside [rho, cap], driven by the device count
  if (int rc = launch_build_fallback(p.cent, p.keys, w.fail_n, w.fail_rows, p.C, p.gs, p.h, p.g, p.d,
                                     p.cap, p.off_begin, p.n_off, scale, w.scratch,
                                     std::max(1, w.scratch_rows), p.rho, p.lists, p.flags, st))
    return rc;
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

}  // namespace ctkv
