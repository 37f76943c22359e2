// Decode tail (bf16 fused step): the per-(b,g) work that nothing later in
// the step reads, run by the engine on a side stream beside the next layers:
//
//   * the full (score desc, recall position asc) order of the unit's L
//     recalled tokens -- an O(L) counting sort over linear bins of the
//     packed score keys plus an exact rank inside each (small) bin
//     (ck/tensor_ops.py:121-141 order on the rerank scores);
//   * the FIFO dynamic centroid update: the top-rho list row, the query
//     rows and their norms into slot fifo_head % C (ck/index.py:103-133);
//   * the ordered sparse ids (RerankResult.sparse_ids, ck/retrieval.py:210-216);
//   * the last unit advances the per-batch cursors and the token counter
//     (ck/index.py:121,133; ck/store.py:125-129).
//
// Inputs come from the chain kernel's workspace: keyg / recg per position,
// uctr[u] = (.., .., L, R).
#include <cfloat>
#include <cmath>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_decode_dev.cuh"
#include "ctkv_internal.h"

namespace ctkv {

constexpr int kTailT = 256;            // threads per tail CTA
constexpr int kTailBins = 1024;        // counting-sort bins

__host__ __device__ inline size_t tail_smem(const DecodeParams& p) {
  const int lmax = p.lmax > 1 ? p.lmax : 1;
  return align16((size_t)lmax * 4) + align16((size_t)2 * lmax * 2) + (size_t)2 * kTailBins * 4;
}

template <typename T, int D>
__global__ void __launch_bounds__(kTailT) tail_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int u = blockIdx.x;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int64_t s_slot;
  __shared__ uint32_t s_mm[2 * (kTailT / 32)];
  const int lmax = p.lmax > 1 ? p.lmax : 1;
  // positions fit 16 bits (lmax = c' * rho <= 32768): 8 B per recall slot
  uint32_t* k32 = reinterpret_cast<uint32_t*>(smem);                          // [lmax] score keys
  uint16_t* binned = reinterpret_cast<uint16_t*>(smem + align16((size_t)lmax * 4));   // [lmax] by bin
  uint16_t* order = binned + lmax;                                            // [lmax] rank -> position
  int* hist = reinterpret_cast<int*>(smem + align16((size_t)lmax * 4) + align16((size_t)2 * lmax * 2));
  int* cur = hist + kTailBins;                                                // [kTailBins]
  pdl_trigger();
  pdl_wait();
  ktl_mark(p.tl, 2, false);
  if (tid == 0) s_slot = p.fifo ? (p.fifo[bi] % p.C) : 0;
  const int L = p.uctr[u * 4 + 2], Rn = p.uctr[u * 4 + 3];
  const bool dcu_here = (p.stages & kStageDcu) && L > 0;
  const bool need_sort = L > 0 && (dcu_here || (p.sparse_ids && p.use_rerank));
  const uint64_t* kg = p.keyg + (int64_t)u * p.lmax;
  const int32_t* rec = p.recg + (int64_t)u * p.lmax;
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  if (need_sort) {
    // full (score desc, position asc) order by a counting sort over linear
    // bins of [min, max] of the score keys, then an exact rank inside each
    // (small) bin -- O(L), no comparison sort
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (int i = tid; i < L; i += kTailT) {
      const uint32_t k = (uint32_t)(__ldcg(kg + i) >> 32);
      k32[i] = k;
      mn = min(mn, k);
      mx = max(mx, k);
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) { s_mm[warp] = mn; s_mm[kTailT / 32 + warp] = mx; }
    for (int b = tid; b < kTailBins; b += kTailT) hist[b] = 0;
    __syncthreads();
    mn = 0xffffffffu;
    mx = 0u;
    for (int w = 0; w < kTailT / 32; ++w) { mn = min(mn, s_mm[w]); mx = max(mx, s_mm[kTailT / 32 + w]); }
    const float fscale = (float)kTailBins / ((float)(mx - mn) + 1.0f);
    auto bin_of = [&](uint32_t k) { return min(kTailBins - 1, (int)((float)(k - mn) * fscale)); };
    for (int i = tid; i < L; i += kTailT) atomicAdd(&hist[bin_of(k32[i])], 1);
    __syncthreads();
    {
      constexpr int BPT = kTailBins / kTailT;
      int loc = 0;
      for (int x = 0; x < BPT; ++x) loc += hist[tid * BPT + x];
      int tot;
      int run = block_exclusive_scan(loc, &tot, reinterpret_cast<double*>(s_mm));
      for (int x = 0; x < BPT; ++x) {
        cur[tid * BPT + x] = run;
        run += hist[tid * BPT + x];
      }
    }
    __syncthreads();
    for (int i = tid; i < L; i += kTailT) binned[atomicAdd(&cur[bin_of(k32[i])], 1)] = (uint16_t)i;
    __syncthreads();
    for (int i = tid; i < L; i += kTailT) {
      const uint32_t k = k32[i];
      const int b = bin_of(k);
      const int e = cur[b], s0 = e - hist[b];
      int r = s0;
      for (int x = s0; x < e; ++x) {
        const int j = binned[x];
        const uint32_t kj = k32[j];
        r += (kj < k) || (kj == k && j < i);
      }
      order[r] = (uint16_t)i;
    }
  }
  __syncthreads();
  auto pos_at = [&](int i) { return order[i]; };
  if (dcu_here) {
    const int64_t slot = s_slot;
    int32_t* row = p.lists + ((int64_t)u * p.C + slot) * p.rho;
    const int keep = min(p.rho, L);
    for (int i = tid; i < p.rho; i += kTailT) row[i] = i < keep ? rec[pos_at(i)] : kEmpty;
    T* cent = static_cast<T*>(p.cent);
    constexpr int VPR = D * int(sizeof(T)) / 16;   // 16-byte pieces per row
    for (int i = tid; i < gs * VPR; i += kTailT) {
      const int hh = i / VPR, e = i % VPR;
      reinterpret_cast<uint4*>(cent + (((int64_t)bi * p.h + gi * gs + hh) * p.C + slot) * D)[e] =
          reinterpret_cast<const uint4*>(q)[i];
    }
    write_slot_norms<T, D>(p, q, bi, gi, slot);
  }
  if (p.sparse_ids)
    for (int i = tid; i < p.sparse_cap; i += kTailT)
      p.sparse_ids[(int64_t)u * p.sparse_cap + i] =
          i < Rn ? rec[p.use_rerank ? pos_at(i) : i] : kEmpty;

  // completion: FIFO cursor advance + total++ by the last unit
  if (p.stages & (kStageDcu | kStageAppendTail)) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (dcu_here) atomicAdd(&p.sync[1 + bi], 1);
      __threadfence();
      const int prev = atomicAdd(&p.sync[0], 1);
      if (prev == p.U - 1) {
        __threadfence();
        for (int b2 = 0; b2 < p.b; ++b2) {
          const int hits = atomicExch(&p.sync[1 + b2], 0);
          if (hits > 0) p.fifo[b2] = p.fifo[b2] % p.C + 1;
        }
        if (p.k_new != nullptr) *p.total = *p.total + 1;
        atomicExch(&p.sync[0], 0);
        __threadfence();
      }
    }
  }
  __syncthreads();
  ktl_mark(p.tl, 2, true);
}

// ------------------------------------------------------------------------
// launcher
// ------------------------------------------------------------------------

template <typename T, int D>
static int launch_tail_t(const DecodeParams& p, cudaStream_t st) {
  const bool any = (p.stages & (kStageDcu | kStageAppendTail)) || p.sparse_ids;
  if (!any) return CTKV_OK;
  auto kt = tail_kernel<T, D>;
  const size_t sm = tail_smem(p);
  if (int rc = set_max_smem_k(kt, sm)) return rc;
  launch_k(kt, dim3(p.U), dim3(kTailT), sm, st, kPrioMid, p);
  return cudaGetLastError() == cudaSuccess ? CTKV_OK : CTKV_ECUDA;
}

bool tail_supported(const DecodeParams& p, int dtype, int D) {
  if (dtype != CTKV_BF16 || (D != 64 && D != 128)) return false;
  if (p.lmax > 65535) return false;   // 16-bit positions
  return tail_smem(p) <= 200 * 1024;
}

int launch_tail(const DecodeParams& p, int dtype, int D, cudaStream_t st) {
  if (dtype != CTKV_BF16) return CTKV_ECONFIG;
  if (D == 128) return launch_tail_t<__nv_bfloat16, 128>(p, st);
  if (D == 64) return launch_tail_t<__nv_bfloat16, 64>(p, st);
  return CTKV_ECONFIG;
}

}  // namespace ctkv
