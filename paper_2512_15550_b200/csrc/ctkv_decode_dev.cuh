// Device helpers shared by the decode-step kernel files (ctkv_decode.cu,
// ctkv_unit_wide.cu): row gathers, weighted row sums, block scans, the
// radix top-R selection and the register bitonic sort of packed keys.
#pragma once

#include "ctkv_common.cuh"
#include "ctkv_internal.h"

namespace ctkv {

template <typename T>
__device__ __forceinline__ const T* kv_row(const T* base, const T* fresh, int64_t cap, int unit,
                                           int64_t id, int64_t t_new, int D) {
  // the token appended by this very step is read from the caller's buffer
  // (the store copy is written concurrently by scan block 0)
  if (fresh != nullptr && id == t_new) return fresh + (int64_t)unit * D;
  return base + ((int64_t)unit * cap + id) * D;
}

// Per-warp weighted row sums: red_warp[hh][:] += sum_t w(hh,t) * row(t)[:]
// for t in [0,n) strided over the block's warps.  Heads are processed four
// at a time so the accumulators stay in registers for any group size; UN
// row passes are loaded before any is consumed (memory-level parallelism).
template <typename T, int D, typename RowFn, typename WFn>
__device__ void accum_weighted_rows(int n, int gs, RowFn rowfn, WFn wfn, float* red_warp) {
  using R = Row<T, D>;
  constexpr int UN = 4;
  const int nwarps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane % R::LPR, rw = lane / R::LPR;
  const int step = nwarps * R::RPW;
  for (int h0 = 0; h0 < gs; h0 += 4) {
    float acc[4][R::EPL];
#pragma unroll
    for (int hh = 0; hh < 4; ++hh)
#pragma unroll
      for (int j = 0; j < R::EPL; ++j) acc[hh][j] = 0.f;
    for (int base = warp * R::RPW; base < n; base += step * UN) {
      float vv[UN][R::EPL];
      bool ok[UN];
#pragma unroll
      for (int u2 = 0; u2 < UN; ++u2) {
        const int t = base + u2 * step + rw;
        const T* row = t < n ? rowfn(t) : nullptr;
        ok[u2] = row != nullptr;
        if (ok[u2]) {
          load_row_slice<T, D>(row, sub, vv[u2]);
        } else {
#pragma unroll
          for (int j = 0; j < R::EPL; ++j) vv[u2][j] = 0.f;
        }
      }
#pragma unroll
      for (int u2 = 0; u2 < UN; ++u2) {
        if (!ok[u2]) continue;
        const int t = base + u2 * step + rw;
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
          if (h0 + hh < gs) {
            const float w = wfn(h0 + hh, t);
#pragma unroll
            for (int j = 0; j < R::EPL; ++j) acc[hh][j] = fmaf(w, vv[u2][j], acc[hh][j]);
          }
        }
      }
    }
#pragma unroll
    for (int hh = 0; hh < 4; ++hh)
#pragma unroll
      for (int j = 0; j < R::EPL; ++j) {
        float x = acc[hh][j];
#pragma unroll
        for (int o = R::LPR; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        acc[hh][j] = x;
      }
    if (rw == 0) {
#pragma unroll
      for (int hh = 0; hh < 4; ++hh)
        if (h0 + hh < gs)
#pragma unroll
          for (int v = 0; v < R::VPL; ++v)
#pragma unroll
            for (int j = 0; j < R::EPV; ++j)
              red_warp[(h0 + hh) * D + R::elem(sub, v) + j] += acc[hh][v * R::EPV + j];
    }
  }
}

struct StaticSpan {
  int64_t n_init, ring_start, n_static;
  __device__ StaticSpan(int64_t total, int init_len, int local_len) {
    n_init = min((int64_t)init_len, total);
    ring_start = max((int64_t)init_len, total - local_len);
    n_static = n_init + (total - ring_start);
  }
  __device__ int64_t id(int64_t i) const { return i < n_init ? i : ring_start + (i - n_init); }
};

// DCU helper: |q_h| of the gs query heads written next to their centroid rows
template <typename T, int D>
__device__ void write_slot_norms(const DecodeParams& p, const T* q, int bi, int gi, int64_t slot) {
  if (p.cnorm == nullptr) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int hh = warp; hh < p.gs; hh += nw) {
    double s = 0.0;
    for (int e = lane; e < D; e += 32) {
      const double v = (double)to_f(q[hh * D + e]);
      s = fma(v, v, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) p.cnorm[((int64_t)bi * p.h + gi * p.gs + hh) * p.C + slot] = (float)sqrt(s);
  }
}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

static __device__ __noinline__ int block_exclusive_scan(int x, int* total, double* scratch) {
  int* ws = reinterpret_cast<int*>(scratch);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  if (warp == 0) {
    int v = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < nw) ws[lane] = v;  // inclusive prefix of warp totals
  }
  __syncthreads();
  const int warp_prefix = warp ? ws[warp - 1] : 0;
  *total = ws[nw - 1];
  return warp_prefix + incl - x;
}

template <int IPT>
__device__ void sort_keys(uint64_t* skey) {
  uint64_t k[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) k[i] = skey[threadIdx.x * IPT + i];
  bitonic_regs<IPT>(k, skey);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) skey[threadIdx.x * IPT + i] = k[i];
  __syncthreads();
}

// positions of the R smallest of the (unique) keys key[0..L) -> spos (any order)
static __device__ int select_smallest(const uint64_t* key, int L, int R, int* spos, int* hist,
                               int* s_state) {
  if (R >= L) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) spos[i] = i;
    __syncthreads();
    return L;
  }
  uint64_t prefix = 0;
  int need = R, shift = 56;
  while (true) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    // warp-aggregated (similar scores share their leading digits)
    for (int i0 = threadIdx.x & ~31; i0 < L; i0 += blockDim.x) {
      const int i = i0 + (threadIdx.x & 31);
      const uint64_t k = i < L ? key[i] : 0ull;
      const bool in = i < L && (shift == 56 || ((k ^ prefix) >> (shift + 8)) == 0);
      const int bin = in ? (int)((k >> shift) & 255) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      if (in && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int sum = 0;
      for (int b = 8 * lane; b < 8 * lane + 8; ++b) sum += hist[b];
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - sum;
      const unsigned bal = __ballot_sync(0xffffffffu, incl >= need && excl < need);
      if (lane == __ffs(bal) - 1) {
        int run = excl;
        for (int b = 8 * lane; b < 8 * lane + 8; ++b) {
          if (run + hist[b] >= need) {
            s_state[0] = b;
            s_state[1] = run;
            s_state[2] = hist[b];
            break;
          }
          run += hist[b];
        }
      }
    }
    __syncthreads();
    const int b = s_state[0], below = s_state[1], cnt = s_state[2];
    prefix |= (uint64_t)b << shift;
    need -= below;
    if (cnt == need || shift == 0) break;
    shift -= 8;
    __syncthreads();
  }
  if (threadIdx.x == 0) s_state[3] = 0;
  __syncthreads();
  const uint64_t lim = prefix >> shift;
  for (int i = threadIdx.x; i < L; i += blockDim.x)
    if ((key[i] >> shift) <= lim) spos[atomicAdd(&s_state[3], 1)] = i;
  __syncthreads();
  return s_state[3];
}

// top-C' centroid slots of unit u from the scan's chunk candidates (value
// desc, slot asc; ck/tensor_ops.py:88-92 on the group-max cosines) -> sel.
// One warp.
static __device__ void warp_top_slots(const DecodeParams& p, int u, int32_t* sel) {
  const int lane = threadIdx.x & 31;
  const int M = p.cos_blocks_per_unit * p.ncand;
  const double* cv = p.cval + (int64_t)u * M;
  const int32_t* ci = p.cidx + (int64_t)u * M;
  constexpr int KR = 8;
  uint64_t rk[KR];
  int ri[KR];
#pragma unroll
  for (int r = 0; r < KR; ++r) {
    const int m = lane + 32 * r;
    rk[r] = m < M ? okey64(__ldcg(cv + m)) : 0ull;
    ri[r] = m < M ? __ldcg(ci + m) : INT32_MAX;
  }
  uint64_t prev_key = ~0ull;
  int prev_idx = -1;
  for (int r = 0; r < p.c_prime; ++r) {
    uint64_t bk = 0;
    int bidx = INT32_MAX;
#pragma unroll
    for (int x = 0; x < KR; ++x) {
      const bool below = rk[x] < prev_key || (rk[x] == prev_key && ri[x] > prev_idx);
      if (below && (rk[x] > bk || (rk[x] == bk && ri[x] < bidx))) { bk = rk[x]; bidx = ri[x]; }
    }
    for (int m = lane + 32 * KR; m < M; m += 32) {
      const uint64_t k = okey64(__ldcg(cv + m));
      const int i = __ldcg(ci + m);
      const bool below = k < prev_key || (k == prev_key && i > prev_idx);
      if (below && (k > bk || (k == bk && i < bidx))) { bk = k; bidx = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (k2 > bk || (k2 == bk && i2 < bidx)) { bk = k2; bidx = i2; }
    }
    if (lane == 0) sel[r] = bidx;
    prev_key = bk;
    prev_idx = bidx;
  }
}

// Top-C' slots of vals[0..C) (value desc, slot asc; ck/tensor_ops.py:121-141
// on the group-max cosines of ck/retrieval.py:145-154) with the whole block,
// by sorting networks over one 64-bit key per entry (no serial arg-max
// rounds, no lane-divergent code around the shuffles):
//   1. each thread keeps a sorted top-K of its strided values (branch-free
//      insertion);
//   2. warps merge lane lists pairwise by butterflies: the top-K of two
//      sorted K-lists is bitonic after one max per position, then a log K
//      half-cleaner sorts it;
//   3. warp 0 merges the warps' lists the same way.
// The key is the value's order key with its low kSlotBits bits replaced by
// (mask - slot): one unsigned compare orders by (value desc, slot asc).
// Values closer than 2^-32 relative compare by slot alone -- far inside the
// north_star's 1e-6 tie window (the cosines themselves carry f32-chunk
// rounding).
constexpr int kSlotBits = 20;                       // C <= 2^20
constexpr uint64_t kSlotMask = (1ull << kSlotBits) - 1;
__device__ __forceinline__ uint64_t slot_key(double v, int slot) {
  return (okey64(v) & ~kSlotMask) | (kSlotMask - (uint64_t)slot);
}
__device__ __forceinline__ int key_slot(uint64_t k) { return (int)(kSlotMask - (k & kSlotMask)); }

template <int K>
__device__ __forceinline__ void topk_insert(uint64_t (&t)[K], uint64_t e) {
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const uint64_t hi = t[r] > e ? t[r] : e;
    e = t[r] > e ? e : t[r];
    t[r] = hi;
  }
}
// merge with the list of lane (lane ^ o): both sorted descending
template <int K>
__device__ __forceinline__ void topk_merge_shfl(uint64_t (&t)[K], int o) {
  uint64_t pt[K];
#pragma unroll
  for (int r = 0; r < K; ++r) pt[r] = __shfl_xor_sync(0xffffffffu, t[r], o);
#pragma unroll
  for (int r = 0; r < K; ++r) t[r] = t[r] > pt[K - 1 - r] ? t[r] : pt[K - 1 - r];
#pragma unroll
  for (int st = K / 2; st > 0; st >>= 1)
#pragma unroll
    for (int r = 0; r < K; ++r)
      if ((r & st) == 0) {
        const uint64_t x = t[r], y = t[r + st];
        t[r] = x > y ? x : y;
        t[r + st] = x > y ? y : x;
      }
}

// top-K keys of vals[lo, hi) (slots are absolute indices); the sorted list
// ends in the registers of lane 0 of warp 0 (lanes < blockDim/32 of warp 0
// hold it too).  scratch: (blockDim/32)*K.
template <int K, int PT = 16>
__device__ void block_top_core(const double* vals, int lo, int hi, uint64_t (&t)[K],
                               uint64_t* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = hi - lo;
#pragma unroll
  for (int r = 0; r < K; ++r) t[r] = 0ull;
  if (n <= PT * (int)blockDim.x) {
    // PT strided values per thread in flight
    double v[PT];
#pragma unroll
    for (int x = 0; x < PT; ++x) {
      const int c = threadIdx.x + x * (int)blockDim.x;
      v[x] = c < n ? __ldcg(vals + lo + c) : 0.0;
    }
    const int per = (n + (int)blockDim.x - 1) / (int)blockDim.x;   // uniform
#pragma unroll
    for (int x = 0; x < PT; ++x) {
      if (x >= per) break;
      const int c = threadIdx.x + x * (int)blockDim.x;
      topk_insert<K>(t, c < n ? slot_key(v[x], lo + c) : 0ull);
    }
  } else {
    for (int c = threadIdx.x; c < n; c += (int)blockDim.x)
      topk_insert<K>(t, slot_key(__ldcg(vals + lo + c), lo + c));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) topk_merge_shfl<K>(t, o);
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < K; ++r) scratch[warp * K + r] = t[r];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int r = 0; r < K; ++r) t[r] = lane < nw ? scratch[lane * K + r] : 0ull;
    for (int o = 16; o > 0; o >>= 1)
      if (o < nw) topk_merge_shfl<K>(t, o);   // (uniform: lanes >= nw hold nothing)
  }
}

template <int K>
__device__ void block_top_k(const double* vals, int C, int cp, int32_t* out, uint64_t* scratch) {
  uint64_t t[K];
  block_top_core<K>(vals, 0, C, t, scratch);
  if (threadIdx.x == 0)
#pragma unroll
    for (int r = 0; r < K; ++r)
      if (r < cp) out[r] = key_slot(t[r]);          // compile-time index: t stays in registers
}

static __device__ __noinline__ void block_top_slots(const double* vals, int C, int cp, int32_t* out,
                                                    uint64_t* scratch) {
  if (cp <= 4) block_top_k<4>(vals, C, cp, out, scratch);
  else block_top_k<8>(vals, C, cp, out, scratch);
}

}  // namespace ctkv
