// v5 decode: the per-(b,g) unit work after the scan, spread over many CTAs.
//
// The scan kernel (ctkv_decode.cu) leaves, per unit, the chunk top-C'
// cosine candidates and the static-partition softmax partials.  What
// follows is a dependency chain per unit -- top-C' slots -> union of their
// lists -> rerank logits -> top-rho' -> sparse attention -> merge -- that a
// single CTA (or CTA pair) per unit runs latency-bound on one SM while the
// rest of the GPU idles.  Here every link of the chain is wide:
//
//   recall_wide_kernel   U x PB CTAs.  Every CTA of a unit recomputes the
//                        top-C' slots and the first-occurrence union
//                        (ck/retrieval.py:144-162; cheap: c'rho ids from L2)
//                        and gathers the rerank logits of its 1/PB slice of
//                        the recall positions (ck/retrieval.py:171-218).  The
//                        unit's last CTA (completion counter) selects the
//                        top-rho' positions (score desc, position asc) and
//                        their per-head logit maxima.
//   attend_wide_kernel   U x PC CTAs: softmax weights + V gather over 1/PC
//                        of the selected tokens (ck/retrieval.py:221-246);
//                        the unit's last CTA merges the PC sparse partials
//                        with the static partials (ck/retrieval.py:275-284).
//   tail_wide_kernel     U CTAs: full (score, position) order, FIFO DCU
//                        write (ck/index.py:103-133), ordered sparse ids,
//                        cursor/total advance.  Nothing later in the step
//                        reads what it writes, so the engine runs it on a
//                        side stream, overlapped with the next layers.
//
// Completion counters (uctr) are zeroed by the scan kernel of the same step.
#include <cfloat>
#include <cmath>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_decode_dev.cuh"
#include "ctkv_internal.h"

namespace ctkv {

constexpr int kWT = 256;               // threads per recall / attend CTA
constexpr int kWWarps = kWT / 32;
constexpr int kWItems = 32;            // union entries per thread (c' rho <= 8192)
constexpr int kWMaxLists = 8;          // c' <= 8
constexpr int kWMaxGs = 8;             // gs <= 8
constexpr int kTailT = 512;            // threads per tail CTA
constexpr int kTailBins = 1024;        // counting-sort bins of the tail ordering

struct WideSmem {
  uint64_t* area;    // union bitmaps [c'-1][words]; finisher: packed keys [lmax]
  int32_t* ids;      // this part's recalled ids; finisher: selected positions
  uint32_t* mark;    // finisher: selection bitmap over positions
  int* hist;         // [256]
  double* scratch;   // [128]
};

__host__ __device__ inline size_t wide_b_layout(const DecodeParams& p, int parts, WideSmem* s,
                                                unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* ptr = base ? base + off : nullptr;
    off += align16(bytes);
    return ptr;
  };
  const int lmax = p.lmax > 1 ? p.lmax : 1;
  const size_t bm = (size_t)(p.c_prime > 1 ? p.c_prime - 1 : 1) * p.bitmap_words * 4;
  const size_t keys = (size_t)lmax * 8;
  const int slice = lmax / parts + 2;
  const int rsel = p.rho_prime < lmax ? p.rho_prime : lmax;
  WideSmem t;
  t.area = reinterpret_cast<uint64_t*>(take(bm > keys ? bm : keys));
  t.ids = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (slice > rsel ? slice : rsel)));
  t.mark = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * ((lmax + 31) / 32)));
  t.hist = reinterpret_cast<int*>(take(sizeof(int) * 256));
  t.scratch = reinterpret_cast<double*>(take(sizeof(double) * 128));
  if (s) *s = t;
  return off;
}

struct WideCSmem {
  float* wts;        // [gs][slice]
  int32_t* vid;      // [slice]
  float* red;        // [warps][gs][D]
  double* scratch;   // [128]
};

__host__ __device__ inline int wide_c_slice(const DecodeParams& p, int parts) {
  const int rsel = p.rho_prime < p.lmax ? p.rho_prime : p.lmax;
  return (rsel > 1 ? rsel : 1) / parts + 2;
}

__host__ __device__ inline size_t wide_c_layout(const DecodeParams& p, int D, int parts,
                                                WideCSmem* s, unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* ptr = base ? base + off : nullptr;
    off += align16(bytes);
    return ptr;
  };
  const int sl = wide_c_slice(p, parts);
  WideCSmem t;
  t.wts = reinterpret_cast<float*>(take(sizeof(float) * p.gs * sl));
  t.vid = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * sl));
  t.red = reinterpret_cast<float*>(take(sizeof(float) * kWWarps * p.gs * D));
  const int nscr = p.gs * (p.ns + 1) > 128 ? p.gs * (p.ns + 1) : 128;
  t.scratch = reinterpret_cast<double*>(take(sizeof(double) * nscr));
  if (s) *s = t;
  return off;
}

__host__ __device__ inline size_t wide_tail_smem(const DecodeParams& p) {
  const int lmax = p.lmax > 1 ? p.lmax : 1;
  return (size_t)3 * lmax * 4 + (size_t)2 * kTailBins * 4;
}

__host__ __device__ inline int wide_tail_npad(int lmax) {
  const int n = next_pow2(lmax > 1 ? lmax : 1);
  return n < kTailT ? kTailT : n;
}

template <typename T, int D>
__global__ void __launch_bounds__(kWT) recall_wide_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int PB = p.wparts_b;
  WideSmem S;
  wide_b_layout(p, PB, &S, smem);
  const int u = blockIdx.x / PB, part = blockIdx.x % PB;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t total = *p.total + (p.k_new != nullptr ? 1 : 0);
  __shared__ __align__(16) T qs[kWMaxGs * D];
  __shared__ int32_t sel[kWMaxLists];
  __shared__ int s_state[4];
  __shared__ int wtot[kWWarps + 1];
  __shared__ int s_last;

  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  if (warp == 0) warp_top_slots(p, u, sel);
  for (int i = tid; i < gs * D; i += kWT) qs[i] = q[i];
  const int nb = p.c_prime - 1;                 // bitmaps of lists 0..c'-2
  uint32_t* bm = reinterpret_cast<uint32_t*>(S.area);
  for (int i = tid; i < nb * p.bitmap_words; i += kWT) bm[i] = 0u;
  __syncthreads();

  // ---- first-occurrence union (every CTA of the unit, identically) --------
  // warp w owns entries [w*P, (w+1)*P) of the (list, position) order,
  // lane-interleaved; ballots give each survivor its recall position.
  const int E = p.c_prime * p.rho;
  const int P = ((E + kWWarps - 1) / kWWarps + 31) & ~31;
  const int nit = P / 32;
  int ids[kWItems];
#pragma unroll
  for (int it = 0; it < kWItems; ++it) {
    ids[it] = kEmpty;
    const int o = warp * P + it * 32 + lane;
    if (it < nit && o < E) {
      const int j = o / p.rho;
      int id = __ldg(p.lists + ((int64_t)u * p.C + sel[j]) * p.rho + (o - j * p.rho));
      if (id != kEmpty && (id < 0 || id >= total)) { set_flag(p.flags, kFlagIdRange); id = kEmpty; }
      ids[it] = id;
      if (id != kEmpty && j < nb) atomicOr(&bm[j * p.bitmap_words + (id >> 5)], 1u << (id & 31));
    }
  }
  __syncthreads();
  uint32_t keepbits = 0;
  int wcount = 0;
#pragma unroll
  for (int it = 0; it < kWItems; ++it) {
    const int o = warp * P + it * 32 + lane;
    bool keep = ids[it] != kEmpty;
    if (keep) {
      const int j = o / p.rho;
      for (int j2 = 0; j2 < j; ++j2)
        keep = keep && !((bm[j2 * p.bitmap_words + (ids[it] >> 5)] >> (ids[it] & 31)) & 1u);
    }
    keepbits |= (keep ? 1u : 0u) << it;
    wcount += __popc(__ballot_sync(0xffffffffu, keep));
  }
  if (lane == 0) wtot[warp] = wcount;
  __syncthreads();
  int base = 0, L = 0;
  for (int w = 0; w < kWWarps; ++w) {
    if (w < warp) base += wtot[w];
    L += wtot[w];
  }
  const int lo = (int)((int64_t)part * L / PB), hi = (int)((int64_t)(part + 1) * L / PB);
  int32_t* recg = p.recg + (int64_t)u * p.lmax;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < kWItems; ++it) {
    const unsigned m = __ballot_sync(0xffffffffu, (keepbits >> it) & 1u);
    if ((m >> lane) & 1u) {
      const int pos = base + __popc(m & lt);
      if (pos >= lo && pos < hi) {
        S.ids[pos - lo] = ids[it];
        recg[pos] = ids[it];
      }
    }
    base += __popc(m);
  }
  __syncthreads();

  // ---- rerank logits of positions [lo, hi) ------------------------------------
  // 8 lanes per key row (two 16-byte chunks each), f32 chunk partials of exact
  // bf16 products, f64 across chunks and lanes; group max packed with the
  // position into an ascending sort key.
  double* lg = p.logits + (int64_t)u * gs * p.lmax;
  uint64_t* kg = p.keyg + (int64_t)u * p.lmax;
  {
    const T* keys = static_cast<const T*>(p.keys) + (int64_t)u * p.cap * D;
    const double scale = 1.0 / sqrt((double)D);
    constexpr int VPR = D * int(sizeof(T)) / 16;
    constexpr int LPRL = 8;
    constexpr int CPL = VPR / LPRL;
    constexpr int RPWL = 32 / LPRL;
    constexpr int UNL = 4;
    const int sub = lane % LPRL, rw = lane / LPRL;
    const int stepw = kWWarps * RPWL;
    for (int b0 = lo + warp * RPWL; b0 < hi; b0 += stepw * UNL) {
      uint4 raw[UNL][CPL];
      int tt[UNL];
#pragma unroll
      for (int x = 0; x < UNL; ++x) {
        tt[x] = b0 + x * stepw + rw;
        if (tt[x] < hi) {
          const uint4* r4 = reinterpret_cast<const uint4*>(keys + (int64_t)S.ids[tt[x] - lo] * D);
#pragma unroll
          for (int c = 0; c < CPL; ++c) raw[x][c] = ldg16(r4 + c * LPRL + sub);
        } else {
#pragma unroll
          for (int c = 0; c < CPL; ++c) raw[x][c] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int x = 0; x < UNL; ++x) {
        double gmax = -INFINITY;
        for (int hh = 0; hh < gs; ++hh) {
          const uint4* q4 = reinterpret_cast<const uint4*>(qs + hh * D);
          double a = 0.0;
#pragma unroll
          for (int c = 0; c < CPL; ++c) a += (double)bf16x8_dot(q4[c * LPRL + sub], raw[x][c], 0.f);
#pragma unroll
          for (int o = 1; o < LPRL; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          a *= scale;
          if (sub == 0 && tt[x] < hi) lg[(int64_t)hh * p.lmax + tt[x]] = a;
          gmax = fmax(gmax, a);
        }
        if (sub == 0 && tt[x] < hi)
          kg[tt[x]] = ((uint64_t)(~okey32((float)gmax)) << 32) | (uint32_t)tt[x];
      }
    }
  }

  // ---- the unit's last CTA: top-rho' positions and per-head maxima ----------
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&p.uctr[u * 4 + 0], 1) == PB - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int Rn = L > 0 ? (p.use_rerank ? min(p.rho_prime, L) : L) : 0;
  int32_t* wsel = p.wsel + (int64_t)u * p.lmax;
  const bool subset = Rn > 0 && Rn < L;
  if (subset) {
    uint64_t* key = S.area;   // bitmaps are dead
    for (int i = tid; i < L; i += kWT) key[i] = __ldcg(kg + i);
    const int nw = (L + 31) / 32;
    for (int i = tid; i < nw; i += kWT) S.mark[i] = 0u;
    __syncthreads();
    const int ns = select_smallest(key, L, Rn, S.ids, S.hist, s_state);
    for (int i = tid; i < ns; i += kWT) atomicOr(&S.mark[S.ids[i] >> 5], 1u << (S.ids[i] & 31));
    __syncthreads();
    // ordered compaction (deterministic summation order downstream)
    const int wpt = (nw + kWT - 1) / kWT;
    const int w0 = min(nw, tid * wpt), w1 = min(nw, w0 + wpt);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(S.mark[w]);
    int tot;
    int o = block_exclusive_scan(cnt, &tot, S.scratch);
    for (int w = w0; w < w1; ++w) {
      uint32_t m = S.mark[w];
      while (m) {
        const int bpos = __ffs(m) - 1;
        m &= m - 1;
        wsel[o++] = w * 32 + bpos;
      }
    }
  } else {
    for (int i = tid; i < Rn; i += kWT) wsel[i] = i;
  }
  // per-head max of the selected logits
  double m8[kWMaxGs];
#pragma unroll
  for (int hh = 0; hh < kWMaxGs; ++hh) m8[hh] = -INFINITY;
  for (int i = tid; i < Rn; i += kWT) {
    const int pos = subset ? S.ids[i] : i;
#pragma unroll
    for (int hh = 0; hh < kWMaxGs; ++hh)
      if (hh < gs) m8[hh] = fmax(m8[hh], __ldcg(lg + (int64_t)hh * p.lmax + pos));
  }
#pragma unroll
  for (int hh = 0; hh < kWMaxGs; ++hh)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m8[hh] = fmax(m8[hh], __shfl_xor_sync(0xffffffffu, m8[hh], o));
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int hh = 0; hh < kWMaxGs; ++hh) S.scratch[warp * kWMaxGs + hh] = m8[hh];
  __syncthreads();
  if (tid < gs) {
    double m = -INFINITY;
    for (int w = 0; w < kWWarps; ++w) m = fmax(m, S.scratch[w * kWMaxGs + tid]);
    p.wmax[(int64_t)u * gs + tid] = m;
  }
  if (tid == 0) {
    p.uctr[u * 4 + 2] = L;
    p.uctr[u * 4 + 3] = Rn;
    if (p.recall_len) p.recall_len[u] = L;
    if (p.sparse_len) p.sparse_len[u] = Rn;
    set_flag(p.flags, L > 0 ? kFlagNonEmptyRecall : kFlagEmptyRecall);
  }
  if (p.selected)
    for (int r = tid; r < p.c_prime; r += kWT) p.selected[(int64_t)u * p.c_prime + r] = sel[r];
}

template <typename T, int D>
__global__ void __launch_bounds__(kWT) attend_wide_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int PC = p.wparts_c;
  WideCSmem S;
  wide_c_layout(p, D, PC, &S, smem);
  const int sl = wide_c_slice(p, PC);
  const int u = blockIdx.x / PC, part = blockIdx.x % PC;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ double msh[kWMaxGs], lsh[kWMaxGs];
  __shared__ int s_last;
  const int Rn = p.uctr[u * 4 + 3];
  const int lo = (int)((int64_t)part * Rn / PC), hi = (int)((int64_t)(part + 1) * Rn / PC);
  const int n = hi - lo;
  const double* lg = p.logits + (int64_t)u * gs * p.lmax;
  const int32_t* wsel = p.wsel + (int64_t)u * p.lmax;
  const int32_t* recg = p.recg + (int64_t)u * p.lmax;
  if (tid < gs) msh[tid] = p.wmax[(int64_t)u * gs + tid];
  for (int i = tid; i < kWWarps * gs * D; i += kWT) S.red[i] = 0.f;
  __syncthreads();
  double l8[kWMaxGs];
#pragma unroll
  for (int hh = 0; hh < kWMaxGs; ++hh) l8[hh] = 0.0;
  for (int i = tid; i < n; i += kWT) {
    const int pos = wsel[lo + i];
    S.vid[i] = recg[pos];
#pragma unroll
    for (int hh = 0; hh < kWMaxGs; ++hh)
      if (hh < gs) {
        const double e = exp(lg[(int64_t)hh * p.lmax + pos] - msh[hh]);
        S.wts[hh * sl + i] = (float)e;
        l8[hh] += e;
      }
  }
#pragma unroll
  for (int hh = 0; hh < kWMaxGs; ++hh)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l8[hh] += __shfl_xor_sync(0xffffffffu, l8[hh], o);
  if (lane == 0)
#pragma unroll
    for (int hh = 0; hh < kWMaxGs; ++hh) S.scratch[warp * kWMaxGs + hh] = l8[hh];
  __syncthreads();
  const T* vals = static_cast<const T*>(p.values) + (int64_t)u * p.cap * D;
  accum_weighted_rows<T, D>(
      n, gs, [&](int t) -> const T* { return vals + (int64_t)S.vid[t] * D; },
      [&](int hh, int t) { return S.wts[hh * sl + t]; }, S.red + (int64_t)warp * gs * D);
  __syncthreads();
  float* apo = p.apo + ((int64_t)u * PC + part) * gs * D;
  for (int i = tid; i < gs * D; i += kWT) {
    float s = 0.f;
    for (int w = 0; w < kWWarps; ++w) s += S.red[(int64_t)w * gs * D + i];
    apo[i] = s;
  }
  if (tid < gs) {
    double l = 0.0;
    for (int w = 0; w < kWWarps; ++w) l += S.scratch[w * kWMaxGs + tid];
    p.apl[((int64_t)u * PC + part) * gs + tid] = l;
  }

  // ---- the unit's last CTA merges sparse and static partials ---------------
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&p.uctr[u * 4 + 1], 1) == PC - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ns = p.ns;
  const int64_t pbase = (int64_t)u * ns;
  double* wj = S.scratch;   // [gs][ns + 1] split weights
  if (tid < gs) {
    const int hh = tid;
    double lsp = 0.0;
    for (int k = 0; k < PC; ++k) lsp += __ldcg(p.apl + ((int64_t)u * PC + k) * gs + hh);
    const double msp = msh[hh];
    double M = lsp > 0.0 ? msp : -INFINITY;
    for (int j = 0; j < ns; ++j)
      if (p.pl[(pbase + j) * gs + hh] > 0.0) M = fmax(M, p.pm[(pbase + j) * gs + hh]);
    double Ls = 0.0;
    for (int j = 0; j < ns; ++j) {
      const double lj = p.pl[(pbase + j) * gs + hh];
      const double w = lj > 0.0 ? exp(p.pm[(pbase + j) * gs + hh] - M) : 0.0;
      wj[hh * (ns + 1) + j] = w;
      Ls += w * lj;
    }
    const double wsp = lsp > 0.0 ? exp(msp - M) : 0.0;
    wj[hh * (ns + 1) + ns] = wsp;
    Ls += wsp * lsp;
    msh[hh] = M;
    lsh[hh] = Ls;
  }
  __syncthreads();
  bool none = false;
  for (int i = tid; i < gs * D; i += kWT) {
    const int hh = i / D, e = i % D;
    float o0 = 0.f;
    for (int k = 0; k < PC; ++k) o0 += __ldcg(p.apo + ((int64_t)u * PC + k) * gs * D + i);
    const double* wh = wj + hh * (ns + 1);
    double O = wh[ns] * (double)o0;
    for (int j = 0; j < ns; ++j) O += wh[j] * (double)p.po[((pbase + j) * gs + hh) * D + e];
    const double Ls = lsh[hh];
    const int64_t oh = (int64_t)bi * p.h + gi * gs + hh;
    if (Ls > 0.0) {
      p.out[oh * D + e] = (float)(O / Ls);
    } else {
      p.out[oh * D + e] = 0.f;
      none = true;
    }
    if (e == 0) {
      if (p.row_max) p.row_max[oh] = msh[hh];
      if (p.denom) p.denom[oh] = Ls;
    }
  }
  if (none) set_flag(p.flags, kFlagNoTokens);
}

template <int IPT>
__device__ void tail_sort(uint64_t* skey) {
  uint64_t k[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) k[i] = skey[threadIdx.x * IPT + i];
  bitonic_regs<IPT>(k, skey);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) skey[threadIdx.x * IPT + i] = k[i];
  __syncthreads();
}

template <typename T, int D>
__global__ void __launch_bounds__(kTailT) tail_wide_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int u = blockIdx.x;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int64_t s_slot;
  __shared__ uint32_t s_mm[2 * (kTailT / 32)];
  const int lmax = p.lmax > 1 ? p.lmax : 1;
  uint32_t* k32 = reinterpret_cast<uint32_t*>(smem);   // [lmax] score keys by position
  int* binned = reinterpret_cast<int*>(k32 + lmax);    // [lmax] positions grouped by bin
  int* order = binned + lmax;                          // [lmax] position of rank r
  int* hist = order + lmax;                            // [kTailBins]
  int* cur = hist + kTailBins;                         // [kTailBins]
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
    for (int i = tid; i < L; i += kTailT) binned[atomicAdd(&cur[bin_of(k32[i])], 1)] = i;
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
      order[r] = i;
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
    for (int i = tid; i < gs * D; i += kTailT) {
      const int hh = i / D, e = i % D;
      cent[(((int64_t)bi * p.h + gi * gs + hh) * p.C + slot) * D + e] = q[i];
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
// launchers
// ------------------------------------------------------------------------

static int wide_parts(const void* fn, size_t smem, int threads, int U) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  const int slots = sms * (occ > 0 ? occ : 1);
  int parts = slots / (U > 0 ? U : 1);
  return parts < 1 ? 1 : (parts > 8 ? 8 : parts);
}

template <typename T, int D>
static int launch_wide_t(DecodeParams p, int what, cudaStream_t st) {
  if (what & 1) {
    auto kb = recall_wide_kernel<T, D>;
    const size_t smem2 = wide_b_layout(p, 2, nullptr, nullptr);
    if (cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2))
      return CTKV_ECUDA;
    p.wparts_b = wide_parts((const void*)kb, smem2, kWT, p.U);
    if (p.wparts_b < 2) p.wparts_b = 2;
    const size_t smemb = wide_b_layout(p, p.wparts_b, nullptr, nullptr);
    kb<<<p.U * p.wparts_b, kWT, smemb, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return CTKV_ECUDA;
    auto kc = attend_wide_kernel<T, D>;
    const size_t smemc2 = wide_c_layout(p, D, 2, nullptr, nullptr);
    if (cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemc2))
      return CTKV_ECUDA;
    p.wparts_c = wide_parts((const void*)kc, smemc2, kWT, p.U);
    if (p.wparts_c < 2) p.wparts_c = 2;
    const size_t smemc = wide_c_layout(p, D, p.wparts_c, nullptr, nullptr);
    kc<<<p.U * p.wparts_c, kWT, smemc, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return CTKV_ECUDA;
  }
  if (what & 2) {
    const bool any = (p.stages & (kStageDcu | kStageAppendTail)) || p.sparse_ids;
    if (!any) return CTKV_OK;
    auto kt = tail_wide_kernel<T, D>;
    const size_t smemt = wide_tail_smem(p);
    if (cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemt))
      return CTKV_ECUDA;
    launch_k(kt, dim3(p.U), dim3(kTailT), smemt, st, kPrioMid, p);
    if (cudaGetLastError() != cudaSuccess) return CTKV_ECUDA;
  }
  return CTKV_OK;
}

bool wide_supported(const DecodeParams& p, int dtype, int D) {
  if (dtype != CTKV_BF16 || (D != 64 && D != 128)) return false;
  if (p.gs > kWMaxGs || p.c_prime > kWMaxLists) return false;
  if ((int64_t)p.c_prime * p.rho > (int64_t)kWWarps * 32 * kWItems) return false;
  if (wide_tail_smem(p) > 200 * 1024) return false;
  if (wide_b_layout(p, 2, nullptr, nullptr) > 200 * 1024) return false;
  return true;
}

int launch_wide(const DecodeParams& p, int dtype, int D, int what, cudaStream_t st) {
  if (dtype != CTKV_BF16) return CTKV_ECONFIG;
  if (D == 128) return launch_wide_t<__nv_bfloat16, 128>(p, what, st);
  if (D == 64) return launch_wide_t<__nv_bfloat16, 64>(p, what, st);
  return CTKV_ECONFIG;
}

}  // namespace ctkv
