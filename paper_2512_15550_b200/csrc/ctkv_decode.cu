// Decode-step kernels for the B200 CTkvr path (sm_100a).
//
// The bf16 fused step is scan2_kernel (here) followed by the cluster chain
// kernel (ctkv_chain.cu) and the deferred tail (ctkv_tail.cu).  This
// file holds the scan, the exact f64 unit kernel of the fp32 parity path and
// the staged API calls, the 2-CTA unit2 kernel (bf16 fallback), and the
// generic id-list attention:
//
//   scan2_kernel  -- every SM streams HBM: (a) per (b,g) unit, the cosine of
//                    the gs query heads against all C centroids with the GQA
//                    group max (Alg. 2 L1-2; ck/retrieval.py:144-145,
//                    ck/tensor_ops.py:190-207); (b) split-K attention partials
//                    over the static partition [0,L_init) U [ring_start,total)
//                    (ck/retrieval.py:341-344).  Block 0 also appends the new
//                    token's K/V (ck/store.py:114-129).
//   unit_kernel   -- (fp32 / staged) one CTA per (b,g) unit: top-C' slots (ties -> smaller
//                    slot), first-occurrence union of their lists through a
//                    shared-memory bitmap (ck/retrieval.py:151-162), gathered
//                    f64 q.k rerank with group max (ck/retrieval.py:171-218),
//                    (score desc, position asc) ordering, the FIFO DCU write
//                    (ck/index.py:103-133), sparse attention reusing the
//                    rerank logits (ck/retrieval.py:221-246), and the exact
//                    merge with the static partials (ck/retrieval.py:275-284).
//
// The same unit_kernel, with stage bits switched off, backs the staged API
// calls (recall / rerank / fifo_update) so every stage is parity-testable
// on its own.  Generic id-list attention (sparse_attention API,
// _partial_over_ids) is attn_split_kernel + attn_merge_kernel.
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_internal.h"
#include "ctkv_decode_dev.cuh"

namespace ctkv {

constexpr int kScanRowsV2 = 256;   // threads (and centroid rows) per v2 scan CTA

// per-CTA scan2 timeline (globaltimer ns), profiling only: [cta][0 start,
// 1 first rows landed, 2 compute done, 3 end]; on while DecodeParams::dbg & 1
constexpr int kS2TlCtas = 4096;
__device__ unsigned long long g_s2tl[kS2TlCtas][8];
int g_host_dbg = 0;
__device__ __forceinline__ void s2mark(const DecodeParams& p, int k) {
#ifdef CTKV_PROFILE
  if ((p.dbg & 1) && threadIdx.x == 0 && blockIdx.x < kS2TlCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_s2tl[blockIdx.x][k] = t;
  }
#endif
}

// Per-CTA phase timestamps of the fused unit kernel (globaltimer, ns), for
// profiling only: [cta][checkpoint].  Written when g_phase_on != 0.
constexpr int kPhaseCtas = 256, kPhases = 12;
__device__ unsigned long long g_phase[kPhaseCtas][kPhases];
__device__ int g_phase_on;
__device__ __forceinline__ void phase_mark(int k) {
#ifdef CTKV_PROFILE
  if (g_phase_on && threadIdx.x == 0 && blockIdx.x < kPhaseCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_phase[blockIdx.x][k] = t;
  }
#endif
}

constexpr int kScanThreads = 256;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kCosChunk = 64;       // centroids per scan CTA (all gs heads)
constexpr int kUnitThreads = 512;
constexpr int kUnitWarps = kUnitThreads / 32;
constexpr int kAttnChunk = 512;     // sparse tokens per weight chunk
constexpr int kAttnSplit = 64;      // tokens per attn_split_kernel CTA


// this lane's partial of q_hh . row in f64 (products of f32-representable
// values are exact in f64; only the summation order differs from numpy)
template <typename T, int D>
__device__ __forceinline__ double lane_dot(const float* qs, int hh, const float* kv, int sub) {
  using R = Row<T, D>;
  double a = 0.0;
#pragma unroll
  for (int v = 0; v < R::VPL; ++v) {
    const float4* qv = reinterpret_cast<const float4*>(qs + hh * D + R::elem(sub, v));
#pragma unroll
    for (int j = 0; j < R::EPV / 4; ++j) {
      const float4 q4 = qv[j];
      const float* x = kv + v * R::EPV + 4 * j;
      a = fma((double)q4.x, (double)x[0], a);
      a = fma((double)q4.y, (double)x[1], a);
      a = fma((double)q4.z, (double)x[2], a);
      a = fma((double)q4.w, (double)x[3], a);
    }
  }
  return a;
}


// ------------------------------------------------------------------------
// scan kernel: cosine chunks + static attention splits (+ append)
// ------------------------------------------------------------------------


// softmax partial (m, l, unnormalised o) of the gs heads over up to
// kAttnSplit tokens whose ids come from `idf(i)`; written to slot `part`.
template <typename T, int D, typename IdFn>
__device__ void attn_partial_block(const DecodeParams& p, int u, int ntok, IdFn idf,
                                   int64_t t_new, int64_t total, double* pm, double* pl, float* po,
                                   unsigned char* smem) {
  using R = Row<T, D>;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int nwarps = blockDim.x >> 5;
  float* qs = reinterpret_cast<float*>(smem);                          // [gs][D]
  double* lg = reinterpret_cast<double*>(qs + kMaxGroup * D);          // [gs][kAttnSplit]
  double* mh = lg + kMaxGroup * kAttnSplit;                            // [gs]
  double* lh = mh + kMaxGroup;                                         // [gs]
  float* red = reinterpret_cast<float*>(lh + kMaxGroup);               // [nwarps][gs][D]
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  for (int i = threadIdx.x; i < gs * D; i += blockDim.x) qs[i] = to_f(q[i]);
  __syncthreads();
  const T* keys = static_cast<const T*>(p.keys);
  const T* vals = static_cast<const T*>(p.values);
  const T* knew = static_cast<const T*>(p.k_new);
  const T* vnew = static_cast<const T*>(p.v_new);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane % R::LPR, rw = lane / R::LPR;
  const double scale = 1.0 / sqrt((double)D);
  // phase 1: logits (f64)
  for (int base = warp * R::RPW; base < ntok; base += nwarps * R::RPW) {
    const int t = base + rw;
    float kv[R::EPL];
    bool ok = t < ntok;
    const int64_t id = ok ? idf(t) : 0;
    if (ok && (id < 0 || id >= total)) {
      set_flag(p.flags, kFlagIdRange);
      ok = false;
    }
    if (ok) {
      load_row_slice<T, D>(kv_row(keys, knew, p.cap, u, id, t_new, D), sub, kv);
    } else {
#pragma unroll
      for (int j = 0; j < R::EPL; ++j) kv[j] = 0.f;
    }
    for (int hh = 0; hh < gs; ++hh) {
      const double a = row_sum<R::LPR>(lane_dot<T, D>(qs, hh, kv, sub));
      if (sub == 0 && t < ntok) lg[hh * kAttnSplit + t] = ok ? a * scale : -INFINITY;
    }
  }
  for (int i = threadIdx.x; i < nwarps * gs * D; i += blockDim.x) red[i] = 0.f;
  __syncthreads();
  // per-head max and exp weights (f64)
  if (threadIdx.x < gs) {
    const int hh = threadIdx.x;
    double m = -INFINITY;
    for (int t = 0; t < ntok; ++t) m = fmax(m, lg[hh * kAttnSplit + t]);
    double l = 0.0;
    for (int t = 0; t < ntok; ++t) {
      const double e = (m == -INFINITY) ? 0.0 : exp(lg[hh * kAttnSplit + t] - m);
      lg[hh * kAttnSplit + t] = e;
      l += e;
    }
    mh[hh] = m;
    lh[hh] = l;
  }
  __syncthreads();
  // phase 2: o[h] = sum_t w[h,t] * V[t]  (unnormalised)
  accum_weighted_rows<T, D>(
      ntok, gs,
      [&](int t) -> const T* {
        const int64_t id = idf(t);
        if (id < 0 || id >= total) return nullptr;
        return kv_row(vals, vnew, p.cap, u, id, t_new, D);
      },
      [&](int hh, int t) { return (float)lg[hh * kAttnSplit + t]; }, red + (int64_t)warp * gs * D);
  __syncthreads();
  for (int i = threadIdx.x; i < gs * D; i += blockDim.x) {
    float s = 0.f;
    for (int w = 0; w < nwarps; ++w) s += red[(int64_t)w * gs * D + i];
    po[i] = s;
  }
  if (threadIdx.x < gs) {
    pm[threadIdx.x] = mh[threadIdx.x];
    pl[threadIdx.x] = lh[threadIdx.x];
  }
}

// ------------------------------------------------------------------------
// v2 scan: one task per CTA, operands pulled with TMA bulk copies into
// shared memory, one row per thread.  For bf16 rows the bf16 x bf16
// products are exact in f32; each 8-element chunk is summed in f32 and the
// chunk partials in f64 (relative error <= 7 * 2^-24 of the chunk's
// absolute sum -- inside the 1e-6 tie window).  f32 rows use f64 products.
// ------------------------------------------------------------------------

template <typename T> struct Prec;
template <> struct Prec<__nv_bfloat16> { static constexpr bool kChunkF32 = true; };
template <> struct Prec<float> { static constexpr bool kChunkF32 = false; };

// dot(q, row) and |row|^2 with rotated 16-byte chunk order (conflict-free
// when consecutive threads own consecutive rows).  `q` has the row's type:
// bf16 rows use the mixed-precision FMA on raw bf16 pairs.
template <typename T, int D, bool kNorm>
__device__ __forceinline__ void row_dot(const T* q, const T* row, int rot, double& dot,
                                        double& nrm) {
  constexpr int EPV = 16 / int(sizeof(T));
  constexpr int VPR = D / EPV;
  const uint4* r4 = reinterpret_cast<const uint4*>(row);
  const uint4* q4 = reinterpret_cast<const uint4*>(q);
  dot = 0.0;
  nrm = 0.0;
#pragma unroll 4
  for (int k = 0; k < VPR; ++k) {
    const int kk = (k + rot) & (VPR - 1);
    const uint4 x = r4[kk];
    if (Prec<T>::kChunkF32) {
      dot += (double)bf16x8_dot(q4[kk], x, 0.f);
      if (kNorm) nrm += (double)bf16x8_dot(x, x, 0.f);
    } else {
      float xf[EPV], qf[EPV];
      unpack16<T>(x, xf);
      unpack16<T>(q4[kk], qf);
#pragma unroll
      for (int j = 0; j < EPV; ++j) {
        dot = fma((double)qf[j], (double)xf[j], dot);
        if (kNorm) nrm = fma((double)xf[j], (double)xf[j], nrm);
      }
    }
  }
}

// |q_j| for the gs query heads staged in shared memory: one warp per head,
// lanes stride over d, f64 squares reduced by shuffles (the reference's
// np.linalg.norm, ck/tensor_ops.py:199-200)
template <typename T, int D>
__device__ __forceinline__ void query_norms(const T* qs, int gs, double* qn, int wid, int nw) {
  const int lane = threadIdx.x & 31;
  for (int j = wid; j < gs; j += nw) {
    double s = 0.0;
    for (int e = lane; e < D; e += 32) {
      const double x = (double)to_f(qs[j * D + e]);
      s = fma(x, x, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) qn[j] = sqrt(s);
  }
}


template <typename T>
__host__ __device__ constexpr int static_tok() { return sizeof(T) == 2 ? 128 : 64; }

template <typename T, int D>
__device__ void cos_task(const DecodeParams& p, int task, unsigned char* smem, uint64_t* bars) {
  constexpr int RB = D * int(sizeof(T));
  const int gs = p.gs, CC = kScanRowsV2 / gs;
  const int cpu = p.cos_blocks_per_unit;
  const int u = task / cpu, chunk = task % cpu;
  const int bi = u / p.g, gi = u % p.g;
  const int c0 = chunk * CC, nc = min(CC, p.C - c0);
  T* rows = reinterpret_cast<T*>(smem);                                   // [gs][CC][D]
  T* qs = reinterpret_cast<T*>(smem + (size_t)kScanRowsV2 * RB);          // [gs][D] raw
  double* qn = reinterpret_cast<double*>(qs + gs * D);                    // [gs]
  double* cosv = qn + gs;                                                 // [gs*CC]
  double* gv = cosv + kScanRowsV2;                                        // [CC] group max
  float* cns = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(gv + CC) + 15) &
                                        ~uintptr_t(15));                  // [gs][CC] |c|
  const T* cent = static_cast<const T*>(p.cent);
  // cached centroid norms ride with the rows when 16-byte aligned
  const bool cn_bulk = p.cnorm != nullptr && (p.C & 3) == 0 && (nc & 3) == 0;
  if (threadIdx.x == 0) {
    // one barrier per head block: rows of head j are computed as soon as they land
    for (int j = 0; j < gs; ++j) {
      bar_init(&bars[j], 1);
      bar_expect(&bars[j], (uint32_t)(nc * RB) + (cn_bulk ? (uint32_t)(nc * 4) : 0u));
      bulk_g2s(rows + (size_t)j * CC * D, cent + (((int64_t)bi * p.h + gi * gs + j) * p.C + c0) * D,
               (uint32_t)(nc * RB), &bars[j]);
      if (cn_bulk)
        bulk_g2s(cns + j * CC, p.cnorm + ((int64_t)bi * p.h + gi * gs + j) * p.C + c0,
                 (uint32_t)(nc * 4), &bars[j]);
    }
  }
  // the rows are in flight; the query may come from the previous kernel and
  // rides its own bulk copy
  pdl_wait();
  uint64_t* barq = &bars[kMaxGroup];   // after the gs (<= kMaxGroup) head barriers
  if (threadIdx.x == 0) {
    bar_init(barq, 1);
    bar_expect(barq, (uint32_t)(gs * D * sizeof(T)));
    bulk_g2s(qs, static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D,
             (uint32_t)(gs * D * sizeof(T)), barq);
  }
  __syncthreads();
  bar_wait(barq, 0);
  query_norms<T, D>(qs, gs, qn, threadIdx.x >> 5, blockDim.x >> 5);
  __syncthreads();
  for (int r = threadIdx.x; r < gs * CC; r += blockDim.x) {
    const int j = r / CC, c = r % CC;
    if (c >= nc) continue;
    bar_wait(&bars[j], 0);
    if (r == 0) s2mark(p, 1);
    double dot, nrm;
    double cn;
    if (p.cnorm != nullptr) {
      row_dot<T, D, false>(qs + j * D, rows + (size_t)r * D, r, dot, nrm);
      cn = cn_bulk ? (double)cns[j * CC + c]
                   : (double)__ldg(p.cnorm + ((int64_t)bi * p.h + gi * gs + j) * p.C + c0 + c);
    } else {
      row_dot<T, D, true>(qs + j * D, rows + (size_t)r * D, r, dot, nrm);
      cn = sqrt(nrm);
    }
    const double den = qn[j] * cn;
    double cv;
    if (den == 0.0) {
      cv = 0.0;
      set_flag(p.flags, kFlagDegenerate);
    } else {
      cv = fmin(fmax(dot / den, -1.0), 1.0);
    }
    cosv[r] = cv;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    double m = cosv[c];
    for (int j = 1; j < gs; ++j) m = fmax(m, cosv[j * CC + c]);
    p.gcos[(int64_t)u * p.C + c0 + c] = m;
    gv[c] = m;
  }
  // v6: the unit's last cosine chunk takes the top-C' of all C group maxima
  // The unit's last chunk is its selector: the other chunks publish with a
  // release fence and a fire-and-forget increment and exit at once (no
  // atomic round trip); the selector acquires the count, then takes the
  // top-C' of all C group maxima.  Lower-numbered CTAs are dispatched first,
  // so the selector only ever waits for CTAs that are already resident.
  if (p.selg != nullptr) {
    __syncthreads();   // this chunk's gcos written
    s2mark(p, 4);
    if (chunk != cpu - 1) {
      if (threadIdx.x == 0)   // release (cumulative over the barrier above) + relaxed increment
        asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(p.selctr + u)
                     : "memory");
      return;
    }
    if (threadIdx.x == 0) {
      int seen;
      for (int spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(p.selctr + u) : "memory");
        if (seen >= cpu - 1) break;
        if (spin > (1 << 24)) {   // ~1 s: never expected; report instead of hanging the GPU
          set_flag(p.flags, kFlagInternal);
          break;
        }
        __nanosleep(64);
      }
      // take this step's cpu-1 arrivals off the counter (0 again in the
      // normal case; after a timeout, late arrivals still net to 0)
      atomicSub(p.selctr + u, cpu - 1);
    }
    __syncthreads();
    s2mark(p, 6);
    block_top_slots(p.gcos + (int64_t)u * p.C, p.C, p.c_prime, p.selg + (int64_t)u * p.c_prime,
                    reinterpret_cast<uint64_t*>(cosv));
    s2mark(p, 7);
    return;
  }
  // chunk-local top-C' candidates (value desc, slot asc): the global top-C'
  // is contained in the union of the chunks' candidates
  if (p.cval != nullptr) {
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint64_t prev_key = ~0ull;
      int prev_idx = -1;
      const int64_t base = ((int64_t)u * cpu + chunk) * p.ncand;
      for (int r = 0; r < p.ncand; ++r) {
        uint64_t bk = 0;
        int bidx = INT32_MAX;
        for (int c = lane; c < nc; c += 32) {
          const uint64_t k = okey64(gv[c]);
          const int i = c0 + c;
          const bool below = k < prev_key || (k == prev_key && i > prev_idx);
          if (below && (k > bk || (k == bk && i < bidx))) { bk = k; bidx = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
          const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
          if (k2 > bk || (k2 == bk && i2 < bidx)) { bk = k2; bidx = i2; }
        }
        if (lane == 0) {
          p.cval[base + r] = bidx == INT32_MAX ? -INFINITY : gv[bidx - c0];
          p.cidx[base + r] = bidx;
        }
        prev_key = bk;
        prev_idx = bidx;
      }
    }
  }
}

// attention partial over static tokens [i0, i0+ST) of the static index space
// (f32, d < 64, or gs = 16; bf16 at d >= 64 and gs <= 8 takes static_task_tc)
template <typename T, int D>
__device__ void static_task(const DecodeParams& p, int task, int64_t t0, int64_t total,
                            unsigned char* smem, uint64_t* bar) {
  constexpr int RB = D * int(sizeof(T));
  constexpr int ST = static_tok<T>();
  const int gs = p.gs;
  const int u = task / p.ns, split = task % p.ns;
  const int bi = u / p.g, gi = u % p.g;
  const StaticSpan span(total, p.init_len, p.local_len);
  const int64_t i0 = (int64_t)split * ST;
  const int nt = (int)max((int64_t)0, min((int64_t)ST, span.n_static - i0));
  T* Ks = reinterpret_cast<T*>(smem);                           // [ST][D]
  T* Vs = Ks + (size_t)ST * D;                                  // [ST][D]
  T* qs = Vs + (size_t)ST * D;                                  // [gs][D] raw
  double* lg = reinterpret_cast<double*>(qs + gs * D);          // [gs][ST]
  float* w = reinterpret_cast<float*>(lg + gs * ST);            // [gs][ST]
  double* ml = reinterpret_cast<double*>(w + gs * ST);          // [2][gs]
  const int64_t slot = (int64_t)u * p.ns + split;
  double* pm = p.pm + slot * gs;
  double* pl = p.pl + slot * gs;
  float* po = p.po + slot * gs * D;
  if (nt == 0) {
    for (int i = threadIdx.x; i < gs * D; i += blockDim.x) po[i] = 0.f;
    if (threadIdx.x < gs) { pm[threadIdx.x] = -INFINITY; pl[threadIdx.x] = 0.0; }
    return;
  }
  const T* keys = static_cast<const T*>(p.keys) + (int64_t)u * p.cap * D;
  const T* vals = static_cast<const T*>(p.values) + (int64_t)u * p.cap * D;
  const bool appending = p.k_new != nullptr;
  uint64_t* barK = bar;
  uint64_t* barV = bar + 1;
  if (threadIdx.x == 0) {
    bar_init(barK, 1);
    bar_init(barV, 1);
    bar_expect(barK, (uint32_t)(nt * RB));
    bar_expect(barV, (uint32_t)(nt * RB));
    // contiguous runs of ids: [i0, n_init) and the ring part
    int64_t i = i0;
    const int64_t i1 = i0 + nt;
    while (i < i1) {
      const int64_t id = span.id(i);
      int64_t run_end = (i < span.n_init) ? min(i1, span.n_init) : i1;
      int64_t n = run_end - i;
      // the token appended by this step comes from the caller's buffer
      const bool has_new = appending && id <= t0 && t0 < id + n;
      if (has_new) n = t0 - id;  // rows before the new token
      if (n > 0) {
        bulk_g2s(Ks + (size_t)(i - i0) * D, keys + id * D, (uint32_t)(n * RB), barK);
        bulk_g2s(Vs + (size_t)(i - i0) * D, vals + id * D, (uint32_t)(n * RB), barV);
      }
      if (has_new) {
        const int64_t at = i + n - i0;
        bulk_g2s(Ks + (size_t)at * D, static_cast<const T*>(p.k_new) + (int64_t)u * D, RB, barK);
        bulk_g2s(Vs + (size_t)at * D, static_cast<const T*>(p.v_new) + (int64_t)u * D, RB, barV);
        n += 1;
      }
      i += n;
    }
  }
  // K/V (and the appended token's rows, from the caller's k_new/v_new) are in
  // flight; the query is read only after the wait (include/ctkv.h, phase bit 16)
  pdl_wait();
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  for (int k = threadIdx.x; k < gs * D; k += blockDim.x) qs[k] = q[k];
  __syncthreads();
  bar_wait(barK, 0);
  s2mark(p, 1);
  const double scale = 1.0 / sqrt((double)D);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // logits: pair (t, j), consecutive threads -> consecutive tokens
  for (int pr = threadIdx.x; pr < nt * gs; pr += blockDim.x) {
    const int t = pr % nt, j = pr / nt;
    double dot, nrm;
    row_dot<T, D, false>(qs + j * D, Ks + (size_t)t * D, t, dot, nrm);
    lg[j * ST + t] = dot * scale;
  }
  __syncthreads();
  s2mark(p, 4);
  // per-head max / exp weights / denominators: one warp per head
  for (int j = warp; j < gs; j += nw) {
    double m = -INFINITY;
    for (int t = lane; t < nt; t += 32) m = fmax(m, lg[j * ST + t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double l = 0.0;
    for (int t = lane; t < nt; t += 32) {
      const double e = sizeof(T) == 2 ? (double)expf((float)(lg[j * ST + t] - m)) : exp(lg[j * ST + t] - m);
      w[j * ST + t] = (float)e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) { ml[j] = m; ml[gs + j] = l; }
  }
  __syncthreads();
  s2mark(p, 5);
  bar_wait(barV, 0);
  s2mark(p, 6);
  if constexpr (sizeof(T) == 2 && D >= 64) {
    // o[j][:] = sum_t w[j][t] V[t][:]: a lane owns a 16-byte chunk (8 dims) of
    // one head for a quarter of the tokens (lanes 0-7 of a quarter read one
    // 128-byte row segment: conflict-free), quarters summed by shuffles
    constexpr int CHN = D / 8;
    const int ch_lo = lane & 7, tq = lane >> 3;
    const int ntask = (CHN / 8) * gs;
    for (int task = warp; task < ntask; task += nw) {
      const int j = task / (CHN / 8), ch = (task % (CHN / 8)) * 8 + ch_lo;
      float a[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = 0.f;
      const float* wj = w + j * ST;
      for (int t = tq; t < nt; t += 4) {
        float f[8];
        unpack16<T>(*reinterpret_cast<const uint4*>(Vs + (size_t)t * D + ch * 8), f);
        const float wt = wj[t];
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = fmaf(wt, f[e], a[e]);
      }
#pragma unroll
      for (int o = 8; o < 32; o <<= 1)
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] += __shfl_xor_sync(0xffffffffu, a[e], o);
      if (tq == 0) {
        float4* dst = reinterpret_cast<float4*>(po + j * D + ch * 8);
        dst[0] = make_float4(a[0], a[1], a[2], a[3]);
        dst[1] = make_float4(a[4], a[5], a[6], a[7]);
      }
    }
  } else
  // o[j][e] = sum_t w[j][t] * V[t][e]; a thread owns two adjacent elements
  for (int pr = threadIdx.x; pr < gs * (D / 2); pr += blockDim.x) {
    const int j = pr / (D / 2), e = 2 * (pr % (D / 2));
    float a0 = 0.f, a1 = 0.f;
    const float* wj = w + j * ST;
    for (int t = 0; t < nt; ++t) {
      const T* vr = Vs + (size_t)t * D + e;
      a0 = fmaf(wj[t], to_f(vr[0]), a0);
      a1 = fmaf(wj[t], to_f(vr[1]), a1);
    }
    po[j * D + e] = a0;
    po[j * D + e + 1] = a1;
  }
  if (threadIdx.x < gs) {
    pm[threadIdx.x] = ml[threadIdx.x];
    pl[threadIdx.x] = ml[gs + threadIdx.x];
  }
}

// bf16, d >= 64, gs <= 8: the static partition on the tensor cores, kept in
// registers between its phases.  One 16-token block per warp (ST = 16 x 8
// warps): logits by mma.m16n8k16 (f32 per 16-element k-step, f64 across, as
// in static_task), the per-head maxima exchanged through shared memory, the
// weights exp(l - m) computed by the lanes that hold the logits and split
// into three bf16 terms hi + mid + lo (exactly the f32 weight), and P.V as
// the GEMM O[gs x D] = W[gs x ST] V[ST x D] on the tensor cores (the bf16 V
// rows are exact operands; products exact in f32, f32 accumulation).  V rows
// land in groups of 16 tokens whose base moves 16 B per group, so an
// ldmatrix.trans reading one row from each group (the MMA's k slots span
// the groups) is conflict-free.  No logits or f32 weight arrays: the
// partition needs 2 x ST x D x 2 B + 128 B of shared memory, which keeps
// the scan at three CTAs per SM at gs = 8.
constexpr int kStGroup = 16;                        // tokens per V row group
template <int RB>
__device__ __forceinline__ uint32_t vrow_off(int t) {
  return (uint32_t)((t >> 4) * (kStGroup * RB + 16) + (t & 15) * RB);
}
constexpr int kWpStride = 128 + 8;                  // bf16 per weight row (bank shift)
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <typename T, int D>
__device__ void static_task_tc(const DecodeParams& p, int task, int64_t t0, int64_t total,
                               unsigned char* smem, uint64_t* bar) {
  static_assert(sizeof(T) == 2 && D >= 64, "bf16, d >= 64");
  constexpr int RB = D * int(sizeof(T));
  constexpr int ST = static_tok<T>();
  static_assert(ST == 16 * (kScanRowsV2 / 32), "one 16-token block per warp");
  static_assert(kWpStride == ST + 8, "weight rows: ST slots + 16 B bank shift");
  static_assert(3 * 8 * kWpStride * 2 <= ST * RB, "the weight terms fit over the K rows");
  const int gs = p.gs;
  const int u = task / p.ns, split = task % p.ns;
  const int bi = u / p.g, gi = u % p.g;
  const StaticSpan span(total, p.init_len, p.local_len);
  const int64_t i0 = (int64_t)split * ST;
  const int nt = (int)max((int64_t)0, min((int64_t)ST, span.n_static - i0));
  T* Ks = reinterpret_cast<T*>(smem);                                      // [ST][D]
  unsigned char* Vb = smem + (size_t)ST * RB;                              // grouped rows
  T* qs = reinterpret_cast<T*>(Vb + (size_t)ST * RB + (ST / kStGroup) * 16);  // [gs][D]
  __nv_bfloat16* Wp = reinterpret_cast<__nv_bfloat16*>(smem);   // [3][8][kWpStride], over Ks
  // per-warp head maxima and partial denominators
  double (*wmax)[8] = reinterpret_cast<double (*)[8]>(
      (reinterpret_cast<uintptr_t>(qs + gs * D) + 15) & ~uintptr_t(15));   // [8 warps][8]
  double (*wsum)[8] = wmax + kScanRowsV2 / 32;                              // [8 warps][8]
  const int64_t slot = (int64_t)u * p.ns + split;
  double* pm = p.pm + slot * gs;
  double* pl = p.pl + slot * gs;
  float* po = p.po + slot * gs * D;
  if (nt == 0) {
    for (int i = threadIdx.x; i < gs * D; i += blockDim.x) po[i] = 0.f;
    if (threadIdx.x < gs) { pm[threadIdx.x] = -INFINITY; pl[threadIdx.x] = 0.0; }
    return;
  }
  const T* keys = static_cast<const T*>(p.keys) + (int64_t)u * p.cap * D;
  const T* vals = static_cast<const T*>(p.values) + (int64_t)u * p.cap * D;
  const bool appending = p.k_new != nullptr;
  uint64_t* barK = bar;
  uint64_t* barV = bar + 1;
  if (threadIdx.x == 0) {
    bar_init(barK, 1);
    bar_init(barV, 1);
    bar_expect(barK, (uint32_t)(nt * RB));
    bar_expect(barV, (uint32_t)(nt * RB));
    // V rows [t, t + n) of the split from `src`, cut at the row groups
    auto copy_v = [&](int t, const T* src, int n) {
      while (n > 0) {
        const int m = min(n, kStGroup - (t & (kStGroup - 1)));
        bulk_g2s(Vb + vrow_off<RB>(t), src, (uint32_t)(m * RB), barV);
        t += m;
        src += (size_t)m * D;
        n -= m;
      }
    };
    // contiguous runs of ids: [i0, n_init) and the ring part
    int64_t i = i0;
    const int64_t i1 = i0 + nt;
    while (i < i1) {
      const int64_t id = span.id(i);
      int64_t run_end = (i < span.n_init) ? min(i1, span.n_init) : i1;
      int64_t n = run_end - i;
      // the token appended by this step comes from the caller's buffer
      const bool has_new = appending && id <= t0 && t0 < id + n;
      if (has_new) n = t0 - id;  // rows before the new token
      if (n > 0) {
        bulk_g2s(Ks + (size_t)(i - i0) * D, keys + id * D, (uint32_t)(n * RB), barK);
        copy_v((int)(i - i0), vals + id * D, (int)n);
      }
      if (has_new) {
        const int64_t at = i + n - i0;
        bulk_g2s(Ks + (size_t)at * D, static_cast<const T*>(p.k_new) + (int64_t)u * D, RB, barK);
        copy_v((int)at, static_cast<const T*>(p.v_new) + (int64_t)u * D, 1);
        n += 1;
      }
      i += n;
    }
  }
  // V rows past the partition's tokens take part in the P.V MMAs with zero
  // weights: make them finite zeros
  for (int x = nt * (RB / 16) + threadIdx.x; x < ST * (RB / 16); x += blockDim.x)
    *reinterpret_cast<uint4*>(Vb + vrow_off<RB>(x / (RB / 16)) + (x % (RB / 16)) * 16) = make_uint4(0, 0, 0, 0);
  // K/V (and the appended token's rows, from the caller's k_new/v_new) are in
  // flight; the query is read only after the wait (include/ctkv.h, phase bit 16)
  pdl_wait();
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  for (int k = threadIdx.x; k < gs * D / 8; k += blockDim.x)   // 16-byte pieces
    reinterpret_cast<uint4*>(qs)[k] = __ldg(reinterpret_cast<const uint4*>(q) + k);
  __syncthreads();
  bar_wait(barK, 0);
  s2mark(p, 1);
  const double scale = 1.0 / sqrt((double)D);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  // ---- logits of tokens r0 = 16 warp + g8 and r1 = r0 + 8, heads 2 t4 + e
  const int r0 = warp * 16 + g8, r1 = r0 + 8;
  double lv[2][2];
  {
    const T* ra = Ks + (size_t)r0 * D + 8 * t4;
    const T* rb = ra + 8 * D;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (warp * 16 < nt) {
#pragma unroll
      for (int s2 = 0; s2 < D / 32; ++s2) {
        const uint4 a = *reinterpret_cast<const uint4*>(ra + s2 * 32);
        const uint4 b = *reinterpret_cast<const uint4*>(rb + s2 * 32);
        const uint4 qv = g8 < gs ? *reinterpret_cast<const uint4*>(qs + g8 * D + s2 * 32 + 8 * t4)
                                 : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float d[4] = {0.f, 0.f, 0.f, 0.f};
          mma_bf16_16816(d, hf ? a.z : a.x, hf ? b.z : b.x, hf ? a.w : a.y, hf ? b.w : b.y,
                         hf ? qv.z : qv.x, hf ? qv.w : qv.y);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[e] += (double)d[e];
        }
      }
    }
    double mloc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool hv = 2 * t4 + e < gs;
      lv[e][0] = (hv && r0 < nt) ? acc[e] * scale : -INFINITY;
      lv[e][1] = (hv && r1 < nt) ? acc[2 + e] * scale : -INFINITY;
      mloc[e] = fmax(lv[e][0], lv[e][1]);
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      mloc[0] = fmax(mloc[0], __shfl_xor_sync(0xffffffffu, mloc[0], o));
      mloc[1] = fmax(mloc[1], __shfl_xor_sync(0xffffffffu, mloc[1], o));
    }
    if (g8 == 0) { wmax[warp][2 * t4] = mloc[0]; wmax[warp][2 * t4 + 1] = mloc[1]; }
  }
  __syncthreads();   // maxima exchanged; every warp is done with Ks
  s2mark(p, 4);
  // ---- weights: exp(l - m) as f32, split hi + mid + lo into Wp (over Ks),
  // k slot of token t in k-step s = t%16 / 2: 8 (t%2) + t/16
  {
    double lsum[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = 2 * t4 + e;
      double m = -INFINITY;
      for (int w2 = 0; w2 < kScanRowsV2 / 32; ++w2) m = fmax(m, wmax[w2][h]);
      lsum[e] = 0.0;
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int t = rr ? r1 : r0;
        const float ef = lv[e][rr] == -INFINITY ? 0.f : expf((float)(lv[e][rr] - m));
        lsum[e] += (double)ef;
        const __nv_bfloat16 w0 = __float2bfloat16_rn(ef);
        const float x1 = ef - __bfloat162float(w0);
        const __nv_bfloat16 w1 = __float2bfloat16_rn(x1);
        const __nv_bfloat16 w2 = __float2bfloat16_rn(x1 - __bfloat162float(w1));
        if (h < 8) {
          const int idx = ((t & 15) >> 1) * 16 + 8 * (t & 1) + (t >> 4);
          Wp[(0 * 8 + h) * kWpStride + idx] = w0;
          Wp[(1 * 8 + h) * kWpStride + idx] = w1;
          Wp[(2 * 8 + h) * kWpStride + idx] = w2;
        }
      }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      lsum[0] += __shfl_xor_sync(0xffffffffu, lsum[0], o);
      lsum[1] += __shfl_xor_sync(0xffffffffu, lsum[1], o);
    }
    if (g8 == 0) { wsum[warp][2 * t4] = lsum[0]; wsum[warp][2 * t4 + 1] = lsum[1]; }
  }
  __syncthreads();   // Wp and the partial denominators complete
  s2mark(p, 5);
  if (threadIdx.x < gs) {
    double m = -INFINITY, l = 0.0;
    for (int w2 = 0; w2 < kScanRowsV2 / 32; ++w2) {
      m = fmax(m, wmax[w2][threadIdx.x]);
      l += wsum[w2][threadIdx.x];
    }
    pm[threadIdx.x] = m;
    pl[threadIdx.x] = l;
  }
  bar_wait(barV, 0);
  s2mark(p, 6);
  // ---- P.V: warp w owns output columns [w D/8, (w+1) D/8) = D/64 n-tiles
  constexpr int NTW = D / 64;                 // n-tiles of 8 columns per warp
  float c[NTW][4];
#pragma unroll
  for (int j = 0; j < NTW; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
  const int n0 = warp * (D / 8);
  const bool arow = g8 < gs;
  const uint32_t wbase = sa(Wp) + (uint32_t)(g8 * kWpStride + 2 * t4) * 2u;
  const int mat = lane >> 3, li = lane & 7;
#pragma unroll 1
  for (int s = 0; s < ST / 16; ++s) {
    uint32_t a[3][2];
#pragma unroll
    for (int tm = 0; tm < 3; ++tm) {
      const uint32_t ad = wbase + (uint32_t)(tm * 8 * kWpStride + s * 16) * 2u;
      a[tm][0] = arow ? ld_shared_u32(ad) : 0u;
      a[tm][1] = arow ? ld_shared_u32(ad + 16u) : 0u;
    }
    // row li of matrix `mat`: token 16 li + 2 s + (mat & 1), columns
    // n0 + 8 (mat >> 1) (+16 per further pair)
    const uint32_t vrow = sa(Vb) + vrow_off<RB>(16 * li + 2 * s + (mat & 1));
    if constexpr (NTW == 1) {
      uint32_t b0, b1;
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                   : "=r"(b0), "=r"(b1)
                   : "r"(vrow + (uint32_t)n0 * 2u));
#pragma unroll
      for (int tm = 0; tm < 3; ++tm) mma_bf16_16816(c[0], a[tm][0], 0u, a[tm][1], 0u, b0, b1);
    } else {
#pragma unroll
      for (int jp = 0; jp < NTW / 2; ++jp) {
        uint32_t b[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                     : "r"(vrow + (uint32_t)(n0 + 16 * jp + 8 * (mat >> 1)) * 2u));
#pragma unroll
        for (int tm = 0; tm < 3; ++tm) {
          mma_bf16_16816(c[2 * jp], a[tm][0], 0u, a[tm][1], 0u, b[0], b[1]);
          mma_bf16_16816(c[2 * jp + 1], a[tm][0], 0u, a[tm][1], 0u, b[2], b[3]);
        }
      }
    }
  }
  if (arow)
#pragma unroll
    for (int j = 0; j < NTW; ++j)
      *reinterpret_cast<float2*>(po + g8 * D + n0 + 8 * j + 2 * t4) = make_float2(c[j][0], c[j][1]);
}

template <typename T, int D>
__global__ void __launch_bounds__(kScanRowsV2, 4) scan2_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[kMaxGroup + 1];
  ktl_mark(p.tl, 0, false);
  s2mark(p, 0);
  const bool appending = p.k_new != nullptr;
  const int ncos = p.do_cos ? p.U * p.cos_blocks_per_unit : 0;
  // the token counter is read only where it is used (static tasks, the
  // append): a cosine CTA issues its centroid copies without that round trip
  if ((int)blockIdx.x < ncos) {
    cos_task<T, D>(p, blockIdx.x, smem, bars);
  } else {
    const int64_t t0 = p.total ? *p.total : p.id_bound;
    if constexpr (sizeof(T) == 2 && D >= 64) {
      if (p.gs <= 8) {
        static_task_tc<T, D>(p, blockIdx.x - ncos, t0, t0 + (appending ? 1 : 0), smem, bars);
      } else {
        static_task<T, D>(p, blockIdx.x - ncos, t0, t0 + (appending ? 1 : 0), smem, bars);
      }
    } else {
      static_task<T, D>(p, blockIdx.x - ncos, t0, t0 + (appending ? 1 : 0), smem, bars);
    }
  }
  s2mark(p, 2);
  if (appending && blockIdx.x == 0) {
    const int64_t t0 = p.total ? *p.total : p.id_bound;
    T* keys = static_cast<T*>(const_cast<void*>(p.keys));
    T* vals = static_cast<T*>(const_cast<void*>(p.values));
    const T* kn = static_cast<const T*>(p.k_new);
    const T* vn = static_cast<const T*>(p.v_new);
    if constexpr (D * sizeof(T) % 16 == 0) {   // 16-byte pieces of each unit's new row
      constexpr int VPR = D * int(sizeof(T)) / 16;
      for (int64_t i = threadIdx.x; i < (int64_t)p.U * VPR; i += blockDim.x) {
        const int64_t uu = i / VPR, e = i % VPR;
        reinterpret_cast<uint4*>(keys + (uu * p.cap + t0) * D)[e] = reinterpret_cast<const uint4*>(kn)[i];
        reinterpret_cast<uint4*>(vals + (uu * p.cap + t0) * D)[e] = reinterpret_cast<const uint4*>(vn)[i];
      }
    } else {
      for (int64_t i = threadIdx.x; i < (int64_t)p.U * D; i += blockDim.x) {
        const int64_t uu = i / D, e = i % D;
        keys[(uu * p.cap + t0) * D + e] = kn[i];
        vals[(uu * p.cap + t0) * D + e] = vn[i];
      }
    }
  }
  __syncthreads();
  ktl_mark(p.tl, 0, true);
  s2mark(p, 3);
}

int scan2_timeline(int on, unsigned long long* out, int n) {
  if (out != nullptr) {
    const int m = n < kS2TlCtas * 8 ? n : kS2TlCtas * 8;
    if (cudaMemcpyFromSymbol(out, g_s2tl, sizeof(unsigned long long) * m) != cudaSuccess) return CTKV_ECUDA;
  }
  if (on >= 0) set_host_dbg(1, on);
  return CTKV_OK;
}

template <typename T, int D>
size_t scan2_smem(int gs) {
  constexpr int RB = D * int(sizeof(T));
  constexpr int ST = static_tok<T>();
  const size_t cosb = (size_t)kScanRowsV2 * RB + sizeof(T) * gs * D + sizeof(double) * gs +
                      sizeof(double) * 2 * kScanRowsV2 + sizeof(float) * kScanRowsV2 + 16;
  // static partitions: static_task_tc (bf16, d >= 64, gs <= 8) keeps logits
  // and weights in registers / over the K rows; static_task stages them
  const bool tc = sizeof(T) == 2 && D >= 64 && gs <= 8;
  const size_t stb = tc ? (size_t)2 * ST * RB + (ST / kStGroup) * 16 + sizeof(T) * gs * D + 16 +
                             2 * sizeof(double) * (kScanRowsV2 / 32) * 8
                        : (size_t)2 * ST * RB + sizeof(float) * gs * D + sizeof(double) * gs * ST +
                              sizeof(float) * gs * ST + sizeof(double) * 2 * gs;
  return cosb > stb ? cosb : stb;
}

// ------------------------------------------------------------------------
// unit kernel: select -> union -> rerank -> order -> DCU -> sparse attend
// ------------------------------------------------------------------------

struct UnitSmem {
  int32_t* sel;      // [c_prime]
  uint32_t* bitmap;  // [nwords]
  int32_t* rec;      // [lmax]
  uint64_t* skey;    // [npad_max]  (reused as the attention reduce area)
  int32_t* sval;     // [npad_max]
  float* wts;        // [gs][kAttnChunk]
  double* scratch;   // [64] reductions
};


__host__ __device__ inline size_t unit_smem_layout(const DecodeParams& p, int D, UnitSmem* s,
                                                   unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* ptr = base ? base + off : nullptr;
    off += align16(bytes);
    return ptr;
  };
  const int npad = next_pow2(max(p.lmax, 1));
  const size_t red_bytes = (size_t)kUnitWarps * p.gs * D * sizeof(float);
  const size_t key_bytes =
      (size_t)npad * sizeof(uint64_t) > red_bytes ? (size_t)npad * sizeof(uint64_t) : red_bytes;
  UnitSmem t;
  t.sel = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * max(p.c_prime, 1)));
  t.bitmap = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * p.bitmap_words));
  t.rec = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * max(p.lmax, 1)));
  t.skey = reinterpret_cast<uint64_t*>(take(key_bytes));
  t.sval = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * npad));
  t.wts = reinterpret_cast<float*>(take(sizeof(float) * p.gs * kAttnChunk));
  t.scratch = reinterpret_cast<double*>(take(sizeof(double) * 128));
  if (s) *s = t;
  return off;
}

size_t unit_smem_bytes(const DecodeParams& p, int D) {
  return unit_smem_layout(p, D, nullptr, nullptr);
}

// block-wide arg-max over (key desc, idx asc) pairs; returns the winner idx
__device__ int block_argmax(uint64_t key, int idx, double* scratch) {
  auto better = [](uint64_t ka, int ia, uint64_t kb, int ib) {
    return ka > kb || (ka == kb && ia < ib);
  };
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (better(k2, i2, key, idx)) { key = k2; idx = i2; }
  }
  uint64_t* sk = reinterpret_cast<uint64_t*>(scratch);  // [33]
  int* si = reinterpret_cast<int*>(sk + 34);            // [33]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) { sk[warp] = key; si[warp] = idx; }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  if (warp == 0) {
    key = lane < nw ? sk[lane] : 0;
    idx = lane < nw ? si[lane] : INT32_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(0xffffffffu, key, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      if (better(k2, i2, key, idx)) { key = k2; idx = i2; }
    }
    if (lane == 0) { sk[32] = key; si[32] = idx; }
  }
  __syncthreads();
  return si[32];
}


__device__ double block_max_f64(double x, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = x;
  __syncthreads();
  double m = -INFINITY;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, scratch[w]);
  return m;
}

__device__ double block_sum_f64(double x, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = x;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += scratch[w];
  return s;
}

template <typename T, int D>
__global__ void __launch_bounds__(kUnitThreads, 1) unit_kernel(DecodeParams p) {
  using R = Row<T, D>;
  extern __shared__ __align__(128) unsigned char smem[];
  UnitSmem S;
  unit_smem_layout(p, D, &S, smem);
  const int u = blockIdx.x;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t t0 = p.total ? *p.total : p.id_bound;
  const bool appending = p.k_new != nullptr;
  const int64_t total = t0 + (appending ? 1 : 0);
  __shared__ int64_t s_slot;
  __shared__ float qs[kMaxGroup * D];
  if (tid == 0) s_slot = p.fifo ? (p.fifo[bi] % p.C) : 0;
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  for (int i = tid; i < gs * D; i += blockDim.x) qs[i] = to_f(q[i]);

  // ---- 1. top-C' centroid slots (ck/retrieval.py:154) -------------------
  int L = 0;
  if (p.stages & kStageSelect) {
    uint64_t prev_key = ~0ull;
    int prev_idx = -1;
    const double* gc = p.gcos + (int64_t)u * p.C;
    for (int r = 0; r < p.c_prime; ++r) {
      uint64_t bk = 0;
      int bidx = INT32_MAX;
      for (int i = tid; i < p.C; i += blockDim.x) {
        const uint64_t k = okey64(gc[i]);
        const bool below = k < prev_key || (k == prev_key && i > prev_idx);
        if (below && (k > bk || (k == bk && i < bidx))) { bk = k; bidx = i; }
      }
      const int w = block_argmax(bk, bidx, S.scratch);
      if (tid == 0) S.sel[r] = w;
      prev_idx = w;
      prev_key = okey64(gc[w]);
    }
    __syncthreads();
    if (p.selected)
      for (int r = tid; r < p.c_prime; r += blockDim.x)
        p.selected[(int64_t)u * p.c_prime + r] = S.sel[r];
  }

  // ---- 2. union of the selected lists, first occurrence kept ------------
  if (p.stages & kStageUnion) {
    const int nwords = (int)((total + 31) >> 5);
    for (int i = tid; i < nwords; i += blockDim.x) S.bitmap[i] = 0u;
    __syncthreads();
    const int per = (p.rho + blockDim.x - 1) / blockDim.x;
    for (int j = 0; j < p.c_prime; ++j) {
      const int32_t* row = p.lists + ((int64_t)u * p.C + S.sel[j]) * p.rho;
      int keep_mask = 0, cnt = 0;
      int ids[8];
      // `per` <= 8 is guaranteed by the host (rho <= 8 * kUnitThreads)
      for (int e = 0; e < per; ++e) {
        const int i = tid * per + e;
        int id = (i < p.rho) ? row[i] : kEmpty;
        if (id != kEmpty && (id < 0 || id >= total)) {
          set_flag(p.flags, kFlagIdRange);
          id = kEmpty;
        }
        ids[e] = id;
        if (id != kEmpty && !((S.bitmap[id >> 5] >> (id & 31)) & 1u)) {
          keep_mask |= 1 << e;
          ++cnt;
        }
      }
      int tot_kept;
      int pos = L + block_exclusive_scan(cnt, &tot_kept, S.scratch);
      for (int e = 0; e < per; ++e)
        if (keep_mask & (1 << e)) S.rec[pos++] = row[tid * per + e];
      __syncthreads();  // every test of list j precedes any set of list j
      for (int e = 0; e < per; ++e)
        if (keep_mask & (1 << e)) {
          const int id = row[tid * per + e];
          atomicOr(&S.bitmap[id >> 5], 1u << (id & 31));
        }
      L += tot_kept;
      __syncthreads();
    }
    if (p.rec_out)
      for (int i = tid; i < p.lmax; i += blockDim.x)
        p.rec_out[(int64_t)u * p.lmax + i] = i < L ? S.rec[i] : kEmpty;
  } else {
    L = p.len_in[u];
    for (int i = tid; i < L; i += blockDim.x) S.rec[i] = p.rec_in[(int64_t)u * p.lmax + i];
  }
  if (p.recall_len && tid == 0) p.recall_len[u] = L;
  if (tid == 0) set_flag(p.flags, L > 0 ? kFlagNonEmptyRecall : kFlagEmptyRecall);
  __syncthreads();

  // ---- 3. rerank logits (f64) + group max -------------------------------
  const int npad = next_pow2(max(L, 1));
  double* lg = p.logits + (int64_t)u * gs * p.lmax;
  const double scale = 1.0 / sqrt((double)D);
  if (L > 0 && (p.stages & kStageScores)) {
    const T* keys = static_cast<const T*>(p.keys);
    const int sub = lane % R::LPR, rw = lane / R::LPR;
    constexpr int U = 4;
    for (int base = warp * R::RPW; base < L; base += kUnitWarps * R::RPW * U) {
      float kv[U][R::EPL];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int t = base + k * kUnitWarps * R::RPW + rw;
        if (t < L) {
          load_row_slice<T, D>(keys + ((int64_t)u * p.cap + S.rec[t]) * D, sub, kv[k]);
        } else {
#pragma unroll
          for (int j = 0; j < R::EPL; ++j) kv[k][j] = 0.f;
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int t = base + k * kUnitWarps * R::RPW + rw;
        double gmax = -INFINITY;
        for (int hh = 0; hh < gs; ++hh) {
          double a = 0.0;
#pragma unroll
          for (int v = 0; v < R::VPL; ++v) {
            const float* qv = qs + hh * D + R::elem(sub, v);
#pragma unroll
            for (int j = 0; j < R::EPV; ++j) a = fma((double)qv[j], (double)kv[k][v * R::EPV + j], a);
          }
          a = row_sum<R::LPR>(a) * scale;
          gmax = fmax(gmax, a);
          if (sub == 0 && t < L) lg[(int64_t)hh * p.lmax + t] = a;
        }
        if (sub == 0 && t < L) {
          S.skey[t] = ~okey64(gmax);
          S.sval[t] = t;
          if (p.grouped_out) p.grouped_out[(int64_t)u * p.lmax + t] = gmax;
        }
      }
    }
  } else if (L > 0 && p.grouped_in != nullptr) {
    // scores supplied by the caller (fifo_update API)
    for (int t = tid; t < L; t += blockDim.x) {
      S.skey[t] = ~okey64(p.grouped_in[(int64_t)u * p.lmax + t]);
      S.sval[t] = t;
    }
  }
  for (int t = L + tid; t < npad; t += blockDim.x) {
    S.skey[t] = ~0ull;
    S.sval[t] = INT32_MAX;
  }

  // ---- 4. order by (score desc, recall position asc) --------------------
  if (L > 0 && (p.stages & kStageSort)) bitonic_sort_pairs(S.skey, S.sval, npad);
  __syncthreads();
  if (p.order_out)
    for (int i = tid; i < p.lmax; i += blockDim.x)
      p.order_out[(int64_t)u * p.lmax + i] = i < L ? S.sval[i] : kEmpty;

  // ---- 5. FIFO dynamic centroid update (ck/index.py:120-133) ------------
  const bool dcu_here = (p.stages & kStageDcu) && (L > 0 || p.dcu_force);
  if (dcu_here) {
    const int64_t slot = s_slot;
    int32_t* row = p.lists + ((int64_t)u * p.C + slot) * p.rho;
    const int keep = min(p.rho, L);
    for (int i = tid; i < p.rho; i += blockDim.x) row[i] = i < keep ? S.rec[S.sval[i]] : kEmpty;
    T* cent = static_cast<T*>(p.cent);
    for (int i = tid; i < gs * D; i += blockDim.x) {
      const int hh = i / D, e = i % D;
      cent[(((int64_t)bi * p.h + gi * gs + hh) * p.C + slot) * D + e] = q[i];
    }
    write_slot_norms<T, D>(p, q, bi, gi, slot);
  }

  // ---- 6. sparse attention over the top rho' (or the whole recall set) ---
  if (p.stages & kStageAttend) {
    const int R_ = (L > 0) ? (p.use_rerank ? min(p.rho_prime, L) : L) : 0;
    auto pos_of = [&](int i) { return p.use_rerank ? S.sval[i] : i; };
    if (p.sparse_ids)
      for (int i = tid; i < p.sparse_cap; i += blockDim.x)
        p.sparse_ids[(int64_t)u * p.sparse_cap + i] = i < R_ ? S.rec[pos_of(i)] : kEmpty;
    if (p.sparse_len && tid == 0) p.sparse_len[u] = R_;
    __shared__ double ms[kMaxGroup], ls[kMaxGroup];
    // per-head max over the sparse logits
    for (int hh = 0; hh < gs; ++hh) {
      double m = -INFINITY;
      for (int i = tid; i < R_; i += blockDim.x) m = fmax(m, lg[(int64_t)hh * p.lmax + pos_of(i)]);
      m = block_max_f64(m, S.scratch);
      if (tid == 0) ms[hh] = m;
    }
    __syncthreads();
    const T* vals = static_cast<const T*>(p.values);
    // sparse set weights, chunk by chunk; accumulators live in the reduce
    // area (aliases the sort keys, dead after ordering)
    float* red = reinterpret_cast<float*>(S.skey);
    for (int i = tid; i < kUnitWarps * gs * D; i += blockDim.x) red[i] = 0.f;
    if (tid < gs) ls[tid] = 0.0;
    for (int c0 = 0; c0 < R_; c0 += kAttnChunk) {
      const int n = min(kAttnChunk, R_ - c0);
      for (int hh = 0; hh < gs; ++hh) {
        double lpart = 0.0;
        for (int i = tid; i < n; i += blockDim.x) {
          const double e = exp(lg[(int64_t)hh * p.lmax + pos_of(c0 + i)] - ms[hh]);
          S.wts[hh * kAttnChunk + i] = (float)e;
          lpart += e;
        }
        lpart = block_sum_f64(lpart, S.scratch);
        if (tid == 0) ls[hh] += lpart;
      }
      __syncthreads();
      accum_weighted_rows<T, D>(
          n, gs,
          [&](int t) -> const T* { return vals + ((int64_t)u * p.cap + S.rec[pos_of(c0 + t)]) * D; },
          [&](int hh, int t) { return S.wts[hh * kAttnChunk + t]; }, red + (int64_t)warp * gs * D);
      __syncthreads();
    }
    // ---- 7. exact merge with the static partials ------------------------
    bool none = false;
    for (int i = tid; i < gs * D; i += blockDim.x) {
      const int hh = i / D;
      float osp = 0.f;
      for (int w = 0; w < kUnitWarps; ++w) osp += red[(int64_t)w * gs * D + i];
      double M = R_ > 0 ? ms[hh] : -INFINITY;
      const int64_t pbase = (int64_t)u * p.ns;
      for (int j = 0; j < p.ns; ++j)
        if (p.pl[(pbase + j) * gs + hh] > 0.0) M = fmax(M, p.pm[(pbase + j) * gs + hh]);
      double Lsum = 0.0, O = 0.0;
      if (R_ > 0) {
        const double w = exp(ms[hh] - M);
        Lsum += w * ls[hh];
        O += w * (double)osp;
      }
      for (int j = 0; j < p.ns; ++j) {
        const double lj = p.pl[(pbase + j) * gs + hh];
        if (lj > 0.0) {
          const double w = exp(p.pm[(pbase + j) * gs + hh] - M);
          Lsum += w * lj;
          O += w * (double)p.po[((pbase + j) * gs + hh) * D + (i % D)];
        }
      }
      const int64_t oh = (int64_t)bi * p.h + gi * gs + hh;
      if (Lsum > 0.0) {
        p.out[oh * D + (i % D)] = (float)(O / Lsum);
      } else {
        p.out[oh * D + (i % D)] = 0.f;
        none = true;
      }
      if (i % D == 0) {
        if (p.row_max) p.row_max[oh] = M;
        if (p.denom) p.denom[oh] = Lsum;
      }
    }
    if (none) set_flag(p.flags, kFlagNoTokens);  // nothing attendable (ck/retrieval.py:355)
  }

  // ---- 8. completion: FIFO cursor advance and total++ by the last CTA ----
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
        if (appending) *p.total = t0 + 1;
        atomicExch(&p.sync[0], 0);
        __threadfence();
      }
    }
  }
}

// ------------------------------------------------------------------------
// v3 fused unit kernel (bf16): a 2-CTA cluster per (b, g) unit.
//   both ranks : top-C' slots from the scan's chunk candidates (one warp),
//                union via per-list bitmaps tested in parallel, rerank
//                logits for half the recalled positions -> packed
//                (score, position) keys in both CTAs' smem (DSMEM)
//   cluster barrier
//   rank 0     : radix-select the top-rho' set, sparse attention over it,
//                exact merge with the (prefetched) static partials -> out
//   rank 1     : full (score desc, position asc) sort, FIFO DCU write,
//                ordered sparse-id outputs
// ------------------------------------------------------------------------

constexpr int kU2Threads = 512;
constexpr int kU2Warps = kU2Threads / 32;
constexpr int kMaxParLists = 8;   // C' lists unioned in parallel (else sequentially)
constexpr int kUnionItems = 16;   // union elements per thread held in registers

struct U2Smem {
  int32_t* sel;      // [c_prime]
  uint32_t* areaA;   // union bitmaps; then static-partial o prefetch + selected positions
  int32_t* rec;      // [lmax]
  uint64_t* skey;    // [npad]; rank 0 reuses it as the attention reduce area
  float* wts;        // [gs][kAttnChunk]
  double* spml;      // [2][ns][gs] static m, l
  int* hist;         // [256]
  double* scratch;   // [128]
};

__host__ __device__ inline int u2_npad(int lmax) {
  const int n = next_pow2(lmax > 1 ? lmax : 1);
  return n < kU2Threads ? kU2Threads : n;
}

__host__ __device__ inline size_t u2_area_a(const DecodeParams& p, int D) {
  const int nb = p.c_prime <= kMaxParLists ? p.c_prime : 1;
  const size_t bm = (size_t)nb * p.bitmap_words * 4;
  const size_t po = (size_t)p.ns * p.gs * D * 4 + (size_t)4 * (p.lmax > 1 ? p.lmax : 1);
  return bm > po ? bm : po;
}

__host__ __device__ inline size_t u2_layout(const DecodeParams& p, int D, U2Smem* s,
                                            unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* ptr = base ? base + off : nullptr;
    off += align16(bytes);
    return ptr;
  };
  const size_t red = (size_t)kU2Warps * p.gs * D * 4;
  const size_t keys = (size_t)u2_npad(p.lmax) * 8;
  U2Smem t;
  t.sel = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (p.c_prime > 1 ? p.c_prime : 1)));
  t.areaA = reinterpret_cast<uint32_t*>(take(u2_area_a(p, D)));
  t.rec = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (p.lmax > 1 ? p.lmax : 1)));
  t.skey = reinterpret_cast<uint64_t*>(take(keys > red ? keys : red));
  t.wts = reinterpret_cast<float*>(take(sizeof(float) * p.gs * kAttnChunk));
  t.spml = reinterpret_cast<double*>(take(sizeof(double) * 2 * (p.ns > 1 ? p.ns : 1) * p.gs));
  t.hist = reinterpret_cast<int*>(take(sizeof(int) * 256));
  const int nscr = p.gs * (p.ns + 1) > 128 ? p.gs * (p.ns + 1) : 128;
  t.scratch = reinterpret_cast<double*>(take(sizeof(double) * nscr));
  if (s) *s = t;
  return off;
}

size_t unit2_smem_bytes(const DecodeParams& p, int D) { return u2_layout(p, D, nullptr, nullptr); }



template <typename T, int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kU2Threads, 1)
    unit2_kernel(DecodeParams p) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  U2Smem S;
  u2_layout(p, D, &S, smem);
  const int u = blockIdx.x >> 1;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t t0 = *p.total;
  const bool appending = p.k_new != nullptr;
  const int64_t total = t0 + (appending ? 1 : 0);
  __shared__ int64_t s_slot;
  __shared__ __align__(16) T qs[kMaxGroup * D];
  __shared__ double ms[kMaxGroup], ls[kMaxGroup];
  __shared__ int s_state[4];
  phase_mark(0);
  if (tid == 0) s_slot = p.fifo ? (p.fifo[bi] % p.C) : 0;
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  for (int i = tid; i < gs * D; i += blockDim.x) qs[i] = q[i];
  const int64_t pbase = (int64_t)u * p.ns;
  if (rank == 0)   // static m, l (ready since the scan kernel finished)
    for (int i = tid; i < p.ns * gs; i += blockDim.x) {
      S.spml[i] = p.pm[pbase * gs + i];
      S.spml[p.ns * gs + i] = p.pl[pbase * gs + i];
    }

  // ---- 1. top-C' slots from the chunk candidates (one warp) -------------
  if (warp == 0) {
    const int M = p.cos_blocks_per_unit * p.ncand;
    const double* cv = p.cval + (int64_t)u * M;
    const int32_t* ci = p.cidx + (int64_t)u * M;
    constexpr int KR = 8;                 // candidates per lane kept in registers
    uint64_t rk[KR];
    int ri[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int m = lane + 32 * r;
      rk[r] = m < M ? okey64(cv[m]) : 0ull;
      ri[r] = m < M ? ci[m] : INT32_MAX;
    }
    uint64_t prev_key = ~0ull;
    int prev_idx = -1;
    for (int r = 0; r < p.c_prime; ++r) {
      uint64_t bk = 0;
      int bidx = INT32_MAX;
#pragma unroll
      for (int x = 0; x < KR; ++x) {
        const uint64_t k = rk[x];
        const int i = ri[x];
        const bool below = k < prev_key || (k == prev_key && i > prev_idx);
        if (below && (k > bk || (k == bk && i < bidx))) { bk = k; bidx = i; }
      }
      for (int m = lane + 32 * KR; m < M; m += 32) {   // only when M > 256
        const uint64_t k = okey64(cv[m]);
        const int i = ci[m];
        const bool below = k < prev_key || (k == prev_key && i > prev_idx);
        if (below && (k > bk || (k == bk && i < bidx))) { bk = k; bidx = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (k2 > bk || (k2 == bk && i2 < bidx)) { bk = k2; bidx = i2; }
      }
      if (lane == 0) S.sel[r] = bidx;
      prev_key = bk;
      prev_idx = bidx;
    }
  }
  __syncthreads();
  phase_mark(1);

  // ---- 2. union of the selected lists, first occurrence kept -------------
  int L = 0;
  const int nwords = (int)((total + 31) >> 5);
  if (p.c_prime <= kMaxParLists && p.c_prime * p.rho <= kU2Threads * kUnionItems) {
    // every list marks its own bitmap, then an id of list j survives iff no
    // earlier list holds it.  Warp w owns the contiguous element range
    // [w*P, (w+1)*P) in (list, position) order, lane-interleaved, so ballots
    // give each survivor its rank without a block-wide scan per list.
    const int nb = p.c_prime;
    const int n = nb * p.rho;
    for (int i = tid; i < nb * p.bitmap_words; i += blockDim.x) S.areaA[i] = 0u;
    const int P = ((n + kU2Warps - 1) / kU2Warps + 31) & ~31;
    const int nit = P / 32;
    int ids[kUnionItems];
    int lst[kUnionItems];
#pragma unroll
    for (int it = 0; it < kUnionItems; ++it) {
      ids[it] = kEmpty;
      lst[it] = 0;
      const int o = warp * P + it * 32 + lane;
      if (it < nit && o < n) {
        const int j = o / p.rho;
        int id = p.lists[((int64_t)u * p.C + S.sel[j]) * p.rho + (o - j * p.rho)];
        if (id != kEmpty && (id < 0 || id >= total)) { set_flag(p.flags, kFlagIdRange); id = kEmpty; }
        ids[it] = id;
        lst[it] = j;
      }
    }
    __syncthreads();   // bitmaps cleared
#pragma unroll
    for (int it = 0; it < kUnionItems; ++it)
      if (ids[it] != kEmpty)
        atomicOr(&S.areaA[lst[it] * p.bitmap_words + (ids[it] >> 5)], 1u << (ids[it] & 31));
    __syncthreads();
    int wcount = 0;
    unsigned keepm[kUnionItems];
#pragma unroll
    for (int it = 0; it < kUnionItems; ++it) {
      bool keep = ids[it] != kEmpty;
      if (keep)
        for (int j2 = 0; j2 < lst[it]; ++j2)
          keep = keep && !((S.areaA[j2 * p.bitmap_words + (ids[it] >> 5)] >> (ids[it] & 31)) & 1u);
      keepm[it] = __ballot_sync(0xffffffffu, keep);
      wcount += __popc(keepm[it]);
    }
    int* wtot = reinterpret_cast<int*>(S.scratch);
    if (lane == 0) wtot[warp] = wcount;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += wtot[w];
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < kU2Warps; ++w) t += wtot[w];
      wtot[kU2Warps] = t;
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < kUnionItems; ++it) {
      if ((keepm[it] >> lane) & 1u) S.rec[base + __popc(keepm[it] & lt)] = ids[it];
      base += __popc(keepm[it]);
    }
    __syncthreads();
    L = wtot[kU2Warps];
    __syncthreads();
  } else {
    uint32_t* bitmap = S.areaA;
    for (int i = tid; i < nwords; i += blockDim.x) bitmap[i] = 0u;
    __syncthreads();
    const int per = (p.rho + blockDim.x - 1) / blockDim.x;
    for (int j = 0; j < p.c_prime; ++j) {
      const int32_t* row = p.lists + ((int64_t)u * p.C + S.sel[j]) * p.rho;
      int keep_mask = 0, cnt = 0;
      for (int e = 0; e < per; ++e) {
        const int i = tid * per + e;
        int id = (i < p.rho) ? row[i] : kEmpty;
        if (id != kEmpty && (id < 0 || id >= total)) { set_flag(p.flags, kFlagIdRange); id = kEmpty; }
        if (id != kEmpty && !((bitmap[id >> 5] >> (id & 31)) & 1u)) { keep_mask |= 1 << e; ++cnt; }
      }
      int tot;
      int pos = L + block_exclusive_scan(cnt, &tot, S.scratch);
      for (int e = 0; e < per; ++e)
        if (keep_mask & (1 << e)) S.rec[pos++] = row[tid * per + e];
      __syncthreads();
      for (int e = 0; e < per; ++e)
        if (keep_mask & (1 << e)) {
          const int id = row[tid * per + e];
          atomicOr(&bitmap[id >> 5], 1u << (id & 31));
        }
      L += tot;
      __syncthreads();
    }
  }
  phase_mark(2);
  const int npad = u2_npad(L);
  // rank 0: prefetch the static partials' o into area A (free after the union)
  float* spo = reinterpret_cast<float*>(S.areaA);
  int* spos = reinterpret_cast<int*>(spo + (size_t)p.ns * gs * D);
  if (rank == 0)
    for (int i = tid; i < p.ns * gs * D; i += blockDim.x) spo[i] = p.po[pbase * gs * D + i];

  // ---- 3. rerank logits for this rank's half -------------------------------
  // 8 lanes per key row (each lane two 16-byte chunks, so a lane group reads
  // one contiguous 128-byte line per load), f32 chunk partials from exact
  // bf16 products, f64 across chunks and lanes.
  double* lg = p.logits + (int64_t)u * gs * p.lmax;
  uint64_t* peer_skey = cl.map_shared_rank(S.skey, rank ^ 1);
  {
    const int half = (L + 1) >> 1;
    const int lo = rank ? half : 0, hi = rank ? L : half;
    const T* keys = static_cast<const T*>(p.keys) + (int64_t)u * p.cap * D;
    const double scale = 1.0 / sqrt((double)D);
    constexpr int VPR = D * int(sizeof(T)) / 16;     // 16 for d=128 bf16
    constexpr int LPRL = 8;                          // lanes per row
    constexpr int CPL = VPR / LPRL;                  // chunks per lane
    constexpr int RPWL = 32 / LPRL;                  // rows per warp pass
    constexpr int UNL = 2;                           // passes in flight
    const int sub = lane % LPRL, rw = lane / LPRL;
    const int stepw = kU2Warps * RPWL;
    for (int base = lo + warp * RPWL; base < hi; base += stepw * UNL) {
      uint4 raw[UNL][CPL];
      int tt[UNL];
#pragma unroll
      for (int u2 = 0; u2 < UNL; ++u2) {
        tt[u2] = base + u2 * stepw + rw;
        if (tt[u2] < hi) {
          const uint4* r4 = reinterpret_cast<const uint4*>(keys + (int64_t)S.rec[tt[u2]] * D);
#pragma unroll
          for (int c = 0; c < CPL; ++c) raw[u2][c] = ldg16(r4 + c * LPRL + sub);
        } else {
#pragma unroll
          for (int c = 0; c < CPL; ++c) raw[u2][c] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u2 = 0; u2 < UNL; ++u2) {
        double gmax = -INFINITY;
        for (int hh = 0; hh < gs; ++hh) {
          const uint4* q4 = reinterpret_cast<const uint4*>(qs + hh * D);
          double a = 0.0;
#pragma unroll
          for (int c = 0; c < CPL; ++c) a += (double)bf16x8_dot(q4[c * LPRL + sub], raw[u2][c], 0.f);
#pragma unroll
          for (int o = 1; o < LPRL; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          a *= scale;
          if (sub == 0 && tt[u2] < hi) lg[(int64_t)hh * p.lmax + tt[u2]] = a;
          gmax = fmax(gmax, a);
        }
        if (sub == 0 && tt[u2] < hi) {
          const uint64_t key = ((uint64_t)(~okey32((float)gmax)) << 32) | (uint32_t)tt[u2];
          S.skey[tt[u2]] = key;
          peer_skey[tt[u2]] = key;
        }
      }
    }
    for (int t = L + tid; t < npad; t += blockDim.x) S.skey[t] = ~0ull;
  }
  phase_mark(3);
  cl.sync();  // keys complete in both CTAs; logits visible in global memory
  phase_mark(4);

  const int Rn = (L > 0) ? (p.use_rerank ? min(p.rho_prime, L) : L) : 0;
  const bool dcu_here = (p.stages & kStageDcu) && L > 0;
  if (rank == 1) {
    // ---- rank 1: full order, DCU, ordered sparse ids -------------------------
    if (L > 0 && (dcu_here || (p.sparse_ids && p.use_rerank))) {
      switch (npad) {
        case 512: sort_keys<1>(S.skey); break;
        case 1024: sort_keys<2>(S.skey); break;
        case 2048: sort_keys<4>(S.skey); break;
        case 4096: sort_keys<8>(S.skey); break;
        default: sort_keys<16>(S.skey); break;
      }
    }
    phase_mark(5);
    auto pos_at = [&](int i) { return (int)(uint32_t)(S.skey[i] & 0xffffffffu); };
    if (dcu_here) {
      const int64_t slot = s_slot;
      int32_t* row = p.lists + ((int64_t)u * p.C + slot) * p.rho;
      const int keep = min(p.rho, L);
      for (int i = tid; i < p.rho; i += blockDim.x) row[i] = i < keep ? S.rec[pos_at(i)] : kEmpty;
      T* cent = static_cast<T*>(p.cent);
      for (int i = tid; i < gs * D; i += blockDim.x) {
        const int hh = i / D, e = i % D;
        cent[(((int64_t)bi * p.h + gi * gs + hh) * p.C + slot) * D + e] = q[i];
      }
      write_slot_norms<T, D>(p, q, bi, gi, slot);
    }
    if (p.sparse_ids)
      for (int i = tid; i < p.sparse_cap; i += blockDim.x)
        p.sparse_ids[(int64_t)u * p.sparse_cap + i] =
            i < Rn ? S.rec[p.use_rerank ? pos_at(i) : i] : kEmpty;
    phase_mark(6);
    return;
  }

  // ---- rank 0: top-rho' set, sparse attention, merge --------------------
  const int nsel = Rn > 0 ? select_smallest(S.skey, L, Rn, spos, S.hist, s_state) : 0;
  phase_mark(5);
  {
    // per-head max over the selected logits: thread-local, warp, then block
    double* wm = S.scratch;             // [kU2Warps][gs] (gs <= 8 here) as doubles
    for (int h0 = 0; h0 < gs; h0 += 4) {
      double m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int i = tid; i < nsel; i += blockDim.x) {
        const int ps = spos[i];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh)
          if (h0 + hh < gs) m4[hh] = fmax(m4[hh], lg[(int64_t)(h0 + hh) * p.lmax + ps]);
      }
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m4[hh] = fmax(m4[hh], __shfl_xor_sync(0xffffffffu, m4[hh], o));
      }
      __syncthreads();
      if (lane == 0)
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) wm[warp * 4 + hh] = m4[hh];
      __syncthreads();
      if (tid < 4 && h0 + tid < gs) {
        double m = -INFINITY;
        for (int w = 0; w < kU2Warps; ++w) m = fmax(m, wm[w * 4 + tid]);
        ms[h0 + tid] = m;
        ls[h0 + tid] = 0.0;
      }
    }
    __syncthreads();
    phase_mark(6);
    float* red = reinterpret_cast<float*>(S.skey);   // keys are dead on rank 0 now
    for (int i = tid; i < kU2Warps * gs * D; i += blockDim.x) red[i] = 0.f;
    const T* vals = static_cast<const T*>(p.values) + (int64_t)u * p.cap * D;
    for (int c0 = 0; c0 < nsel; c0 += kAttnChunk) {
      const int n = min(kAttnChunk, nsel - c0);
      for (int h0 = 0; h0 < gs; h0 += 4) {
        double l4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i = tid; i < n; i += blockDim.x) {
          const int ps = spos[c0 + i];
#pragma unroll
          for (int hh = 0; hh < 4; ++hh)
            if (h0 + hh < gs) {
              const double e = exp(lg[(int64_t)(h0 + hh) * p.lmax + ps] - ms[h0 + hh]);
              S.wts[(h0 + hh) * kAttnChunk + i] = (float)e;
              l4[hh] += e;
            }
        }
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) l4[hh] += __shfl_xor_sync(0xffffffffu, l4[hh], o);
        }
        __syncthreads();
        if (lane == 0)
#pragma unroll
          for (int hh = 0; hh < 4; ++hh) S.scratch[warp * 4 + hh] = l4[hh];
        __syncthreads();
        if (tid < 4 && h0 + tid < gs) {
          double l = 0.0;
          for (int w = 0; w < kU2Warps; ++w) l += S.scratch[w * 4 + tid];
          ls[h0 + tid] += l;
        }
      }
      __syncthreads();
      accum_weighted_rows<T, D>(
          n, gs, [&](int t) -> const T* { return vals + (int64_t)S.rec[spos[c0 + t]] * D; },
          [&](int hh, int t) { return S.wts[hh * kAttnChunk + t]; }, red + (int64_t)warp * gs * D);
      __syncthreads();
    }
    phase_mark(7);
    // exact merge with the static partials: per head the running max M and
    // the split weights exp(m_j - M) once, then a weighted sum per element
    double* wj = S.scratch;   // [gs][ns + 1]: w_static_j ..., w_sparse ; Ls at [gs*(ns+1)+hh]
    const int ns = p.ns;
    __syncthreads();
    if (tid < gs) {
      const int hh = tid;
      double M = ls[hh] > 0.0 ? ms[hh] : -INFINITY;
      for (int j = 0; j < ns; ++j)
        if (S.spml[ns * gs + j * gs + hh] > 0.0) M = fmax(M, S.spml[j * gs + hh]);
      double Ls = 0.0;
      for (int j = 0; j < ns; ++j) {
        const double lj = S.spml[ns * gs + j * gs + hh];
        const double w = lj > 0.0 ? exp(S.spml[j * gs + hh] - M) : 0.0;
        wj[hh * (ns + 1) + j] = w;
        Ls += w * lj;
      }
      const double wsp = ls[hh] > 0.0 ? exp(ms[hh] - M) : 0.0;
      wj[hh * (ns + 1) + ns] = wsp;
      Ls += wsp * ls[hh];
      ms[hh] = M;          // reuse: merged statistics
      ls[hh] = Ls;
    }
    __syncthreads();
    bool none = false;
    for (int i = tid; i < gs * D; i += blockDim.x) {
      const int hh = i / D, e = i % D;
      float o0 = 0.f;
      for (int w = 0; w < kU2Warps; ++w) o0 += red[(int64_t)w * gs * D + i];
      const double* wh = wj + hh * (ns + 1);
      double O = wh[ns] * (double)o0;
      for (int j = 0; j < ns; ++j) O += wh[j] * (double)spo[(j * gs + hh) * D + e];
      const double Ls = ls[hh];
      const int64_t oh = (int64_t)bi * p.h + gi * gs + hh;
      if (Ls > 0.0) {
        p.out[oh * D + e] = (float)(O / Ls);
      } else {
        p.out[oh * D + e] = 0.f;
        none = true;
      }
      if (e == 0) {
        if (p.row_max) p.row_max[oh] = ms[hh];
        if (p.denom) p.denom[oh] = Ls;
      }
    }
    if (none) set_flag(p.flags, kFlagNoTokens);
  }
  phase_mark(8);
  if (p.selected)
    for (int r = tid; r < p.c_prime; r += blockDim.x) p.selected[(int64_t)u * p.c_prime + r] = S.sel[r];
  if (p.recall_len && tid == 0) p.recall_len[u] = L;
  if (p.sparse_len && tid == 0) p.sparse_len[u] = Rn;
  if (tid == 0) set_flag(p.flags, L > 0 ? kFlagNonEmptyRecall : kFlagEmptyRecall);

  // ---- completion: FIFO cursor advance + total++ by the last unit ----------
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
        if (appending) *p.total = t0 + 1;
        atomicExch(&p.sync[0], 0);
        __threadfence();
      }
    }
  }
}

// ------------------------------------------------------------------------
// generic id-list attention (sparse_attention API): split-K partials + merge
// ------------------------------------------------------------------------

template <typename T, int D>
__global__ void __launch_bounds__(kScanThreads) attn_split_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int64_t total = *p.total;
  const int per_unit = p.ns;  // splits per unit (list splits first, then static)
  const int u = blockIdx.x / per_unit, split = blockIdx.x % per_unit;
  const int slot = u * per_unit + split;
  const int list_splits = p.list_splits;
  if (split < list_splits) {
    const int len = p.ids_shared ? p.len_in[0] : p.len_in[u];
    const int32_t* ids = p.rec_in + (p.ids_shared ? 0 : (int64_t)u * p.lmax);
    const int i0 = split * kAttnSplit;
    const int ntok = max(0, min(kAttnSplit, len - i0));
    attn_partial_block<T, D>(p, u, ntok, [&](int t) { return (int64_t)ids[i0 + t]; }, -1, total,
                             p.pm + (int64_t)slot * p.gs, p.pl + (int64_t)slot * p.gs,
                             p.po + (int64_t)slot * p.gs * D, smem);
  } else {
    const StaticSpan span(total, p.init_len, p.local_len);
    const int64_t i0 = (int64_t)(split - list_splits) * kAttnSplit;
    const int ntok = (int)max((int64_t)0, min((int64_t)kAttnSplit, span.n_static - i0));
    attn_partial_block<T, D>(p, u, ntok, [&](int t) { return span.id(i0 + t); }, -1, total,
                             p.pm + (int64_t)slot * p.gs, p.pl + (int64_t)slot * p.gs,
                             p.po + (int64_t)slot * p.gs * D, smem);
  }
}

// one thread per (unit, head, e): combine split partials
__global__ void attn_merge_kernel(DecodeParams p, int D) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)p.U * p.gs * D;
  if (i >= n) return;
  const int e = (int)(i % D);
  const int hh = (int)((i / D) % p.gs);
  const int u = (int)(i / ((int64_t)D * p.gs));
  const int bi = u / p.g, gi = u % p.g;
  double M = -INFINITY;
  for (int j = 0; j < p.ns; ++j) {
    const int64_t s = ((int64_t)u * p.ns + j) * p.gs + hh;
    if (p.pl[s] > 0.0) M = fmax(M, p.pm[s]);
  }
  double Lsum = 0.0, O = 0.0;
  for (int j = 0; j < p.ns; ++j) {
    const int64_t s = ((int64_t)u * p.ns + j) * p.gs + hh;
    if (p.pl[s] > 0.0) {
      const double w = exp(p.pm[s] - M);
      Lsum += w * p.pl[s];
      O += w * (double)p.po[s * D + e];
    }
  }
  const int64_t oh = (int64_t)bi * p.h + gi * p.gs + hh;
  p.out[oh * D + e] = Lsum > 0.0 ? (float)(O / Lsum) : 0.f;
  if (e == 0) {
    if (p.row_max) p.row_max[oh] = M;
    if (p.denom) p.denom[oh] = Lsum;
  }
}

__global__ void merge2_kernel(int64_t rows, int D, const float* oa, const double* ma,
                              const double* la, const float* ob, const double* mb,
                              const double* lb, float* out, double* mo, double* lo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * D) return;
  const int64_t r = i / D;
  const double m = fmax(ma[r], mb[r]);
  const double wa = exp(ma[r] - m) * la[r];
  const double wb = exp(mb[r] - m) * lb[r];
  const double den = wa + wb;
  out[i] = (float)(((double)oa[i] * wa + (double)ob[i] * wb) / den);
  if (i % D == 0) {
    if (mo) mo[r] = m;
    if (lo) lo[r] = den;
  }
}

template <typename T>
__global__ void append_kernel(T* keys, T* vals, const T* kn, const T* vn, int64_t* total,
                              int64_t units, int64_t cap, int D) {
  const int64_t t0 = *total;
  for (int64_t i = threadIdx.x; i < units * D; i += blockDim.x) {
    const int64_t u = i / D, e = i % D;
    keys[(u * cap + t0) * D + e] = kn[i];
    vals[(u * cap + t0) * D + e] = vn[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) *total = t0 + 1;
}

// ------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------

size_t scan_smem_bytes(const DecodeParams& p, int D) {
  const size_t cosb = sizeof(float) * kMaxGroup * D + sizeof(double) * kMaxGroup +
                      sizeof(double) * kMaxGroup * kCosChunk;
  const size_t attb = sizeof(float) * kMaxGroup * D + sizeof(double) * kMaxGroup * kAttnSplit +
                      2 * sizeof(double) * kMaxGroup + sizeof(float) * kScanWarps * p.gs * D;
  return std::max(cosb, attb);
}


template <typename T, int D>
static int launch_scan_t(const DecodeParams& p0, int nblocks, cudaStream_t st) {
  DecodeParams p = p0;
  p.dbg = g_host_dbg;
  const size_t sm = scan2_smem<T, D>(p.gs);
  auto k = scan2_kernel<T, D>;
  if (int rc = set_max_smem_k(k, sm)) return rc;
  if (nblocks > 0) launch_k(k, dim3(nblocks), dim3(kScanRowsV2), sm, st, kPrioLow, p);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

template <typename T, int D>
static int launch_unit2_t(const DecodeParams& p, cudaStream_t st) {
  const size_t sm = unit2_smem_bytes(p, D);
  if (sm > 200 * 1024) return CTKV_ECONFIG;
  auto k = unit2_kernel<T, D>;
  if (int rc = set_max_smem_k(k, sm)) return rc;
  k<<<2 * p.U, kU2Threads, sm, st>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

template <typename T, int D>
static int launch_unit_t(const DecodeParams& p, cudaStream_t st) {
  const size_t sm = unit_smem_bytes(p, D);
  if (sm > 220 * 1024) return CTKV_ECONFIG;
  auto k = unit_kernel<T, D>;
  if (int rc = set_max_smem_k(k, sm)) return rc;
  k<<<p.U, kUnitThreads, sm, st>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

template <typename T, int D>
static int launch_attn_t(const DecodeParams& p, cudaStream_t st) {
  const size_t sm = scan_smem_bytes(p, D);
  auto k = attn_split_kernel<T, D>;
  if (int rc = set_max_smem_k(k, sm)) return rc;
  k<<<p.U * p.ns, kScanThreads, sm, st>>>(p);
  const int64_t n = (int64_t)p.U * p.gs * D;
  attn_merge_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, D);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

#define CTKV_DISPATCH(DTYPE, DIM, FN, ...)                                              \
  [&]() -> int {                                                                        \
    if ((DTYPE) == CTKV_BF16) {                                                         \
      switch (DIM) {                                                                    \
        case 16: return FN<__nv_bfloat16, 16>(__VA_ARGS__);                             \
        case 32: return FN<__nv_bfloat16, 32>(__VA_ARGS__);                             \
        case 64: return FN<__nv_bfloat16, 64>(__VA_ARGS__);                             \
        case 128: return FN<__nv_bfloat16, 128>(__VA_ARGS__);                           \
        case 256: return FN<__nv_bfloat16, 256>(__VA_ARGS__);                           \
      }                                                                                 \
    } else {                                                                            \
      switch (DIM) {                                                                    \
        case 16: return FN<float, 16>(__VA_ARGS__);                                     \
        case 32: return FN<float, 32>(__VA_ARGS__);                                     \
        case 64: return FN<float, 64>(__VA_ARGS__);                                     \
        case 128: return FN<float, 128>(__VA_ARGS__);                                   \
        case 256: return FN<float, 256>(__VA_ARGS__);                                   \
      }                                                                                 \
    }                                                                                   \
    return (int)CTKV_ESHAPE;                                                            \
  }()

int launch_scan(const DecodeParams& p, int dtype, int D, int nblocks, cudaStream_t st) {
  return CTKV_DISPATCH(dtype, D, launch_scan_t, p, nblocks, st);
}
int launch_unit(const DecodeParams& p, int dtype, int D, cudaStream_t st) {
  return CTKV_DISPATCH(dtype, D, launch_unit_t, p, st);
}
int launch_unit2(const DecodeParams& p, int dtype, int D, cudaStream_t st) {
  if (dtype != CTKV_BF16) return CTKV_ECONFIG;
  switch (D) {
    case 64: return launch_unit2_t<__nv_bfloat16, 64>(p, st);
    case 128: return launch_unit2_t<__nv_bfloat16, 128>(p, st);
    case 256: return launch_unit2_t<__nv_bfloat16, 256>(p, st);
  }
  return CTKV_ESHAPE;
}
int phase_timing(int on, unsigned long long* out, int n) {
  if (out != nullptr) {
    const int m = n < kPhaseCtas * kPhases ? n : kPhaseCtas * kPhases;
    if (cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * m) != cudaSuccess) return CTKV_ECUDA;
  }
  if (on >= 0) {
    if (cudaMemcpyToSymbol(g_phase_on, &on, sizeof(int)) != cudaSuccess) return CTKV_ECUDA;
  }
  return 0;
}
int kernel_timeline(int on) {   // host switch; on < 0 queries
  static int v = 0;
  if (on >= 0) v = on;
  return v;
}

// Launch priorities: the latency-bound chain kernels are dispatched first,
// the bandwidth-bound scans and the deferred tails after them (a ready chain
// otherwise waits ~16 us behind queued scan CTAs).
int launch_priority(LaunchPrio pr) {
  static int lo = 1, hi = 0, init = 0;
  if (!init) {
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) { lo = 0; hi = 0; }
    init = 1;
  }
  return pr == kPrioHigh ? hi : lo;   // numerically lower = higher priority
}

// Programmatic dependent launch, for callers that allow it (phase bit 16):
// on the chain launch (scan CTAs trigger by exiting, so the chain's launch is
// processed while the scan drains, without resident CTAs waiting) and on the
// scan launch (the previous chain triggers after its compaction; the scan's
// centroid TMA loads start before its griddepcontrol wait).
thread_local int t_pdl_ok = 0;

// 16-byte copy by a kernel (either side may be mapped pinned host memory):
// every load of a thread issued before its stores, so a PCIe read stream has
// many requests in flight
__global__ void __launch_bounds__(256) stage_copy_kernel(uint4* __restrict__ dst,
                                                         const uint4* __restrict__ src, int64_t n) {
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) r[u] = src[i0 + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) dst[i0 + u * stride] = r[u];
  }
}

int launch_stage_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  const int64_t n = (int64_t)(bytes / 16);
  const int64_t blocks = std::min<int64_t>((n + 1023) / 1024, 4 * 148);
  stage_copy_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(
      static_cast<uint4*>(dst), static_cast<const uint4*>(src), n);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

// |row| for rows of D elements: one warp per row, f64 squares (exact for
// bf16 and f32 inputs), rounded to f32
template <typename T, int D>
__global__ void row_norms_kernel(const T* __restrict__ rows, int64_t n, float* __restrict__ out) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const T* x = rows + r * D;
  double s = 0.0;
  for (int e = lane; e < D; e += 32) {
    const double v = (double)to_f(x[e]);
    s = fma(v, v, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = (float)sqrt(s);
}

template <typename T, int D>
static int launch_norms_t(const void* cent, int64_t rows, float* out, cudaStream_t st) {
  if (rows == 0) return 0;
  const int64_t threads = rows * 32;
  row_norms_kernel<T, D><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      static_cast<const T*>(cent), rows, out);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

int launch_centroid_norms(int dtype, int D, const void* cent, int64_t rows, float* out,
                          cudaStream_t st) {
  return CTKV_DISPATCH(dtype, D, launch_norms_t, cent, rows, out, st);
}

int static_tok_for(int dtype) { return dtype == CTKV_BF16 ? static_tok<__nv_bfloat16>() : static_tok<float>(); }
int launch_attn(const DecodeParams& p, int dtype, int D, cudaStream_t st) {
  return CTKV_DISPATCH(dtype, D, launch_attn_t, p, st);
}
int launch_merge2(int64_t rows, int D, const float* oa, const double* ma, const double* la,
                  const float* ob, const double* mb, const double* lb, float* out, double* mo,
                  double* lo, cudaStream_t st) {
  const int64_t n = rows * D;
  if (n == 0) return 0;
  merge2_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rows, D, oa, ma, la, ob, mb, lb, out,
                                                              mo, lo);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}
int launch_append(int dtype, void* keys, void* vals, const void* kn, const void* vn,
                  int64_t* total, int64_t units, int64_t cap, int D, cudaStream_t st) {
  if (dtype == CTKV_BF16)
    append_kernel<__nv_bfloat16><<<1, 256, 0, st>>>(
        (__nv_bfloat16*)keys, (__nv_bfloat16*)vals, (const __nv_bfloat16*)kn,
        (const __nv_bfloat16*)vn, total, units, cap, D);
  else
    append_kernel<float><<<1, 256, 0, st>>>((float*)keys, (float*)vals, (const float*)kn,
                                            (const float*)vn, total, units, cap, D);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

}  // namespace ctkv
