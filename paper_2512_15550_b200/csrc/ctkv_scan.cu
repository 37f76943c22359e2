// v6 scan: a persistent, warp-specialised streaming kernel for the
// bandwidth-bound half of a decode layer (bf16 stores).
//
// Work items ("tasks"), handed out dynamically with one atomic counter so
// that concurrently running launches (the engine's micro-batch lanes) and
// late-starting CTAs balance themselves:
//   cos(u, chunk)   64 centroids x gs query heads of unit u = 64 KB of rows:
//                   cosine q.c / (|q||c|) per (head, centroid), clipped, then
//                   the GQA group max (ck/tensor_ops.py:190-207,
//                   ck/retrieval.py:144-145) -> gcos[u][c] (f64)
//   static(u, s)    128 static tokens (K and V, 64 KB) of unit u: split-K
//                   attention partial (m, l, o) over the static partition
//                   (ck/retrieval.py:341-344, ck/store.py:94-96)
// Cosine tasks come first (in unit order), static tasks after them.
//
// Roles: warp 0 is the producer -- lane 0 claims a task, waits for a free
// stage and issues TMA bulk copies (rows, the unit's query heads, the cached
// centroid norms); lanes 1..gs compute the exact f64 query norms of the
// task's heads into the stage header.  Warps 1..8 consume: a cosine task
// needs no block barrier (thread = (centroid, head), group max by
// shuffles); every consumer warp releases the stage on its own
// (the chain kernel selects each unit's top-C' slots from gcos).  Static
// tasks use a named barrier among the consumers.
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_decode_dev.cuh"
#include "ctkv_internal.h"

namespace ctkv {

// per-CTA task timeline (globaltimer, ns), profiling only
constexpr int kS4TlCtas = 160, kS4TlSlots = 64;
__device__ unsigned long long g_s4tl[kS4TlCtas][kS4TlSlots];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kS4Stages = 3;
constexpr int kS4Cons = 512;                     // consumer threads (16 warps)
constexpr int kS4Threads = 32 + kS4Cons;
constexpr int kS4Rows = 256;                     // rows per cosine task
constexpr int kS4Tok = 128;                      // static tokens per task
constexpr int kS4Data = 64 * 1024;               // row bytes per stage
constexpr int kS4Q = 2048;                       // query heads (gs <= 8, d <= 128 bf16)
constexpr int kS4Cn = 1024;                      // cached norms [gs][CC] f32
constexpr int kS4Hdr = 128;                      // task id + f64 query norms
constexpr int kS4Stage = kS4Data + kS4Q + kS4Cn + kS4Hdr;

__device__ __forceinline__ void s4_cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kS4Cons) : "memory");
}
__device__ __forceinline__ void s4_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(bar)) : "memory");
}

struct S4Hdr {
  int task;
  int pad;
  double qn[8];
};

template <int D>
__device__ void s4_issue(const DecodeParams& p, int task, int ncos, int64_t t0, int64_t total,
                         unsigned char* stage, uint64_t* full) {
  using T = __nv_bfloat16;
  constexpr int RB = D * 2;
  const int gs = p.gs;
  unsigned char* qdst = stage + kS4Data;
  const T* qsrc;
  if (task < ncos) {
    const int CC = kS4Rows / gs, cpu = p.cos_blocks_per_unit;
    const int u = task / cpu, chunk = task % cpu;
    const int bi = u / p.g, gi = u % p.g;
    const int c0 = chunk * CC, nc = min(CC, p.C - c0);
    const bool cn = p.cnorm != nullptr && (p.C & 3) == 0 && (nc & 3) == 0;
    qsrc = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
    bar_expect(full, (uint32_t)(gs * nc * RB + gs * RB + (cn ? gs * nc * 4 : 0)));
    const T* cent = static_cast<const T*>(p.cent);
    for (int j = 0; j < gs; ++j) {
      const int64_t row0 = ((int64_t)bi * p.h + gi * gs + j) * p.C + c0;
      bulk_g2s(stage + (size_t)j * CC * RB, cent + row0 * D, (uint32_t)(nc * RB), full);
      if (cn) bulk_g2s(stage + kS4Data + kS4Q + j * CC * 4, p.cnorm + row0, (uint32_t)(nc * 4), full);
    }
  } else {
    const int st = task - ncos;
    const int u = st / p.ns, split = st % p.ns;
    const int bi = u / p.g, gi = u % p.g;
    qsrc = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
    const StaticSpan span(total, p.init_len, p.local_len);
    const int64_t i0 = (int64_t)split * kS4Tok;
    const int nt = (int)max((int64_t)0, min((int64_t)kS4Tok, span.n_static - i0));
    bar_expect(full, (uint32_t)(2 * nt * RB + gs * RB));
    const T* keys = static_cast<const T*>(p.keys) + (int64_t)u * p.cap * D;
    const T* vals = static_cast<const T*>(p.values) + (int64_t)u * p.cap * D;
    unsigned char* Ks = stage;
    unsigned char* Vs = stage + (size_t)kS4Tok * RB;
    int64_t i = i0;
    const int64_t i1 = i0 + nt;
    while (i < i1) {
      const int64_t id = span.id(i);
      const int64_t run_end = (i < span.n_init) ? min(i1, span.n_init) : i1;
      int64_t n = run_end - i;
      // the token appended by this step comes from the caller's buffer
      const bool has_new = p.k_new != nullptr && id <= t0 && t0 < id + n;
      if (has_new) n = t0 - id;
      if (n > 0) {
        bulk_g2s(Ks + (size_t)(i - i0) * RB, keys + id * D, (uint32_t)(n * RB), full);
        bulk_g2s(Vs + (size_t)(i - i0) * RB, vals + id * D, (uint32_t)(n * RB), full);
      }
      if (has_new) {
        const int64_t at = i + n - i0;
        bulk_g2s(Ks + (size_t)at * RB, static_cast<const T*>(p.k_new) + (int64_t)u * D, RB, full);
        bulk_g2s(Vs + (size_t)at * RB, static_cast<const T*>(p.v_new) + (int64_t)u * D, RB, full);
        n += 1;
      }
      i += n;
    }
  }
  bulk_g2s(qdst, qsrc, (uint32_t)(gs * RB), full);
}

// cosine task, one consumer thread per (centroid, head) row; no block barrier
template <int D>
__device__ void s4_cos(const DecodeParams& p, int task, const unsigned char* stage, uint64_t* empty) {
  using T = __nv_bfloat16;
  constexpr int RB = D * 2, CH = RB / 16;
  const int ct = threadIdx.x - 32, lane = threadIdx.x & 31;
  const int gs = p.gs, CC = kS4Rows / gs, cpu = p.cos_blocks_per_unit;
  const int u = task / cpu, chunk = task % cpu;
  const int c0 = chunk * CC, nc = min(CC, p.C - c0);
  // two threads per (centroid, head) row, each half of the chunks
  const int rowi = ct >> 1, half = ct & 1;
  const int c = rowi / gs, j = rowi % gs;
  const bool live = c < nc;
  const bool cn_bulk = p.cnorm != nullptr && (p.C & 3) == 0 && (nc & 3) == 0;
  // exact f64 |q_j|^2 (np.linalg.norm, ck/tensor_ops.py:199-200): the 32/gs
  // lanes of this warp that hold head j square a few chunks each, then a
  // butterfly over them -- no block barrier
  double qq = 0.0;
  {
    const uint4* qj = reinterpret_cast<const uint4*>(stage + kS4Data + (size_t)j * RB);
    const int nl = 32 / gs, sub = (lane / (2 * gs)) * 2 + half;
    for (int i = sub; i < CH; i += nl) {
      float f[8];
      unpack16<T>(qj[i], f);
#pragma unroll
      for (int x = 0; x < 8; ++x) qq = fma((double)f[x], (double)f[x], qq);
    }
    qq += __shfl_xor_sync(0xffffffffu, qq, 1);
    for (int o = 2 * gs; o < 32; o <<= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
  }
  double dot = 0.0, nrm = 0.0;
  if (live) {
    constexpr int HC = CH / 2;
    const uint4* r4 = reinterpret_cast<const uint4*>(stage + (size_t)(j * CC + c) * RB) + half * HC;
    const uint4* q4 = reinterpret_cast<const uint4*>(stage + kS4Data + (size_t)j * RB) + half * HC;
#pragma unroll
    for (int k = 0; k < HC; ++k) {
      const int kk = (k + rowi) & (HC - 1);
      const uint4 x = r4[kk];
      dot += (double)bf16x8_dot(q4[kk], x, 0.f);
      if (p.cnorm == nullptr) nrm += (double)bf16x8_dot(x, x, 0.f);
    }
  }
  dot += __shfl_xor_sync(0xffffffffu, dot, 1);
  if (p.cnorm == nullptr) nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
  double cv = -INFINITY;
  if (live) {
    double cn;
    if (p.cnorm == nullptr) {
      cn = sqrt(nrm);
    } else {
      const int bi = u / p.g, gi = u % p.g;
      cn = cn_bulk ? (double)reinterpret_cast<const float*>(stage + kS4Data + kS4Q)[j * CC + c]
                   : (double)__ldg(p.cnorm + ((int64_t)bi * p.h + gi * gs + j) * p.C + c0 + c);
    }
    const double den = sqrt(qq) * cn;
    if (den == 0.0) {
      cv = 0.0;
      if (half == 0) set_flag(p.flags, kFlagDegenerate);
    } else {
      cv = fmin(fmax(dot / den, -1.0), 1.0);
    }
  }
  __syncwarp();
  if (lane == 0) s4_arrive(empty);   // this warp is done with the stage
  // GQA group max over the gs heads of a centroid (adjacent lane pairs)
  for (int o = 2; o < 2 * gs; o <<= 1) cv = fmax(cv, __shfl_xor_sync(0xffffffffu, cv, o));
  if (j == 0 && half == 0 && live) p.gcos[(int64_t)u * p.C + c0 + c] = cv;
}

// static-attention task over up to 128 tokens (named barrier among consumers)
template <int D>
__device__ void s4_static(const DecodeParams& p, int st, int64_t total, const unsigned char* stage,
                          double* lg, float* w, double* ml) {
  using T = __nv_bfloat16;
  constexpr int RB = D * 2;
  const int ct = threadIdx.x - 32;
  const int gs = p.gs;
  const int u = st / p.ns, split = st % p.ns;
  const StaticSpan span(total, p.init_len, p.local_len);
  const int64_t i0 = (int64_t)split * kS4Tok;
  const int nt = (int)max((int64_t)0, min((int64_t)kS4Tok, span.n_static - i0));
  const int64_t slot = (int64_t)u * p.ns + split;
  double* pm = p.pm + slot * gs;
  double* pl = p.pl + slot * gs;
  float* po = p.po + slot * gs * D;
  if (nt == 0) {
    for (int i = ct; i < gs * D; i += kS4Cons) po[i] = 0.f;
    if (ct < gs) { pm[ct] = -INFINITY; pl[ct] = 0.0; }
    return;
  }
  const T* Ks = reinterpret_cast<const T*>(stage);
  const T* Vs = reinterpret_cast<const T*>(stage + (size_t)kS4Tok * RB);
  const uint4* q4 = reinterpret_cast<const uint4*>(stage + kS4Data);
  constexpr int CH = RB / 16;
  const double scale = 1.0 / sqrt((double)D);
  for (int pr = ct; pr < nt * gs; pr += kS4Cons) {
    const int t = pr % nt, j = pr / nt;
    const uint4* r4 = reinterpret_cast<const uint4*>(Ks + (size_t)t * D);
    double dot = 0.0;
#pragma unroll 4
    for (int k = 0; k < CH; ++k) {
      const int kk = (k + t) & (CH - 1);
      dot += (double)bf16x8_dot(q4[j * CH + kk], r4[kk], 0.f);
    }
    lg[j * kS4Tok + t] = dot * scale;
  }
  s4_cons_sync();
  const int warp = ct >> 5, lane = ct & 31;
  for (int j = warp; j < gs; j += kS4Cons / 32) {
    double m = -INFINITY;
    for (int t = lane; t < nt; t += 32) m = fmax(m, lg[j * kS4Tok + t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double l = 0.0;
    for (int t = lane; t < nt; t += 32) {
      const double e = exp(lg[j * kS4Tok + t] - m);
      w[j * kS4Tok + t] = (float)e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) { ml[j] = m; ml[gs + j] = l; }
  }
  s4_cons_sync();
  for (int pr = ct; pr < gs * (D / 2); pr += kS4Cons) {
    const int j = pr / (D / 2), e = 2 * (pr % (D / 2));
    float a0 = 0.f, a1 = 0.f;
    const float* wj = w + j * kS4Tok;
    for (int t = 0; t < nt; ++t) {
      const uint32_t v2 = *reinterpret_cast<const uint32_t*>(Vs + (size_t)t * D + e);
      a0 = fmaf(wj[t], __uint_as_float(v2 << 16), a0);
      a1 = fmaf(wj[t], __uint_as_float(v2 & 0xffff0000u), a1);
    }
    po[j * D + e] = a0;
    po[j * D + e + 1] = a1;
  }
  if (ct < gs) {
    pm[ct] = ml[ct];
    pl[ct] = ml[gs + ct];
  }
}

template <int D>
__global__ void __launch_bounds__(kS4Threads, 1) scan4_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[kS4Stages], empty[kS4Stages];
  const int64_t t0 = *p.total;
  const bool appending = p.k_new != nullptr;
  const int64_t total = t0 + (appending ? 1 : 0);
  const int ncos = p.U * p.cos_blocks_per_unit;
  const int ntasks = ncos + p.U * p.ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* scratch = smem + (size_t)kS4Stages * kS4Stage;
  if ((p.dbg & 4) && threadIdx.x == 0 && blockIdx.x < kS4TlCtas) g_s4tl[blockIdx.x][0] = gtimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS4Stages; ++s) {
      bar_init(&full[s], 1);                // producer lane 0 (+tx)
      bar_init(&empty[s], kS4Cons / 32);    // one arrival per consumer warp
    }
  }
  __syncthreads();
  if (warp == 0) {
    // ---- producer -------------------------------------------------------
    if (lane == 0) {
      // static round-robin assignment (a contended per-task atomic claim
      // costs more than the imbalance it would remove)
      int next = blockIdx.x;
      for (int k = 0;; ++k) {
        const int stage = k % kS4Stages;
        const uint32_t ph = (uint32_t)(k / kS4Stages) & 1u;
        unsigned char* st = smem + (size_t)stage * kS4Stage;
        S4Hdr* hdr = reinterpret_cast<S4Hdr*>(st + kS4Data + kS4Q + kS4Cn);
        const int task = next;
        bar_wait(&empty[stage], ph ^ 1u);
        hdr->task = task;
        if (task >= ntasks) {
          s4_arrive(&full[stage]);   // sentinel: no tx
          break;
        }
        s4_issue<D>(p, task, ncos, t0, total, st, &full[stage]);
        next += gridDim.x;
      }
    }
  } else {
    // ---- consumers ------------------------------------------------------
    if (appending && blockIdx.x == gridDim.x - 1) {   // the step's KV append (16-byte rows pieces)
      constexpr int V = D * 2 / 16;
      uint4* keys = static_cast<uint4*>(const_cast<void*>(p.keys));
      uint4* vals = static_cast<uint4*>(const_cast<void*>(p.values));
      const uint4* kn = static_cast<const uint4*>(p.k_new);
      const uint4* vn = static_cast<const uint4*>(p.v_new);
      for (int i = threadIdx.x - 32; i < p.U * V; i += kS4Cons) {
        const int64_t uu = i / V, e = i % V;
        keys[(uu * p.cap + t0) * V + e] = kn[i];
        vals[(uu * p.cap + t0) * V + e] = vn[i];
      }
    }
    double* lg = reinterpret_cast<double*>(scratch);          // [8][kS4Tok]
    float* w = reinterpret_cast<float*>(lg + 8 * kS4Tok);     // [8][kS4Tok]
    double* ml = reinterpret_cast<double*>(w + 8 * kS4Tok);   // [2][8]
    for (int k = 0;; ++k) {
      const int stage = k % kS4Stages;
      const uint32_t ph = (uint32_t)(k / kS4Stages) & 1u;
      bar_wait(&full[stage], ph);
      const unsigned char* st = smem + (size_t)stage * kS4Stage;
      const S4Hdr* hdr = reinterpret_cast<const S4Hdr*>(st + kS4Data + kS4Q + kS4Cn);
      const int task = hdr->task;
      if ((p.dbg & 4) && threadIdx.x == 32 && blockIdx.x < kS4TlCtas && 2 + k < kS4TlSlots)
        g_s4tl[blockIdx.x][2 + k] = gtimer();
      if (task >= ntasks) break;
      if (task < ncos) {
        s4_cos<D>(p, task, st, &empty[stage]);
      } else {
        s4_static<D>(p, task - ncos, total, st, lg, w, ml);
        s4_cons_sync();   // every consumer is done with the stage and the scratch
        if (lane == 0) s4_arrive(&empty[stage]);
      }
    }
  }
  if ((p.dbg & 4) && threadIdx.x == 32 && blockIdx.x < kS4TlCtas) g_s4tl[blockIdx.x][1] = gtimer();
}

int scan4_timeline(int on, unsigned long long* out, int n) {
  if (out != nullptr) {
    const int m = n < kS4TlCtas * kS4TlSlots ? n : kS4TlCtas * kS4TlSlots;
    if (cudaMemcpyFromSymbol(out, g_s4tl, sizeof(unsigned long long) * m) != cudaSuccess) return CTKV_ECUDA;
  }
  if (on >= 0) set_host_dbg(4, on);
  return CTKV_OK;
}

static size_t scan4_smem() {
  return (size_t)kS4Stages * kS4Stage + sizeof(double) * 8 * kS4Tok + sizeof(float) * 8 * kS4Tok +
         sizeof(double) * 16;
}

bool scan4_supported(const DecodeParams& p, int dtype, int D) {
  if (dtype != CTKV_BF16 || (D != 64 && D != 128)) return false;
  if (p.gs != 1 && p.gs != 2 && p.gs != 4 && p.gs != 8) return false;
  return p.c_prime <= 8 && p.total != nullptr &&
         p.ns * kS4Tok >= 0;
}

template <int D>
static int launch_scan4_t(const DecodeParams& p0, cudaStream_t st) {
  DecodeParams p = p0;
  p.dbg = g_host_dbg;
  const size_t sm = scan4_smem();
  auto k = scan4_kernel<D>;
  static bool set = false;
  if (!set) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))
      return CTKV_ECUDA;
    set = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntasks = p.U * p.cos_blocks_per_unit + p.U * p.ns;
  const int grid = ntasks < sms ? ntasks : sms;
  if (grid > 0) k<<<grid, kS4Threads, sm, st>>>(p);
  return cudaGetLastError() == cudaSuccess ? CTKV_OK : CTKV_ECUDA;
}

int launch_scan4(const DecodeParams& p, int dtype, int D, cudaStream_t st) {
  if (dtype != CTKV_BF16) return CTKV_ECONFIG;
  if (D == 128) return launch_scan4_t<128>(p, st);
  if (D == 64) return launch_scan4_t<64>(p, st);
  return CTKV_ESHAPE;
}

}  // namespace ctkv
