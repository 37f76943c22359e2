// v6 decode: the per-(b,g) unit chain after the scan, on a 4-CTA cluster.
//
// After the scan kernel (ctkv_decode.cu) each unit is a dependency chain:
// top-C' slots -> first-occurrence union of their lists -> rerank logits of
// the recalled keys -> top-rho' -> attention over the selected V rows ->
// merge with the static partials.  On one SM every link is a latency-bound
// gather; here the four CTAs of a cluster split every link and exchange
// the small cross-CTA state through distributed shared memory:
//
//   1. every CTA: top-C' slots from the scan's chunk candidates
//      (ck/retrieval.py:144-154, ties -> smaller slot)
//   2. CTA r owns lists r, r+4, ...: loads them, marks a bitmap over token
//      ids; cluster barrier; an entry of list j survives iff no list j' < j
//      holds it (bits read from the owners' shared memory) -- the
//      np.unique(return_index) first-occurrence order of
//      ck/retrieval.py:156-162; per-list survivor counts are broadcast
//   3. the recall positions [0, L) are split evenly over the CTAs; each
//      pulls its slice's ids from the owners and gathers the K rows with
//      TMA bulk copies, then computes the gs-head rerank logits (f32 sums of
//      exact bf16 products per 8-element chunk, f64 across chunks, x 1/sqrt(d);
//      ck/retrieval.py:171-193) and the packed key (~f32(group max), pos)
//   4. every CTA pulls all L keys and radix-selects the rho'-th smallest:
//      the top-rho' set by (score desc, position asc) (ck/retrieval.py:210-216)
//   5. each CTA attends over its slice's selected tokens (V rows by TMA bulk
//      copy; f64 softmax statistics, f32 weighted sums; ck/retrieval.py:221-246)
//      and sends its partial (m, l, o) to CTA 0
//   6. CTA 0 merges the sparse partials with the static partials exactly
//      (ck/retrieval.py:275-284) and writes out / row_max / denom.
//
// The unit's keys and recall ids go to global memory for the deferred tail
// kernel (full order, FIFO DCU, ordered sparse ids, cursor advance --
// tail_wide_kernel in ctkv_unit_wide.cu), which runs on a side stream.
#include <cfloat>
#include <cmath>

#include <cooperative_groups.h>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_decode_dev.cuh"
#include "ctkv_internal.h"

namespace ctkv {

namespace cg = cooperative_groups;

// per-CTA phase timestamps (globaltimer, ns), profiling only: [cta][mark]
constexpr int kCPhaseCtas = 512, kCPhases = 12;
__device__ unsigned long long g_cphase[kCPhaseCtas][kCPhases];
__device__ int g_cphase_on;
__device__ __forceinline__ void cmark(int k) {
  if (g_cphase_on && threadIdx.x == 0 && blockIdx.x < kCPhaseCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cphase[blockIdx.x][k] = t;
  }
}

// generic-proxy accesses of shared memory before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

constexpr int kCL = 4;           // CTAs per unit (cluster size)
constexpr int kCT = 256;         // threads per CTA
constexpr int kCB = 256;         // rows per gather batch
constexpr int kCMaxGs = 8;       // query heads per kv head
constexpr int kCMaxLists = 8;    // c' <= 8
constexpr int kCMaxOwn = 32;     // list entries per thread held in registers

struct ChainSmem {
  unsigned char* rows;   // [kCB][D] gathered K (then V) rows; later the row-group sums
  uint32_t* bm;          // [nlo][words] bitmaps of this CTA's lists  } area A; CTA 0 reuses it
  int32_t* recl;         // [nlo][rho] this CTA's lists, survivors    } for the static partials
  uint64_t* keys;        // [lmax] packed keys of all recall positions
  int32_t* sid;          // [scap] ids of this CTA's slice
  double* slg;           // [gs][scap] rerank logits of the slice
  int32_t* spos;         // [scap] selected slice offsets, ascending
  float* wts;            // [gs][kCB] attention weights of a batch
  float* cpo;            // CTA 0: [kCL][gs][D] sparse partial sums from the cluster
  double* cpml;          // CTA 0: [2][kCL][gs] their (m, l)
  int* hist;             // [256]
  double* scratch;       // [128]
  size_t area_a;
};

__host__ __device__ inline int chain_nlo(int c_prime) { return (c_prime + kCL - 1) / kCL; }
__host__ __device__ inline int chain_scap(int lmax) { return (lmax + kCL - 1) / kCL + 1; }

__host__ __device__ inline size_t chain_layout(const DecodeParams& p, int D, int esize, ChainSmem* s,
                                               unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* ptr = base ? base + off : nullptr;
    off += align16(bytes);
    return ptr;
  };
  const int nlo = chain_nlo(p.c_prime);
  const int scap = chain_scap(p.lmax);
  const int lmax = p.lmax > 1 ? p.lmax : 1;
  const size_t a_lists = (size_t)nlo * p.bitmap_words * 4 + align16((size_t)nlo * p.rho * 4);
  const size_t a_static = (size_t)p.ns * p.gs * D * 4 + align16((size_t)2 * p.ns * p.gs * 8);
  ChainSmem t;
  t.area_a = a_lists > a_static ? a_lists : a_static;
  const size_t rows = (size_t)kCB * D * esize;
  const size_t red = (size_t)(kCT / (D / 4)) * p.gs * D * 4;
  t.rows = take(rows > red ? rows : red);
  unsigned char* a = take(t.area_a);
  t.bm = reinterpret_cast<uint32_t*>(a);
  t.recl = a ? reinterpret_cast<int32_t*>(a + align16((size_t)nlo * p.bitmap_words * 4)) : nullptr;
  t.keys = reinterpret_cast<uint64_t*>(take((size_t)lmax * 8));
  t.sid = reinterpret_cast<int32_t*>(take((size_t)scap * 4));
  t.slg = reinterpret_cast<double*>(take((size_t)p.gs * scap * 8));
  t.spos = reinterpret_cast<int32_t*>(take((size_t)scap * 4));
  t.wts = reinterpret_cast<float*>(take((size_t)p.gs * kCB * 4));
  t.cpo = reinterpret_cast<float*>(take((size_t)kCL * p.gs * D * 4));
  t.cpml = reinterpret_cast<double*>(take((size_t)2 * kCL * p.gs * 8));
  t.hist = reinterpret_cast<int*>(take(256 * 4));
  const int nscr = p.gs * (p.ns + kCL) > 128 ? p.gs * (p.ns + kCL) : 128;
  t.scratch = reinterpret_cast<double*>(take((size_t)nscr * 8));
  if (s) *s = t;
  return off;
}

// the R-th smallest of the unique keys key[0..L): on return every selected
// key satisfies (key >> st[1]) <= lim (st[0..1] = lim lo/hi word, shift)
__device__ void chain_threshold(const uint64_t* key, int L, int R, int* hist, int* st,
                                uint64_t* lim_out, int* shift_out) {
  uint64_t prefix = 0;
  int need = R, shift = 56;
  while (true) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    // warp-aggregated: the leading digits of similar scores coincide, so
    // per-key atomics would serialise on a few bins
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
            st[0] = b;
            st[1] = run;
            st[2] = hist[b];
            break;
          }
          run += hist[b];
        }
      }
    }
    __syncthreads();
    const int b = st[0], below = st[1], cnt = st[2];
    prefix |= (uint64_t)b << shift;
    need -= below;
    __syncthreads();
    if (cnt == need || shift == 0) break;
    shift -= 8;
  }
  *lim_out = prefix >> shift;
  *shift_out = shift;
}

template <typename T, int D>
__global__ void __cluster_dims__(kCL, 1, 1) __launch_bounds__(kCT, 1) chain_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  ChainSmem S;
  chain_layout(p, D, sizeof(T), &S, smem);
  const int u = blockIdx.x / kCL;
  const int bi = u / p.g, gi = u % p.g, gs = p.gs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int RB = D * int(sizeof(T));
  constexpr int CH = RB / 16;                 // 16-byte chunks per row
  const int64_t total = *p.total + (p.k_new != nullptr ? 1 : 0);
  const int scap = chain_scap(p.lmax);
  __shared__ __align__(16) T qs[kCMaxGs * D];
  __shared__ int32_t sel[kCMaxLists];
  __shared__ int lcnt[kCMaxLists];
  __shared__ int sbase[kCMaxLists + 1];
  __shared__ int s_state[4];
  __shared__ uint64_t bar_rows, bar_st;
  __shared__ double hm[kCMaxGs], hl[kCMaxGs];

  cmark(0);
  if (tid == 0) {
    bar_init(&bar_rows, 1);
    bar_init(&bar_st, 1);
  }
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  for (int i = tid; i < gs * D; i += kCT) qs[i] = q[i];

  // ---- 1. top-C' slots (every CTA) ------------------------------------------
  if (warp == 0) warp_top_slots(p, u, sel);

  // ---- 2. own lists: load, bitmap, first-occurrence test ----------------------
  const int nlo = chain_nlo(p.c_prime);
  const int nown = (p.c_prime - r + kCL - 1) / kCL;     // lists r, r + kCL, ... < c'
  const int per = (p.rho + kCT - 1) / kCT;              // entries per thread per list
  __syncthreads();                                      // sel, bar init
  cmark(1);
  // entry x of this thread: list slot x / per, position tid * per + x % per
  int ids[kCMaxOwn];
#pragma unroll
  for (int x = 0; x < kCMaxOwn; ++x) {
    ids[x] = kEmpty;
    const int sl = x / per, i = tid * per + x % per;
    if (sl < nown && i < p.rho) {
      int id = __ldg(p.lists + ((int64_t)u * p.C + sel[r + kCL * sl]) * p.rho + i);
      if (id != kEmpty && (id < 0 || id >= total)) { set_flag(p.flags, kFlagIdRange); id = kEmpty; }
      ids[x] = id;
    }
  }
  for (int i = tid; i < nlo * p.bitmap_words; i += kCT) S.bm[i] = 0u;
  __syncthreads();
#pragma unroll
  for (int x = 0; x < kCMaxOwn; ++x)
    if (ids[x] != kEmpty) atomicOr(&S.bm[(x / per) * p.bitmap_words + (ids[x] >> 5)], 1u << (ids[x] & 31));
  cl.sync();   // #1: every list's bitmap is complete
  cmark(2);
  // survivors, compacted in position order per list
  for (int sl = 0; sl < nown; ++sl) {
    const int j = r + kCL * sl;
    unsigned keepm = 0;
    int cnt = 0;
#pragma unroll
    for (int x = 0; x < kCMaxOwn; ++x) {
      if (x / per != sl) continue;
      const int id = ids[x];
      bool keep = id != kEmpty;
      for (int j2 = 0; keep && j2 < j; ++j2) {
        const uint32_t* obm = cl.map_shared_rank(S.bm, j2 % kCL) + (j2 / kCL) * p.bitmap_words;
        keep = !((obm[id >> 5] >> (id & 31)) & 1u);
      }
      keepm |= (keep ? 1u : 0u) << x;
      cnt += keep;
    }
    int tot;
    int o = block_exclusive_scan(cnt, &tot, S.scratch);
#pragma unroll
    for (int x = 0; x < kCMaxOwn; ++x)
      if ((keepm >> x) & 1u) S.recl[sl * p.rho + o++] = ids[x];
    if (tid < kCL) {
      int* peer = cl.map_shared_rank(lcnt, tid);
      peer[j] = tot;
    }
  }
  cl.sync();   // #2: survivor counts everywhere, survivors compacted
  cmark(3);

  if (tid == 0) {
    sbase[0] = 0;
    for (int j = 0; j < kCMaxLists; ++j) sbase[j + 1] = sbase[j] + (j < p.c_prime ? lcnt[j] : 0);
  }
  __syncthreads();
  const int L = sbase[kCMaxLists];
  const int lo = (int)((int64_t)r * L / kCL), hi = (int)((int64_t)(r + 1) * L / kCL);
  const int n_sl = hi - lo;
  int32_t* recg = p.recg + (int64_t)u * p.lmax;
  uint64_t* kg = p.keyg + (int64_t)u * p.lmax;
  for (int i = tid; i < n_sl; i += kCT) {
    const int pos = lo + i;
    int j = 0;
    while (j + 1 < p.c_prime && pos >= sbase[j + 1]) ++j;
    const int32_t* orecl = cl.map_shared_rank(S.recl, j % kCL);
    const int id = orecl[(j / kCL) * p.rho + (pos - sbase[j])];
    S.sid[i] = id;
    recg[pos] = id;
  }
  __syncthreads();

  cmark(4);
  // ---- 3. rerank logits of the slice ---------------------------------------------
  const double scale = 1.0 / sqrt((double)D);
  const T* keys_g = static_cast<const T*>(p.keys) + (int64_t)u * p.cap * D;
  T* rows = reinterpret_cast<T*>(S.rows);
  uint32_t ph = 0;
  for (int b0 = 0; b0 < n_sl; b0 += kCB) {
    const int n = min(kCB, n_sl - b0);
    if (tid == 0) bar_expect(&bar_rows, (uint32_t)(n * RB));
    fence_proxy_async();
    __syncthreads();
    if (tid < n) bulk_g2s(rows + (size_t)tid * D, keys_g + (int64_t)S.sid[b0 + tid] * D, RB, &bar_rows);
    bar_wait(&bar_rows, ph);
    ph ^= 1u;
    if (tid < n) {
      double acc[kCMaxGs];
#pragma unroll
      for (int hh = 0; hh < kCMaxGs; ++hh) acc[hh] = 0.0;
      const uint4* r4 = reinterpret_cast<const uint4*>(rows + (size_t)tid * D);
      const uint4* q4 = reinterpret_cast<const uint4*>(qs);
#pragma unroll 4
      for (int c = 0; c < CH; ++c) {
        const int cc = (c + tid) & (CH - 1);
        const uint4 x = r4[cc];
#pragma unroll
        for (int hh = 0; hh < kCMaxGs; ++hh)
          if (hh < gs) acc[hh] += (double)bf16x8_dot(q4[hh * CH + cc], x, 0.f);
      }
      double gmax = -INFINITY;
#pragma unroll
      for (int hh = 0; hh < kCMaxGs; ++hh)
        if (hh < gs) {
          const double a = acc[hh] * scale;
          S.slg[hh * scap + b0 + tid] = a;
          gmax = fmax(gmax, a);
        }
      const int pos = lo + b0 + tid;
      const uint64_t key = ((uint64_t)(~okey32((float)gmax)) << 32) | (uint32_t)pos;
      S.keys[pos] = key;
      kg[pos] = key;
    }
    __syncthreads();   // rows reused by the next batch
  }
  cl.sync();   // #3: every slice's keys are complete
  cmark(5);

  // CTA 0: prefetch the static partials into area A (its lists are dead)
  const int ns = p.ns;
  float* spo = reinterpret_cast<float*>(S.bm);
  double* spml = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(S.bm) +
                                           align16((size_t)ns * gs * D * 4));
  const int64_t pbase = (int64_t)u * ns;
  if (r == 0) {
    fence_proxy_async();
    if (tid == 0) {
      const uint32_t ob = (uint32_t)(ns * gs * D * 4);
      bar_expect(&bar_st, ob);
      bulk_g2s(spo, p.po + pbase * gs * D, ob, &bar_st);
    }
    for (int i = tid; i < ns * gs; i += kCT) {
      cp_async8(spml + i, p.pm + pbase * gs + i);
      cp_async8(spml + ns * gs + i, p.pl + pbase * gs + i);
    }
    cp_async_commit();
  }

  // ---- 4. top-rho' threshold over all L keys ----------------------------------------
  for (int pos = tid; pos < L; pos += kCT) {
    if (pos >= lo && pos < hi) continue;
    int o = 0;
    while ((int)((int64_t)(o + 1) * L / kCL) <= pos) ++o;
    S.keys[pos] = cl.map_shared_rank(S.keys, o)[pos];
  }
  __syncthreads();
  cmark(6);
  const int Rn = L > 0 ? (p.use_rerank ? min(p.rho_prime, L) : L) : 0;
  uint64_t lim = ~0ull;
  int shift = 0;
  if (Rn > 0 && Rn < L) chain_threshold(S.keys, L, Rn, S.hist, s_state, &lim, &shift);

  cmark(7);
  // ---- 5. attention over this slice's selected tokens --------------------------------
  // ordered compaction of the selected slice offsets
  {
    const int pt = (n_sl + kCT - 1) / kCT;
    int cnt = 0;
    for (int e = 0; e < pt; ++e) {
      const int i = tid * pt + e;
      cnt += (i < n_sl && (S.keys[lo + i] >> shift) <= lim);
    }
    int tot;
    int o = block_exclusive_scan(cnt, &tot, S.scratch);
    for (int e = 0; e < pt; ++e) {
      const int i = tid * pt + e;
      if (i < n_sl && (S.keys[lo + i] >> shift) <= lim) S.spos[o++] = i;
    }
    if (tid == 0) s_state[3] = tot;
    __syncthreads();
  }
  const int nsel = s_state[3];
  // per-head max of the selected logits
  {
    double m8[kCMaxGs];
#pragma unroll
    for (int hh = 0; hh < kCMaxGs; ++hh) m8[hh] = -INFINITY;
    for (int k = tid; k < nsel; k += kCT) {
      const int i = S.spos[k];
#pragma unroll
      for (int hh = 0; hh < kCMaxGs; ++hh)
        if (hh < gs) m8[hh] = fmax(m8[hh], S.slg[hh * scap + i]);
    }
#pragma unroll
    for (int hh = 0; hh < kCMaxGs; ++hh)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m8[hh] = fmax(m8[hh], __shfl_xor_sync(0xffffffffu, m8[hh], o));
    if (lane == 0)
#pragma unroll
      for (int hh = 0; hh < kCMaxGs; ++hh) S.scratch[warp * kCMaxGs + hh] = m8[hh];
    __syncthreads();
    if (tid < gs) {
      double m = -INFINITY;
      for (int w = 0; w < kCT / 32; ++w) m = fmax(m, S.scratch[w * kCMaxGs + tid]);
      hm[tid] = m;
      hl[tid] = 0.0;
    }
    __syncthreads();
  }
  constexpr int DQ = D / 4;              // 4-element column groups
  constexpr int RG = kCT / DQ;           // row groups
  const int dq = tid % DQ, rg = tid / DQ;
  float acc[kCMaxGs][4];
#pragma unroll
  for (int hh = 0; hh < kCMaxGs; ++hh)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[hh][e] = 0.f;
  const T* vals_g = static_cast<const T*>(p.values) + (int64_t)u * p.cap * D;
  double l8[kCMaxGs];
#pragma unroll
  for (int hh = 0; hh < kCMaxGs; ++hh) l8[hh] = 0.0;
  for (int b0 = 0; b0 < nsel; b0 += kCB) {
    const int n = min(kCB, nsel - b0);
    if (tid == 0) bar_expect(&bar_rows, (uint32_t)(n * RB));
    fence_proxy_async();
    __syncthreads();
    if (tid < n)
      bulk_g2s(rows + (size_t)tid * D, vals_g + (int64_t)S.sid[S.spos[b0 + tid]] * D, RB, &bar_rows);
    if (tid < n) {
      const int i = S.spos[b0 + tid];
#pragma unroll
      for (int hh = 0; hh < kCMaxGs; ++hh)
        if (hh < gs) {
          const double e = exp(S.slg[hh * scap + i] - hm[hh]);
          S.wts[hh * kCB + tid] = (float)e;
          l8[hh] += e;
        }
    }
    bar_wait(&bar_rows, ph);
    ph ^= 1u;
    __syncthreads();   // weights visible
    for (int k = rg; k < n; k += RG) {
      const uint2 raw = *reinterpret_cast<const uint2*>(rows + (size_t)k * D + 4 * dq);
      const float v0 = __uint_as_float(raw.x << 16), v1 = __uint_as_float(raw.x & 0xffff0000u);
      const float v2 = __uint_as_float(raw.y << 16), v3 = __uint_as_float(raw.y & 0xffff0000u);
#pragma unroll
      for (int hh = 0; hh < kCMaxGs; ++hh)
        if (hh < gs) {
          const float w = S.wts[hh * kCB + k];
          acc[hh][0] = fmaf(w, v0, acc[hh][0]);
          acc[hh][1] = fmaf(w, v1, acc[hh][1]);
          acc[hh][2] = fmaf(w, v2, acc[hh][2]);
          acc[hh][3] = fmaf(w, v3, acc[hh][3]);
        }
    }
    __syncthreads();   // rows and weights reused by the next batch
  }
  // l per head: block reduce
#pragma unroll
  for (int hh = 0; hh < kCMaxGs; ++hh)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l8[hh] += __shfl_xor_sync(0xffffffffu, l8[hh], o);
  if (lane == 0)
#pragma unroll
    for (int hh = 0; hh < kCMaxGs; ++hh) S.scratch[warp * kCMaxGs + hh] = l8[hh];
  // row-group partial sums -> rows area, then reduce over the row groups
  float* red = reinterpret_cast<float*>(S.rows);
#pragma unroll
  for (int hh = 0; hh < kCMaxGs; ++hh)
    if (hh < gs)
      *reinterpret_cast<float4*>(red + ((size_t)rg * gs + hh) * D + 4 * dq) =
          make_float4(acc[hh][0], acc[hh][1], acc[hh][2], acc[hh][3]);
  __syncthreads();
  float* cpo0 = cl.map_shared_rank(S.cpo, 0);
  double* cpml0 = cl.map_shared_rank(S.cpml, 0);
  for (int i = tid; i < gs * D; i += kCT) {
    float s = 0.f;
    for (int g2 = 0; g2 < RG; ++g2) s += red[(size_t)g2 * gs * D + i];
    cpo0[(size_t)r * gs * D + i] = s;
  }
  if (tid < gs) {
    double l = 0.0;
    for (int w = 0; w < kCT / 32; ++w) l += S.scratch[w * kCMaxGs + tid];
    cpml0[r * gs + tid] = nsel > 0 ? hm[tid] : -INFINITY;
    cpml0[kCL * gs + r * gs + tid] = nsel > 0 ? l : 0.0;
  }
  cmark(8);
  cl.sync();   // #4: all sparse partials are in CTA 0
  cmark(9);
  if (r != 0) return;

  // ---- 6. CTA 0: exact merge with the static partials ---------------------------------
  bar_wait(&bar_st, 0);
  cp_async_wait_all();
  __syncthreads();
  double* wj = S.scratch;   // [gs][ns + kCL] split weights
  const int nsp = ns + kCL;
  if (tid < gs) {
    const int hh = tid;
    double M = -INFINITY;
    for (int j = 0; j < ns; ++j)
      if (spml[ns * gs + j * gs + hh] > 0.0) M = fmax(M, spml[j * gs + hh]);
    for (int k = 0; k < kCL; ++k)
      if (S.cpml[kCL * gs + k * gs + hh] > 0.0) M = fmax(M, S.cpml[k * gs + hh]);
    double Ls = 0.0;
    for (int j = 0; j < ns; ++j) {
      const double lj = spml[ns * gs + j * gs + hh];
      const double w = lj > 0.0 ? exp(spml[j * gs + hh] - M) : 0.0;
      wj[hh * nsp + j] = w;
      Ls += w * lj;
    }
    for (int k = 0; k < kCL; ++k) {
      const double lk = S.cpml[kCL * gs + k * gs + hh];
      const double w = lk > 0.0 ? exp(S.cpml[k * gs + hh] - M) : 0.0;
      wj[hh * nsp + ns + k] = w;
      Ls += w * lk;
    }
    hm[hh] = M;
    hl[hh] = Ls;
  }
  __syncthreads();
  bool none = false;
  for (int i = tid; i < gs * D; i += kCT) {
    const int hh = i / D, e = i % D;
    const double* wh = wj + hh * nsp;
    double O = 0.0;
    for (int j = 0; j < ns; ++j) O += wh[j] * (double)spo[(j * gs + hh) * D + e];
    for (int k = 0; k < kCL; ++k) O += wh[ns + k] * (double)S.cpo[((size_t)k * gs + hh) * D + e];
    const double Ls = hl[hh];
    const int64_t oh = (int64_t)bi * p.h + gi * gs + hh;
    if (Ls > 0.0) {
      p.out[oh * D + e] = (float)(O / Ls);
    } else {
      p.out[oh * D + e] = 0.f;
      none = true;
    }
    if (e == 0) {
      if (p.row_max) p.row_max[oh] = hm[hh];
      if (p.denom) p.denom[oh] = Ls;
    }
  }
  if (none) set_flag(p.flags, kFlagNoTokens);
  if (tid == 0) {
    p.uctr[u * 4 + 2] = L;
    p.uctr[u * 4 + 3] = Rn;
    if (p.recall_len) p.recall_len[u] = L;
    if (p.sparse_len) p.sparse_len[u] = Rn;
    set_flag(p.flags, L > 0 ? kFlagNonEmptyRecall : kFlagEmptyRecall);
  }
  if (p.selected)
    for (int k = tid; k < p.c_prime; k += kCT) p.selected[(int64_t)u * p.c_prime + k] = sel[k];
  cmark(10);
}

// ------------------------------------------------------------------------
// launcher
// ------------------------------------------------------------------------

template <typename T, int D>
static int launch_chain_t(const DecodeParams& p, cudaStream_t st) {
  const size_t sm = chain_layout(p, D, sizeof(T), nullptr, nullptr);
  auto k = chain_kernel<T, D>;
  static size_t configured = 0;
  if (sm > configured) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))
      return CTKV_ECUDA;
    configured = sm;
  }
  k<<<p.U * kCL, kCT, sm, st>>>(p);
  return cudaGetLastError() == cudaSuccess ? CTKV_OK : CTKV_ECUDA;
}

int chain_phase_timing(int on, unsigned long long* out, int n) {
  if (out != nullptr) {
    const int m = n < kCPhaseCtas * kCPhases ? n : kCPhaseCtas * kCPhases;
    if (cudaMemcpyFromSymbol(out, g_cphase, sizeof(unsigned long long) * m) != cudaSuccess)
      return CTKV_ECUDA;
  }
  if (on >= 0 && cudaMemcpyToSymbol(g_cphase_on, &on, sizeof(int)) != cudaSuccess) return CTKV_ECUDA;
  return CTKV_OK;
}

bool chain_supported(const DecodeParams& p, int dtype, int D) {
  if (dtype != CTKV_BF16 || (D != 64 && D != 128)) return false;
  if (p.gs > kCMaxGs || p.c_prime > kCMaxLists) return false;
  const int per = (p.rho + kCT - 1) / kCT;
  if (chain_nlo(p.c_prime) * per > kCMaxOwn) return false;
  return chain_layout(p, D, 2, nullptr, nullptr) <= 220 * 1024;
}

int launch_chain(const DecodeParams& p, int dtype, int D, cudaStream_t st) {
  if (dtype != CTKV_BF16) return CTKV_ECONFIG;
  if (D == 128) return launch_chain_t<__nv_bfloat16, 128>(p, st);
  if (D == 64) return launch_chain_t<__nv_bfloat16, 64>(p, st);
  return CTKV_ESHAPE;
}

}  // namespace ctkv
