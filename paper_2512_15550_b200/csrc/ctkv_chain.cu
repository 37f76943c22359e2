// v6 decode: the per-(b,g) unit chain after the scan, on a CL-CTA cluster.
//
// After the scan kernel (ctkv_decode.cu) each unit is a dependency chain:
// top-C' slots -> first-occurrence union of their lists -> rerank logits of
// the recalled keys -> top-rho' -> attention over the selected V rows ->
// merge with the static partials.  Its gathers are random 256-byte rows,
// which one SM pulls at only ~27 GB/s (measured, scripts/micro), so the CL
// CTAs of a cluster split every gather and exchange the small cross-CTA
// state through distributed shared memory.  Each CTA is small (~64 KB of
// shared memory, <= 80 registers) so three fit an SM next to other work:
// the engine's micro-batch lanes overlap one lane's chains with another
// lane's bandwidth-bound scan.
//
//   1. the scan's last cosine CTA of the unit already wrote its top-C'
//      slots (ck/retrieval.py:144-154, ties -> smaller slot)
//   2. CTA r owns lists r, r+CL, ...: loads them, marks a bitmap over token
//      ids; cluster barrier; an entry of list j survives iff no list j' < j
//      holds it (bits read from the owners' shared memory) -- the
//      np.unique(return_index) first-occurrence order of
//      ck/retrieval.py:156-162; per-list survivor counts are broadcast
//   3. the recall positions [0, L) are split evenly over the CTAs; each
//      pulls its slice's ids from the owners and gathers the K rows into
//      registers (8 lanes x 32 B per row, 128 rows in flight), computing the
//      gs-head rerank logits (f32 sums of exact bf16 products per 8-element
//      chunk, f64 across chunks, x 1/sqrt(d); ck/retrieval.py:171-193)
//   4. every CTA pulls all L score keys and radix-selects the top-rho' set
//      by (score desc, position asc) (ck/retrieval.py:210-216)
//   5. the selected tokens, in position order, are split evenly over the
//      CTAs; each gathers its V rows into registers and accumulates an
//      online-softmax partial (f64 statistics, f32 weighted sums;
//      ck/retrieval.py:221-246) that goes to CTA 0
//   6. CTA 0 merges the sparse partials with the static partials exactly
//      (ck/retrieval.py:275-284) and writes out / row_max / denom.
//
// The unit's keys and recall ids go to global memory for the deferred tail
// kernel (full order, FIFO DCU, ordered sparse ids, cursor advance --
// tail_kernel in ctkv_tail.cu), which runs on a side stream.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_decode_dev.cuh"
#include "ctkv_internal.h"

namespace ctkv {

namespace cg = cooperative_groups;

// per-CTA phase timestamps (globaltimer, ns), profiling only: [cta][mark]
constexpr int kCPhaseCtas = 512, kCPhases = 16;
__device__ unsigned long long g_cphase[kCPhaseCtas][kCPhases];
__device__ __forceinline__ void cmark(const DecodeParams& p, int k) {
#ifdef CTKV_PROFILE
  if ((p.dbg & 2) && threadIdx.x == 0 && blockIdx.x < kCPhaseCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cphase[blockIdx.x][k] = t;
  }
#endif
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ uint32_t dsmem_addr(const void* ptr, int rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(sa(ptr)), "r"(rank));
  return a;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// f64 exp out of line: one copy of its ~200 instructions per kernel
__device__ __noinline__ double dexp(double x) { return exp(x); }
__device__ __forceinline__ double warp_max_f64(double m) {
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}
__device__ __forceinline__ double warp_sum_f64(double m) {
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  return m;
}

constexpr int kCT = 256;         // threads per CTA
constexpr int kCW = kCT / 32;
constexpr int kCB = 128;         // selected rows per attention batch
constexpr int kCMaxLists = 8;    // c' <= 8
constexpr int kCMaxPer = 32;     // list entries per thread (keep mask bits)
constexpr int kVUn = 8;          // V-row passes in flight per warp (2 rows each; gs <= 4)
constexpr int kCBins = 1024;     // top-rho' selection: histogram bins
constexpr int kCBnd = 256;       // ... and keys ranked exactly in the boundary bin
constexpr int kRedHeads = 4;     // heads per pass of the cross-warp V-sum reduction

struct ChainSmem {
  uint32_t* bm;          // [words] OR of the lists before an owned one } area A; CTA 0
  int32_t* recl;         // [nlo][rho] this CTA's lists, survivors     } later: static partials
  float* spo;            // CTA 0, after the union: [ns][gs][D] static o
  double* spml;          //                          [2][ns][gs] static (m, l)
  uint32_t* keys;        // [lmax] score keys ~f32(group max) by position } area B: later the
  float* red;            // [kCW][gs][D] per-warp partial sums           } per-warp V sums
  int32_t* sid;          // [scap] ids of this CTA's slice
  int32_t* spos;         // [scap] this CTA's selected positions, in position order
  int32_t* vid;          // [kCB] ids of an attention batch
  float* wts;            // [gs][kCB] weights of an attention batch
  double* lgs;           // [gs][kCB] logits / f64 weights of an attention batch
  float* cpo;            // CTA 0: [CL][gs][D] sparse partial sums from the cluster
  double* cpml;          // CTA 0: [2][CL][gs] their (m, l)
  int* hist;             // [kCBins] selection histogram
  double* scratch;       // [max(128, gs * (ns + CL))]
};

__host__ __device__ inline int chain_nlo(int c_prime, int CL) { return (c_prime + CL - 1) / CL; }
__host__ __device__ inline int chain_scap(int lmax, int CL) { return (lmax + CL - 1) / CL + 1; }

__host__ __device__ inline size_t chain_layout(const DecodeParams& p, int D, int CL, ChainSmem* s,
                                               unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* ptr = base ? base + off : nullptr;
    off += align16(bytes);
    return ptr;
  };
  const int nlo = chain_nlo(p.c_prime, CL);
  const int scap = chain_scap(p.lmax, CL);
  const int lmax = p.lmax > 1 ? p.lmax : 1;
  const size_t bm_b = align16((size_t)p.bitmap_words * 4);   // one OR-bitmap
  const size_t a_lists = bm_b + align16((size_t)nlo * p.rho * 4);
  const size_t spo_b = align16((size_t)p.ns * p.gs * D * 4);
  const size_t a_static = spo_b + align16((size_t)2 * p.ns * p.gs * 8);
  // per-warp V sums of at most kRedHeads heads at a time (gs = 8 reduces in
  // two passes, so the chain stays at two CTAs per SM)
  const size_t keys_b = (size_t)lmax * 4, red_b = (size_t)kCW * min(p.gs, kRedHeads) * D * 4;
  ChainSmem t;
  unsigned char* a = take(a_lists > a_static ? a_lists : a_static);
  t.bm = reinterpret_cast<uint32_t*>(a);
  t.recl = a ? reinterpret_cast<int32_t*>(a + bm_b) : nullptr;
  t.spo = reinterpret_cast<float*>(a);
  t.spml = a ? reinterpret_cast<double*>(a + spo_b) : nullptr;
  unsigned char* b = take(keys_b > red_b ? keys_b : red_b);
  t.keys = reinterpret_cast<uint32_t*>(b);
  t.red = reinterpret_cast<float*>(b);
  t.sid = reinterpret_cast<int32_t*>(take((size_t)scap * 4));
  t.spos = reinterpret_cast<int32_t*>(take((size_t)(scap > 2 * kCBnd ? scap : 2 * kCBnd) * 4));
  t.vid = reinterpret_cast<int32_t*>(take((size_t)kCB * 4));
  t.wts = reinterpret_cast<float*>(take((size_t)p.gs * kCB * 4));
  t.lgs = reinterpret_cast<double*>(take((size_t)p.gs * kCB * 8));
  t.cpo = reinterpret_cast<float*>(take((size_t)CL * p.gs * D * 4));
  t.cpml = reinterpret_cast<double*>(take((size_t)2 * CL * p.gs * 8));
  t.hist = reinterpret_cast<int*>(take(kCBins * 4));
  const int nscr = p.gs * (p.ns + CL) > 128 ? p.gs * (p.ns + CL) : 128;
  t.scratch = reinterpret_cast<double*>(take((size_t)nscr * 8));
  if (s) *s = t;
  return off;
}

// Boundary of the R smallest 64-bit keys (key[i] << 32 | i), i < L, i.e. the
// top-R by (score desc, position asc): returns v and need such that the
// selected positions are {i : key[i] < v} plus the first `need` positions
// (in position order) with key[i] == v.  Radix over the 32-bit score keys,
// warp-aggregated histogram (similar scores share leading digits).
__device__ void chain_boundary(const uint32_t* key, int L, int R, int* hist, int* st, uint32_t* v_out,
                               int* need_out) {
  uint32_t prefix = 0;
  int need = R;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i0 = threadIdx.x & ~31; i0 < L; i0 += blockDim.x) {
      const int i = i0 + (threadIdx.x & 31);
      const uint32_t k = i < L ? key[i] : 0u;
      const bool in = i < L && (shift == 24 || ((k ^ prefix) >> (shift + 8)) == 0);
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
            break;
          }
          run += hist[b];
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)st[0] << shift;
    need -= st[1];
    __syncthreads();
  }
  *v_out = prefix;
  *need_out = need;
}

// Boundary (vk, vpos) of the top-R of L packed keys (key[i] << 32 | i):
// selected(i) <=> key[i] < vk || (key[i] == vk && i <= vpos).  One histogram
// pass over [min, max] of the keys (1024 linear bins), then an exact rank
// of the few keys in the boundary bin; degenerate distributions (more than
// kCBnd keys in that bin) fall back to the 8-bit radix passes.
// `mn`/`mx` are the keys' min and max and `hist` is zeroed (the chain
// gathers both while the keys are produced).
__device__ void chain_select(const uint32_t* key, int L, int R, uint32_t mn, uint32_t mx, int* hist,
                             uint64_t* bnd, int* st, uint32_t* red, uint32_t* vk_out, int* vpos_out) {
  const int tid = threadIdx.x;
  if (mn == mx) {   // all scores equal: the first R positions
    *vk_out = mn;
    *vpos_out = R - 1;
    return;
  }
  // monotone bin map (the same float expression in both passes)
  const float fscale = (float)kCBins / ((float)(mx - mn) + 1.0f);
  auto bin_of = [&](uint32_t k) { return min(kCBins - 1, (int)((float)(k - mn) * fscale)); };
  for (int i = tid; i < L; i += blockDim.x) atomicAdd(&hist[bin_of(key[i])], 1);
  __syncthreads();
  // boundary bin: the first whose cumulative count reaches R
  constexpr int BPT = kCBins / 256;
  int loc = 0;
  for (int b = 0; b < BPT && tid < 256; ++b) loc += hist[tid * BPT + b];
  int tot;
  int run = block_exclusive_scan(tid < 256 ? loc : 0, &tot, reinterpret_cast<double*>(red));
  if (tid < 256 && run < R && run + loc >= R) {
    for (int b = tid * BPT;; ++b) {
      if (run + hist[b] >= R) { st[0] = b; st[1] = run; break; }
      run += hist[b];
    }
  }
  if (tid == 0) st[2] = 0;
  __syncthreads();
  const int bb = st[0], below = st[1];
  if (hist[bb] > kCBnd) {   // degenerate: radix passes over the raw keys
    uint32_t vb;
    int need;
    chain_boundary(key, L, R, hist, st, &vb, &need);
    // the need-th key equal to vb in position order: per-thread counts over
    // contiguous chunks, an exclusive scan, then the owning thread walks its
    // chunk (a single-thread walk over L cost up to ~25 us at large L)
    const int pt = (L + (int)blockDim.x - 1) / (int)blockDim.x;
    int c = 0;
    for (int e = 0; e < pt; ++e) {
      const int i = tid * pt + e;
      c += (i < L && key[i] == vb) ? 1 : 0;
    }
    int tot;
    const int before = block_exclusive_scan(c, &tot, reinterpret_cast<double*>(red));
    if (before < need && before + c >= need) {
      int cc = before;
      for (int e = 0; e < pt; ++e) {
        const int i = tid * pt + e;
        if (i < L && key[i] == vb && ++cc == need) { st[3] = i; break; }
      }
    }
    __syncthreads();
    *vk_out = vb;
    *vpos_out = st[3];
    return;
  }
  for (int i = tid; i < L; i += blockDim.x) {
    const uint32_t k = key[i];
    if (bin_of(k) == bb) bnd[atomicAdd(&st[2], 1)] = ((uint64_t)k << 32) | (uint32_t)i;
  }
  __syncthreads();
  const int nb = st[2], need = R - below;   // 1 <= need <= nb
  for (int t = tid; t < nb; t += blockDim.x) {
    const uint64_t me = bnd[t];
    int rank = 0;
    for (int x = 0; x < nb; ++x) rank += bnd[x] < me;
    if (rank == need - 1) { st[0] = (int)(me >> 32); st[1] = (int)(uint32_t)me; }
  }
  __syncthreads();
  *vk_out = (uint32_t)st[0];
  *vpos_out = st[1];
}

template <typename T, int D, int CL, int GS>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kCT, 2) chain_kernel(DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  ChainSmem S;
  chain_layout(p, D, CL, &S, smem);
  const int u = blockIdx.x / CL;
  const int bi = u / p.g, gi = u % p.g;
  constexpr int gs = GS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int CH = D * int(sizeof(T)) / 16;   // 16-byte chunks per row (16 at d=128)
  static_assert(CH == 16 || CH == 8, "d = 64 or 128 (bf16)");
  const int64_t total = *p.total + (p.k_new != nullptr ? 1 : 0);
  const int ns = p.ns;
  __shared__ __align__(16) T qs[GS * D];
  __shared__ int32_t sel[kCMaxLists];
  __shared__ int lcnt[kCMaxLists];
  __shared__ int sbase[kCMaxLists + 1];
  __shared__ int s_state[4];
  __shared__ uint32_t s_kmm[2];   // min / max of all L score keys (every cluster CTA)
  __shared__ double hm[GS], hl[GS], hnew[GS], hresc[GS];

  cmark(p, 0);
  // #0 (split): every CTA of the cluster has started before any DSMEM access
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  ktl_mark(p.tl, 1, false);
  ktl_mark(p.tl, 3, true);   // the last CTA start (slot 3 end = max start)
  pdl_wait();      // the scan's outputs (gcos / slots, static partials) are complete
  const T* q = static_cast<const T*>(p.q) + ((int64_t)bi * p.h + (int64_t)gi * gs) * D;
  for (int i = tid; i < gs * D / 8; i += kCT)   // 16-byte pieces (q is 16-byte aligned: the scan bulk-copies it)
    reinterpret_cast<uint4*>(qs)[i] = __ldg(reinterpret_cast<const uint4*>(q) + i);
  if (tid < p.c_prime) sel[tid] = __ldcg(p.selg + (int64_t)u * p.c_prime + tid);
  __syncthreads();
  cmark(p, 1);

  // ---- 2. own lists: first-occurrence survivors ---------------------------------
  // CTA r owns lists j = r, r+CL, ...  An entry of list j survives iff no list
  // j' < j holds it (np.unique(return_index) order, ck/retrieval.py:156-162),
  // tested against a local bitmap that ORs lists 0..j-1.  Lists 0..jmax are
  // staged in area B by TMA bulk copies issued together (one L2/HBM round
  // trip however many lists precede the owned one).
  const int nown = (p.c_prime - r + CL - 1) / CL;      // lists r, r + CL, ... < c'
  const int jmax = r + CL * (nown - 1);                // last owned list
  int32_t* stage = reinterpret_cast<int32_t*>(S.keys);   // area B: [jmax + 1][rho] raw ids
  const int per = (p.rho + kCT - 1) / kCT;             // entries per thread per list
  auto list_row = [&](int j) { return p.lists + ((int64_t)u * p.C + sel[j]) * p.rho; };
  const bool bulk = (p.rho & 3) == 0 && (reinterpret_cast<uintptr_t>(p.lists) & 15) == 0;
  __shared__ __align__(8) uint64_t lbar;
  if (nown > 0) {
    if (bulk) {
      if (tid == 0) {
        bar_init(&lbar, 1);
        bar_expect(&lbar, (uint32_t)((jmax + 1) * p.rho * 4));
        for (int j = 0; j <= jmax; ++j) bulk_g2s(stage + j * p.rho, list_row(j), p.rho * 4, &lbar);
      }
    } else {
      for (int i = tid; i < (jmax + 1) * p.rho; i += kCT)
        stage[i] = __ldg(list_row(i / p.rho) + i % p.rho);
    }
  }
  for (int i = tid; i < p.bitmap_words; i += kCT) S.bm[i] = 0u;
  __syncthreads();   // barrier initialised, bitmap cleared (and the plain-load stage written)
  if (nown > 0 && bulk) bar_wait(&lbar, 0);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // #0: the survivor counts go remote below
  int jdone = 0;                                        // lists already in the bitmap
  for (int sl = 0; sl < nown; ++sl) {
    const int j = r + CL * sl;
    if (sl > 0) __syncthreads();                        // previous tests done
    for (; jdone < j; ++jdone) {                        // OR lists jdone .. j-1 into the bitmap
      const int32_t* row = stage + jdone * p.rho;
      for (int i = tid; i < p.rho; i += kCT) {
        const int v = row[i];
        if (v >= 0 && v < total) atomicOr(&S.bm[v >> 5], 1u << (v & 31));
      }
    }
    __syncthreads();
    const int32_t* rl = stage + j * p.rho;
    unsigned keepm = 0;
    int cnt = 0;
#pragma unroll 4
    for (int e = 0; e < per; ++e) {
      const int i = tid * per + e;
      int id = i < p.rho ? rl[i] : kEmpty;
      if (id != kEmpty && (id < 0 || id >= total)) { set_flag(p.flags, kFlagIdRange); id = kEmpty; }
      const bool keep = id != kEmpty && !((S.bm[id >> 5] >> (id & 31)) & 1u);
      keepm |= (keep ? 1u : 0u) << e;
      cnt += keep;
    }
    int tot;
    int o = block_exclusive_scan(cnt, &tot, S.scratch);
#pragma unroll 1
    for (int e = 0; e < per; ++e)
      if ((keepm >> e) & 1u) S.recl[sl * p.rho + o++] = rl[tid * per + e];
    if (tid < CL) cl.map_shared_rank(lcnt, tid)[j] = tot;
  }
  cmark(p, 2);
  if (tid == 0) { s_kmm[0] = 0xffffffffu; s_kmm[1] = 0u; }   // key min / max (filled remotely below)
  for (int b = tid; b < kCBins; b += kCT) S.hist[b] = 0;
  cl.sync();   // #2: survivor counts everywhere, survivors compacted
  cmark(p, 3);

  if (tid == 0) {
    sbase[0] = 0;
    for (int j = 0; j < kCMaxLists; ++j) sbase[j + 1] = sbase[j] + (j < p.c_prime ? lcnt[j] : 0);
  }
  __syncthreads();
  const int L = sbase[kCMaxLists];
  const int lo = (int)((int64_t)r * L / CL), hi = (int)((int64_t)(r + 1) * L / CL);
  const int n_sl = hi - lo;
  int32_t* recg = p.recg + (int64_t)u * p.lmax;
  uint64_t* kg = p.keyg + (int64_t)u * p.lmax;
  double* lgg = p.logits + (int64_t)u * gs * p.lmax;
  for (int i = tid; i < n_sl; i += kCT) {
    const int pos = lo + i;
    int j = 0;
    while (j + 1 < p.c_prime && pos >= sbase[j + 1]) ++j;
    const int id = cl.map_shared_rank(S.recl, j % CL)[(j / CL) * p.rho + (pos - sbase[j])];
    S.sid[i] = id;
    recg[pos] = id;
  }
  __syncthreads();
  cmark(p, 4);

  // ---- 3. rerank logits of the slice (K rows gathered into registers) ----------
  {
    // Tensor-core form: per warp, 16-row blocks of the slice as the A operand
    // of mma.m16n8k16 (bf16 products exact, f32 sum per 16-element k-step,
    // f64 across the k-steps), the gs query heads as the B columns.  The
    // order of near-equal scores can differ from the SIMT form's (both lie
    // well inside the north_star's 1e-6 tie window; tests/test_parity_gpu.py).  A lane
    // loads 16 B pieces of rows g and g+8; the dot product is invariant to
    // a common permutation of k, so each piece is used as the k-step
    // fragment as loaded and q is permuted the same way.
    const double scale = 1.0 / sqrt((double)D);
    const T* keys_g = static_cast<const T*>(p.keys) + (int64_t)u * p.cap * D;
    constexpr int KS2 = D / 32;            // 32-element k pairs per row
    constexpr int NB = GS >= 8 ? 1 : 2;    // 16-row blocks in flight per warp (1 at gs = 8: registers)
    const int g8 = lane >> 2, t4 = lane & 3;
    const T* qf_base = qs + (g8 < GS ? g8 : 0) * D + 8 * t4;   // B fragments re-read from smem per k-step
    uint32_t rkeys[CL > 1 ? CL - 1 : 1];   // shared::cluster addresses of the other CTAs' keys
#pragma unroll
    for (int o = 0; o < CL - 1; ++o) rkeys[o] = dsmem_addr(S.keys, (r + 1 + o) % CL);
    const int h0 = 2 * t4;                 // this lane's D columns: heads h0, h0 + 1
    // rows past the first round: into L2 now, so the second round is an L2 hit
    constexpr int R1 = kCW * NB * 16;
    for (int i = tid; i < 2 * (n_sl - R1); i += kCT)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(keys_g + (int64_t)S.sid[R1 + (i >> 1)] * D + (i & 1) * (D / 2)));
    uint32_t kmn = 0xffffffffu, kmx = 0u;   // this thread's key range
    for (int bk0 = warp * NB; bk0 * 16 < n_sl; bk0 += kCW * NB) {
      uint4 ra[NB][KS2], rb[NB][KS2];
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int r0 = (bk0 + nb) * 16 + g8, r1 = r0 + 8;
        const T* k0 = keys_g + (int64_t)(r0 < n_sl ? S.sid[r0] : 0) * D + 8 * t4;
        const T* k1 = keys_g + (int64_t)(r1 < n_sl ? S.sid[r1] : 0) * D + 8 * t4;
#pragma unroll
        for (int s2 = 0; s2 < KS2; ++s2) {
          ra[nb][s2] = r0 < n_sl ? ldg16(reinterpret_cast<const uint4*>(k0 + s2 * 32)) : make_uint4(0, 0, 0, 0);
          rb[nb][s2] = r1 < n_sl ? ldg16(reinterpret_cast<const uint4*>(k1 + s2 * 32)) : make_uint4(0, 0, 0, 0);
        }
      }
      if (bk0 == warp * NB) cmark(p, 12);
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        if (nb == 1 && bk0 == warp * NB) cmark(p, 13);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int s2 = 0; s2 < KS2; ++s2) {
          const uint4 qv = g8 < GS ? *reinterpret_cast<const uint4*>(qf_base + s2 * 32) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {   // 16-element k-steps: (.x .y) then (.z .w) of the pieces
            const uint32_t a0 = hf ? ra[nb][s2].z : ra[nb][s2].x, a1 = hf ? rb[nb][s2].z : rb[nb][s2].x;
            const uint32_t a2 = hf ? ra[nb][s2].w : ra[nb][s2].y, a3 = hf ? rb[nb][s2].w : rb[nb][s2].y;
            const uint32_t b0 = hf ? qv.z : qv.x, b1 = hf ? qv.w : qv.y;
            float d0, d1, d2, d3;
            asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%10,%10,%10,%10};"
                : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3)
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
            acc[0] += (double)d0;
            acc[1] += (double)d1;
            acc[2] += (double)d2;
            acc[3] += (double)d3;
          }
        }
        // acc[0..1]: row r0, heads h0, h0+1; acc[2..3]: row r1
        const int r0 = (bk0 + nb) * 16 + g8, r1 = r0 + 8;
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int hh = h0 + e;
          if (hh < GS) {
            const double l0 = acc[e] * scale, l1 = acc[2 + e] * scale;
            if (r0 < n_sl) lgg[(int64_t)hh * p.lmax + lo + r0] = l0;
            if (r1 < n_sl) lgg[(int64_t)hh * p.lmax + lo + r1] = l1;
            m0 = fmaxf(m0, (float)l0);
            m1 = fmaxf(m1, (float)l1);
          }
        }
        // group max over the row's heads (lanes t4 = 0..3; max commutes with the f32 rounding)
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
          m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
        }
        if (t4 < 2) {
          const int rr = t4 == 0 ? r0 : r1;
          const float gm = t4 == 0 ? m0 : m1;
          if (rr < n_sl) {
            const uint32_t k32 = ~okey32(gm);
            kmn = min(kmn, k32);
            kmx = max(kmx, k32);
            S.keys[lo + rr] = k32;
#pragma unroll
            for (int o = 0; o < CL - 1; ++o) st_cluster_u32(rkeys[o] + 4u * (uint32_t)(lo + rr), k32);
            kg[lo + rr] = ((uint64_t)k32 << 32) | (uint32_t)(lo + rr);
          }
        }
      }
      if (bk0 == warp * NB) cmark(p, 14);
    }
    // the slice's key range into every cluster CTA (the top-rho' histogram
    // needs the min / max of all L keys; barrier #3 publishes them)
    kmn = __reduce_min_sync(0xffffffffu, kmn);
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    if (lane == 0 && kmn <= kmx)
#pragma unroll
      for (int o = 0; o < CL; ++o) {
        uint32_t* rm = cl.map_shared_rank(s_kmm, o);
        atomicMin(rm, kmn);
        atomicMax(rm + 1, kmx);
      }
  }
  cmark(p, 5);
  cl.sync();   // #3: every slice's keys are complete (and its logits/ids in L2)
  cmark(p, 6);

  // CTA 0: prefetch the static partials into area A (its lists are dead)
  if (r == 0) {
    for (int i = tid; i < ns * gs * D / 4; i += kCT)
      cp_async16(S.spo + 4 * i, p.po + (int64_t)u * ns * gs * D + 4 * i);
    for (int i = tid; i < ns * gs; i += kCT) {
      cp_async8(S.spml + i, p.pm + (int64_t)u * ns * gs + i);
      cp_async8(S.spml + ns * gs + i, p.pl + (int64_t)u * ns * gs + i);
    }
    cp_async_commit();
  }

  // ---- 4. top-rho' boundary over all L keys (pushed here before barrier #3) ----
  cmark(p, 7);
  const int Rn = L > 0 ? (p.use_rerank ? min(p.rho_prime, L) : L) : 0;
  uint32_t vk = 0xffffffffu;
  int vpos = L;
  if (Rn > 0 && Rn < L)
    chain_select(S.keys, L, Rn, s_kmm[0], s_kmm[1], S.hist, reinterpret_cast<uint64_t*>(S.spos),
                 s_state, reinterpret_cast<uint32_t*>(S.scratch), &vk, &vpos);
  cmark(p, 8);
  // this CTA's share of the selected positions: ranks [Rn*r/CL, Rn*(r+1)/CL)
  // in position order (ordered compaction)
  const int rlo = (int)((int64_t)Rn * r / CL), rhi = (int)((int64_t)Rn * (r + 1) / CL);
  {
    const int pt = (L + kCT - 1) / kCT;
    int nsel = 0;
    for (int e = 0; e < pt; ++e) {
      const int i = tid * pt + e;
      if (i < L) {
        const uint32_t k = S.keys[i];
        nsel += (k < vk) || (k == vk && i <= vpos);
      }
    }
    int tot;
    int rk = block_exclusive_scan(nsel, &tot, S.scratch);
    for (int e = 0; e < pt; ++e) {
      const int i = tid * pt + e;
      if (i < L) {
        const uint32_t k = S.keys[i];
        if ((k < vk) || (k == vk && i <= vpos)) {
          if (rk >= rlo && rk < rhi) S.spos[rk - rlo] = i;
          ++rk;
        }
      }
    }
  }
  __syncthreads();   // keys dead from here: area B becomes the per-warp V sums
  // the stream's next kernel (the next layer's scan) may start launching now:
  // its CTAs stage their centroid rows while this chain attends and merges
  pdl_trigger();
  const int nmy = rhi - rlo;
  cmark(p, 9);

  // ---- 5. attention over this CTA's selected tokens (online softmax) ------------
  constexpr int VL = CH;                     // lanes per V row (one 16-byte chunk each)
  constexpr int VR = 32 / VL;                // rows per warp pass
  const int vsub = lane % VL, vrw = lane / VL;
  float acc[GS][8];
#pragma unroll
  for (int hh = 0; hh < GS; ++hh)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[hh][e] = 0.f;
  if (tid < GS) {
    hm[tid] = -INFINITY;
    hl[tid] = 0.0;
  }
  const T* vals_g = static_cast<const T*>(p.values) + (int64_t)u * p.cap * D;
  for (int b0 = 0; b0 < nmy; b0 += kCB) {
    const int n = min(kCB, nmy - b0);
    __syncthreads();   // previous batch's weights and ids consumed; hm/hl current
    double* lgs = S.lgs;   // [GS][kCB] this batch's logits, then their exp weights
    for (int i = tid; i < n; i += kCT) {
      const int pos = S.spos[b0 + i];
      S.vid[i] = __ldcg(recg + pos);
#pragma unroll
      for (int hh = 0; hh < GS; ++hh) lgs[hh * kCB + i] = __ldcg(lgg + (int64_t)hh * p.lmax + pos);
    }
    __syncthreads();
    // the first round of V rows is in flight while the weights are computed
    // V-row passes in flight per warp: at gs = 8 the 64 accumulators leave
    // room for 4 (8 there cost 3 %: cfg3 3,607 vs 3,709 tok/s; 2 also lost)
    constexpr int VUN = GS >= 8 ? 4 : kVUn;
    uint4 rawv[VUN];
    const int t00 = warp * VR;
#pragma unroll
    for (int x = 0; x < VUN; ++x) {
      const int t = t00 + x * kCW * VR + vrw;
      rawv[x] = t < n ? ldg16(reinterpret_cast<const uint4*>(vals_g + (int64_t)S.vid[t] * D) + vsub)
                      : make_uint4(0, 0, 0, 0);
    }
    // running max per head (warp hh), then one exp per (head, token)
    for (int hh = warp; hh < GS; hh += kCW) {
      double m = -INFINITY;
      for (int i = lane; i < n; i += 32) m = fmax(m, lgs[hh * kCB + i]);
      m = warp_max_f64(m);
      if (lane == 0) {
        const double mn = fmax(m, hm[hh]);
        hresc[hh] = hm[hh] == -INFINITY ? 0.0 : dexp(hm[hh] - mn);
        hnew[hh] = mn;
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int i = tid; i < GS * n; i += kCT) {
      const int hh = i / n, k = i - hh * n;
      const double e = (double)expf((float)(lgs[hh * kCB + k] - hnew[hh]));   // f32 exp: ~1e-7 rel. weights
      lgs[hh * kCB + k] = e;
      S.wts[hh * kCB + k] = (float)e;
    }
    __syncthreads();
    for (int hh = warp; hh < GS; hh += kCW) {
      double l = 0.0;
      for (int i = lane; i < n; i += 32) l += lgs[hh * kCB + i];
      l = warp_sum_f64(l);
      if (lane == 0) {
        hl[hh] = hl[hh] * hresc[hh] + l;
        hm[hh] = hnew[hh];
      }
    }
    float resc[GS];
#pragma unroll
    for (int hh = 0; hh < GS; ++hh) resc[hh] = (float)hresc[hh];
#pragma unroll
    for (int hh = 0; hh < GS; ++hh)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[hh][e] *= resc[hh];
    // weighted V rows: VL lanes per row, VUN passes in flight
    for (int t0 = t00; t0 < n; t0 += kCW * VR * VUN) {
      if (t0 != t00) {
#pragma unroll
        for (int x = 0; x < VUN; ++x) {
          const int t = t0 + x * kCW * VR + vrw;
          rawv[x] = t < n ? ldg16(reinterpret_cast<const uint4*>(vals_g + (int64_t)S.vid[t] * D) + vsub)
                          : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int x = 0; x < VUN; ++x) {
        const int t = t0 + x * kCW * VR + vrw;
        if (t >= n) continue;
        float f[8];
        unpack16<T>(rawv[x], f);
#pragma unroll
        for (int hh = 0; hh < GS; ++hh)
          if (hh < gs) {
            const float w = S.wts[hh * kCB + t];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[hh][e] = fmaf(w, f[e], acc[hh][e]);
          }
      }
    }
  }
  // rows of a warp pass -> one partial per warp, then over the warps
#pragma unroll
  for (int hh = 0; hh < GS; ++hh)
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int o = VL; o < 32; o <<= 1) acc[hh][e] += __shfl_xor_sync(0xffffffffu, acc[hh][e], o);
  float* cpo0 = cl.map_shared_rank(S.cpo, 0);
  double* cpml0 = cl.map_shared_rank(S.cpml, 0);
  constexpr int RH = GS < kRedHeads ? GS : kRedHeads;   // heads per reduction pass
#pragma unroll
  for (int h0 = 0; h0 < GS; h0 += RH) {
    __syncthreads();   // (previous pass's) sums consumed
    if (vrw == 0)
#pragma unroll
      for (int hh = h0; hh < h0 + RH; ++hh)
        if (hh < gs) {
          float4* dst = reinterpret_cast<float4*>(S.red + ((size_t)warp * RH + (hh - h0)) * D + 8 * vsub);
          dst[0] = make_float4(acc[hh][0], acc[hh][1], acc[hh][2], acc[hh][3]);
          dst[1] = make_float4(acc[hh][4], acc[hh][5], acc[hh][6], acc[hh][7]);
        }
    __syncthreads();
    const int nh = min(RH, gs - h0);
    for (int i = tid; i < nh * D; i += kCT) {
      float s = 0.f;
      for (int w = 0; w < kCW; ++w) s += S.red[(size_t)w * RH * D + i];
      cpo0[(size_t)r * gs * D + (size_t)h0 * D + i] = s;
    }
  }
  if (tid < gs) {
    cpml0[r * gs + tid] = nmy > 0 ? hm[tid] : -INFINITY;
    cpml0[CL * gs + r * gs + tid] = nmy > 0 ? hl[tid] : 0.0;
  }
  cmark(p, 10);
  cl.sync();   // #4: all sparse partials are in CTA 0
  if (r != 0) {
    ktl_mark(p.tl, 1, true);
    return;
  }

  // ---- 6. CTA 0: exact merge with the static partials ---------------------------------
  cp_async_wait_all();
  __syncthreads();
  double* wj = S.scratch;   // [gs][ns + CL] split weights
  const int nsp = ns + CL;
  if (nsp <= 32) {   // a warp per head, a lane per split: max, weights, denominator
    for (int hh = warp; hh < gs; hh += kCW) {
      const int j = lane;
      double mj = -INFINITY, lj = 0.0;
      if (j < ns) {
        mj = S.spml[j * gs + hh];
        lj = S.spml[ns * gs + j * gs + hh];
      } else if (j < nsp) {
        mj = S.cpml[(j - ns) * gs + hh];
        lj = S.cpml[CL * gs + (j - ns) * gs + hh];
      }
      double M = lj > 0.0 ? mj : -INFINITY;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
      const double w = lj > 0.0 ? dexp(mj - M) : 0.0;
      double Ls = w * lj;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Ls += __shfl_xor_sync(0xffffffffu, Ls, o);
      if (j < nsp) wj[hh * nsp + j] = w;
      if (lane == 0) {
        hm[hh] = M;
        hl[hh] = Ls;
      }
    }
    __syncthreads();
  } else {
  if (tid < gs) {
    const int hh = tid;
    double M = -INFINITY;
#pragma unroll 1
    for (int j = 0; j < ns; ++j)
      if (S.spml[ns * gs + j * gs + hh] > 0.0) M = fmax(M, S.spml[j * gs + hh]);
    for (int c = 0; c < CL; ++c)
      if (S.cpml[CL * gs + c * gs + hh] > 0.0) M = fmax(M, S.cpml[c * gs + hh]);
    hm[hh] = M;
  }
  __syncthreads();
  for (int i = tid; i < gs * nsp; i += kCT) {   // one exp per (head, split), in parallel
    const int hh = i / nsp, j = i % nsp;
    const double mj = j < ns ? S.spml[j * gs + hh] : S.cpml[(j - ns) * gs + hh];
    const double lj = j < ns ? S.spml[ns * gs + j * gs + hh] : S.cpml[CL * gs + (j - ns) * gs + hh];
    wj[i] = lj > 0.0 ? dexp(mj - hm[hh]) : 0.0;
  }
  __syncthreads();
  if (tid < gs) {
    const int hh = tid;
    double Ls = 0.0;
#pragma unroll 1
    for (int j = 0; j < ns; ++j) Ls += wj[hh * nsp + j] * S.spml[ns * gs + j * gs + hh];
    for (int c = 0; c < CL; ++c) Ls += wj[hh * nsp + ns + c] * S.cpml[CL * gs + c * gs + hh];
    hl[hh] = Ls;
  }
  __syncthreads();
  }
  bool none = false;
#pragma unroll 1
  for (int i = tid; i < gs * D; i += kCT) {
    const int hh = i / D, e = i % D;
    const double* wh = wj + hh * nsp;
    double O = 0.0;
#pragma unroll 1
    for (int j = 0; j < ns; ++j) O += wh[j] * (double)S.spo[(j * gs + hh) * D + e];
    for (int c = 0; c < CL; ++c) O += wh[ns + c] * (double)S.cpo[((size_t)c * gs + hh) * D + e];
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
    for (int k2 = tid; k2 < p.c_prime; k2 += kCT) p.selected[(int64_t)u * p.c_prime + k2] = sel[k2];
  cmark(p, 11);
  __syncthreads();
  ktl_mark(p.tl, 1, true);
}

// ------------------------------------------------------------------------
// launcher
// ------------------------------------------------------------------------

// CTAs per unit (cluster size).  A step of few units (<= 16: small
// batches, e.g. one GPU's slice of cfg5 at B <= 16) is latency-bound and
// splits each unit's gathers and selection over 8 CTAs (+4-6 % at cfg5
// B = 1..16); larger steps share the GPU between lanes and keep 4 (8 lost at
// cfg5 B = 32 and at cfg2).  The lanes engine passes its whole-batch choice
// (phase bits 32/64) so every lane of a step uses the same size.
constexpr int kChainCL = 4, kChainCLSmall = 8, kChainSmallUnits = 16;
static int chain_cl(const DecodeParams& p) {
  if (p.chain_cl) return p.chain_cl;
  return p.U <= kChainSmallUnits ? kChainCLSmall : kChainCL;
}

template <typename T, int D, int CL, int GS>
static int launch_chain_t(const DecodeParams& p0, cudaStream_t st) {
  DecodeParams p = p0;
  p.dbg = g_host_dbg;
  const size_t sm = chain_layout(p, D, CL, nullptr, nullptr);
  auto k = chain_kernel<T, D, CL, GS>;
  if (int rc = set_max_smem_k(k, sm)) return rc;
  launch_k(k, dim3(p.U * CL), dim3(kCT), sm, st, kPrioHigh, p);
  return cudaGetLastError() == cudaSuccess ? CTKV_OK : CTKV_ECUDA;
}

int chain_phase_timing(int on, unsigned long long* out, int n) {
  if (out != nullptr) {
    const int m = n < kCPhaseCtas * kCPhases ? n : kCPhaseCtas * kCPhases;
    if (cudaMemcpyFromSymbol(out, g_cphase, sizeof(unsigned long long) * m) != cudaSuccess)
      return CTKV_ECUDA;
  }
  if (on >= 0) set_host_dbg(2, on);
  return CTKV_OK;
}

bool chain_supported(const DecodeParams& p, int dtype, int D) {
  if (dtype != CTKV_BF16 || (D != 64 && D != 128)) return false;
  if ((p.gs != 1 && p.gs != 2 && p.gs != 4 && p.gs != 8) || p.c_prime > kCMaxLists) return false;
  if ((p.rho + kCT - 1) / kCT > kCMaxPer) return false;
  return chain_layout(p, D, chain_cl(p), nullptr, nullptr) <= 200 * 1024;
}

template <int D, int CL>
static int launch_chain_g(const DecodeParams& p, cudaStream_t st) {
  switch (p.gs) {
    case 1: return launch_chain_t<__nv_bfloat16, D, CL, 1>(p, st);
    case 2: return launch_chain_t<__nv_bfloat16, D, CL, 2>(p, st);
    case 4: return launch_chain_t<__nv_bfloat16, D, CL, 4>(p, st);
    case 8: return launch_chain_t<__nv_bfloat16, D, CL, 8>(p, st);
  }
  return CTKV_ESHAPE;
}

int launch_chain(const DecodeParams& p, int dtype, int D, cudaStream_t st) {
  if (dtype != CTKV_BF16) return CTKV_ECONFIG;
  const bool small = chain_cl(p) == kChainCLSmall;
  if (D == 128) return small ? launch_chain_g<128, kChainCLSmall>(p, st) : launch_chain_g<128, kChainCL>(p, st);
  if (D == 64) return small ? launch_chain_g<64, kChainCLSmall>(p, st) : launch_chain_g<64, kChainCL>(p, st);
  return CTKV_ESHAPE;
}

}  // namespace ctkv
