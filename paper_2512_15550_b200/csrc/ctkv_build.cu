// Prefill index build (Alg. 1; ck/index.py:59-99) -- SIMT path.
//
//   scores_kernel  -- grouped scores S[c, j] = f32(max_h (q_{h,c} . k_j) / sqrt(d))
//                     for a chunk of centroid rows against the offloaded keys,
//                     accumulated in ACC (double: the exact parity mode whose
//                     rounding matches the reference's f64 matmul + f32 cast,
//                     ck/tensor_ops.py:88-92; float: the fast SIMT mode).
//   topk_rows_kernel -- per row, the exact top-k by (value desc, index asc)
//                     (ck/tensor_ops.py:144-169) with a 3-pass 11/11/10-bit
//                     radix select on order-preserving u32 keys, an ordered
//                     tie pass when ties straddle the k-th value, and a
//                     shared-memory bitonic sort of the k survivors.
//
// The tensor-core build (ctkv_build_tc.cu) reuses topk_rows_kernel.
#include <cfloat>
#include <cmath>

#include "ctkv.h"
#include "ctkv_common.cuh"
#include "ctkv_internal.h"

namespace ctkv {

constexpr int kSC = 32;        // centroids per scores tile
constexpr int kSD = 32;        // d chunk staged in smem
constexpr int kSThreads = 256; // 32 centroids x 8 key groups
// keys per thread (accumulators GS x KPT stay in registers) and per tile
template <int GS> struct STile {
  static constexpr int KPT = GS >= 8 ? 4 : 8;
  static constexpr int SK = 8 * KPT;
};

// out[(c - c_lo), j] for c in [c_lo, c_lo + nc), j in [0, n)  (grouped=1), or
// out[(hh, c - c_lo), j] per head (grouped=0, used by ctkv_scores)
template <typename T, int GS, typename ACC>
__global__ void __launch_bounds__(kSThreads) scores_kernel(
    const T* __restrict__ cent, int64_t cent_unit_stride /*elements between (b,g) head groups*/,
    int64_t cent_row_stride /*between consecutive centroids*/, int64_t cent_head_stride,
    const T* __restrict__ keys, int64_t key_unit_stride, int64_t key_row_stride, int d, int nc,
    int64_t n, int grouped, float* __restrict__ out, int64_t out_unit_stride, int64_t out_ld) {
  constexpr int kSKPT = STile<GS>::KPT, kSK = STile<GS>::SK;
  __shared__ float As[kSC * GS][kSD + 1];
  __shared__ float Bs[kSK][kSD + 1];
  const int unit = blockIdx.z;
  const int c0 = blockIdx.y * kSC;
  const int64_t j0 = (int64_t)blockIdx.x * kSK;
  const T* A = cent + unit * cent_unit_stride;
  const T* B = keys + unit * key_unit_stride;
  const int tid = threadIdx.x;
  const int tc = tid / 8, tk = tid % 8;
  ACC acc[GS][kSKPT];
#pragma unroll
  for (int hh = 0; hh < GS; ++hh)
#pragma unroll
    for (int j = 0; j < kSKPT; ++j) acc[hh][j] = ACC(0);
  for (int e0 = 0; e0 < d; e0 += kSD) {
    __syncthreads();
    for (int i = tid; i < kSC * GS * kSD; i += kSThreads) {
      const int r = i / kSD, e = i % kSD;
      const int hh = r / kSC, c = r % kSC;
      float v = 0.f;
      if (c0 + c < nc && e0 + e < d)
        v = to_f(A[hh * cent_head_stride + (int64_t)(c0 + c) * cent_row_stride + e0 + e]);
      As[hh * kSC + c][e] = v;
    }
    for (int i = tid; i < kSK * kSD; i += kSThreads) {
      const int r = i / kSD, e = i % kSD;
      float v = 0.f;
      if (j0 + r < n && e0 + e < d) v = to_f(B[(j0 + r) * key_row_stride + e0 + e]);
      Bs[r][e] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int e = 0; e < kSD; ++e) {
      ACC a[GS], bv[kSKPT];
#pragma unroll
      for (int hh = 0; hh < GS; ++hh) a[hh] = (ACC)As[hh * kSC + tc][e];
#pragma unroll
      for (int j = 0; j < kSKPT; ++j) bv[j] = (ACC)Bs[tk + 8 * j][e];
#pragma unroll
      for (int hh = 0; hh < GS; ++hh)
#pragma unroll
        for (int j = 0; j < kSKPT; ++j) acc[hh][j] = fma(a[hh], bv[j], acc[hh][j]);
    }
  }
  if (c0 + tc >= nc) return;
  const ACC scale = ACC(1.0 / sqrt((double)d));
  float* O = out + unit * out_unit_stride;
#pragma unroll
  for (int j = 0; j < kSKPT; ++j) {
    const int64_t col = j0 + tk + 8 * j;
    if (col >= n) continue;
    if (grouped) {
      ACC m = acc[0][j] * scale;
#pragma unroll
      for (int hh = 1; hh < GS; ++hh) m = fmax(m, acc[hh][j] * scale);
      float* o = O + (int64_t)(c0 + tc) * out_ld + col;
      // grouped == 2: second half of a 16-head group, max into the first's
      // (rounding to f32 is monotonic, so this equals f32 of the f64 max)
      *o = grouped == 2 ? fmaxf(*o, (float)m) : (float)m;
    } else {
#pragma unroll
      for (int hh = 0; hh < GS; ++hh)
        O[((int64_t)hh * nc + c0 + tc) * out_ld + col] = (float)(acc[hh][j] * scale);
    }
  }
}

// ------------------------------------------------------------------------
// exact row top-k
// ------------------------------------------------------------------------

constexpr int kTThreads = 512;
constexpr int kTBins = 2048;

// Warp 0 finds the bin where the descending cumulative count reaches `k`;
// returns (bin, count strictly above the bin).
__device__ void find_bin(const int* hist, int nbins, int k, int* s_bin, int* s_above) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int per = nbins / 32;
  // lane L owns bins [nbins - (L+1)*per, nbins - L*per) : lane 0 = top bins
  const int hi = nbins - lane * per;
  int sum = 0;
  for (int b = hi - 1; b >= hi - per; --b) sum += hist[b];
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int excl = incl - sum;
  const unsigned ballot = __ballot_sync(0xffffffffu, incl >= k && excl < k);
  const int owner = __ffs(ballot) - 1;
  if (lane == owner) {
    int run = excl;
    for (int b = hi - 1; b >= hi - per; --b) {
      if (run + hist[b] >= k) {
        *s_bin = b;
        *s_above = run;
        break;
      }
      run += hist[b];
    }
  }
}

// Exact top-k of one row v[0..n) (value desc, index asc) into dst[0..k),
// ids + add; the whole block cooperates.  smem: hist [kTBins] int, cand
// [next_pow2(k)] u64, then (kSmemRow) the row's n u32 keys.
template <bool kSmemRow>
__device__ void topk_row_body(const float* __restrict__ v, int64_t n, int k,
                              int32_t* __restrict__ dst, int32_t add, unsigned char* smem) {
  int* hist = reinterpret_cast<int*>(smem);                        // [kTBins]
  uint64_t* cand = reinterpret_cast<uint64_t*>(hist + kTBins);     // [next_pow2(k)]
  const int kp = next_pow2(k);
  uint32_t* rowk = reinterpret_cast<uint32_t*>(cand + kp);         // [n] (kSmemRow)
  __shared__ int s_bin, s_above, s_cnt;
  const int tid = threadIdx.x;
  auto key_at = [&](int64_t i) -> uint32_t {
    if (kSmemRow) return rowk[i];
    return okey32(v[i]);
  };
  if (kSmemRow) {
    for (int64_t i = tid; i < n; i += kTThreads) rowk[i] = okey32(v[i]);
  }
  // radix passes: 11 / 11 / 10 bits
  uint32_t prefix = 0;
  int above = 0;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
  for (int pass = 0; pass < 3; ++pass) {
    const int sh = shifts[pass];
    const int nb = 1 << widths[pass];
    for (int i = tid; i < kTBins; i += kTThreads) hist[i] = 0;
    __syncthreads();
    const int hsh = sh + widths[pass];  // bits above the current digit
    for (int64_t i = tid; i < n; i += kTThreads) {
      const uint32_t key = key_at(i);
      const bool match = pass == 0 || (key >> hsh) == (prefix >> hsh);
      if (match) atomicAdd(&hist[(key >> sh) & (nb - 1)], 1);
    }
    __syncthreads();
    find_bin(hist, nb, k - above, &s_bin, &s_above);
    __syncthreads();
    prefix |= (uint32_t)s_bin << sh;
    above += s_above;
  }
  const uint32_t T = prefix;          // the k-th largest key
  const int need = k - above;         // ties at T to take (>= 1)
  const int ties = hist[T & 1023];    // pass-3 histogram count of key == T
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (int64_t i = tid; i < n; i += kTThreads) {
    const uint32_t key = key_at(i);
    if (key > T || (key == T && ties == need)) {
      const int slot = atomicAdd(&s_cnt, 1);
      cand[slot] = ((uint64_t)(~key) << 32) | (uint32_t)i;
    }
  }
  __syncthreads();
  if (ties != need && tid < 32) {
    // ties straddle the k-th value: take the `need` smallest indices
    int taken = 0;
    const int base = s_cnt;
    for (int64_t i0 = 0; i0 < n && taken < need; i0 += 32) {
      const int64_t i = i0 + tid;
      const bool t = i < n && key_at(i) == T;
      const unsigned b = __ballot_sync(0xffffffffu, t);
      const int r = __popc(b & ((1u << tid) - 1));
      if (t && taken + r < need) cand[base + taken + r] = ((uint64_t)(~T) << 32) | (uint32_t)i;
      taken += __popc(b);
    }
  }
  __syncthreads();
  for (int i = k + tid; i < kp; i += kTThreads) cand[i] = ~0ull;
  bitonic_sort_u64(cand, kp);
  for (int i = tid; i < k; i += kTThreads) dst[i] = (int32_t)(cand[i] & 0xffffffffu) + add;
  __syncthreads();
}

template <bool kSmemRow>
__global__ void __launch_bounds__(kTThreads) topk_rows_kernel(const float* __restrict__ vals,
                                                              int64_t n, int64_t ld, int k,
                                                              int32_t* __restrict__ idx_out,
                                                              int64_t out_ld, int32_t add,
                                                              int64_t rows_per_group,
                                                              int64_t group_stride,
                                                              const int32_t* row_map) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t row = blockIdx.x;
  int32_t* dst = row_map ? idx_out + (int64_t)row_map[row] * out_ld
                        : idx_out + (row / rows_per_group) * group_stride + (row % rows_per_group) * out_ld;
  topk_row_body<kSmemRow>(vals + row * ld, n, k, dst, add, smem);
}

// Exact fallback of the tensor-core build for the rows its select pass could
// not finish (candidate count outside [rho, cap]): a fixed grid walks the
// device-side failure list (no host round trip, so the build stays
// graph-capturable); per row, f32 SIMT group-max scores of every offloaded
// key into this CTA's scratch row, then the exact top-rho of that row.
__global__ void __launch_bounds__(kTThreads) build_fallback_kernel(
    const __nv_bfloat16* __restrict__ cent, const __nv_bfloat16* __restrict__ keys,
    const int32_t* __restrict__ fail_n, const int32_t* __restrict__ fail_rows, int C, int gs,
    int h, int g, int d, int64_t cap, int64_t off, int64_t n, float scale,
    float* __restrict__ scratch, int rho, int32_t* __restrict__ lists, int32_t* flags) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ float qs[16 * 256];
  const int nf = *fail_n;
  if (nf > 0 && blockIdx.x == 0 && threadIdx.x == 0) set_flag(flags, kFlagBuildFallback);
  float* sc = scratch + (int64_t)blockIdx.x * n;
  for (int f = blockIdx.x; f < nf; f += gridDim.x) {
    const int r = fail_rows[f];
    const int u = r / C, c = r % C;
    const int bi = u / g, gi = u % g;
    for (int i = threadIdx.x; i < gs * d; i += blockDim.x) {
      const int j = i / d, e = i % d;
      qs[i] = __bfloat162float(cent[(((int64_t)bi * h + gi * gs + j) * C + c) * d + e]);
    }
    __syncthreads();
    for (int64_t key = threadIdx.x; key < n; key += blockDim.x) {
      const __nv_bfloat16* kr = keys + ((int64_t)u * cap + off + key) * d;
      float m = -INFINITY;
      for (int j = 0; j < gs; ++j) {
        float a = 0.f;
        for (int e = 0; e < d; ++e) a = fmaf(qs[j * d + e], __bfloat162float(kr[e]), a);
        m = fmaxf(m, a);
      }
      sc[key] = m * scale;
    }
    __syncthreads();
    topk_row_body<false>(sc, n, rho, lists + (int64_t)r * rho, (int32_t)off, smem);
  }
}

int launch_build_fallback(const void* cent, const void* keys, const int32_t* fail_n,
                          const int32_t* fail_rows, int C, int gs, int h, int g, int d, int64_t cap,
                          int64_t off, int64_t n, float scale, float* scratch, int grid, int rho,
                          int32_t* lists, int32_t* flags, cudaStream_t st) {
  const size_t sm = sizeof(int) * kTBins + sizeof(uint64_t) * next_pow2(rho);
  if (sm > 200 * 1024 || gs * d > 16 * 256) return CTKV_ECONFIG;
  if (int rc = set_max_smem_k(build_fallback_kernel, sm)) return rc;
  build_fallback_kernel<<<grid, kTThreads, sm, st>>>(
      static_cast<const __nv_bfloat16*>(cent), static_cast<const __nv_bfloat16*>(keys), fail_n,
      fail_rows, C, gs, h, g, d, cap, off, n, scale, scratch, rho, lists, flags);
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

// ------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------

static size_t topk_smem(int64_t n, int k, bool smem_row) {
  return sizeof(int) * kTBins + sizeof(uint64_t) * next_pow2(k) +
         (smem_row ? sizeof(uint32_t) * (size_t)n : 0);
}

int topk_launch(const float* v, int64_t rows, int64_t n, int64_t ld, int k, int32_t* out,
                int64_t out_ld, int32_t add, cudaStream_t st, int64_t rows_per_group,
                int64_t group_stride, const int32_t* row_map) {
  if (rows_per_group <= 0) {
    rows_per_group = rows > 0 ? rows : 1;
    group_stride = 0;
  }
  if (rows == 0 || k == 0) return 0;
  const bool smem_row = topk_smem(n, k, true) <= 200 * 1024;
  const size_t sm = topk_smem(n, k, smem_row);
  if (sm > 220 * 1024) return CTKV_ECONFIG;
  if (smem_row) {
    if (int rc = set_max_smem_k(topk_rows_kernel<true>, sm)) return rc;
    topk_rows_kernel<true><<<(unsigned)rows, kTThreads, sm, st>>>(v, n, ld, k, out, out_ld, add,
                                                                  rows_per_group, group_stride,
                                                                  row_map);
  } else {
    if (int rc = set_max_smem_k(topk_rows_kernel<false>, sm)) return rc;
    topk_rows_kernel<false><<<(unsigned)rows, kTThreads, sm, st>>>(v, n, ld, k, out, out_ld, add,
                                                                  rows_per_group, group_stride,
                                                                  row_map);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

size_t topk_workspace_bytes(int64_t, int64_t, int) { return 0; }

int launch_topk_rows(const float* v, int64_t rows, int64_t n, int k, int32_t* idx, void*, size_t,
                     cudaStream_t st) {
  return topk_launch(v, rows, n, n, k, idx, k, 0, st, -1, 0, nullptr);
}

template <typename T, typename ACC>
static int scores_dispatch(int gs, dim3 grid_in, cudaStream_t st, const T* cent, int64_t cus,
                           int64_t crs, int64_t chs, const T* keys, int64_t kus, int64_t krs,
                           int d, int nc, int64_t n, int grouped, float* out, int64_t ous,
                           int64_t old_) {
#define CTKV_SC(G)                                                                            \
  grid.x = (unsigned)((n + STile<G>::SK - 1) / STile<G>::SK);                                  \
  scores_kernel<T, G, ACC><<<grid, kSThreads, 0, st>>>(cent, cus, crs, chs, keys, kus, krs, d, \
                                                       nc, n, grouped, out, ous, old_);        \
  break;
#define CTKV_SC_16(CENT, GROUPED, OUT)                                                        \
  grid.x = (unsigned)((n + STile<8>::SK - 1) / STile<8>::SK);                                  \
  scores_kernel<T, 8, ACC><<<grid, kSThreads, 0, st>>>(CENT, cus, crs, chs, keys, kus, krs, d, \
                                                       nc, n, GROUPED, OUT, ous, old_);
  dim3 grid = grid_in;
  switch (gs) {
    case 1: CTKV_SC(1)
    case 2: CTKV_SC(2)
    case 4: CTKV_SC(4)
    case 8: CTKV_SC(8)
    case 16: {
      // two 8-head passes: heads 0-7, then 8-15 max-combined (grouped) or
      // written after the first eight heads' rows (per head)
      CTKV_SC_16(cent, grouped, out)
      CTKV_SC_16(cent + 8 * chs, grouped ? 2 : 0, grouped ? out : out + 8 * (int64_t)nc * old_)
      break;
    }
    default: return CTKV_ESHAPE;
  }
#undef CTKV_SC
#undef CTKV_SC_16
  return cudaGetLastError() == cudaSuccess ? 0 : CTKV_ECUDA;
}

// grouped scores for centroids [c_lo, c_lo+nc) of every (b,g) unit into
// out[unit][c][n] (ld = n)
static int scores_chunk(const BuildParams& p, int dtype, int c_lo, int nc, float* out,
                        bool exact, cudaStream_t st) {
  const int U = p.b * p.g;
  dim3 grid(1, (unsigned)((nc + kSC - 1) / kSC), (unsigned)U);
  const int64_t d = p.d;
  // centroids [b,h,C,d]; unit (b,g) heads start at ((b*h + g*gs) * C + c_lo) * d
  // unit stride in elements for z = b*g + gi : heads of unit u start at u*gs*C*d
  const int64_t cus = (int64_t)p.gs * p.C * d, crs = d, chs = (int64_t)p.C * d;
  const int64_t kus = p.cap * d, krs = d;
  if (dtype == CTKV_BF16) {
    auto* c = static_cast<const __nv_bfloat16*>(p.cent) + (int64_t)c_lo * d;
    auto* k = static_cast<const __nv_bfloat16*>(p.keys) + p.off_begin * d;
    return exact ? scores_dispatch<__nv_bfloat16, double>(p.gs, grid, st, c, cus, crs, chs, k, kus, krs,
                                                          p.d, nc, p.n_off, 1, out,
                                                          (int64_t)nc * p.n_off, p.n_off)
                 : scores_dispatch<__nv_bfloat16, float>(p.gs, grid, st, c, cus, crs, chs, k, kus, krs,
                                                         p.d, nc, p.n_off, 1, out,
                                                         (int64_t)nc * p.n_off, p.n_off);
  }
  auto* c = static_cast<const float*>(p.cent) + (int64_t)c_lo * d;
  auto* k = static_cast<const float*>(p.keys) + p.off_begin * d;
  return exact ? scores_dispatch<float, double>(p.gs, grid, st, c, cus, crs, chs, k, kus, krs, p.d,
                                                nc, p.n_off, 1, out, (int64_t)nc * p.n_off, p.n_off)
               : scores_dispatch<float, float>(p.gs, grid, st, c, cus, crs, chs, k, kus, krs, p.d,
                                               nc, p.n_off, 1, out, (int64_t)nc * p.n_off, p.n_off);
}

// rows of the materialised chunk that fit the workspace
static int chunk_rows(const BuildParams& p, size_t ws_bytes) {
  const int U = p.b * p.g;
  const size_t per_c = (size_t)U * p.n_off * sizeof(float);
  if (per_c == 0) return p.C;
  size_t c = ws_bytes / per_c;
  if (c > (size_t)p.C) c = p.C;
  return (int)c;
}

bool build_tc_supported(const BuildParams& p, int dtype);
size_t build_tc_workspace_bytes(const BuildParams& p);
int build_tc(const BuildParams& p, int dtype, void* ws, size_t ws_bytes, cudaStream_t st);

size_t build_simt_workspace_bytes(const BuildParams& p);

size_t build_workspace_bytes(const BuildParams& p) {
  size_t b = build_simt_workspace_bytes(p);
  if (p.mode == CTKV_BUILD_FAST && build_tc_supported(p, p.dtype)) {
    const size_t t = build_tc_workspace_bytes(p);
    if (t > b) b = t;
  }
  return b;
}

size_t build_simt_workspace_bytes(const BuildParams& p) {
  // one materialised chunk of up to 64 centroids (or all C when smaller),
  // capped at 2 GiB
  const int U = p.b * p.g;
  const size_t per_c = (size_t)U * p.n_off * sizeof(float);
  size_t c = 64;
  if (c > (size_t)p.C) c = p.C;
  while (c > 1 && c * per_c > (2ull << 30)) c >>= 1;
  return c * per_c;
}

int launch_build(const BuildParams& p, int dtype, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (p.rho == 0 || p.C == 0) return 0;
  if (p.mode == CTKV_BUILD_FAST && build_tc_supported(p, dtype) &&
      build_tc_workspace_bytes(p) <= ws_bytes)
    return build_tc(p, dtype, ws, ws_bytes, st);
  const int U = p.b * p.g;
  const int cr = chunk_rows(p, ws_bytes);
  if (cr < 1) return CTKV_EWORKSPACE;
  float* S = static_cast<float*>(ws);
  const bool exact = p.mode == CTKV_BUILD_EXACT;
  for (int c_lo = 0; c_lo < p.C; c_lo += cr) {
    const int nc = std::min(cr, p.C - c_lo);
    int rc = scores_chunk(p, dtype, c_lo, nc, S, exact, st);
    if (rc) return rc;
    // lists[u][c_lo + r][:] = off_begin + topk(S[u][r][:]), one launch
    rc = topk_launch(S, (int64_t)U * nc, p.n_off, p.n_off, p.rho, p.lists + (int64_t)c_lo * p.rho,
                     p.rho, (int32_t)p.off_begin, st, nc, (int64_t)p.C * p.rho, nullptr);
    if (rc) return rc;
  }
  return 0;
}

int launch_scores(int dtype, int b, int h, int g, int d, const void* q, int64_t m, const void* k,
                  int64_t n, int64_t k_row_stride, int grouped, float* out, cudaStream_t st) {
  const int gs = h / g;
  const int U = b * g;
  dim3 grid(1, (unsigned)((m + kSC - 1) / kSC), (unsigned)U);
  // q [b,h,m,d] -> unit u's heads start at u*gs*m*d; k [b,g,*,k_row_stride/d ...]
  const int64_t cus = (int64_t)gs * m * d, crs = d, chs = m * (int64_t)d;
  const int64_t kus = k_row_stride, krs = d;
  const int64_t ous = grouped ? m * n : (int64_t)gs * m * n;
  if (dtype == CTKV_BF16)
    return scores_dispatch<__nv_bfloat16, double>(gs, grid, st, (const __nv_bfloat16*)q, cus, crs, chs,
                                                  (const __nv_bfloat16*)k, kus, krs, d, (int)m, n,
                                                  grouped, out, ous, n);
  return scores_dispatch<float, double>(gs, grid, st, (const float*)q, cus, crs, chs, (const float*)k,
                                        kus, krs, d, (int)m, n, grouped, out, ous, n);
}

}  // namespace ctkv
