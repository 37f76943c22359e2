// Shared device helpers for the CTkvr sm_100a kernels.
//
// Row model: every K/V/centroid/query row is `D` contiguous elements of T
// (float or bf16), i.e. D*sizeof(T) bytes, read with 128-bit vector loads.
// A row is covered by LPR lanes, each holding VPL 16-byte vectors, so one
// warp pass covers RPW rows.  Scores that drive a selection are accumulated
// in float64 (bf16*bf16 and f32*f32 products are exact in f64), which keeps
// every top-k decision aligned with the reference's f64 arithmetic
// (ck/tensor_ops.py:88-92, :196-207; ck/retrieval.py:185-187).
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ctkv {

constexpr int kMaxGroup = 16;   // query heads per kv head supported
constexpr int32_t kEmpty = -1;  // ck/index.py:32

// sticky status bits written to the caller's flags word
enum : int32_t {
  kFlagDegenerate = 1,    // zero-norm query/centroid (DegenerateQueryWarning)
  kFlagEmptyRecall = 2,   // a (b,g) unit recalled nothing
  kFlagNonEmptyRecall = 4,
  kFlagIdRange = 8,       // a token id outside [0, total)  (IndexError)
  kFlagCapacity = 16,     // internal buffer limit exceeded
  kFlagDupIds = 32,       // duplicate ids in an attention set
  kFlagBuildFallback = 64 // build rows that needed the exact fallback path
};

template <typename T, int D>
struct Row {
  static constexpr int EPV = 16 / int(sizeof(T));   // elements per 16B vector
  static constexpr int VPR = D / EPV;               // vectors per row
  static constexpr int LPR = VPR >= 32 ? 32 : VPR;  // lanes per row
  static constexpr int VPL = VPR / LPR;             // vectors per lane
  static constexpr int RPW = 32 / LPR;              // rows per warp pass
  static constexpr int EPL = VPL * EPV;             // elements per lane
  static_assert(D % EPV == 0, "head_dim must fill whole 16B vectors");
  static_assert((LPR & (LPR - 1)) == 0, "lanes per row must be a power of two");
  static_assert(VPR % LPR == 0, "row vectors must split evenly over lanes");
  // element offset of vector v of sub-lane `sub`
  __device__ __forceinline__ static int elem(int sub, int v) { return (v * LPR + sub) * EPV; }
};

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// 16 bytes -> EPV floats
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& u, float* f);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
}
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint4 ldg16(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
// streaming load: bypass L1 (bulk data read once)
__device__ __forceinline__ uint4 ldg16_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Load this lane's slice of a row as floats.
template <typename T, int D, bool kStream = false>
__device__ __forceinline__ void load_row_slice(const T* row, int sub, float* f) {
  using R = Row<T, D>;
#pragma unroll
  for (int v = 0; v < R::VPL; ++v) {
    const uint4 u = kStream ? ldg16_stream(row + R::elem(sub, v)) : ldg16(row + R::elem(sub, v));
    unpack16<T>(u, f + v * R::EPV);
  }
}

// sum over the LPR lanes that share a row (xor butterfly stays inside the
// aligned lane group because LPR is a power of two)
template <int LPR>
__device__ __forceinline__ double row_sum(double x) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
template <int LPR>
__device__ __forceinline__ float row_sum(float x) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Order-preserving map of a double to u64 (larger value -> larger key);
// -0.0 folds onto +0.0 so numerically equal values tie, like numpy compares.
__device__ __forceinline__ uint64_t okey64(double v) {
  v = v + 0.0;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey64_inv(uint64_t k) {
  const uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ uint32_t okey32(float v) {
  v = v + 0.0f;
  uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float okey32_inv(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(b);
}

// In-shared-memory bitonic sort, ascending on (key, val) pairs with n a power
// of two.  Used with key = ~okey(score) so ascending order means
// (score desc, val asc) -- the reference's tie-break (ck/tensor_ops.py:121-169).
template <typename K>
__device__ void bitonic_sort_pairs(K* key, int32_t* val, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const K ka = key[lo], kb = key[hi];
        const int32_t va = val[lo], vb = val[hi];
        const bool a_gt_b = (ka > kb) || (ka == kb && va > vb);
        if (a_gt_b == up) {
          key[lo] = kb; key[hi] = ka;
          val[lo] = vb; val[hi] = va;
        }
      }
    }
  }
  __syncthreads();
}

// bitonic sort of packed u64 keys (ascending)
__device__ inline void bitonic_sort_u64(uint64_t* key, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const uint64_t a = key[lo], b = key[hi];
        if ((a > b) == up) { key[lo] = b; key[hi] = a; }
      }
    }
  }
  __syncthreads();
}

__host__ __device__ inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// programmatic dependent launch (no-ops when launched without the attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// debug kernel timeline: CTA spans folded into [kind][start, end] (atomic
// min/max); tl is null unless ctkv_debug_kernel_timeline(1) is on
__device__ __forceinline__ void ktl_mark(unsigned long long* tl, int kind, bool end) {
#ifdef CTKV_PROFILE
  if (tl != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (end) atomicMax(tl + 2 * kind + 1, t);
    else atomicMin(tl + 2 * kind, t);
  }
#endif
}

__device__ __forceinline__ void set_flag(int32_t* flags, int32_t bit) {
  if (flags) atomicOr(flags, bit);
}

// ---- bf16 x bf16 -> f32 mixed-precision FMA (sm_100 FHFMA.BF16) -----------
// acc + sum_i q_i * x_i over the 8 bf16 lanes of a 16-byte chunk; every
// product is exact and every add rounds once to f32, exactly like
// unpack-to-f32 + FFMA, without the unpack instructions.
__device__ __forceinline__ float bf16x8_dot(const uint4& q, const uint4& x, float acc) {
  const uint32_t qa[4] = {q.x, q.y, q.z, q.w}, xa[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("{.reg .b16 ql, qh, xl, xh;\n\t"
        "mov.b32 {ql, qh}, %1;\n\t"
        "mov.b32 {xl, xh}, %2;\n\t"
        "fma.rn.f32.bf16 %0, ql, xl, %0;\n\t"
        "fma.rn.f32.bf16 %0, qh, xh, %0;}"
        : "+f"(acc)
        : "r"(qa[i]), "r"(xa[i]));
  return acc;
}

// ---- async-proxy helpers (mbarrier + TMA bulk copies) ----------------------

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "BW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra BD_%=;\n\t"
      "bra BW_%=;\n\t"
      "BD_%=:\n\t}" ::"r"(sa(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (16 B aligned, multiple of 16 B)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(bar))
      : "memory");
}

// Register bitonic sort of packed u64 keys across a block: element
// t*IPT + i lives in thread t, register i; strides inside a thread are
// register swaps, inside a warp shuffles, beyond a warp go through `xch`
// (blockDim*IPT u64 of shared memory).  Ascending.
template <int IPT>
__device__ void bitonic_regs(uint64_t (&k)[IPT], uint64_t* xch) {
  const int t = threadIdx.x;
  const int n = blockDim.x * IPT;
  for (int size = 2; size <= n; size <<= 1) {
    // strides >= IPT: partner in another lane (shuffle) or another warp (smem)
    for (int stride = size >> 1; stride >= IPT; stride >>= 1) {
      if (stride < 32 * IPT) {
        const int lm = stride / IPT;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const int e = t * IPT + i;
          const bool up = (e & size) == 0;
          const bool lower = (e & stride) == 0;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, k[i], lm);
          const uint64_t mn = o < k[i] ? o : k[i], mx = o < k[i] ? k[i] : o;
          k[i] = (lower == up) ? mn : mx;
        }
      } else {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; ++i) xch[t * IPT + i] = k[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const int e = t * IPT + i;
          const bool up = (e & size) == 0;
          const bool lower = (e & stride) == 0;
          const uint64_t o = xch[e ^ stride];
          const uint64_t mn = o < k[i] ? o : k[i], mx = o < k[i] ? k[i] : o;
          k[i] = (lower == up) ? mn : mx;
        }
      }
    }
    // strides < IPT: compile-time register pairs
#pragma unroll
    for (int stride = IPT / 2; stride > 0; stride >>= 1) {
      if (stride < size) {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = ((t * IPT + i) & size) == 0;
            const uint64_t a = k[i], b = k[j];
            const bool sw = (a > b) == up;
            k[i] = sw ? b : a;
            k[j] = sw ? a : b;
          }
        }
      }
    }
  }
}

}  // namespace ctkv
