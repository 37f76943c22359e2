// Internal host<->device parameter blocks shared by the kernel files and
// the C-ABI layer.  Not part of the public ABI (include/ctkv.h is).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

namespace ctkv {

enum : int32_t {
  kStageSelect = 1,      // top-C' slots from gcos
  kStageUnion = 2,       // union of the selected lists (else rec_in/len_in)
  kStageScores = 4,      // rerank logits + group max (else grouped_in)
  kStageSort = 8,        // (score desc, position asc) order
  kStageDcu = 16,        // FIFO dynamic centroid update
  kStageAttend = 32,     // sparse attention + merge with static partials
  kStageAppendTail = 64  // last CTA advances *total (fused append)
};

constexpr int32_t kFlagNoTokens = 128;  // nothing attendable (ConfigError)
constexpr int32_t kFlagInternal = 256;  // a device-side wait timed out (RuntimeError)

struct DecodeParams {
  // layout
  int b, h, g, gs, U;  // U = b * g units
  int64_t cap;
  int init_len, local_len;
  // store
  const void* keys;
  const void* values;
  int64_t* total;      // device scalar; nullptr -> id_bound is used instead
  int64_t id_bound;
  const void* k_new;  // fused append (nullable)
  const void* v_new;
  // index
  void* cent;
  int32_t* lists;
  int64_t* fifo;
  int32_t* sync;
  float* cnorm;       // [b,h,C] centroid norms (nullable)
  int C, rho;
  // step
  const void* q;
  int c_prime, rho_prime, use_rerank, dcu_force;
  int stages;
  int do_cos;
  int cos_blocks_per_unit;
  int ns;           // partial slots per unit (static splits, or list+static splits)
  int list_splits;  // attn_split_kernel: leading splits that read id lists
  int ids_shared;
  int bitmap_words;
  int lmax;
  // workspace
  double* gcos;     // [U][C]
  double* pm;       // [U][ns][gs]
  double* pl;       // [U][ns][gs]
  float* po;        // [U][ns][gs][D]
  double* logits;   // [U][gs][lmax]
  double* cval;     // [U][cos_blocks_per_unit][ncand] chunk top-C' cosines
  int32_t* cidx;    // [U][cos_blocks_per_unit][ncand] their centroid slots
  int ncand;        // min(C', centroids per cos chunk)
  // chain -> tail hand-off (per unit, by recall position)
  int32_t* recg;    // [U][lmax] recalled ids, first-occurrence order
  uint64_t* keyg;   // [U][lmax] packed (~f32 score, position) rerank keys
  int* uctr;        // [U][4]: [2] = L (recall length), [3] = R (sparse length)
  unsigned long long* tl;  // [4 kinds][start, end] globaltimer span of this step's kernels (debug)
  int wparts_b, wparts_c;
  // v6 chain: the scan's last cosine CTA of a unit writes its top-C' slots
  int32_t* selg;    // [U][c'] top-C' slots (ties -> smaller slot)
  int* selctr;      // [U] cosine-chunk completion counters (reset by the last CTA)
  int chain_cl;     // chain cluster size chosen by the caller (0: by this launch's units)
  int dbg;          // profiling builds only (-DCTKV_PROFILE): timestamp mark bits
                    // (1 scan2, 2 chain), a kernel parameter, so marks that are off
                    // cost no global load
  // staged io
  const int32_t* rec_in;
  const int32_t* len_in;
  const double* grouped_in;
  int32_t* rec_out;
  double* grouped_out;
  int32_t* order_out;
  // outputs
  float* out;
  double* row_max;
  double* denom;
  int32_t* selected;
  int32_t* recall_len;
  int32_t* sparse_ids;
  int32_t* sparse_len;
  int sparse_cap;
  int32_t* flags;
};

size_t scan_smem_bytes(const DecodeParams& p, int D);
size_t unit_smem_bytes(const DecodeParams& p, int D);
int launch_scan(const DecodeParams& p, int dtype, int D, int nblocks, cudaStream_t st);
int launch_unit(const DecodeParams& p, int dtype, int D, cudaStream_t st);
int launch_unit2(const DecodeParams& p, int dtype, int D, cudaStream_t st);
size_t unit2_smem_bytes(const DecodeParams& p, int D);
int static_tok_for(int dtype);
int phase_timing(int on, unsigned long long* out, int n);
int kernel_timeline(int on);
extern int g_host_dbg;   // debug mark bits the launchers copy into DecodeParams::dbg
inline void set_host_dbg(int bit, int on) { g_host_dbg = on ? (g_host_dbg | bit) : (g_host_dbg & ~bit); }
bool tail_supported(const DecodeParams& p, int dtype, int D);
// the deferred tail of the fused step: order, DCU, sparse ids, cursor/total (ctkv_tail.cu)
int launch_tail(const DecodeParams& p, int dtype, int D, cudaStream_t st);
bool chain_supported(const DecodeParams& p, int dtype, int D);
// v6: the unit chain on a 4-CTA cluster per unit (ctkv_chain.cu)
int scan2_timeline(int on, unsigned long long* out, int n);
int chain_phase_timing(int on, unsigned long long* out, int n);
int launch_chain(const DecodeParams& p, int dtype, int D, cudaStream_t st);
int launch_centroid_norms(int dtype, int D, const void* cent, int64_t rows, float* out, cudaStream_t st);
int launch_attn(const DecodeParams& p, int dtype, int D, cudaStream_t st);
int launch_merge2(int64_t rows, int D, const float* oa, const double* ma, const double* la,
                  const float* ob, const double* mb, const double* lb, float* out, double* mo,
                  double* lo, cudaStream_t st);
int launch_append(int dtype, void* keys, void* vals, const void* kn, const void* vn,
                  int64_t* total, int64_t units, int64_t cap, int D, cudaStream_t st);

// Programmatic dependent launch: a kernel launched with it may start (its
// prologue, e.g. TMA loads of data no earlier kernel writes) while its
// stream predecessor finishes; it calls pdl_wait() (griddepcontrol.wait)
// before touching anything the predecessor produced.
// Programmatic dependent launch is used only inside a ctkv_decode_step_phase
// call whose caller set phase bit 16 (see include/ctkv.h); this host-thread
// flag carries that permission to launch_k for the duration of the call.
extern thread_local int t_pdl_ok;
struct PdlScope {
  explicit PdlScope(bool ok) { t_pdl_ok = ok ? 1 : 0; }
  ~PdlScope() { t_pdl_ok = 0; }
};
// Launch priorities (CTA dispatch order when several kernels wait for SMs):
// the latency-critical chain kernels go first, the bandwidth-bound scans
// last.
enum LaunchPrio { kPrioLow = 0, kPrioMid = 1, kPrioHigh = 2 };
int launch_priority(LaunchPrio pr);
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                           cudaStream_t st, LaunchPrio pr, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributePriority;
  attr[n].val.priority = launch_priority(pr);
  ++n;
  if (t_pdl_ok && (pr == kPrioHigh || pr == kPrioLow)) {   // chain and scan launches
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int kCosChunkHost = 64;
constexpr int kStaticSplitHost = 64;
constexpr int kAttnSplitHost = 64;

// ---- build ---------------------------------------------------------------
struct BuildParams {
  int b, h, g, gs, d;
  int64_t cap;            // key rows per (b,g)
  const void* cent;       // [b,h,C,d]
  const void* keys;       // [b,g,cap,d]
  int64_t off_begin, n_off;
  int C, rho;
  int32_t* lists;         // [b,g,C,rho]
  int32_t* flags;
  int mode;
  int dtype;
};

size_t build_workspace_bytes(const BuildParams& p);
// exact recompute of the tensor-core build's unfinished rows (ctkv_build.cu)
int launch_build_fallback(const void* cent, const void* keys, const int32_t* fail_n,
                          const int32_t* fail_rows, int C, int gs, int h, int g, int d, int64_t cap,
                          int64_t off, int64_t n, float scale, float* scratch, int grid, int rho,
                          int32_t* lists, int32_t* flags, cudaStream_t st);
int launch_build(const BuildParams& p, int dtype, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_scores(int dtype, int b, int h, int g, int d, const void* q, int64_t m, const void* k,
                  int64_t n, int64_t k_row_stride, int grouped, float* out, cudaStream_t st);
size_t topk_workspace_bytes(int64_t rows, int64_t n, int k);
int launch_topk_rows(const float* v, int64_t rows, int64_t n, int k, int32_t* idx, void* ws,
                     size_t ws_bytes, cudaStream_t st);

int launch_stage_copy(void* dst, const void* src, size_t bytes, cudaStream_t st);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more than it was last given on this device (the per-call API otherwise
// pays the attribute call on every launch)
int set_max_smem(const void* kernel, size_t bytes);
template <typename K>
inline int set_max_smem_k(K* kernel, size_t bytes) {
  return set_max_smem(reinterpret_cast<const void*>(kernel), bytes);
}

}  // namespace ctkv
