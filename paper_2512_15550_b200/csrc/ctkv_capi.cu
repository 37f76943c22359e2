// extern "C" entry points of libctkv.so (declared in include/ctkv.h).
// Validation mirrors the reference's exception contract: shape problems
// -> CTKV_ESHAPE (ShapeError), precondition violations -> CTKV_ECONFIG
// (ConfigError, e.g. ck/retrieval.py:136-139), CUDA failures -> CTKV_ECUDA.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#include "ctkv.h"
#include "ctkv_internal.h"

using namespace ctkv;

namespace {

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

bool dim_ok(int d) { return d == 16 || d == 32 || d == 64 || d == 128 || d == 256; }

int check_layout(const ctkv_layout* L) {
  if (!L) return CTKV_ESHAPE;
  if (L->batch < 1 || L->query_heads < 1 || L->kv_heads < 1) return CTKV_ESHAPE;
  if (L->query_heads % L->kv_heads) return CTKV_ESHAPE;
  const int gs = L->query_heads / L->kv_heads;
  if (gs > 16) return CTKV_ESHAPE;
  if (!dim_ok(L->head_dim)) return CTKV_ESHAPE;
  if (L->dtype != CTKV_F32 && L->dtype != CTKV_BF16) return CTKV_ESHAPE;
  if (L->capacity < 0 || L->init_len < 0 || L->local_len < 0) return CTKV_ECONFIG;
  return CTKV_OK;
}

// static-partition partial slots of the fused scan kernel (dtype-sized splits)
int static_slots(const ctkv_layout* L) {
  const int64_t n = (int64_t)L->init_len + L->local_len;
  const int st = static_tok_for(L->dtype);
  return (int)((n + st - 1) / st);
}

// static slots of the generic attend kernel (64-token splits)
int attend_static_slots(const ctkv_layout* L) {
  const int64_t n = (int64_t)L->init_len + L->local_len;
  return (int)((n + kAttnSplitHost - 1) / kAttnSplitHost);
}

struct DecodeWs {
  double* gcos;
  double* pm;
  double* pl;
  float* po;
  double* logits;
  double* cval;
  int32_t* cidx;
  int32_t* recg;
  uint64_t* keyg;
  int* uctr;
  unsigned long long* tl;
  int32_t* selg;
  int* selctr;
  size_t bytes;
};

// chunk-local top-C' candidates the fused scan writes: [U][C / (256/gs)][min(C', 256/gs)]
int ncand_for(const ctkv_layout* L, int c_prime) {
  const int cc = 256 / (L->query_heads / L->kv_heads);
  return c_prime < cc ? c_prime : cc;
}

DecodeWs carve_decode(const ctkv_layout* L, int C, int lmax, int ns, void* base, int c_prime = 0) {
  const int U = L->batch * L->kv_heads;
  const int gs = L->query_heads / L->kv_heads;
  const int d = L->head_dim;
  size_t off = 0;
  auto take = [&](size_t b) {
    char* p = base ? static_cast<char*>(base) + off : nullptr;
    off += a256(b);
    return p;
  };
  DecodeWs w;
  w.gcos = reinterpret_cast<double*>(take(sizeof(double) * (size_t)U * std::max(C, 1)));
  w.pm = reinterpret_cast<double*>(take(sizeof(double) * (size_t)U * std::max(ns, 1) * gs));
  w.pl = reinterpret_cast<double*>(take(sizeof(double) * (size_t)U * std::max(ns, 1) * gs));
  w.po = reinterpret_cast<float*>(take(sizeof(float) * (size_t)U * std::max(ns, 1) * gs * d));
  w.logits = reinterpret_cast<double*>(take(sizeof(double) * (size_t)U * gs * std::max(lmax, 1)));
  const int cc = 256 / gs;
  const size_t ncand_total =
      c_prime > 0 ? (size_t)U * ((std::max(C, 1) + cc - 1) / cc) * ncand_for(L, c_prime) : 1;
  w.cval = reinterpret_cast<double*>(take(sizeof(double) * ncand_total));
  w.cidx = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * ncand_total));
  const size_t lm = (size_t)std::max(lmax, 1);
  w.recg = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (size_t)U * lm));
  w.keyg = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * (size_t)U * lm));
  w.uctr = reinterpret_cast<int*>(take(sizeof(int) * 4 * (size_t)U));
  w.tl = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * 8));
  w.selg = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (size_t)U * std::max(c_prime, 1)));
  w.selctr = reinterpret_cast<int*>(take(sizeof(int) * (size_t)U));
  w.bytes = off;
  return w;
}

void fill_layout(DecodeParams& p, const ctkv_layout* L) {
  std::memset(&p, 0, sizeof(p));
  p.b = L->batch;
  p.h = L->query_heads;
  p.g = L->kv_heads;
  p.gs = p.h / p.g;
  p.U = p.b * p.g;
  p.cap = L->capacity;
  p.init_len = L->init_len;
  p.local_len = L->local_len;
  p.bitmap_words = (int)((L->capacity + 31) / 32);
}


}  // namespace

namespace ctkv {
int set_max_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> given;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return CTKV_ECUDA;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = given[{dev, kernel}];
  if (bytes <= have) return CTKV_OK;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return CTKV_ECUDA;
  have = bytes;
  return CTKV_OK;
}
}  // namespace ctkv

extern "C" {

int ctkv_abi_version(void) { return CTKV_ABI_VERSION; }

const char* ctkv_status_string(int s) {
  switch (s) {
    case CTKV_OK: return "ok";
    case CTKV_ESHAPE: return "shape error (unsupported or inconsistent dimensions)";
    case CTKV_ECONFIG: return "config error (precondition violated or device limit exceeded)";
    case CTKV_EINDEX: return "token id out of range";
    case CTKV_ECUDA: return "CUDA error";
    case CTKV_EWORKSPACE: return "workspace too small";
  }
  return "unknown status";
}

int ctkv_device_ok(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return 0;
  return major == 10 && minor == 0 ? 1 : 0;
}

int ctkv_append(const ctkv_layout* L, ctkv_store S, const void* k_new, const void* v_new,
                void* stream) {
  if (int rc = check_layout(L)) return rc;
  if (!S.keys || !S.values || !S.total || !k_new || !v_new) return CTKV_ECONFIG;
  return launch_append(L->dtype, S.keys, S.values, k_new, v_new, S.total,
                       (int64_t)L->batch * L->kv_heads, L->capacity, L->head_dim,
                       static_cast<cudaStream_t>(stream));
}

size_t ctkv_build_workspace_bytes(const ctkv_layout* L, int32_t capacity, int32_t rho,
                                  int64_t n_off, int32_t mode) {
  if (check_layout(L)) return 0;
  BuildParams p{};
  p.b = L->batch;
  p.h = L->query_heads;
  p.g = L->kv_heads;
  p.gs = p.h / p.g;
  p.d = L->head_dim;
  p.C = capacity;
  p.rho = rho;
  p.n_off = n_off;
  p.mode = mode;
  p.dtype = L->dtype;
  p.cap = L->capacity;
  return build_workspace_bytes(p);
}

int ctkv_build_lists(const ctkv_layout* L, const void* centroids, const void* keys,
                     int64_t off_begin, int64_t n_off, int32_t capacity, int32_t rho,
                     int32_t mode, int32_t* lists, int32_t* flags, void* workspace,
                     size_t workspace_bytes, void* stream) {
  if (int rc = check_layout(L)) return rc;
  if (capacity < 1 || rho < 0 || rho > n_off || n_off < 0 || off_begin < 0 ||
      off_begin + n_off > L->capacity)
    return CTKV_ECONFIG;
  if (rho > 8192) return CTKV_ECONFIG;
  const int gs = L->query_heads / L->kv_heads;
  if (gs != 1 && gs != 2 && gs != 4 && gs != 8 && gs != 16) return CTKV_ESHAPE;
  BuildParams p{};
  p.b = L->batch;
  p.h = L->query_heads;
  p.g = L->kv_heads;
  p.gs = gs;
  p.d = L->head_dim;
  p.cap = L->capacity;
  p.cent = centroids;
  p.keys = keys;
  p.off_begin = off_begin;
  p.n_off = n_off;
  p.C = capacity;
  p.rho = rho;
  p.lists = lists;
  p.flags = flags;
  p.mode = mode;
  p.dtype = L->dtype;
  return launch_build(p, L->dtype, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

size_t ctkv_decode_workspace_bytes(const ctkv_layout* L, int32_t capacity, int32_t rho,
                                   int32_t c_prime, int32_t) {
  if (check_layout(L)) return 0;
  return carve_decode(L, capacity, c_prime * rho, static_slots(L), nullptr, c_prime).bytes;
}

int ctkv_decode_step(const ctkv_layout* L, ctkv_store S, ctkv_index I, const ctkv_step_args* A,
                     void* workspace, size_t workspace_bytes, void* stream) {
  return ctkv_decode_step_phase(L, S, I, A, 3, workspace, workspace_bytes, stream);
}

int ctkv_decode_step_phase(const ctkv_layout* L, ctkv_store S, ctkv_index I,
                           const ctkv_step_args* A, int32_t phase, void* workspace,
                           size_t workspace_bytes, void* stream) {
  if (phase < 1 || phase > 127) return CTKV_ECONFIG;
  const PdlScope pdl_scope((phase & 16) != 0);   // 16: the caller allows programmatic dependent launch
  // 32: the caller picks the chain's cluster size -- 8 CTAs per unit if 64
  // is set, else 4 (a lanes engine decides from its whole batch, so a step's
  // result does not depend on how the batch is split into lanes)
  const int chain_cl = (phase & 32) ? ((phase & 64) ? 8 : 4) : 0;
  phase &= 15;
  if (phase < 1) return CTKV_ECONFIG;
  if (int rc = check_layout(L)) return rc;
  if (!A || !A->query || !A->out || !S.keys || !S.values || !S.total) return CTKV_ECONFIG;
  if (I.capacity < 1 || I.capacity > (1 << 20)) return CTKV_ECONFIG;   // slot keys: 20 bits                            // "recall: empty index"
  if (A->c_prime < 1 || A->c_prime > I.capacity) return CTKV_ECONFIG;  // ck/retrieval.py:138
  if (A->rho_prime < 1) return CTKV_ECONFIG;
  if (I.rho < 0 || I.rho > 8 * 512) return CTKV_ECONFIG;
  if ((A->k_new == nullptr) != (A->v_new == nullptr)) return CTKV_ECONFIG;
  if (A->use_dcu && (!I.fifo_head || !I.sync)) return CTKV_ECONFIG;
  if (A->k_new && !I.sync) return CTKV_ECONFIG;
  const int ns = static_slots(L);
  const int lmax = A->c_prime * I.rho;
  DecodeWs w = carve_decode(L, I.capacity, lmax, ns, workspace, A->c_prime);
  if (w.bytes > workspace_bytes) return CTKV_EWORKSPACE;
  DecodeParams p;
  fill_layout(p, L);
  p.keys = S.keys;
  p.values = S.values;
  p.total = S.total;
  p.k_new = A->k_new;
  p.v_new = A->v_new;
  p.cent = I.centroids;
  p.lists = I.lists;
  p.fifo = I.fifo_head;
  p.sync = I.sync;
  p.cnorm = I.cnorm;
  p.C = I.capacity;
  p.rho = I.rho;
  p.q = A->query;
  p.c_prime = A->c_prime;
  p.rho_prime = A->rho_prime;
  p.use_rerank = A->use_rerank;
  p.stages = kStageSelect | kStageUnion | kStageScores | kStageSort | kStageAttend |
             (A->use_dcu ? kStageDcu : 0) | (A->k_new ? kStageAppendTail : 0);
  p.do_cos = 1;
  p.cos_blocks_per_unit = (I.capacity + (256 / p.gs) - 1) / (256 / p.gs);
  p.ns = ns;
  p.lmax = lmax;
  p.gcos = w.gcos;
  p.pm = w.pm;
  p.pl = w.pl;
  p.po = w.po;
  p.logits = w.logits;
  p.cval = w.cval;
  p.cidx = w.cidx;
  p.ncand = ncand_for(L, A->c_prime);
  p.recg = w.recg;
  p.keyg = w.keyg;
  p.uctr = w.uctr;
  p.tl = ctkv::kernel_timeline(-1) ? w.tl : nullptr;
  p.out = A->out;
  p.row_max = A->row_max;
  p.denom = A->denom;
  p.selected = A->selected;
  p.recall_len = A->recall_len;
  p.sparse_ids = A->sparse_ids;
  p.sparse_len = A->sparse_len;
  p.sparse_cap = A->sparse_ids ? A->sparse_cap : 0;
  p.chain_cl = chain_cl;
  p.flags = A->flags;
  // bf16: 2-CTA cluster unit kernel (f32-chunked logits); f32: exact f64 unit kernel
  const bool v2 = L->dtype == CTKV_BF16 && L->head_dim >= 64 && p.gs <= 8 && I.rho <= 4096 &&
                  unit2_smem_bytes(p, L->head_dim) <= 200 * 1024;
  if (!v2) p.cval = nullptr;   // the f64 unit kernel selects from gcos directly
  if (!v2 && unit_smem_bytes(p, L->head_dim) > 220 * 1024) return CTKV_ECONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // bf16 at d = 64/128, gs <= 8, c' <= 8: the scan, then the 4-CTA cluster
  // chain kernel; its tail (DCU, sparse ids, cursor/total) can be deferred
  // (phase bit 8) and enqueued separately (phase 4) on another stream.
  // Other bf16 geometries: scan + the 2-CTA cluster unit2 kernel; f32: scan
  // + the f64-exact unit kernel (both run their tail inside phase 2).
  if (v2 && chain_supported(p, L->dtype, L->head_dim) && tail_supported(p, L->dtype, L->head_dim)) {
    p.selg = w.selg;
    p.selctr = w.selctr;
    const int nblocks = p.U * p.cos_blocks_per_unit + p.U * ns;
    if (phase & 1)
      if (int rc = launch_scan(p, L->dtype, L->head_dim, nblocks, st)) return rc;
    if (phase & 2)
      if (int rc = launch_chain(p, L->dtype, L->head_dim, st)) return rc;
    const bool tail = (phase & 4) || ((phase & 2) && !(phase & 8));
    return tail ? launch_tail(p, L->dtype, L->head_dim, st) : CTKV_OK;
  }
  p.uctr = nullptr;
  const int nblocks = p.U * p.cos_blocks_per_unit + p.U * ns;
  if (phase & 1)
    if (int rc = launch_scan(p, L->dtype, L->head_dim, nblocks, st)) return rc;
  if (phase & 2) return v2 ? launch_unit2(p, L->dtype, L->head_dim, st)
                           : launch_unit(p, L->dtype, L->head_dim, st);
  return CTKV_OK;
}

int ctkv_recall(const ctkv_layout* L, ctkv_index I, int64_t id_bound, const void* query,
                int32_t c_prime, int32_t* selected, int32_t* recalled, int32_t* recall_len,
                int32_t* flags, void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_layout(L)) return rc;
  if (I.capacity < 1 || I.capacity > (1 << 20)) return CTKV_ECONFIG;   // slot keys: 20 bits
  if (c_prime < 1 || c_prime > I.capacity) return CTKV_ECONFIG;
  if (I.rho < 0 || I.rho > 8 * 512) return CTKV_ECONFIG;
  const int lmax = c_prime * I.rho;
  DecodeWs w = carve_decode(L, I.capacity, lmax, 0, workspace);
  if (w.bytes > workspace_bytes) return CTKV_EWORKSPACE;
  if (id_bound < 0) return CTKV_ECONFIG;
  DecodeParams p;
  fill_layout(p, L);
  p.total = nullptr;
  p.id_bound = id_bound;
  p.bitmap_words = (int)((id_bound + 31) / 32);
  p.cent = I.centroids;
  p.lists = I.lists;
  p.cnorm = I.cnorm;
  p.C = I.capacity;
  p.rho = I.rho;
  p.q = query;
  p.c_prime = c_prime;
  p.stages = kStageSelect | kStageUnion;
  p.do_cos = 1;
  p.cos_blocks_per_unit = (I.capacity + (256 / p.gs) - 1) / (256 / p.gs);
  p.ns = 0;
  p.lmax = lmax;
  p.gcos = w.gcos;
  p.logits = w.logits;
  p.selected = selected;
  p.rec_out = recalled;
  p.recall_len = recall_len;
  p.flags = flags;
  if (unit_smem_bytes(p, L->head_dim) > 220 * 1024) return CTKV_ECONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = launch_scan(p, L->dtype, L->head_dim, p.U * p.cos_blocks_per_unit, st)) return rc;
  return launch_unit(p, L->dtype, L->head_dim, st);
}

int ctkv_rerank(const ctkv_layout* L, ctkv_store S, const void* query, const int32_t* recalled,
                const int32_t* recall_len, int32_t lmax, double* grouped, int32_t* order,
                int32_t* flags, void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_layout(L)) return rc;
  if (lmax < 0 || !recalled || !recall_len) return CTKV_ECONFIG;
  DecodeWs w = carve_decode(L, 0, lmax, 0, workspace);
  if (w.bytes > workspace_bytes) return CTKV_EWORKSPACE;
  DecodeParams p;
  fill_layout(p, L);
  p.keys = S.keys;
  p.values = S.values;
  p.total = S.total;
  p.q = query;
  p.C = 1;
  p.stages = kStageScores | kStageSort;
  p.lmax = lmax;
  p.rec_in = recalled;
  p.len_in = recall_len;
  p.logits = w.logits;
  p.grouped_out = grouped;
  p.order_out = order;
  p.flags = flags;
  p.c_prime = 1;
  if (unit_smem_bytes(p, L->head_dim) > 220 * 1024) return CTKV_ECONFIG;
  return launch_unit(p, L->dtype, L->head_dim, static_cast<cudaStream_t>(stream));
}

int ctkv_fifo_update(const ctkv_layout* L, ctkv_index I, const void* query,
                     const int32_t* recalled, const int32_t* recall_len, int32_t lmax,
                     const double* grouped, void* workspace, size_t workspace_bytes,
                     void* stream) {
  if (int rc = check_layout(L)) return rc;
  if (I.capacity < 1 || !I.fifo_head || !I.sync || !recalled || !recall_len || !grouped)
    return CTKV_ECONFIG;
  DecodeWs w = carve_decode(L, 0, lmax, 0, workspace);
  if (w.bytes > workspace_bytes) return CTKV_EWORKSPACE;
  DecodeParams p;
  fill_layout(p, L);
  p.cent = I.centroids;
  p.lists = I.lists;
  p.fifo = I.fifo_head;
  p.sync = I.sync;
  p.cnorm = I.cnorm;
  p.C = I.capacity;
  p.rho = I.rho;
  p.q = query;
  p.c_prime = 1;
  p.dcu_force = 1;
  p.stages = kStageSort | kStageDcu;
  p.lmax = lmax;
  p.rec_in = recalled;
  p.len_in = recall_len;
  p.grouped_in = grouped;
  p.logits = w.logits;
  p.total = nullptr;  // the DCU-only pass never reads the store
  if (unit_smem_bytes(p, L->head_dim) > 220 * 1024) return CTKV_ECONFIG;
  return launch_unit(p, L->dtype, L->head_dim, static_cast<cudaStream_t>(stream));
}

size_t ctkv_attend_workspace_bytes(const ctkv_layout* L, int32_t lmax, int32_t with_static) {
  if (check_layout(L)) return 0;
  const int ns = (lmax + kAttnSplitHost - 1) / kAttnSplitHost + (with_static ? attend_static_slots(L) : 0);
  return carve_decode(L, 0, 0, ns, nullptr).bytes;
}

int ctkv_attend(const ctkv_layout* L, ctkv_store S, const void* query, const int32_t* ids,
                const int32_t* ids_len, int32_t lmax, int32_t ids_shared, int32_t with_static,
                float* out, double* row_max, double* denom, int32_t* flags, void* workspace,
                size_t workspace_bytes, void* stream) {
  if (int rc = check_layout(L)) return rc;
  if (!out || lmax < 0 || (lmax > 0 && (!ids || !ids_len))) return CTKV_ECONFIG;
  const int list_splits = lmax > 0 ? (lmax + kAttnSplitHost - 1) / kAttnSplitHost : 0;
  const int ns = list_splits + (with_static ? attend_static_slots(L) : 0);
  if (ns == 0) return CTKV_ECONFIG;
  DecodeWs w = carve_decode(L, 0, 0, ns, workspace);
  if (w.bytes > workspace_bytes) return CTKV_EWORKSPACE;
  DecodeParams p;
  fill_layout(p, L);
  p.keys = S.keys;
  p.values = S.values;
  p.total = S.total;
  p.q = query;
  p.ns = ns;
  p.list_splits = list_splits;
  p.ids_shared = ids_shared;
  p.lmax = lmax;
  p.rec_in = ids;
  p.len_in = ids_len;
  p.pm = w.pm;
  p.pl = w.pl;
  p.po = w.po;
  p.out = out;
  p.row_max = row_max;
  p.denom = denom;
  p.flags = flags;
  return launch_attn(p, L->dtype, L->head_dim, static_cast<cudaStream_t>(stream));
}

int ctkv_merge(int64_t rows, int32_t head_dim, const float* out_a, const double* max_a,
               const double* den_a, const float* out_b, const double* max_b,
               const double* den_b, float* out, double* row_max, double* denom, void* stream) {
  if (rows < 0 || head_dim < 1) return CTKV_ESHAPE;
  return launch_merge2(rows, head_dim, out_a, max_a, den_a, out_b, max_b, den_b, out, row_max,
                       denom, static_cast<cudaStream_t>(stream));
}

int ctkv_scores(const ctkv_layout* L, const void* q, int64_t m, const void* k, int64_t n,
                int64_t k_row_stride, int32_t grouped, float* out, void* stream) {
  // any head_dim works here (the SIMT scores kernel tiles d generically)
  if (!L || L->head_dim < 1) return CTKV_ESHAPE;
  ctkv_layout l2 = *L;
  l2.head_dim = 16;
  if (int rc = check_layout(&l2)) return rc;
  const int gs = L->query_heads / L->kv_heads;
  if (gs != 1 && gs != 2 && gs != 4 && gs != 8 && gs != 16) return CTKV_ESHAPE;
  if (m < 0 || n < 0) return CTKV_ESHAPE;
  if (m == 0 || n == 0) return CTKV_OK;
  return launch_scores(L->dtype, L->batch, L->query_heads, L->kv_heads, L->head_dim, q, m, k, n,
                       k_row_stride, grouped, out, static_cast<cudaStream_t>(stream));
}

size_t ctkv_topk_workspace_bytes(int64_t rows, int64_t n, int32_t k) {
  return topk_workspace_bytes(rows, n, k);
}

int ctkv_topk_rows(const float* values, int64_t rows, int64_t n, int32_t k, int32_t* idx,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (rows < 0 || n < 0 || k < 0) return CTKV_ESHAPE;
  if (k > n) k = (int32_t)n;
  if (k > 8192) return CTKV_ECONFIG;
  return launch_topk_rows(values, rows, n, k, idx, workspace, workspace_bytes,
                          static_cast<cudaStream_t>(stream));
}

int ctkv_centroid_norms(const ctkv_layout* L, const void* centroids, int32_t capacity,
                        float* cnorm, void* stream) {
  if (int rc = check_layout(L)) return rc;
  if (!centroids || !cnorm || capacity < 0) return CTKV_ECONFIG;
  const int64_t rows = (int64_t)L->batch * L->query_heads * capacity;
  return launch_centroid_norms(L->dtype, L->head_dim, centroids, rows, cnorm,
                               static_cast<cudaStream_t>(stream));
}

int ctkv_stage_copy(void* dst, const void* src, size_t bytes, void* stream) {
  if ((bytes & 15) || ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15))
    return CTKV_ECONFIG;
  if (bytes == 0) return CTKV_OK;
  if (!dst || !src) return CTKV_ECONFIG;
  return launch_stage_copy(dst, src, bytes, static_cast<cudaStream_t>(stream));
}

int ctkv_debug_kernel_timeline(int32_t on) {
#ifndef CTKV_PROFILE
  return CTKV_ECONFIG;   // profiling builds only (make -C csrc profile)
#endif
  return ctkv::kernel_timeline(on);
}

int ctkv_debug_timeline_rw(const ctkv_layout* L, int32_t capacity, int32_t rho, int32_t c_prime,
                           void* workspace, uint64_t* host_out, int32_t reset) {
#ifndef CTKV_PROFILE
  return CTKV_ECONFIG;   // profiling builds only (make -C csrc profile)
#endif
  if (int rc = check_layout(L)) return rc;
  DecodeWs w = carve_decode(L, capacity, c_prime * rho, static_slots(L), workspace, c_prime);
  if (host_out && cudaMemcpy(host_out, w.tl, 64, cudaMemcpyDeviceToHost) != cudaSuccess) return CTKV_ECUDA;
  if (reset) {
    unsigned long long init[8];
    for (int k = 0; k < 4; ++k) { init[2 * k] = ~0ull; init[2 * k + 1] = 0ull; }
    if (cudaMemcpy(w.tl, init, 64, cudaMemcpyHostToDevice) != cudaSuccess) return CTKV_ECUDA;
  }
  return CTKV_OK;
}

int ctkv_debug_scan_timeline(int32_t on, uint64_t* host_out, int32_t n) {
#ifndef CTKV_PROFILE
  return CTKV_ECONFIG;   // profiling builds only (make -C csrc profile)
#endif
  return ctkv::scan2_timeline(on, reinterpret_cast<unsigned long long*>(host_out), n);
}

int ctkv_debug_phase_timing(int32_t on, uint64_t* host_out, int32_t n) {
#ifndef CTKV_PROFILE
  return CTKV_ECONFIG;   // profiling builds only (make -C csrc profile)
#endif
  // the chain kernel's marks (bf16 d = 64/128); the unit kernels' otherwise
  const int rc = ctkv::chain_phase_timing(on, reinterpret_cast<unsigned long long*>(host_out), n);
  if (rc) return rc;
  return ctkv::phase_timing(on, nullptr, 0);
}

}  // extern "C"
