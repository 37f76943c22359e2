/*
 * ctkv.h -- C ABI of the B200 (sm_100a) CTkvr hot path.
 *
 * Drop-in boundary for the reference package `centroidkv` 0.1.0, whose
 * public hot-path API is Python (ck/__init__.py:10-35; ck = the package at
 * /root/reference/pkg/src/centroidkv).  The reference has no FFI, so each
 * entry point below names the Python function it replaces; the Python
 * mirror in paper_2512_15550_b200/ binds these through ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless documented otherwise; calls
 *    are asynchronous on the caller's stream (a cudaStream_t passed as
 *    void*; NULL = legacy default stream).
 *  - Caller allocates everything, including a workspace whose size the
 *    matching *_workspace_bytes() query returns.  No hidden allocation.
 *  - Status is returned as int (CTKV_OK == 0); nothing throws across C.
 *    Data-dependent conditions found on the device (empty recall, zero
 *    norms, ids out of range) are reported through a caller-provided
 *    int32 `flags` word (CTKV_FLAG_*), sticky (OR-ed).
 *  - Tensor layouts follow the reference exactly: K/V [b,g,cap,d]
 *    token-major per (b,g) (ck/store.py:41-44), centroids [b,h,C,d],
 *    lists [b,g,C,rho] int32 with -1 = empty (ck/index.py:35-55),
 *    fifo_head [b] int64.
 *  - Scores that drive selections accumulate in float64; attention outputs
 *    are float32 [b,h,d] with float64 row_max / denom
 *    (ck/retrieval.py:50-58).
 */
#ifndef CTKV_H
#define CTKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTKV_ABI_VERSION 1

enum ctkv_dtype { CTKV_F32 = 0, CTKV_BF16 = 1 };

enum ctkv_status {
  CTKV_OK = 0,
  CTKV_ESHAPE = 1,     /* -> ShapeError     (ck/errors.py:8-9)   */
  CTKV_ECONFIG = 2,    /* -> ConfigError    (ck/errors.py:12-13) */
  CTKV_EINDEX = 3,     /* -> IndexError     (ck/store.py:146-147) */
  CTKV_ECUDA = 4,      /* -> RuntimeError                         */
  CTKV_EWORKSPACE = 5  /* workspace too small -> RuntimeError      */
};

enum ctkv_flag {
  CTKV_FLAG_DEGENERATE = 1,      /* zero-norm vector: DegenerateQueryWarning (ck/tensor_ops.py:202-206) */
  CTKV_FLAG_EMPTY_RECALL = 2,    /* some (b,g) recalled nothing                */
  CTKV_FLAG_NONEMPTY_RECALL = 4, /* some (b,g) recalled something; both set => the
                                    reference's "mixed empty/nonempty" ConfigError
                                    (ck/retrieval.py:326-327)                    */
  CTKV_FLAG_ID_RANGE = 8,        /* token id outside [0,total): IndexError       */
  CTKV_FLAG_CAPACITY = 16,       /* device buffer limit hit (see ctkv_status_string) */
  CTKV_FLAG_DUP_IDS = 32,        /* duplicate ids in an attention set (ck/retrieval.py:261-262) */
  CTKV_FLAG_BUILD_FALLBACK = 64, /* build rows re-done on the exact fallback path (info) */
  CTKV_FLAG_NO_TOKENS = 128,     /* nothing attendable: ConfigError (ck/retrieval.py:355) */
  CTKV_FLAG_INTERNAL = 256       /* a device-side wait timed out (internal error, RuntimeError) */
};

/* Dimensions shared by every call (ck/tensor_ops.py:25-55 HeadLayout plus
 * the partition lengths of ck/store.py:34-39). */
typedef struct ctkv_layout {
  int32_t batch;        /* b  (the local shard's batch) */
  int32_t query_heads;  /* h */
  int32_t kv_heads;     /* g  (h % g == 0, h/g <= 16) */
  int32_t head_dim;     /* d in {16,32,64,128,256} */
  int64_t capacity;     /* token rows allocated per (b,g) in K and V */
  int32_t dtype;        /* enum ctkv_dtype of K, V, queries and centroids */
  int32_t init_len;     /* L_init */
  int32_t local_len;    /* L_local */
  int32_t reserved;
} ctkv_layout;

/* Device state of one QueryCentroidIndex (ck/index.py:35-55). */
typedef struct ctkv_index {
  void* centroids;      /* [b,h,C,d] dtype, raw (not normalised) queries */
  int32_t* lists;       /* [b,g,C,rho] int32, -1 = empty */
  int64_t* fifo_head;   /* [b] FIFO cursor (ck/index.py:55,121,133) */
  int32_t* sync;        /* [1+b] int32 scratch, zero-initialised once, owned by the index */
  float* cnorm;         /* [b,h,C] |centroid| (f32 of the exact f64 norm) or NULL; kept
                           current by ctkv_centroid_norms and every DCU write */
  int32_t capacity;     /* C */
  int32_t rho;          /* list length */
} ctkv_index;

/* Device state of one KvStore (ck/store.py:23-44). */
typedef struct ctkv_store {
  void* keys;           /* [b,g,capacity,d] */
  void* values;         /* [b,g,capacity,d] */
  int64_t* total;       /* device scalar: tokens stored (ck/store.py:75-76) */
} ctkv_store;

/* One fused decode step (replaces ck/retrieval.py:304-378 decode_step,
 * preceded by ck/store.py:114-129 append when k_new != NULL, exactly the
 * order of ck/session.py:58-60 run_decode). */
typedef struct ctkv_step_args {
  const void* query;    /* [b,h,d] dtype */
  const void* k_new;    /* [b,g,d] dtype or NULL (no append this step) */
  const void* v_new;    /* [b,g,d] dtype or NULL */
  int32_t c_prime;      /* C'  (1 <= C' <= C) */
  int32_t rho_prime;    /* rho' */
  int32_t use_dcu;      /* FIFO dynamic centroid update (ck/index.py:103-133) */
  int32_t use_rerank;   /* 0: attend the whole recall set (ck/retrieval.py:334-337) */
  /* outputs; every one but `out` may be NULL */
  float* out;           /* [b,h,d] merged attention output */
  double* row_max;      /* [b,h] merged running max */
  double* denom;        /* [b,h] merged denominator */
  int32_t* selected;    /* [b,g,C'] centroid slots, cosine-descending */
  int32_t* recall_len;  /* [b,g] */
  int32_t* sparse_ids;  /* [b,g,sparse_cap] score-descending (recall order when !use_rerank) */
  int32_t* sparse_len;  /* [b,g] */
  int32_t sparse_cap;   /* row stride of sparse_ids */
  int32_t* flags;       /* sticky CTKV_FLAG_* word (device) or NULL */
} ctkv_step_args;

int ctkv_abi_version(void);
const char* ctkv_status_string(int status);
/* 1 if the current device is sm_100 and the kernels load; else 0. */
int ctkv_device_ok(void);

/* ---- storage (ck/store.py) -------------------------------------------- */

/* KvStore.append (ck/store.py:114-129): write [b,g,d] rows at *total, ++*total. */
int ctkv_append(const ctkv_layout* L, ctkv_store S, const void* k_new, const void* v_new,
                void* stream);

/* ---- prefill index build (ck/index.py:59-99, Alg. 1) --------------------- */

enum ctkv_build_mode {
  CTKV_BUILD_EXACT = 0,  /* SIMT float64-accumulating scores (fp32 parity config) */
  CTKV_BUILD_FAST = 1    /* tensor-core bf16 scores, fp32 accumulation */
};

size_t ctkv_build_workspace_bytes(const ctkv_layout* L, int32_t capacity, int32_t rho,
                                  int64_t n_off, int32_t mode);
/* QueryCentroidIndex.build: for each (b,g,c) write the top-rho token ids of
 * keys[b,g,off_begin:off_begin+n_off] by GQA group-max of
 * f32((centroids[b,h,c] . k) / sqrt(d)), ordered (score desc, id asc). */
int ctkv_build_lists(const ctkv_layout* L, const void* centroids, const void* keys,
                     int64_t off_begin, int64_t n_off, int32_t capacity, int32_t rho,
                     int32_t mode, int32_t* lists, int32_t* flags, void* workspace,
                     size_t workspace_bytes, void* stream);

/* |c| for every centroid row (the recall cosine's denominator,
 * ck/tensor_ops.py:199-200), exact f64 from the stored values, rounded to
 * f32: cnorm [b,h,C]. */
int ctkv_centroid_norms(const ctkv_layout* L, const void* centroids, int32_t capacity,
                        float* cnorm, void* stream);

/* Copy `bytes` (a multiple of 16, 16-byte aligned pointers) by a kernel
 * rather than a DMA: either side may be pinned (page-locked) host memory,
 * addressed through unified virtual addressing.  The engine's host-I/O step
 * graph stages its inputs and outputs with it (kernel nodes instead of host
 * memcpy nodes, which make every graph launch hundreds of us slower). */
int ctkv_stage_copy(void* dst, const void* src, size_t bytes, void* stream);

/* ---- decode (ck/retrieval.py) --------------------------------------------- */

/* The decode workspace must be zero-filled before its first use; the
 * kernels' completion counters are left at zero by the CTAs that consume
 * them, so a workspace is reusable across steps without clearing. */
size_t ctkv_decode_workspace_bytes(const ctkv_layout* L, int32_t capacity, int32_t rho,
                                   int32_t c_prime, int32_t rho_prime);

/* decode_step (+ append): recall -> rerank -> sparse + static attention ->
 * merge -> DCU, all on the device, no host synchronisation. */
int ctkv_decode_step(const ctkv_layout* L, ctkv_store S, ctkv_index I, const ctkv_step_args* A,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Same step split by kernel.  `phase` is a bit set: 1 = scan kernel
 * (cosine vs all centroids + static-partition attention partials +
 * append); 2 = unit kernels (select, union, rerank, sparse attention,
 * merge) followed by the tail (ordering, FIFO DCU, sparse ids, cursor and
 * total advance); 8 = with 2, leave the tail out; 4 = the tail only.  3 is
 * the whole step.  Phase 2 must follow phase 1 of the same step; a
 * deferred tail (4) must follow that step's phase 2 and precede the next
 * step's phase 1 for the same layer, and may run on another stream
 * concurrently with other layers' work (it writes only this layer's index,
 * total and outputs, and reads this call's workspace).  Paths without a
 * separate tail run it inside phase 2 and treat 4 as a no-op.
 * 16 (with any of the above): programmatic dependent launch.  The scan and
 * chain may then start before the kernel launched last on `stream` has
 * finished, and read or write before their grid-dependency wait:
 *   scan:  reads centroids, centroid norms, *total, the static partition's
 *          K/V rows and k_new/v_new; writes the static partial slots of its
 *          workspace for splits with no tokens;
 *   chain: reads *total.
 * Everything else (the query, lists, FIFO cursor, the rest of the
 * workspace; every output) is touched only after the wait.  The caller
 * guarantees that the previous kernel on `stream` writes none of the
 * pre-wait inputs and does not read this call's workspace.  In the engine
 * the kernel before a scan is the previous layer's chain (another layer's
 * state) and the kernel before a chain is the same layer's scan, which does
 * not write *total; k_new/v_new arrive from a copy stream through an event
 * (a full dependency).
 * 32 (with any of the above): the caller chooses the chain kernel's cluster
 * size -- 8 CTAs per (b, kv head) unit when 64 is also set, else 4.  Without
 * 32 the library uses 8 when the call covers at most 16 units, else 4.  The
 * cluster size changes the f32 summation grouping of the sparse attention
 * (results agree to ~1e-8), so a caller that splits one batch over several
 * calls (the lanes engine) passes the choice for the whole batch. */
int ctkv_decode_step_phase(const ctkv_layout* L, ctkv_store S, ctkv_index I,
                           const ctkv_step_args* A, int32_t phase, void* workspace,
                           size_t workspace_bytes, void* stream);

/* recall (ck/retrieval.py:132-168): selected [b,g,C'], recalled
 * [b,g,C'*rho] first-occurrence order, recall_len [b,g].  Like the
 * reference it needs no store: `id_bound` is an exclusive upper bound of
 * the token ids held in the lists (the store's total at build time; DCU
 * only ever re-lists recalled ids, so it never grows). */
int ctkv_recall(const ctkv_layout* L, ctkv_index I, int64_t id_bound, const void* query,
                int32_t c_prime, int32_t* selected, int32_t* recalled, int32_t* recall_len,
                int32_t* flags, void* workspace, size_t workspace_bytes, void* stream);

/* rerank scores + order (ck/retrieval.py:171-218): grouped [b,g,lmax] f64
 * group-max logits of the recalled ids; order [b,g,lmax] = positions into
 * `recalled` sorted (score desc, position asc). */
int ctkv_rerank(const ctkv_layout* L, ctkv_store S, const void* query, const int32_t* recalled,
                const int32_t* recall_len, int32_t lmax, double* grouped, int32_t* order,
                int32_t* flags, void* workspace, size_t workspace_bytes, void* stream);

/* attention partial over per-(b,g) id lists (ck/retrieval.py:221-264);
 * ids [b,g,lmax] (or [lmax] when ids_shared), optionally united with the
 * static partition (ck/store.py:94-96) -- the merge is exact. */
size_t ctkv_attend_workspace_bytes(const ctkv_layout* L, int32_t lmax, int32_t with_static);
int ctkv_attend(const ctkv_layout* L, ctkv_store S, const void* query, const int32_t* ids,
                const int32_t* ids_len, int32_t lmax, int32_t ids_shared, int32_t with_static,
                float* out, double* row_max, double* denom, int32_t* flags, void* workspace,
                size_t workspace_bytes, void* stream);

/* merge (ck/retrieval.py:275-284) of two partials over `rows` = b*h rows. */
int ctkv_merge(int64_t rows, int32_t head_dim, const float* out_a, const double* max_a,
               const double* den_a, const float* out_b, const double* max_b,
               const double* den_b, float* out, double* row_max, double* denom, void* stream);

/* fifo_update (ck/index.py:103-133): slot = fifo_head[b] % C gets the
 * query and, per kv head, the top-min(rho, L) recalled ids by `grouped`. */
int ctkv_fifo_update(const ctkv_layout* L, ctkv_index I, const void* query,
                     const int32_t* recalled, const int32_t* recall_len, int32_t lmax,
                     const double* grouped, void* workspace, size_t workspace_bytes,
                     void* stream);

/* dot_scores + group_max (ck/tensor_ops.py:72-118) as a device primitive:
 * out [b,g,m,n] f32 (grouped=1) or [b,h,m,n] (grouped=0). */
int ctkv_scores(const ctkv_layout* L, const void* q, int64_t m, const void* k, int64_t n,
                int64_t k_row_stride, int32_t grouped, float* out, void* stream);

/* top_k_rows (ck/tensor_ops.py:144-169) on the device: rows [r,n] f32 ->
 * idx [r,k] int32 ordered (value desc, index asc). */
size_t ctkv_topk_workspace_bytes(int64_t rows, int64_t n, int32_t k);
int ctkv_topk_rows(const float* values, int64_t rows, int64_t n, int32_t k, int32_t* idx,
                   void* workspace, size_t workspace_bytes, void* stream);

/* Profiling aid: on=1/0 switches per-CTA phase timestamps of the fused unit
 * kernel on/off (on<0 leaves it); host_out (may be NULL) receives up to n
 * u64 globaltimer stamps laid out [256 CTAs][12 checkpoints]. */
int ctkv_debug_phase_timing(int32_t on, uint64_t* host_out, int32_t n);
/* Profiling only: per-CTA task timeline of the persistent scan kernel
 * ([cta][slot] globaltimer ns: 0 start, 1 end, 2+k task k ready). */
int ctkv_debug_scan_timeline(int32_t on, uint64_t* host_out, int32_t n);
/* Profiling only: when on, decode launches record their kernels' spans
 * (globaltimer min start / max end per kind: scan, chain, tail) in the last
 * 64 bytes of the workspace reserved for it (read with ctkv_debug_timeline_rw;
 * see scripts/kernel_timeline.py). */
int ctkv_debug_kernel_timeline(int32_t on);
/* Read (8 x u64) and optionally reset a decode workspace's kernel spans. */
int ctkv_debug_timeline_rw(const ctkv_layout* L, int32_t capacity, int32_t rho, int32_t c_prime,
                           void* workspace, uint64_t* host_out, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* CTKV_H */
