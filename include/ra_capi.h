/* ra_capi.h — C ABI of the B200-native RetrievalAttention decode hot path.
 *
 * One shared library (paper_2409_10516_b200/libra_b200.so), sm_100a only.
 * Plain pointers, sizes and an opaque stream (cudaStream_t passed as void*);
 * no C++ or torch types cross this boundary. Every call returns ra_status;
 * on failure ra_last_error() (thread-local) holds the message, which for
 * argument errors is the reference's exact exception text, so an adapter can
 * rethrow the same std::invalid_argument / std::runtime_error.
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   ra_graph_build          <- ood_build / OODGraph::OODGraph     include/attnindex/index_oodgraph.hpp:35-36,78-81
 *   ra_graph_deserialize    <- OODGraph(keys, blob) / load        include/attnindex/index_oodgraph.hpp:40,63-64
 *   ra_graph_serialize      <- OODGraph::serialize / save         include/attnindex/index_oodgraph.hpp:61-62
 *   ra_graph_* accessors    <- entry_point/degree/neighbors/...    include/attnindex/index_oodgraph.hpp:49-59
 *   ra_graph_search_batch   <- SearchIndex::search (OODGraph)      include/attnindex/index.hpp:41-42
 *   ra_flat_search_batch    <- FlatIndex::search                   include/attnindex/index_flat.hpp:14-15
 *   ra_ivf_build / _search_batch <- IVFIndex / IVFIndex::search     include/attnindex/index_ivf.hpp:17-37
 *   ra_partial_attention    <- partial_attention                   include/attnindex/attention.hpp:47-50
 *   ra_merge / _host        <- merge_gammas + merge                include/attnindex/attention.hpp:52-60
 *   ra_partial_attention_host <- partial_attention (host buffers)  include/attnindex/attention.hpp:47-50
 *   ra_static_partition     <- static_partition                    include/attnindex/attention.hpp:44-45
 *   ra_engine_* / decode    <- engine_init / decode_step           include/attnindex/engine.hpp:103-111
 *
 * Memory: "host" pointers are ordinary CPU memory (pinned recommended);
 * "device" pointers are CUDA global memory on the context's device. Each
 * function documents which it takes. Handles are immutable after creation
 * and may be used from several threads; an ra_ctx (stream + scratch) must
 * not be shared between threads concurrently.
 */
#ifndef RA_CAPI_H
#define RA_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RA_OK = 0,
  RA_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  RA_ERR_RUNTIME = 2,          /* reference: std::runtime_error (blob errors) */
  RA_ERR_CUDA = 3,             /* CUDA failure, no usable device, or missing sm_100a */
  RA_ERR_CAPACITY = 4          /* internal capacity exceeded (never silent) */
} ra_status;

typedef struct ra_ctx ra_ctx;     /* device + stream + scratch arena */
typedef struct ra_kv ra_kv;       /* one KV group resident in HBM (refcounted) */
typedef struct ra_graph ra_graph; /* one query head's OODGraph on the device */
typedef struct ra_engine ra_engine;

/* OODGraphBuildParams (index_oodgraph.hpp:17-27); ra_build_params_default
 * fills the reference defaults 32/32/128/8, Medoid, Euclidean, ef 128. */
typedef struct {
  uint32_t k_train;
  uint32_t max_degree;
  uint32_t ef_construction;
  uint32_t edge_window;
  int32_t entry_maxnorm;       /* 0 = EntryStrategy::Medoid, 1 = MaxNorm */
  int32_t prune_inner_product; /* 0 = PruneRule::Euclidean, 1 = InnerProduct */
  uint32_t default_ef;
} ra_build_params;

/* Per-build diagnostics (not part of the reference API). */
typedef struct {
  uint64_t knn_rows;          /* training queries processed in phase 1 */
  uint64_t knn_rows_widened;  /* rows whose approximate top-k had to be rescanned */
  uint64_t candidate_edges;   /* unique (src,dst) proposals after phase 2 */
  uint64_t repair_rounds;     /* phase-4 iterations */
  uint64_t repaired_nodes;    /* nodes attached by phase 4 */
  double ms_knn, ms_edges, ms_prune, ms_entry, ms_repair;
  double ms_knn_tensor;       /* tcgen05 filter GEMM inside ms_knn (0 on the f64 path) */
} ra_build_stats;

const char* ra_last_error(void);
const char* ra_version(void);

/* ---- context ------------------------------------------------------------ */
ra_status ra_ctx_create(int device, ra_ctx** out);
void ra_ctx_destroy(ra_ctx* ctx);
/* stream: a cudaStream_t (NULL = legacy default). Kernels of this ctx are
 * enqueued on it; calls taking host buffers synchronize it before returning. */
ra_status ra_ctx_set_stream(ra_ctx* ctx, void* stream);
ra_status ra_ctx_synchronize(ra_ctx* ctx);
/* Page-locked, device-mapped host memory (for zero-copy ra_engine_step_host
 * staging); free with ra_host_free. */
ra_status ra_host_alloc(size_t bytes, void** out);
void ra_host_free(void* p);
/* Graph-search kernel variant for this ctx (overrides RA_SEARCH_KERNEL):
 * "auto" (latency mode up to 2 x SMs queries, then throughput mode: DUO
 * while the batch fits one wave, else TPS, else TP), "lat", "duo"
 * (throughput, a commit warp + an expansion warp per query), "tp", "tps"
 * (throughput, shared-memory visited bits + TMA row tiles), "tpr"
 * (throughput, register rows), "cta", "warp"; NULL = default.
 * Every variant returns identical results. Engines read it at creation. */
ra_status ra_ctx_set_search_kernel(ra_ctx* ctx, const char* name);

/* ---- KV groups (types.hpp:18-35, 54-61) ------------------------------------
 * keys/values: n x d f32 row-major; values may be NULL (search-only).
 * on_device = 0: host pointers, copied in; 1: device pointers, copied too
 * (the ra_kv owns its HBM). The handle is shared by all query heads of the
 * GQA group (refcount), mirroring the shared_ptr<const VectorSet>. */
ra_status ra_kv_create(ra_ctx* ctx, const float* keys, const float* values, uint64_t n,
                       uint32_t d, int on_device, ra_kv** out);
/* bf16 KV group: keys and values also kept rounded to bf16 (nearest even).
 * attention_only = 0: search and attention read the bf16 rows - exactly the
 *   reference's arithmetic on the rounded inputs (half the decode bytes);
 * attention_only = 1: the search keeps the exact f32 keys (retrieved ids
 *   identical to f32), the sparse attention reads bf16 K/V.
 * ra_kv_is_bf16: 0 = f32, 1 = bf16, 2 = bf16 attention only. */
ra_status ra_kv_create_bf16(ra_ctx* ctx, const float* keys, const float* values, uint64_t n,
                            uint32_t d, int on_device, int attention_only, ra_kv** out);
int ra_kv_is_bf16(const ra_kv* kv);
/* Uploads the values of a keys-only f32 group (n must equal its size): the
 * group's graphs and engines then attend over them. Errors: already has
 * values, n mismatch ("keys and values must have equal n"). */
ra_status ra_kv_attach_values(ra_ctx* ctx, ra_kv* kv, const float* values, uint64_t n,
                              int on_device);
int ra_kv_has_values(const ra_kv* kv);
void ra_kv_retain(ra_kv* kv);
void ra_kv_release(ra_kv* kv);
uint64_t ra_kv_size(const ra_kv* kv);
uint32_t ra_kv_dim(const ra_kv* kv);
const float* ra_kv_keys_device(const ra_kv* kv);
const float* ra_kv_values_device(const ra_kv* kv);

/* ---- graph index ------------------------------------------------------------ */
void ra_build_params_default(ra_build_params* p);
/* ood_build: train_q nq x d f32, host (on_device = 0) or device (1). Not
 * stored. stats may be NULL. Errors: "empty keys", "too many keys",
 * "k_train must be >= 1", "max_degree must be >= 1",
 * "ef_construction must be >= 1", "query dimension mismatch". */
ra_status ra_graph_build(ra_ctx* ctx, ra_kv* keys, const float* train_q, uint64_t nq,
                         uint32_t q_dim, int on_device, const ra_build_params* params,
                         ra_build_stats* stats, ra_graph** out);
/* OODG v1 blob (host bytes). Errors are the reference's runtime_error texts. */
ra_status ra_graph_deserialize(ra_ctx* ctx, ra_kv* keys, const char* blob, uint64_t size,
                               ra_graph** out);
/* Writes when buf != NULL and cap >= size; always sets *size. */
ra_status ra_graph_serialize(const ra_graph* g, char* buf, uint64_t cap, uint64_t* size);
void ra_graph_free(ra_graph* g);
uint64_t ra_graph_size(const ra_graph* g);
uint64_t ra_graph_entry_point(const ra_graph* g);
uint32_t ra_graph_max_degree_bound(const ra_graph* g);
uint32_t ra_graph_default_ef(const ra_graph* g);
uint32_t ra_graph_degree(const ra_graph* g, uint64_t u);
/* copies neighbors(u) (at most cap) into out (host); returns the degree */
uint32_t ra_graph_neighbors(const ra_graph* g, uint64_t u, uint32_t* out, uint32_t cap);
uint64_t ra_graph_reachable_count(const ra_graph* g);
/* OODGraph::memory_bytes (index_oodgraph.cpp:413-415): CSR u64 offsets + u32 adjacency */
uint64_t ra_graph_memory_bytes(const ra_graph* g);
/* HBM actually held by the device-side adjacency */
uint64_t ra_graph_device_bytes(const ra_graph* g);
/* Copies the reference CSR (offsets_[n+1] u64, adjacency_ u32) into host
 * arrays sized from ra_graph_size / ra_graph_memory_bytes
 * (index_oodgraph.hpp:74-75); either pointer may be NULL (not copied). */
ra_status ra_graph_csr(const ra_graph* g, uint64_t* offsets, uint32_t* adjacency);

/* ---- search (OODGraph::search, index_oodgraph.cpp:357-411) -----------------
 * B queries; query b searches graphs[b] (graphs may repeat) with q + b*d.
 * All array arguments are DEVICE pointers: q [B][d] f32; mask: sorted,
 * duplicate-free excluded ids shared by the batch (mask_n may be 0).
 * ef < 0 selects each graph's default_ef. Outputs: ids/scores [B][k]
 * (slots past n_out padded with UINT32_MAX / NaN), n_out, scanned, truncated
 * [B]; expanded [B] (optional, NULL ok) counts frontier pops.
 * Errors: "k must be >= 1", "ef must be >= k", "query dimension mismatch". */
ra_status ra_graph_search_batch(ra_ctx* ctx, const ra_graph* const* graphs, uint32_t B,
                                const float* q, uint32_t q_dim, uint32_t k, int64_t ef,
                                const uint32_t* mask, uint64_t mask_n, uint32_t* ids,
                                float* scores, uint32_t* n_out, uint64_t* scanned,
                                uint8_t* truncated, uint32_t* expanded);

/* Single query on HOST buffers (synchronous): the exact shape of
 * SearchIndex::search for FFI callers (index.hpp:41-42). ids/scores hold k;
 * *n_out receives the number written. ef < 0 selects default_ef. */
ra_status ra_graph_search_host(ra_ctx* ctx, const ra_graph* g, const float* q, uint32_t q_dim,
                               uint32_t k, int64_t ef, const uint32_t* mask, uint64_t mask_n,
                               uint32_t* ids, float* scores, uint32_t* n_out, uint64_t* scanned,
                               uint8_t* truncated);

/* FlatIndex::search (index_flat.cpp:22-43): exact top-k by f64 inner product
 * with the same (score desc, id asc) order. Device pointers as above. */
ra_status ra_flat_search_batch(ra_ctx* ctx, ra_kv* keys, uint32_t B, const float* q,
                               uint32_t k, const uint32_t* mask, uint64_t mask_n,
                               uint32_t* ids, float* scores, uint64_t* scanned);

/* ---- IVF index (index_ivf.cpp; contrast baseline) --------
 * IVFIndex ctor / ivf_build (index_ivf.cpp:56-151): nlist 0 = ceil(sqrt(n));
 * errors "empty keys", "nlist out of range". Arithmetic in the reference's
 * Eigen expression order (fma chains from 0.0, sums in id order). */
typedef struct ra_ivf ra_ivf;
ra_status ra_ivf_build(ra_ctx* ctx, ra_kv* keys, uint32_t nlist, uint64_t seed, uint32_t iters,
                       uint32_t default_nprobe, ra_ivf** out);
void ra_ivf_free(ra_ivf* ivf);
uint32_t ra_ivf_nlist(const ra_ivf* ivf);
uint32_t ra_ivf_default_nprobe(const ra_ivf* ivf);
/* host copies: centroids nlist x d f32, offsets nlist + 1, ids n (ascending per list) */
ra_status ra_ivf_export(const ra_ivf* ivf, float* centroids, uint32_t* offsets, uint32_t* ids);
uint64_t ra_ivf_memory_bytes(const ra_ivf* ivf);
/* IVFIndex::search (index_ivf.cpp:153-181), B queries, device pointers;
 * nprobe < 0 = the index default. Errors "query dimension mismatch",
 * "nprobe out of range", "k out of range". */
ra_status ra_ivf_search_batch(ra_ctx* ctx, const ra_ivf* ivf, uint32_t B, const float* q,
                              uint32_t q_dim, uint32_t k, int64_t nprobe, const uint32_t* mask,
                              uint64_t mask_n, uint32_t* ids, float* scores, uint32_t* n_out,
                              uint64_t* scanned, uint8_t* truncated);

/* ---- attention (attention.cpp:87-157) ------------------------------------- */
/* static_partition into host arrays (either may be NULL to just count). */
ra_status ra_static_partition(uint64_t t, uint64_t s_init, uint64_t s_local,
                              uint32_t* static_ids, uint64_t* n_static, uint32_t* pool_ids,
                              uint64_t* n_pool);
/* partial_attention for B queries against one KV group. Device pointers:
 * q [B][d], idx [B][m_stride] (row b uses its first m[b] entries; m[b] = 0
 * yields an empty partial), out [B][d] f64, zmax/expsum [B] f64. Errors:
 * "keys and values must have equal n" (values missing), "index out of range". */
ra_status ra_partial_attention(ra_ctx* ctx, ra_kv* kv, uint32_t B, const float* q,
                               const uint32_t* idx, uint32_t m_stride, const uint32_t* m,
                               double* out, double* zmax, double* expsum);
/* partial_attention on HOST buffers, one query (attention.cpp:102-128):
 * keys/values n x d f32; the rows named by idx[0..m) are staged in idx order
 * and reduced on the device (in-order f64 dots, max-subtracted exps, the
 * reference's accumulation order). Errors: "query dimension mismatch",
 * "keys and values must have equal n", "empty index set",
 * "index out of range". out [d] f64. */
ra_status ra_partial_attention_host(ra_ctx* ctx, const float* q, uint32_t q_dim,
                                    const float* keys, uint64_t n_keys, const float* values,
                                    uint64_t n_values, uint32_t d, const uint32_t* idx,
                                    uint64_t m, double* out, double* zmax, double* expsum);
/* merge_gammas + merge of ONE partial pair on HOST buffers
 * (attention.cpp:136-157): out [d]; gw / go may be NULL. An empty side
 * returns the other side exactly; both empty: "empty attention support". */
ra_status ra_merge_host(ra_ctx* ctx, uint32_t d, const double* ow, double zw, double sw,
                        int w_empty, const double* oo, double zo, double so, int o_empty,
                        double* out, double* gw, double* go);
/* merge of B partial pairs (device arrays; *_empty [B] u8 flags). Error
 * "empty attention support" if both sides of any row are empty. */
ra_status ra_merge(ra_ctx* ctx, uint32_t B, uint32_t d, const double* ow, const double* zw,
                   const double* sw, const uint8_t* w_empty, const double* oo,
                   const double* zo, const double* so, const uint8_t* o_empty, double* out,
                   double* gw, double* go);

/* ---- decode engine (engine.cpp:23-115) ------------------------------------------
 * n_heads query heads over n_groups KV groups (head h -> group
 * h / (n_heads / n_groups)), one graph per head, frozen static partition at
 * t = kv size. ef < 0 selects default_ef. */
typedef struct {
  uint64_t s_init;   /* 128 */
  uint64_t s_local;  /* 512 */
  uint32_t top_k;    /* 100 */
  int64_t ef;        /* search_param; < 0 = index default */
} ra_engine_config;

ra_status ra_engine_create(ra_ctx* ctx, ra_kv* const* groups, uint32_t n_groups,
                           ra_graph* const* head_graphs, uint32_t n_heads,
                           const ra_engine_config* cfg, ra_engine** out);
void ra_engine_destroy(ra_engine* e);
/* decode_step on DEVICE buffers: q [H][d] f32 -> out [H][d] f64; omega
 * [H][k] u32 with row stride k = ra_engine_k(e) = min(top_k, |dynamic pool|)
 * (UINT32_MAX padded past a head's n_out) and scanned [H] u64 may be NULL. */
ra_status ra_engine_step_device(ra_engine* e, const float* q, double* out, uint32_t* omega,
                                uint64_t* scanned);
/* Row stride of the omega output: min(top_k, |dynamic pool|) (engine.cpp:80). */
uint32_t ra_engine_k(const ra_engine* e);
/* decode_step on HOST buffers (same shapes as ra_engine_step_device): q in,
 * out/omega/scanned back, synchronized.
 * This is the drop-in call a CPU-side engine makes. When every buffer is
 * page-locked host memory (cudaHostAlloc / cudaHostRegister / torch
 * pin_memory) the kernels read q and write the results across the bus
 * themselves (zero-copy, no separate copy operations; RA_NO_ZERO_COPY=1
 * disables); otherwise q is copied in and the results copied out. */
ra_status ra_engine_step_host(ra_engine* e, const float* q, double* out, uint32_t* omega,
                              uint64_t* scanned);
/* device-side counters of the last step (for roofline accounting) */
ra_status ra_engine_last_stats(ra_engine* e, uint64_t* total_scanned,
                               uint64_t* total_expanded);
/* CUDA-event durations of the last step's search kernel and of its
 * attention + merge kernels (recorded on the ctx stream). Synchronizes. */
ra_status ra_engine_last_timing(ra_engine* e, float* search_ms, float* attention_ms);
/* Kernel launches per decode step: 1 when the search kernel also computes the
 * attention (fused step: f32 groups, latency-mode batch), else 3 (W partials,
 * search, Omega partial + merge). RA_FUSED_ATTN=0 disables fusion. */
uint32_t ra_engine_kernels_per_step(const ra_engine* e);
/* Profiling aid: search-kernel counters of the last step summed over heads:
 * {rounds, cycles pre-expanding, cycles committing, commits, commit-phase
 * cycles in argmax / stop test / packet apply / add+compact / select, 0,0,0}. */
ra_status ra_engine_debug_counters(ra_engine* e, uint64_t* out12);
/* Profiling aid: the same 12 counters per head (out = n_heads x 12). */
ra_status ra_engine_debug_counters_per_head(ra_engine* e, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* RA_CAPI_H */
