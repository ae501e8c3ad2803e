/* CPU restatement of the RetrievalAttention decode hot path (plain C11).
 *
 * TEST INFRASTRUCTURE ONLY — the parity checker. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this; the product (paper_2409_10516_b200/) never does.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj) with the same arithmetic order, so that results are
 * bit-identical to the reference compiled with oracle/shim (pinned by
 * tests/test_oracle.py against oracle/_ref and tests/golden/).
 */
#ifndef RA_ORACLE_H
#define RA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* util.hpp:13-18 */
uint64_t ora_splitmix64(uint64_t* state);
/* util.hpp:21-28 */
uint64_t ora_mix_seed(uint64_t seed, uint64_t a, uint64_t b);

/* generate_workload (workload.cpp:102-203); output layout as
 * ref_generate_workload in oracle/ref_capi.cpp. Returns 0 or -1. */
int ora_generate_workload(uint64_t n_ctx, uint32_t d_model, uint32_t d_head,
                          uint32_t n_heads, uint32_t n_kv_groups, uint64_t seed,
                          double ood_strength, double concentration, uint64_t n_decode,
                          float* prefill_q, float* decode_q, float* keys, float* values);

typedef struct {
  uint64_t n;
  uint32_t d;
  uint32_t max_degree;
  uint32_t default_ef;
  uint64_t entry;
  uint64_t* offsets;   /* n+1 */
  uint32_t* adjacency; /* offsets[n] */
} ora_graph;

typedef struct {
  uint32_t k_train, max_degree, ef_construction, edge_window;
  int entry_maxnorm, prune_inner_product;
  uint32_t default_ef;
} ora_build_params;

/* Phase 1 alone (index_oodgraph.cpp:104-128): knn[nq][min(kt,n)] ranked
 * (score desc, id asc). */
void ora_training_knn(const float* keys, uint64_t n, uint32_t d, const float* tq,
                      uint64_t nq, uint32_t kt, uint32_t* knn);

/* OODGraph ctor + build (index_oodgraph.cpp:67-355). Returns 0, or -1 with
 * ora_last_error() = the reference's exception message. */
int ora_graph_build(const float* keys, uint64_t n, uint32_t d, const float* tq,
                    uint64_t nq, const ora_build_params* p, ora_graph* out);
void ora_graph_free(ora_graph* g);
/* OODG v1 (index_oodgraph.cpp:435-449 / 468-495). serialize returns the
 * size and writes when cap suffices; from_blob returns 0 or -1. */
uint64_t ora_graph_serialize(const ora_graph* g, char* buf, uint64_t cap);
int ora_graph_from_blob(uint64_t n_keys, uint32_t d, const char* blob, uint64_t size,
                        ora_graph* out);

/* OODGraph::search (index_oodgraph.cpp:357-411). ef < 0 => default_ef.
 * n_out = number of ids written (<= k). Optional expanded = pops. */
int ora_graph_search(const ora_graph* g, const float* keys, const float* q, uint64_t k,
                     const uint32_t* mask, uint64_t mask_n, int64_t ef, uint32_t* ids,
                     float* scores, uint64_t* n_out, uint64_t* scanned,
                     uint8_t* truncated, uint64_t* expanded);

/* FlatIndex::search (index_flat.cpp:22-43) */
int ora_flat_search(const float* keys, uint64_t n, uint32_t d, const float* q, uint64_t k,
                    const uint32_t* mask, uint64_t mask_n, uint32_t* ids, float* scores,
                    uint64_t* n_out, uint64_t* scanned);

/* partial_attention (attention.cpp:102-128) */
int ora_partial_attention(const float* q, const float* keys, const float* values,
                          uint64_t n, uint32_t d, const uint32_t* idx, uint64_t m,
                          double* out, double* zmax, double* expsum);
/* merge_gammas + merge (attention.cpp:136-157); *_empty selects empty_partial */
int ora_merge(uint32_t d, const double* ow, double zw, double sw, int w_empty,
              const double* oo, double zo, double so, int o_empty, double* out,
              double* gw, double* go);
/* static_partition (attention.cpp:87-100) */
int ora_static_partition(uint64_t t, uint64_t s_init, uint64_t s_local,
                         uint32_t* static_ids, uint64_t* n_static, uint32_t* pool_ids,
                         uint64_t* n_pool);

/* run_head (engine.cpp:69-101) without the reference MSE: search with
 * Mask{W}, partial over W and over Omega, merge. omega padded with
 * UINT32_MAX to top_k. */
int ora_run_head(const ora_graph* g, const float* keys, const float* values, uint64_t t,
                 uint32_t d, const float* q, uint64_t s_init, uint64_t s_local,
                 uint32_t top_k, int64_t ef, double* out, uint32_t* omega,
                 uint64_t* scanned);

const char* ora_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
