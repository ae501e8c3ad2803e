// C-ABI shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/ (as the parity checker) and by
// bench.py's cpu_baseline / --impl reference legs (as the timed reference
// CPU path). Nothing in paper_2409_10516_b200/ links or loads this.
//
// Every entry point returns 0 on success or -1 with ref_last_error() set to
// the reference exception's what() — the same messages the reference tests
// assert (e.g. test_index_oodgraph.cpp:384-400).
#include <chrono>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <set>
#include <cstring>
#include <memory>
#include <numeric>
#include <optional>
#include <span>
#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "attnindex/attention.hpp"
#include "attnindex/engine.hpp"
#include "attnindex/index_flat.hpp"
#include "attnindex/index_oodgraph.hpp"
#include "attnindex/util.hpp"
#include "attnindex/index_ivf.hpp"
#include "attnindex/io.hpp"
#include "attnindex/workload.hpp"

#include <json.hpp>

using namespace attnindex;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
  } catch (const std::runtime_error& e) {
    g_err = std::string("runtime_error: ") + e.what();
  } catch (const std::exception& e) {
    g_err = std::string("exception: ") + e.what();
  }
  return -1;
}

std::shared_ptr<const VectorSet> make_set(Role role, const float* p, uint64_t n,
                                          uint32_t d) {
  auto s = std::make_shared<VectorSet>(role, n, d);
  if (n) std::memcpy(s->data.data(), p, sizeof(float) * n * d);
  return s;
}

struct RefGraph {
  std::shared_ptr<const VectorSet> keys;
  std::unique_ptr<OODGraph> g;
};

void copy_result(const SearchResult& r, uint32_t* ids, float* scores,
                 uint64_t* n_out, uint64_t* scanned, uint8_t* truncated) {
  std::copy(r.ids.begin(), r.ids.end(), ids);
  std::copy(r.scores.begin(), r.scores.end(), scores);
  *n_out = r.ids.size();
  *scanned = r.scanned;
  *truncated = r.truncated ? 1 : 0;
}

// Decode-step harness for the CPU baseline: engine_init's per-head state,
// but with graphs loaded from OODG blobs (index_oodgraph.hpp:40) so 128K
// graphs need not be rebuilt on the CPU.
struct RefEngine {
  EngineState st;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_splitmix64(uint64_t* state) { return splitmix64(*state); }

// generate_workload (workload.cpp:102-203). Outputs, all f32 row-major:
// prefill_q[n_heads][n_ctx][d_head], decode_q[n_heads][n_decode][d_head],
// keys[n_kv_groups][n_ctx][d_head], values[n_kv_groups][n_ctx][d_head].
int ref_generate_workload(uint64_t n_ctx, uint32_t d_model, uint32_t d_head,
                          uint32_t n_heads, uint32_t n_kv_groups, uint64_t seed,
                          double ood_strength, double concentration, uint64_t n_decode,
                          int n_threads, float* prefill_q, float* decode_q, float* keys,
                          float* values) {
  return guard([&] {
    WorkloadSpec s;
    s.n_ctx = n_ctx;
    s.d_model = d_model;
    s.d_head = d_head;
    s.n_heads = n_heads;
    s.n_kv_groups = n_kv_groups;
    s.seed = seed;
    s.ood_strength = ood_strength;
    s.concentration = concentration;
    s.n_decode = n_decode;
    auto heads = generate_workload(s, n_threads);
    const size_t per_ctx = size_t(n_ctx) * d_head, per_dec = size_t(n_decode) * d_head;
    for (uint32_t h = 0; h < n_heads; ++h) {
      std::memcpy(prefill_q + h * per_ctx, heads[h].prefill_queries.data.data(),
                  per_ctx * sizeof(float));
      std::memcpy(decode_q + h * per_dec, heads[h].decode_queries.data.data(),
                  per_dec * sizeof(float));
      const uint32_t g = heads[h].kv_group_id;
      std::memcpy(keys + g * per_ctx, heads[h].keys->data.data(), per_ctx * sizeof(float));
      std::memcpy(values + g * per_ctx, heads[h].values->data.data(),
                  per_ctx * sizeof(float));
    }
  });
}

// generate_workload + save_workloads (io.cpp:143-177) into dir: the KVD1
// byte-format fixture for tests/test_kvd1.py
int ref_save_workloads(uint64_t n_ctx, uint32_t d_model, uint32_t d_head, uint32_t n_heads,
                       uint32_t n_kv_groups, uint64_t seed, uint64_t n_decode, const char* dir) {
  return guard([&] {
    WorkloadSpec s;
    s.n_ctx = n_ctx;
    s.d_model = d_model;
    s.d_head = d_head;
    s.n_heads = n_heads;
    s.n_kv_groups = n_kv_groups;
    s.seed = seed;
    s.n_decode = n_decode;
    auto heads = generate_workload(s, 1);
    save_workloads(heads, n_kv_groups, dir);
  });
}

// load_workloads + load_vectors error text for a file (empty on success)
int ref_load_vectors_check(const char* path) {
  return guard([&] { (void)load_vectors(path); });
}

int ref_graph_build(const float* keys, uint64_t n, uint32_t d, const float* train_q,
                    uint64_t nq, uint32_t k_train, uint32_t max_degree,
                    uint32_t ef_construction, uint32_t edge_window, int entry_maxnorm,
                    int prune_inner_product, uint32_t default_ef, int n_threads,
                    void** out) {
  return guard([&] {
    auto h = std::make_unique<RefGraph>();
    h->keys = make_set(Role::Key, keys, n, d);
    VectorSet tq(Role::Query, nq, d);
    if (nq) std::memcpy(tq.data.data(), train_q, sizeof(float) * nq * d);
    OODGraphBuildParams p;
    p.k_train = k_train;
    p.max_degree = max_degree;
    p.ef_construction = ef_construction;
    p.edge_window = edge_window;
    p.entry_strategy = entry_maxnorm ? EntryStrategy::MaxNorm : EntryStrategy::Medoid;
    p.prune_rule = prune_inner_product ? PruneRule::InnerProduct : PruneRule::Euclidean;
    p.default_ef = default_ef;
    h->g = ood_build(h->keys, tq, p, n_threads);
    *out = h.release();
  });
}

int ref_graph_from_blob(const float* keys, uint64_t n, uint32_t d, const char* blob,
                        uint64_t size, void** out) {
  return guard([&] {
    auto h = std::make_unique<RefGraph>();
    h->keys = make_set(Role::Key, keys, n, d);
    h->g = std::make_unique<OODGraph>(h->keys, std::string(blob, size));
    *out = h.release();
  });
}

void ref_graph_free(void* g) { delete static_cast<RefGraph*>(g); }

// Writes the OODG v1 blob (index_oodgraph.cpp:435-449) when cap suffices;
// always reports the size.
int ref_graph_serialize(void* g, char* buf, uint64_t cap, uint64_t* size) {
  return guard([&] {
    const std::string b = static_cast<RefGraph*>(g)->g->serialize();
    *size = b.size();
    if (buf && cap >= b.size()) std::memcpy(buf, b.data(), b.size());
  });
}

uint64_t ref_graph_entry(void* g) { return static_cast<RefGraph*>(g)->g->entry_point(); }

int ref_graph_search(void* g, const float* q, uint32_t d, uint64_t k,
                     const uint32_t* mask, uint64_t mask_n, int64_t ef, uint32_t* ids,
                     float* scores, uint64_t* n_out, uint64_t* scanned,
                     uint8_t* truncated) {
  return guard([&] {
    const auto& G = *static_cast<RefGraph*>(g)->g;
    std::optional<uint32_t> ef_opt;
    if (ef >= 0) ef_opt = uint32_t(ef);
    auto r = G.search(std::span<const float>(q, d), k,
                      Mask{std::span<const uint32_t>(mask, mask_n)}, ef_opt);
    copy_result(r, ids, scores, n_out, scanned, truncated);
  });
}

int ref_flat_search(const float* keys, uint64_t n, uint32_t d, const float* q, uint64_t k,
                    const uint32_t* mask, uint64_t mask_n, uint32_t* ids, float* scores,
                    uint64_t* n_out, uint64_t* scanned) {
  return guard([&] {
    auto ks = make_set(Role::Key, keys, n, d);
    FlatIndex f(ks);
    auto r = f.search(std::span<const float>(q, d), k,
                      Mask{std::span<const uint32_t>(mask, mask_n)});
    uint8_t t;
    copy_result(r, ids, scores, n_out, scanned, &t);
  });
}

// partial_attention (attention.cpp:102-128); out has d doubles.
int ref_partial_attention(const float* q, const float* keys, const float* values,
                          uint64_t n, uint32_t d, const uint32_t* idx, uint64_t m,
                          double* out, double* zmax, double* expsum) {
  return guard([&] {
    VectorSet K(Role::Key, n, d), V(Role::Value, n, d);
    std::memcpy(K.data.data(), keys, sizeof(float) * n * d);
    std::memcpy(V.data.data(), values, sizeof(float) * n * d);
    auto p = partial_attention(std::span<const float>(q, d), K, V,
                               std::span<const uint32_t>(idx, m));
    std::copy(p.out.begin(), p.out.end(), out);
    *zmax = p.zmax;
    *expsum = p.expsum;
  });
}

// merge (attention.cpp:149-157); a side with empty != 0 is empty_partial(d).
int ref_merge(uint32_t d, const double* ow, double zw, double sw, int w_empty,
              const double* oo, double zo, double so, int o_empty, double* out,
              double* gw, double* go) {
  return guard([&] {
    PartialAttention pw, po;
    pw.out.assign(ow, ow + d);
    pw.zmax = zw;
    pw.expsum = sw;
    pw.empty = w_empty != 0;
    po.out.assign(oo, oo + d);
    po.zmax = zo;
    po.expsum = so;
    po.empty = o_empty != 0;
    if (pw.empty) pw = empty_partial(d);
    if (po.empty) po = empty_partial(d);
    auto [a, b] = merge_gammas(pw, po);
    *gw = a;
    *go = b;
    auto r = merge(pw, po);
    std::copy(r.begin(), r.end(), out);
  });
}

int ref_static_partition(uint64_t t, uint64_t s_init, uint64_t s_local,
                         uint32_t* static_ids, uint64_t* n_static, uint32_t* pool_ids,
                         uint64_t* n_pool) {
  return guard([&] {
    auto p = static_partition(t, s_init, s_local);
    if (static_ids) std::copy(p.static_set.begin(), p.static_set.end(), static_ids);
    if (pool_ids) std::copy(p.dynamic_pool.begin(), p.dynamic_pool.end(), pool_ids);
    *n_static = p.static_set.size();
    *n_pool = p.dynamic_pool.size();
  });
}

// ---- decode engine over blob-loaded graphs (engine.cpp:69-115) -------------
// keys/values: [n_groups][t][d]; head h uses group h / (n_heads / n_groups);
// blobs: concatenated OODG blobs, one per head, sizes in blob_sizes.
int ref_engine_create(const float* keys, const float* values, uint64_t t, uint32_t d,
                      uint32_t n_heads, uint32_t n_groups, const char* blobs,
                      const uint64_t* blob_sizes, uint64_t s_init, uint64_t s_local,
                      uint32_t top_k, int64_t ef, int n_threads, void** out) {
  return guard([&] {
    auto e = std::make_unique<RefEngine>();
    EngineConfig& c = e->st.config;
    c.s_init = s_init;
    c.s_local = s_local;
    c.top_k = top_k;
    c.index_kind = IndexKind::OODGraph;
    if (ef >= 0) c.search_param = uint32_t(ef);
    c.n_threads = n_threads;
    e->st.t = t;
    std::vector<std::shared_ptr<const VectorSet>> K(n_groups), V(n_groups);
    for (uint32_t g = 0; g < n_groups; ++g) {
      K[g] = make_set(Role::Key, keys + size_t(g) * t * d, t, d);
      V[g] = make_set(Role::Value, values + size_t(g) * t * d, t, d);
    }
    const uint32_t per = n_heads / n_groups;
    size_t off = 0;
    e->st.heads.resize(n_heads);
    for (uint32_t h = 0; h < n_heads; ++h) {
      HeadState& hs = e->st.heads[h];
      hs.head_id = h;
      hs.kv_group_id = h / per;
      hs.partition = static_partition(t, s_init, s_local);
      hs.keys = K[h / per];
      hs.values = V[h / per];
      hs.index = std::make_unique<OODGraph>(hs.keys, std::string(blobs + off, blob_sizes[h]));
      off += blob_sizes[h];
    }
    *out = e.release();
  });
}

// The reference's whole decode setup, nothing from this repo:
// generate_workload (workload.cpp:102-203) + engine_init (engine.cpp:23-65,
// OODGraph kind: static_partition + ood_build per head over the group's
// shared keys). build_workers <= 1 is engine_init itself (heads built one
// after another, each ood_build with n_threads); build_workers > 1 builds
// that many heads at once through the same public ood_build
// (index_oodgraph.hpp:78-81), n_threads / build_workers threads each, to
// overlap the builder's serial phase-2 sort. decode_q receives
// [n_heads][n_decode][d_head]; keys / values (nullable) [n_groups][n_ctx][d].
int ref_engine_from_workload(uint64_t n_ctx, uint32_t n_heads, uint32_t n_kv_groups,
                             uint64_t seed, uint64_t n_decode, uint32_t k_train,
                             uint32_t max_degree, uint32_t ef_construction,
                             uint32_t edge_window, uint64_t s_init, uint64_t s_local,
                             uint32_t top_k, int64_t ef, int n_threads, int build_workers,
                             float* decode_q, float* keys, float* values, double* ms_gen,
                             double* ms_build, void** out) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    WorkloadSpec s;
    s.n_ctx = n_ctx;
    s.n_heads = n_heads;
    s.n_kv_groups = n_kv_groups;
    s.seed = seed;
    s.n_decode = n_decode;
    auto t0 = clk::now();
    auto w = generate_workload(s, n_threads);
    auto t1 = clk::now();
    EngineConfig c;
    c.s_init = s_init;
    c.s_local = s_local;
    c.top_k = top_k;
    c.index_kind = IndexKind::OODGraph;
    c.graph.k_train = k_train;
    c.graph.max_degree = max_degree;
    c.graph.ef_construction = ef_construction;
    c.graph.edge_window = edge_window;
    if (ef >= 0) c.search_param = uint32_t(ef);
    c.n_threads = n_threads;
    auto e = std::make_unique<RefEngine>();
    if (build_workers <= 1) {
      e->st = engine_init(w, c);
    } else {
      e->st.config = c;
      e->st.t = n_ctx;
      e->st.heads.resize(w.size());
      for (size_t h = 0; h < w.size(); ++h) {
        HeadState& hs = e->st.heads[h];
        hs.head_id = w[h].head_id;
        hs.kv_group_id = w[h].kv_group_id;
        hs.partition = static_partition(n_ctx, s_init, s_local);
        hs.keys = w[h].keys;
        hs.values = w[h].values;
        e->st.decode_queries.push_back(w[h].decode_queries);
      }
      const int per = std::max(1, n_threads / build_workers);
      parallel_for(w.size(), build_workers, [&](size_t h) {
        e->st.heads[h].index = ood_build(w[h].keys, w[h].prefill_queries, c.graph, per);
      });
    }
    auto t2 = clk::now();
    const uint32_t d = s.d_head;
    const size_t per_dec = size_t(n_decode) * d, per_ctx = size_t(n_ctx) * d;
    for (uint32_t h = 0; h < n_heads; ++h) {
      std::memcpy(decode_q + h * per_dec, w[h].decode_queries.data.data(),
                  per_dec * sizeof(float));
      const uint32_t g = w[h].kv_group_id;
      if (keys)
        std::memcpy(keys + g * per_ctx, w[h].keys->data.data(), per_ctx * sizeof(float));
      if (values)
        std::memcpy(values + g * per_ctx, w[h].values->data.data(), per_ctx * sizeof(float));
    }
    if (ms_gen) *ms_gen = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (ms_build) *ms_build = std::chrono::duration<double, std::milli>(t2 - t1).count();
    *out = e.release();
  });
}

// OODG blob of head h of an engine (the parity artefact of its graph)
int ref_engine_graph_serialize(void* e, uint32_t h, char* buf, uint64_t cap, uint64_t* size) {
  return guard([&] {
    const auto& st = static_cast<RefEngine*>(e)->st;
    const auto* g = dynamic_cast<const OODGraph*>(st.heads.at(h).index.get());
    if (!g) throw std::runtime_error("not an OODGraph head");
    const std::string b = g->serialize();
    *size = b.size();
    if (buf && cap >= b.size()) std::memcpy(buf, b.data(), b.size());
  });
}

void ref_engine_free(void* e) { delete static_cast<RefEngine*>(e); }

// One decode_step over all heads: q [n_heads][d] -> out [n_heads][d] f64,
// omega ids [n_heads][top_k] (UINT32_MAX padded), scanned [n_heads].
int ref_engine_step(void* e, const float* q, uint64_t step, double* out, uint32_t* omega,
                    uint64_t* scanned) {
  return guard([&] {
    const auto& st = static_cast<RefEngine*>(e)->st;
    const uint32_t d = st.heads[0].keys->d;
    std::vector<std::span<const float>> qs(st.heads.size());
    for (size_t h = 0; h < qs.size(); ++h) qs[h] = std::span<const float>(q + h * d, d);
    auto entries = decode_step(st, qs, step);
    const uint32_t k = st.config.top_k;
    for (size_t h = 0; h < entries.size(); ++h) {
      if (out) std::copy(entries[h].out.begin(), entries[h].out.end(), out + h * d);
      if (omega) {
        for (uint32_t i = 0; i < k; ++i)
          omega[h * k + i] = i < entries[h].omega.size() ? entries[h].omega[i] : UINT32_MAX;
      }
      if (scanned) scanned[h] = entries[h].scanned;
    }
  });
}

// decode_run (engine.cpp:117-155) over stored decode queries
// [n_heads][n_steps][d]: the trace JSONL (to_jsonl) and summary JSON (to_json)
// copied into caller buffers (lengths returned; call with cap 0 to size).
int ref_engine_run(void* e, const float* dq, uint64_t n_steps, int compute_reference,
                   int include_omega, char* jsonl, uint64_t cap1, uint64_t* len1,
                   char* summary, uint64_t cap2, uint64_t* len2, double* mse_out) {
  return guard([&] {
    auto& st = static_cast<RefEngine*>(e)->st;
    const uint32_t d = st.heads[0].keys->d;
    st.config.compute_reference = compute_reference != 0;
    st.decode_queries.clear();
    for (size_t h = 0; h < st.heads.size(); ++h)
      st.decode_queries.push_back(*make_set(Role::Query, dq + h * n_steps * d, n_steps, d));
    auto r = decode_run(st, n_steps);
    const std::string a = r.trace.to_jsonl(include_omega != 0), b = r.summary.to_json();
    *len1 = a.size();
    *len2 = b.size();
    if (jsonl && cap1 >= a.size()) std::memcpy(jsonl, a.data(), a.size());
    if (summary && cap2 >= b.size()) std::memcpy(summary, b.data(), b.size());
    if (mse_out)
      for (size_t i = 0; i < r.trace.entries.size(); ++i)
        mse_out[i] = r.trace.entries[i].mse ? *r.trace.entries[i].mse : -1.0;
  });
}

// IVFIndex (index_ivf.cpp): build, export (centroids, offsets, ids), search
int ref_ivf_build(const float* keys, uint64_t n, uint32_t d, uint32_t nlist, uint64_t seed,
                  uint32_t iters, uint32_t default_nprobe, void** out) {
  return guard([&] {
    IVFBuildParams p;
    p.nlist = nlist;
    p.seed = seed;
    p.iters = iters;
    p.default_nprobe = default_nprobe;
    auto ks = make_set(Role::Key, keys, n, d);
    *out = ivf_build(ks, p).release();
  });
}
void ref_ivf_free(void* h) { delete static_cast<IVFIndex*>(h); }
uint32_t ref_ivf_nlist(void* h) { return static_cast<IVFIndex*>(h)->nlist(); }
int ref_ivf_export(void* h, float* cent, uint32_t* offsets, uint32_t* ids) {
  return guard([&] {
    auto* ix = static_cast<IVFIndex*>(h);
    const uint32_t d = ix->keys()->d;
    uint32_t o = 0;
    for (uint32_t c = 0; c < ix->nlist(); ++c) {
      auto cr = ix->centroid(c);
      std::copy(cr.begin(), cr.end(), cent + size_t(c) * d);
      offsets[c] = o;
      for (uint32_t id : ix->list(c)) ids[o++] = id;
    }
    offsets[ix->nlist()] = o;
  });
}
int ref_ivf_search(void* h, const float* q, uint32_t d, uint64_t k, const uint32_t* mask,
                   uint64_t mask_n, int64_t nprobe, uint32_t* ids, float* scores,
                   uint64_t* n_out, uint64_t* scanned, uint8_t* truncated) {
  return guard([&] {
    auto* ix = static_cast<IVFIndex*>(h);
    std::optional<uint32_t> np;
    if (nprobe >= 0) np = uint32_t(nprobe);
    auto r = ix->search(std::span<const float>(q, d), k,
                        Mask{std::span<const uint32_t>(mask, mask_n)}, np);
    std::copy(r.ids.begin(), r.ids.end(), ids);
    std::copy(r.scores.begin(), r.scores.end(), scores);
    *n_out = r.ids.size();
    *scanned = r.scanned;
    *truncated = r.truncated;
  });
}

// cmd_build (tools/main.cpp:401-480) restated over the reference library:
// the workload comes from manifest_path (acquire_workloads' manifest branch,
// main.cpp:344-358), every head's index is built with the reference's own
// builders (build_index, main.cpp:360-374), artifacts and build_report.json
// go to out_dir. kind: 0 flat, 1 ivf, 2 oodgraph. Verify counters are the
// VerifyLog's (main.cpp:308-321): checks made, checks failed.
int ref_build_report(const char* manifest_path, const char* out_dir, int kind, uint32_t k_train,
                     uint32_t max_degree, uint32_t ef_construction, uint32_t edge_window,
                     uint32_t nlist, uint64_t seed, uint32_t iters, uint32_t default_nprobe,
                     int n_threads, int verify, uint64_t* checks, uint64_t* failures) {
  namespace fs = std::filesystem;
  using nlohmann::json;
  return guard([&] {
    uint64_t n_checks = 0, n_fail = 0;
    auto check = [&](bool ok) {
      if (!verify) return;
      ++n_checks;
      n_fail += !ok;
    };
    auto heads = load_workloads(manifest_path);
    if (heads.empty()) throw std::runtime_error("workload has no heads");
    fs::path dir(out_dir);
    fs::create_directories(dir);
    const IndexKind ik = kind == 0 ? IndexKind::Flat : kind == 1 ? IndexKind::IVF : IndexKind::OODGraph;
    json report;
    report["kind"] = std::string(index_kind_name(ik));
    report["n_heads"] = heads.size();
    report["n_keys"] = heads[0].keys->n;
    json per_head = json::array();
    std::set<const VectorSet*> counted;
    size_t kv_bytes = 0, index_bytes = 0;
    for (const auto& h : heads) {
      std::unique_ptr<SearchIndex> idx;
      if (ik == IndexKind::Flat) {
        idx = flat_build(h.keys);
      } else if (ik == IndexKind::IVF) {
        IVFBuildParams p;
        p.nlist = nlist;
        p.seed = seed;
        p.iters = iters;
        p.default_nprobe = default_nprobe;
        idx = ivf_build(h.keys, p);
      } else {
        OODGraphBuildParams p;
        p.k_train = k_train;
        p.max_degree = max_degree;
        p.ef_construction = ef_construction;
        p.edge_window = edge_window;
        idx = ood_build(h.keys, h.prefill_queries, p, n_threads);
      }
      json entry;
      entry["head"] = h.head_id;
      entry["kv_group"] = h.kv_group_id;
      if (const auto* g = dynamic_cast<const OODGraph*>(idx.get())) {
        std::string name = "head" + std::to_string(h.head_id) + ".oodg";
        g->save(dir / name);
        entry["artifact"] = name;
        uint64_t edges = 0;
        std::vector<uint64_t> hist(g->max_degree_bound() + 1, 0);
        for (uint64_t u = 0; u < g->size(); ++u) {
          edges += g->degree(u);
          hist[g->degree(u)] += 1;
        }
        entry["edges"] = edges;
        entry["degree_histogram"] = hist;
        entry["entry_point"] = g->entry_point();
        check(g->reachable_count() == g->size());
        auto back = OODGraph::load(h.keys, dir / name);
        check(back->serialize() == g->serialize());
      } else if (const auto* ivf = dynamic_cast<const IVFIndex*>(idx.get())) {
        entry["artifact"] = nullptr;
        entry["nlist"] = ivf->nlist();
        std::vector<char> seen(ivf->size(), 0);
        uint64_t total = 0;
        bool ok = true;
        for (uint32_t c = 0; c < ivf->nlist(); ++c)
          for (uint32_t id : ivf->list(c)) {
            if (id >= ivf->size() || seen[id]) ok = false;
            else seen[id] = 1;
            ++total;
          }
        check(ok && total == ivf->size());
      } else {
        entry["artifact"] = nullptr;
        entry["note"] = "no preprocessing";
      }
      entry["memory_bytes"] = idx->memory_bytes();
      index_bytes += idx->memory_bytes();
      if (counted.insert(h.keys.get()).second) kv_bytes += h.keys->data.size() * sizeof(float);
      if (counted.insert(h.values.get()).second) kv_bytes += h.values->data.size() * sizeof(float);
      per_head.push_back(std::move(entry));
    }
    report["heads"] = std::move(per_head);
    report["kv_bytes"] = kv_bytes;
    report["index_bytes"] = index_bytes;
    std::ofstream out(dir / "build_report.json", std::ios::binary | std::ios::trunc);
    out << report.dump(2) + "\n";
    if (!out) throw std::runtime_error("write failed");
    *checks = n_checks;
    *failures = n_fail;
  });
}

// recall_sweep + SweepReport::to_csv / to_jsonl (diagnostics.cpp:132-225)
// restated over the reference library (diagnostics.cpp itself needs Eigen
// LLT / HouseholderQR for its Mahalanobis parts, which the shim lacks).
// kind: 0 flat, 1 ivf, 2 oodgraph. Writes the CSV then the JSONL, each
// NUL-terminated, into buf (cap bytes).
int ref_recall_sweep(const float* keys, uint64_t n, uint32_t d, const float* pq, uint64_t npq,
                     const float* dq, uint64_t nq, int kind, const uint32_t* grid, uint32_t ngrid,
                     uint64_t k, uint32_t nlist, uint64_t seed, uint32_t iters, uint32_t nprobe,
                     uint32_t k_train, uint32_t max_degree, uint32_t efc, uint32_t window,
                     int n_threads, char* buf, uint64_t cap) {
  return guard([&] {
    auto ks = make_set(Role::Key, keys, n, d);
    VectorSet pre(Role::Query, npq, d), dec(Role::Query, nq, d);
    if (npq) std::memcpy(pre.data.data(), pq, sizeof(float) * npq * d);
    if (nq) std::memcpy(dec.data.data(), dq, sizeof(float) * nq * d);
    if (nq == 0) throw std::invalid_argument("no decode queries");
    if (k < 1 || k > n) throw std::invalid_argument("k out of range");
    auto recall = [](std::span<const uint32_t> got, std::span<const uint32_t> truth) {
      std::vector<uint32_t> sorted(truth.begin(), truth.end());
      std::sort(sorted.begin(), sorted.end());
      size_t hits = 0;
      for (uint32_t id : got)
        if (std::binary_search(sorted.begin(), sorted.end(), id)) ++hits;
      return double(hits) / double(truth.size());
    };
    FlatIndex flat(ks);
    std::vector<std::vector<uint32_t>> truth(nq);
    for (uint64_t i = 0; i < nq; ++i) truth[i] = flat.search(dec.row(i), k).ids;
    struct Row { std::string kind; uint32_t param; double rec, scan; uint64_t nq; };
    std::vector<Row> rows;
    auto add_rows = [&](const SearchIndex& idx, std::vector<uint32_t> g) {
      for (uint32_t param : g) {
        std::vector<double> rec(nq), scan(nq);
        for (uint64_t i = 0; i < nq; ++i) {
          auto r = idx.search(dec.row(i), k, {},
                              param ? std::optional<uint32_t>(param) : std::nullopt);
          rec[i] = recall(r.ids, truth[i]);
          scan[i] = double(r.scanned) / double(n);
        }
        rows.push_back({std::string(idx.kind()), param,
                        std::accumulate(rec.begin(), rec.end(), 0.0) / double(nq),
                        std::accumulate(scan.begin(), scan.end(), 0.0) / double(nq), nq});
      }
    };
    std::vector<uint32_t> gv(grid, grid + ngrid);
    if (kind == 0) {
      add_rows(flat, {0u});
    } else {
      if (gv.empty()) throw std::invalid_argument("empty parameter grid");
      for (uint32_t g : gv)
        if (g < 1) throw std::invalid_argument("grid values must be >= 1");
      if (kind == 1) {
        IVFBuildParams p;
        p.nlist = nlist, p.seed = seed, p.iters = iters, p.default_nprobe = nprobe;
        auto idx = ivf_build(ks, p);
        add_rows(*idx, gv);
      } else {
        OODGraphBuildParams p;
        p.k_train = k_train, p.max_degree = max_degree, p.ef_construction = efc;
        p.edge_window = window;
        auto idx = ood_build(ks, pre, p, n_threads);
        add_rows(*idx, gv);
      }
    }
    auto fmt = [](double v) {
      char b[40];
      std::snprintf(b, sizeof b, "%.10g", v);
      return std::string(b);
    };
    std::string csv = "index_kind,param,recall_at_k,scan_fraction,n_queries\n", jl;
    for (const auto& r : rows) {
      csv += r.kind + ',' + std::to_string(r.param) + ',' + fmt(r.rec) + ',' + fmt(r.scan) + ',' +
             std::to_string(r.nq) + '\n';
      nlohmann::ordered_json j;
      j["index_kind"] = r.kind;
      j["param"] = r.param;
      j["recall_at_k"] = r.rec;
      j["scan_fraction"] = r.scan;
      j["n_queries"] = r.nq;
      jl += j.dump() + '\n';
    }
    if (csv.size() + jl.size() + 2 > cap) throw std::runtime_error("buffer too small");
    std::memcpy(buf, csv.c_str(), csv.size() + 1);
    std::memcpy(buf + csv.size() + 1, jl.c_str(), jl.size() + 1);
  });
}

}  // extern "C"
