// Drop-in GPU backend for the reference's attnindex::OODGraph.
//
// A maintainer replaces src/index_oodgraph.cpp with this file in the
// reference build (header unchanged: include/attnindex/index_oodgraph.hpp)
// and links libra_b200.so. Every member the header declares is defined
// here: the build (index_oodgraph.cpp:67-81, 89-355) and search (:357-411)
// run on the B200 through include/ra_capi.h; the CSR members the header's
// inline accessors read (offsets_, adjacency_, entry_point_, max_degree_)
// are mirrored from the GPU result, so degree()/neighbors()/serialize()
// behave exactly as before. Exceptions keep the reference's types and texts
// (ra_status INVALID_ARGUMENT -> std::invalid_argument, RUNTIME ->
// std::runtime_error).
//
// Device state: the key set is uploaded ONCE per VectorSet (gpu_registry:
// the GQA heads of a group share it, as their shared_ptr does); each
// OODGraph object's device graph lives in a registry keyed by the object
// address, validated against the object's CSR identity before use, and freed
// once the object's key set has expired. search() is re-entrant: each
// calling thread gets its own ra_ctx (stream + scratch).
#include <cstring>
#include <fstream>
#include <iterator>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "attnindex/index_oodgraph.hpp"
#include "gpu_registry.hpp"
#include "ra_capi.h"

namespace attnindex {
namespace {

using gpu::check;
using gpu::thread_ctx;

struct DevGraph {
  std::weak_ptr<const VectorSet> keys;  // the object's key set (expiry => object gone)
  const VectorSet* keys_id = nullptr;   // identity of the object's CSR + keys
  const uint32_t* adj_data = nullptr;
  size_t adj_size = 0;
  uint64_t entry = 0;
  ra_graph* g = nullptr;  // holds a reference on its ra_kv
};

std::mutex g_mu;
std::unordered_map<const void*, DevGraph> g_graphs;  // per OODGraph object

void purge_locked() {
  for (auto it = g_graphs.begin(); it != g_graphs.end();) {
    if (it->second.keys.expired()) {
      ra_graph_free(it->second.g);
      it = g_graphs.erase(it);
    } else {
      ++it;
    }
  }
}

void attach(const void* self, DevGraph d) {
  std::lock_guard<std::mutex> lk(g_mu);
  purge_locked();
  auto it = g_graphs.find(self);
  if (it != g_graphs.end() && it->second.g) ra_graph_free(it->second.g);
  g_graphs[self] = std::move(d);
}

// the attached graph if it still describes this object's CSR
ra_graph* lookup(const void* self, const std::shared_ptr<const VectorSet>& keys,
                 const std::vector<uint32_t>& adjacency, uint64_t entry) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_graphs.find(self);
  if (it != g_graphs.end() && it->second.keys_id == keys.get() &&
      it->second.keys.lock() == keys && it->second.adj_data == adjacency.data() &&
      it->second.adj_size == adjacency.size() && it->second.entry == entry)
    return it->second.g;
  return nullptr;
}

}  // namespace

OODGraph::OODGraph(std::shared_ptr<const VectorSet> keys, const VectorSet& train_queries,
                   const OODGraphBuildParams& params, int n_threads)
    : SearchIndex(std::move(keys)) {
  if (!keys_ || keys_->n == 0) throw std::invalid_argument("empty keys");
  build(train_queries, params, n_threads);
}

OODGraph::OODGraph(std::shared_ptr<const VectorSet> keys, const std::string& blob)
    : SearchIndex(std::move(keys)) {
  if (!keys_ || keys_->n == 0) throw std::invalid_argument("empty keys");
  from_blob(blob);
}

// the whole build runs on the GPU (ra_graph_build validates with the
// reference's messages); the finished CSR is mirrored into the members
void OODGraph::build(const VectorSet& tq, const OODGraphBuildParams& p, int /*n_threads*/) {
  ra_build_params bp{p.k_train,
                     p.max_degree,
                     p.ef_construction,
                     p.edge_window,
                     p.entry_strategy == EntryStrategy::MaxNorm ? 1 : 0,
                     p.prune_rule == PruneRule::InnerProduct ? 1 : 0,
                     p.default_ef};
  ra_graph* g = nullptr;
  ra_kv* kv = gpu::keys_kv(keys_);
  const ra_status st = ra_graph_build(thread_ctx(), kv, tq.n ? tq.data.data() : nullptr, tq.n,
                                      tq.d, 0, &bp, nullptr, &g);
  ra_kv_release(kv);  // the graph holds its own reference
  check(st);
  max_degree_ = p.max_degree;
  default_ef_ = p.default_ef;
  entry_point_ = ra_graph_entry_point(g);
  offsets_.assign(keys_->n + 1, 0);
  adjacency_.resize((ra_graph_memory_bytes(g) - offsets_.size() * 8) / 4);
  check(ra_graph_csr(g, offsets_.data(), adjacency_.data()));
  attach(this, DevGraph{keys_, keys_.get(), adjacency_.data(), adjacency_.size(), entry_point_, g});
}

// strict OODG v1 validation happens in ra_graph_deserialize (same texts)
void OODGraph::from_blob(const std::string& blob) {
  ra_graph* g = nullptr;
  ra_kv* kv = gpu::keys_kv(keys_);
  const ra_status st = ra_graph_deserialize(thread_ctx(), kv, blob.data(), blob.size(), &g);
  ra_kv_release(kv);
  check(st);
  max_degree_ = ra_graph_max_degree_bound(g);
  entry_point_ = ra_graph_entry_point(g);
  offsets_.assign(keys_->n + 1, 0);
  adjacency_.resize((ra_graph_memory_bytes(g) - offsets_.size() * 8) / 4);
  check(ra_graph_csr(g, offsets_.data(), adjacency_.data()));
  attach(this, DevGraph{keys_, keys_.get(), adjacency_.data(), adjacency_.size(), entry_point_, g});
}

namespace gpu {
// the object's CSR identity through its public accessors (adjacency_ starts
// at neighbors(0); its size follows from memory_bytes(), :413-415)
ra_graph* device_graph(const OODGraph& og) {
  const auto& keys = og.keys();
  const uint32_t* adj = og.neighbors(0).data();
  const size_t adj_size = (og.memory_bytes() - (keys->n + 1) * sizeof(uint64_t)) / 4;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_graphs.find(&og);
    if (it != g_graphs.end() && it->second.keys_id == keys.get() &&
        it->second.keys.lock() == keys && it->second.adj_data == adj &&
        it->second.adj_size == adj_size && it->second.entry == og.entry_point())
      return it->second.g;
  }
  // e.g. a copied object: upload its CSR once
  const std::string blob = og.serialize();
  ra_graph* g = nullptr;
  ra_kv* kv = keys_kv(keys);
  const ra_status st = ra_graph_deserialize(thread_ctx(), kv, blob.data(), blob.size(), &g);
  ra_kv_release(kv);
  check(st);
  attach(&og, DevGraph{keys, keys.get(), adj, adj_size, og.entry_point(), g});
  return g;
}
}  // namespace gpu

SearchResult OODGraph::search(std::span<const float> q, size_t k, Mask mask,
                              std::optional<uint32_t> ef) const {
  if (q.size() != keys_->d) throw std::invalid_argument("query dimension mismatch");
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  const size_t e = ef ? size_t(*ef) : size_t(default_ef_);
  if (e < k) throw std::invalid_argument("ef must be >= k");
  ra_graph* g = gpu::device_graph(*this);
  std::vector<uint32_t> ids(k);
  std::vector<float> scores(k);
  uint32_t n_out = 0;
  uint64_t scanned = 0;
  uint8_t truncated = 0;
  check(ra_graph_search_host(thread_ctx(), g, q.data(), uint32_t(q.size()), uint32_t(k),
                             int64_t(e), mask.ids.data(), mask.ids.size(), ids.data(),
                             scores.data(), &n_out, &scanned, &truncated));
  SearchResult r;
  r.ids.assign(ids.begin(), ids.begin() + n_out);
  r.scores.assign(scores.begin(), scores.begin() + n_out);
  r.scanned = scanned;
  r.truncated = truncated != 0;
  return r;
}

size_t OODGraph::memory_bytes() const {
  return offsets_.size() * sizeof(uint64_t) + adjacency_.size() * sizeof(uint32_t);
}

uint64_t OODGraph::reachable_count() const {
  std::vector<uint8_t> seen(keys_->n, 0);
  std::vector<uint32_t> todo{uint32_t(entry_point_)};
  seen[entry_point_] = 1;
  uint64_t reached = 1;
  while (!todo.empty()) {
    const uint32_t u = todo.back();
    todo.pop_back();
    for (uint64_t j = offsets_[u]; j < offsets_[u + 1]; ++j) {
      const uint32_t v = adjacency_[j];
      if (!seen[v]) {
        seen[v] = 1;
        ++reached;
        todo.push_back(v);
      }
    }
  }
  return reached;
}

std::string OODGraph::serialize() const {
  ra_graph* g = lookup(this, keys_, adjacency_, entry_point_);
  if (g) {  // byte format produced by the library (OODG v1)
    uint64_t size = 0;
    check(ra_graph_serialize(g, nullptr, 0, &size));
    std::string out(size, '\0');
    check(ra_graph_serialize(g, out.data(), size, &size));
    return out;
  }
  std::string out;  // host-only object: encode the mirrored CSR directly
  auto put = [&](const void* p, size_t b) { out.append(static_cast<const char*>(p), b); };
  const uint32_t version = 1;
  const uint64_t n = keys_->n;
  put("OODG", 4);
  put(&version, 4);
  put(&n, 8);
  put(&max_degree_, 4);
  put(&entry_point_, 8);
  for (uint64_t u = 0; u < n; ++u) {
    const uint32_t deg = degree(u);
    put(&deg, 4);
    for (uint32_t v : neighbors(u)) {
      const uint64_t w = v;
      put(&w, 8);
    }
  }
  return out;
}

void OODGraph::save(const std::filesystem::path& path) const {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw std::runtime_error("cannot open " + path.string());
  const std::string b = serialize();
  f.write(b.data(), std::streamsize(b.size()));
  if (!f) throw std::runtime_error("write failed: " + path.string());
}

std::unique_ptr<OODGraph> OODGraph::load(std::shared_ptr<const VectorSet> keys,
                                         const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path.string());
  std::string blob((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  return std::make_unique<OODGraph>(std::move(keys), blob);
}

std::unique_ptr<OODGraph> ood_build(std::shared_ptr<const VectorSet> keys,
                                    const VectorSet& train_queries,
                                    const OODGraphBuildParams& params, int n_threads) {
  return std::make_unique<OODGraph>(std::move(keys), train_queries, params, n_threads);
}

}  // namespace attnindex
