// Drop-in GPU backend for the reference's decode engine
// (include/attnindex/engine.hpp, header unchanged): a maintainer replaces
// src/engine.cpp with this file (next to attnindex_oodgraph_gpu.cpp and
// attnindex_attention_gpu.cpp) and links libra_b200.so.
//
// decode_step (engine.cpp:105-115) for an OODGraph engine is ONE batched
// device step over every head: search with the static set masked, partial
// attention over W and over the retrieved ids, exact merge
// (ra_engine_step_host, page-locked staging so the kernels read the queries
// and write the results across the bus). The ra_engine is created on the
// first decode_step of an EngineState and cached, keyed by the state's
// address and validated on every call against its heads' index objects and
// key / value sets (weak references). GQA heads share one device KV group
// (gpu_registry: one upload per VectorSet). Engines whose heads use the
// reference's Flat / IVF indexes run run_head's sequence per head with the
// device attention of attnindex_attention_gpu.cpp.
//
// engine_init (:23-65), decode_run (:117-155), the trace / summary writers
// (:157-181) and engine_memory (:183-194) keep the reference's behaviour
// and texts; graphs are built by ood_build, i.e. on the GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>

#include <json.hpp>

#include "attnindex/engine.hpp"
#include "attnindex/index_flat.hpp"
#include "attnindex/util.hpp"
#include "gpu_registry.hpp"
#include "ra_capi.h"

namespace attnindex {

std::string_view index_kind_name(IndexKind kind) {
  switch (kind) {
    case IndexKind::Flat: return "flat";
    case IndexKind::IVF: return "ivf";
    case IndexKind::OODGraph: return "oodgraph";
  }
  throw std::invalid_argument("bad index kind");
}

EngineState engine_init(const std::vector<HeadWorkload>& workloads, const EngineConfig& config) {
  if (workloads.empty()) throw std::invalid_argument("no heads");
  if (config.top_k < 1) throw std::invalid_argument("top_k must be >= 1");
  const uint64_t t = workloads[0].keys->n;
  if (t == 0) throw std::invalid_argument("empty context");
  for (const auto& w : workloads)
    if (w.keys->n != t || w.values->n != t)
      throw std::invalid_argument("context length mismatch across heads");
  EngineState st;
  st.config = config;
  st.t = t;
  st.heads.resize(workloads.size());
  st.decode_queries.reserve(workloads.size());
  for (size_t h = 0; h < workloads.size(); ++h) {
    const HeadWorkload& w = workloads[h];
    HeadState& hs = st.heads[h];
    hs.head_id = w.head_id;
    hs.kv_group_id = w.kv_group_id;
    hs.partition = static_partition(t, config.s_init, config.s_local);
    hs.keys = w.keys;
    hs.values = w.values;
    if (config.index_kind == IndexKind::Flat) {
      hs.index = flat_build(w.keys);
    } else if (config.index_kind == IndexKind::IVF) {
      IVFBuildParams p = config.ivf;
      p.seed = config.seed;
      hs.index = ivf_build(w.keys, p);
    } else {
      hs.index = ood_build(w.keys, w.prefill_queries, config.graph, config.n_threads);
    }
    st.decode_queries.push_back(w.decode_queries);
  }
  return st;
}

namespace {

using gpu::check;

// one cached device engine per EngineState
struct DevEngine {
  std::vector<const SearchIndex*> index;  // identity of the state's heads
  std::vector<std::weak_ptr<const VectorSet>> keys, values;
  ra_engine* e = nullptr;
  std::vector<ra_kv*> groups;  // our references
  uint32_t H = 0, d = 0, k = 0;
  // page-locked staging (zero-copy step); ra_engine_step_host also accepts
  // pageable memory if registration is unavailable
  float* q = nullptr;
  double* out = nullptr;
  uint32_t* omega = nullptr;
  uint64_t* scanned = nullptr;
  std::vector<uint8_t> pageable;
  bool pinned = false;
  std::mutex step_mu;  // one step at a time per engine (shared staging)

  ~DevEngine() {
    if (e) ra_engine_destroy(e);
    for (ra_kv* g : groups) ra_kv_release(g);
    if (pinned) ra_host_free(q);
  }
};

std::mutex g_mu;
std::map<const EngineState*, std::unique_ptr<DevEngine>> g_engines;

bool still_valid(const DevEngine& de, const EngineState& st) {
  if (de.index.size() != st.heads.size()) return false;
  for (size_t h = 0; h < st.heads.size(); ++h) {
    const HeadState& hs = st.heads[h];
    if (de.index[h] != hs.index.get() || de.keys[h].lock() != hs.keys ||
        de.values[h].lock() != hs.values)
      return false;
  }
  return true;
}

// nullptr when the heads are not all device-backed OODGraphs (or share a
// key set with different value sets): those states take the per-head path
std::unique_ptr<DevEngine> make_engine(const EngineState& st) {
  const size_t H = st.heads.size();
  std::vector<ra_graph*> graphs(H);
  for (size_t h = 0; h < H; ++h) {
    const auto* og = dynamic_cast<const OODGraph*>(st.heads[h].index.get());
    if (!og) return nullptr;
    graphs[h] = gpu::device_graph(*og);
    if (!graphs[h]) return nullptr;
  }
  auto de = std::make_unique<DevEngine>();
  de->H = uint32_t(H);
  de->d = st.heads[0].keys->d;
  for (const HeadState& hs : st.heads) {
    de->index.push_back(hs.index.get());
    de->keys.push_back(hs.keys);
    de->values.push_back(hs.values);
  }
  // GQA: contiguous runs of heads over one key set, all runs the same
  // length -> one KV group per run; anything else -> one group per head
  size_t per = 1;
  while (per < H && st.heads[per].keys == st.heads[0].keys) ++per;
  bool grouped = H % per == 0;
  for (size_t h = 0; grouped && h < H; ++h) {
    const HeadState& b = st.heads[(h / per) * per];
    grouped = st.heads[h].keys == b.keys && st.heads[h].values == b.values;
  }
  if (!grouped) per = 1;
  for (size_t g = 0; g < H / per; ++g) {
    ra_kv* kv = gpu::kv_with_values(st.heads[g * per].keys, st.heads[g * per].values);
    if (!kv) return nullptr;
    de->groups.push_back(kv);
  }
  const ra_engine_config cfg{st.config.s_init, st.config.s_local, st.config.top_k,
                             st.config.search_param ? int64_t(*st.config.search_param) : -1};
  check(ra_engine_create(gpu::thread_ctx(), de->groups.data(), uint32_t(de->groups.size()),
                         graphs.data(), uint32_t(H), &cfg, &de->e));
  de->k = ra_engine_k(de->e);
  const size_t kk = std::max<uint32_t>(de->k, 1);
  const size_t bytes = H * de->d * 4 + H * de->d * 8 + H * kk * 4 + H * 8 + 64;
  void* p = nullptr;
  de->pinned = ra_host_alloc(bytes, &p) == RA_OK;
  uint8_t* base;
  if (de->pinned) {
    base = static_cast<uint8_t*>(p);
  } else {
    de->pageable.resize(bytes);
    base = de->pageable.data();
  }
  de->q = reinterpret_cast<float*>(base);
  de->out = reinterpret_cast<double*>(base + ((H * de->d * 4 + 7) & ~size_t(7)));
  de->omega = reinterpret_cast<uint32_t*>(de->out + H * de->d);
  de->scanned = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(de->omega + H * kk) + 7) & ~uintptr_t(7));
  return de;
}

DevEngine* engine_for(const EngineState& st) {
  std::lock_guard<std::mutex> lk(g_mu);
  // drop engines whose state's key sets are gone
  for (auto it = g_engines.begin(); it != g_engines.end();) {
    bool dead = !it->second;
    if (!dead)
      for (auto& w : it->second->keys) dead = dead || w.expired();
    it = dead && it->first != &st ? g_engines.erase(it) : std::next(it);
  }
  auto it = g_engines.find(&st);
  if (it != g_engines.end() && it->second && still_valid(*it->second, st))
    return it->second.get();
  auto de = make_engine(st);
  DevEngine* raw = de.get();
  g_engines[&st] = std::move(de);
  return raw;
}

// run_head (engine.cpp:69-101) for heads without a device engine: the
// head's own index, then the device attention and merge
TraceEntry run_head_generic(const EngineState& st, uint32_t h, std::span<const float> q,
                            uint64_t step) {
  const HeadState& hs = st.heads[h];
  const auto& W = hs.partition.static_set;
  const auto& pool = hs.partition.dynamic_pool;
  TraceEntry e;
  e.step = step;
  e.head = h;
  e.w_size = W.size();
  if (!pool.empty()) {
    const size_t k = std::min<size_t>(st.config.top_k, pool.size());
    auto r = hs.index->search(q, k, Mask{W}, st.config.search_param);
    e.omega = std::move(r.ids);
    e.scanned = r.scanned;
  }
  const uint32_t d = hs.keys->d;
  const PartialAttention pw =
      W.empty() ? empty_partial(d) : partial_attention(q, *hs.keys, *hs.values, W);
  const PartialAttention po =
      e.omega.empty() ? empty_partial(d) : partial_attention(q, *hs.keys, *hs.values, e.omega);
  e.out = merge(pw, po);
  if (st.config.compute_reference) e.mse = mse(e.out, full_attention(q, *hs.keys, *hs.values));
  return e;
}

}  // namespace

std::vector<TraceEntry> decode_step(const EngineState& state,
                                    std::span<const std::span<const float>> queries,
                                    uint64_t step) {
  if (queries.size() != state.heads.size())
    throw std::invalid_argument("one query per head required");
  const size_t H = state.heads.size();
  DevEngine* de = engine_for(state);
  std::vector<TraceEntry> entries(H);
  if (!de) {
    parallel_for(H, state.config.n_threads, [&](size_t h) {
      entries[h] = run_head_generic(state, uint32_t(h), queries[h], step);
    });
    return entries;
  }
  const uint32_t d = de->d;
  for (size_t h = 0; h < H; ++h)
    if (queries[h].size() != d) throw std::invalid_argument("query dimension mismatch");
  std::lock_guard<std::mutex> lk(de->step_mu);
  for (size_t h = 0; h < H; ++h) std::memcpy(de->q + h * d, queries[h].data(), size_t(d) * 4);
  check(ra_engine_step_host(de->e, de->q, de->out, de->omega, de->scanned));
  const uint32_t k = de->k, kk = std::max<uint32_t>(k, 1);
  for (size_t h = 0; h < H; ++h) {
    TraceEntry& e = entries[h];
    e.step = step;
    e.head = uint32_t(h);
    e.w_size = state.heads[h].partition.static_set.size();
    const uint32_t* om = de->omega + h * kk;
    uint32_t n = 0;
    while (n < k && om[n] != 0xFFFFFFFFu) ++n;
    e.omega.assign(om, om + n);
    e.scanned = k ? size_t(de->scanned[h]) : 0;
    e.out.assign(de->out + h * d, de->out + (h + 1) * d);
  }
  if (state.config.compute_reference) {
    for (size_t h = 0; h < H; ++h) {
      const HeadState& hs = state.heads[h];
      entries[h].mse = mse(entries[h].out, full_attention(queries[h], *hs.keys, *hs.values));
    }
  }
  return entries;
}

DecodeResult decode_run(const EngineState& state, uint64_t n_steps) {
  for (const auto& dq : state.decode_queries)
    if (dq.n < n_steps) throw std::invalid_argument("insufficient decode queries");
  DecodeResult res;
  res.summary.n_heads = uint32_t(state.heads.size());
  res.summary.n_steps = n_steps;
  for (uint64_t s = 0; s < n_steps; ++s) {
    std::vector<std::span<const float>> qs(state.heads.size());
    for (size_t h = 0; h < qs.size(); ++h) qs[h] = state.decode_queries[h].row(s);
    for (auto& e : decode_step(state, qs, s)) res.trace.entries.push_back(std::move(e));
  }
  // summary in (step, head) order (:132-154)
  DecodeSummary& sm = res.summary;
  size_t n_mse = 0;
  for (const TraceEntry& e : res.trace.entries) {
    const uint64_t pool = state.t - e.w_size;
    sm.total_scanned += e.scanned;
    sm.mean_scanned += double(e.scanned);
    if (pool > 0) sm.mean_scan_fraction += double(e.scanned) / double(pool);
    if (e.mse) {
      ++n_mse;
      sm.mean_mse += *e.mse;
      sm.max_mse = std::max(sm.max_mse, *e.mse);
    }
  }
  const size_t n = res.trace.entries.size();
  if (n > 0) {
    sm.mean_scanned /= double(n);
    sm.mean_scan_fraction /= double(n);
  }
  if (n_mse > 0) sm.mean_mse /= double(n_mse);
  return res;
}

std::string DecodeTrace::to_jsonl(bool include_omega) const {
  std::string s;
  for (const TraceEntry& e : entries) {
    nlohmann::ordered_json j;
    j["step"] = e.step;
    j["head"] = e.head;
    if (include_omega) j["omega_ids"] = e.omega;
    j["scanned"] = e.scanned;
    if (e.mse) j["mse"] = *e.mse;
    s += j.dump();
    s += '\n';
  }
  return s;
}

std::string DecodeSummary::to_json() const {
  nlohmann::ordered_json j;
  j["n_steps"] = n_steps;
  j["n_heads"] = n_heads;
  j["mean_scan_fraction"] = mean_scan_fraction;
  j["mean_scanned"] = mean_scanned;
  j["total_scanned"] = total_scanned;
  j["mean_mse"] = mean_mse;
  j["max_mse"] = max_mse;
  return j.dump(2);
}

MemoryReport engine_memory(const EngineState& state) {
  MemoryReport r;
  std::set<const VectorSet*> seen;  // KV payload counted once per group
  for (const HeadState& hs : state.heads) {
    for (const VectorSet* v : {hs.keys.get(), hs.values.get()})
      if (seen.insert(v).second) r.kv_bytes += v->data.size() * sizeof(float);
    r.index_bytes += hs.index->memory_bytes();
  }
  return r;
}

}  // namespace attnindex
