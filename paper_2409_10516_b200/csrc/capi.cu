// C ABI of libra_b200.so (include/ra_capi.h): handles, validation with the
// reference's error texts, OODG v1 (de)serialization, and the decode engine
// that strings K6 (search) and K7 (partials + merge) together per step.
#include <algorithm>
#include <cstring>
#include <memory>
#include <cmath>
#include <numeric>

#include "common.cuh"

namespace ra {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

void graph_upload(ra_ctx* ctx, ra_graph* g) {
  const uint64_t n = g->n;
  const uint32_t M = g->max_degree;
  std::vector<uint32_t> rows(size_t(n) * M, kSentinel);
  for (uint64_t u = 0; u < n; ++u)
    std::copy(g->adjacency.begin() + g->offsets[u], g->adjacency.begin() + g->offsets[u + 1],
              rows.begin() + u * M);
  if (g->adj.n != rows.size()) g->adj.alloc(rows.size());  // (a build re-uploads in place)
  RA_CUDA(cudaMemcpyAsync(g->adj.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice,
                          ctx->stream));
  RA_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace ra

// the reference CSR from the device rows (kSentinel-padded), once
void ra_graph::host_mirror() const {
  std::call_once(host_once, [this] {
    if (offsets.size() == n + 1) return;  // deserialized: the mirror came first
    std::vector<uint32_t> rows(size_t(n) * max_degree);
    {
      ra::DeviceGuard dg(kv ? kv->device : 0);  // (a build synchronizes its stream before returning)
      RA_CUDA(cudaMemcpy(rows.data(), adj.p, rows.size() * 4, cudaMemcpyDeviceToHost));
    }
    offsets.assign(size_t(n) + 1, 0);
    adjacency.clear();
    adjacency.reserve(n_edges);
    for (uint64_t u = 0; u < n; ++u) {
      const uint32_t* r = rows.data() + u * max_degree;
      uint32_t dg = 0;
      while (dg < max_degree && r[dg] != ra::kSentinel) adjacency.push_back(r[dg++]);
      offsets[u + 1] = offsets[u] + dg;
    }
  });
}

namespace ra {

static void check_ctx(ra_ctx* ctx) {
  if (!ctx) invalid("null context");
}

}  // namespace ra

using namespace ra;

extern "C" {

const char* ra_last_error(void) { return g_last_error.c_str(); }
const char* ra_version(void) { return "ra_b200 0.1 (sm_100a)"; }

// ---- context ----------------------------------------------------------------
ra_status ra_ctx_create(int device, ra_ctx** out) {
  return guard([&] {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw Error(RA_ERR_CUDA, "no CUDA device available (libra_b200 has no CPU fallback)");
    if (device < 0 || device >= count) invalid("device index out of range");
    cudaDeviceProp prop{};
    RA_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw Error(RA_ERR_CUDA, std::string("libra_b200 is built for sm_100a; device is ") +
                                   prop.name);
    auto c = std::make_unique<ra_ctx>();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    // stream-ordered scratch (DevBuf(count, stream)) stays cached in the
    // default pool between calls instead of going back to the driver
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = 32ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = c.release();
  });
}

void ra_ctx_destroy(ra_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dg(ctx->device, true);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->side) cudaStreamSynchronize(ctx->side), cudaStreamDestroy(ctx->side);
  if (ctx->side_fork) cudaEventDestroy(ctx->side_fork);
  if (ctx->side_join) cudaEventDestroy(ctx->side_join);
  delete ctx;
}

ra_status ra_ctx_set_stream(ra_ctx* ctx, void* stream) {
  return guard([&] {
    check_ctx(ctx);
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

ra_status ra_host_alloc(size_t bytes, void** out) {
  return guard([&] {
    if (!out) invalid("null output");
    *out = nullptr;
    RA_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocMapped | cudaHostAllocPortable));
  });
}

void ra_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

ra_status ra_ctx_set_search_kernel(ra_ctx* ctx, const char* name) {
  return guard([&] {
    check_ctx(ctx);
    if (!name) {
      ctx->search_kernel = -1;
      return;
    }
    const int v = ra::search_variant_of(name);
    if (v < 0) invalid("unknown search kernel");
    ctx->search_kernel = v;
  });
}

ra_status ra_ctx_synchronize(ra_ctx* ctx) {
  return guard([&] {
    check_ctx(ctx);
    DeviceGuard dg(ctx->device);
    RA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---- KV groups ------------------------------------------------------------------
ra_status ra_kv_create(ra_ctx* ctx, const float* keys, const float* values, uint64_t n,
                       uint32_t d, int on_device, ra_kv** out) {
  return guard([&] {
    check_ctx(ctx);
    if (d < 1) invalid("VectorSet.d must be >= 1");
    DeviceGuard dg(ctx->device);
    auto kv = std::make_unique<ra_kv>();
    kv->device = ctx->device;
    kv->n = n;
    kv->d = d;
    const auto kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    kv->keys.alloc(size_t(n) * d);
    if (n) RA_CUDA(cudaMemcpyAsync(kv->keys.p, keys, size_t(n) * d * 4, kind, ctx->stream));
    if (values) {
      kv->values.alloc(size_t(n) * d);
      if (n)
        RA_CUDA(cudaMemcpyAsync(kv->values.p, values, size_t(n) * d * 4, kind, ctx->stream));
    }
    RA_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = kv.release();
  });
}

namespace {
__global__ void k_to_bf16(float* x, uint16_t* y, uint64_t n, int round_f32) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t u = __float_as_uint(x[i]);
    u += 0x7FFFu + ((u >> 16) & 1u);  // round to nearest even (finite inputs)
    y[i] = uint16_t(u >> 16);
    if (round_f32) x[i] = __uint_as_float(uint32_t(y[i]) << 16);
  }
}
}  // namespace

ra_status ra_kv_attach_values(ra_ctx* ctx, ra_kv* kv, const float* values, uint64_t n,
                              int on_device) {
  return guard([&] {
    check_ctx(ctx);
    if (!kv || !values) invalid("null kv or values");
    if (n != kv->n) invalid("keys and values must have equal n");
    if (kv->values.p) invalid("kv group already has values");
    if (kv->bf16 || kv->bf16_attn) invalid("attach values to f32 groups only");
    DeviceGuard dg(ctx->device);
    kv->values.alloc(size_t(n) * kv->d);
    if (n)
      RA_CUDA(cudaMemcpyAsync(kv->values.p, values, size_t(n) * kv->d * 4,
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              ctx->stream));
    RA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ra_kv_has_values(const ra_kv* kv) { return kv && kv->values.p ? 1 : 0; }

ra_status ra_kv_create_bf16(ra_ctx* ctx, const float* keys, const float* values, uint64_t n,
                            uint32_t d, int on_device, int attention_only, ra_kv** out) {
  return guard([&] {
    ra_kv* kv = nullptr;
    if (ra_kv_create(ctx, keys, values, n, d, on_device, &kv) != RA_OK)
      throw Error(RA_ERR_INVALID_ARGUMENT, ra_last_error());
    std::unique_ptr<ra_kv, void (*)(ra_kv*)> hold(kv, ra_kv_release);
    DeviceGuard dg(ctx->device);
    kv->bf16 = !attention_only;
    kv->bf16_attn = true;
    const uint64_t m = n * d;
    const int rnd = attention_only ? 0 : 1;
    kv->keys16.alloc(std::max<uint64_t>(m, 1));
    if (m) k_to_bf16<<<1024, 256, 0, ctx->stream>>>(kv->keys.p, kv->keys16.p, m, rnd);
    if (kv->values.p) {
      kv->values16.alloc(std::max<uint64_t>(m, 1));
      if (m) k_to_bf16<<<1024, 256, 0, ctx->stream>>>(kv->values.p, kv->values16.p, m, rnd);
    }
    RA_LAUNCH_CHECK();
    RA_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = hold.release();
  });
}

int ra_kv_is_bf16(const ra_kv* kv) { return !kv ? 0 : kv->bf16 ? 1 : kv->bf16_attn ? 2 : 0; }

void ra_kv_retain(ra_kv* kv) {
  if (kv) kv->refs.fetch_add(1);
}
void ra_kv_release(ra_kv* kv) {
  if (kv && kv->refs.fetch_sub(1) == 1) {
    DeviceGuard dg(kv->device, true);
    delete kv;
  }
}
uint64_t ra_kv_size(const ra_kv* kv) { return kv ? kv->n : 0; }
uint32_t ra_kv_dim(const ra_kv* kv) { return kv ? kv->d : 0; }
const float* ra_kv_keys_device(const ra_kv* kv) { return kv ? kv->keys.p : nullptr; }
const float* ra_kv_values_device(const ra_kv* kv) { return kv ? kv->values.p : nullptr; }

// ---- graphs -------------------------------------------------------------------------
void ra_build_params_default(ra_build_params* p) {
  p->k_train = 32;
  p->max_degree = 32;
  p->ef_construction = 128;
  p->edge_window = 8;
  p->entry_maxnorm = 0;
  p->prune_inner_product = 0;
  p->default_ef = 128;
}

// OODGraph::from_blob (index_oodgraph.cpp:468-495), same checks and messages
ra_status ra_graph_deserialize(ra_ctx* ctx, ra_kv* keys, const char* blob, uint64_t size,
                               ra_graph** out) {
  return guard([&] {
    check_ctx(ctx);
    if (!keys || keys->n == 0) invalid("empty keys");
    if (size < 4 || std::memcmp(blob, "OODG", 4) != 0) runtime("bad graph magic");
    uint64_t pos = 4;
    auto rd = [&](void* dst, size_t bytes) {
      if (pos + bytes > size) runtime("truncated graph blob");
      std::memcpy(dst, blob + pos, bytes);
      pos += bytes;
    };
    uint32_t version;
    rd(&version, 4);
    if (version != 1) runtime("unsupported graph version");
    uint64_t n;
    rd(&n, 8);
    if (n != keys->n) runtime("graph/key count mismatch");
    auto g = std::make_unique<ra_graph>();
    rd(&g->max_degree, 4);
    if (g->max_degree < 1) runtime("bad degree bound");
    rd(&g->entry, 8);
    if (g->entry >= n) runtime("entry point out of range");
    g->n = n;
    g->offsets.assign(n + 1, 0);
    for (uint64_t u = 0; u < n; ++u) {
      uint32_t deg;
      rd(&deg, 4);
      if (deg > g->max_degree) runtime("degree exceeds bound");
      g->offsets[u + 1] = g->offsets[u] + deg;
      for (uint32_t j = 0; j < deg; ++j) {
        uint64_t v;
        rd(&v, 8);
        if (v >= n) runtime("neighbor id out of range");
        if (v == u) runtime("self loop");
        g->adjacency.push_back(uint32_t(v));
      }
    }
    if (pos != size) runtime("trailing bytes in graph blob");
    g->n_edges = g->adjacency.size();
    DeviceGuard dg(ctx->device);
    graph_upload(ctx, g.get());
    ra_kv_retain(keys);
    g->kv = keys;
    *out = g.release();
  });
}

// OODGraph::serialize (index_oodgraph.cpp:435-449)
ra_status ra_graph_serialize(const ra_graph* g, char* buf, uint64_t cap, uint64_t* size) {
  return guard([&] {
    if (!g) invalid("null graph");
    const uint64_t n = g->n;
    const uint64_t total = 28 + 4 * n + 8 * g->n_edges;
    *size = total;
    if (!buf || cap < total) return;
    g->host_mirror();
    char* p = buf;
    auto put = [&](const void* v, size_t b) {
      std::memcpy(p, v, b);
      p += b;
    };
    const uint32_t ver = 1;
    put("OODG", 4);
    put(&ver, 4);
    put(&n, 8);
    put(&g->max_degree, 4);
    put(&g->entry, 8);
    for (uint64_t u = 0; u < n; ++u) {
      const uint32_t deg = uint32_t(g->offsets[u + 1] - g->offsets[u]);
      put(&deg, 4);
      for (uint64_t j = g->offsets[u]; j < g->offsets[u + 1]; ++j) {
        const uint64_t v = g->adjacency[j];
        put(&v, 8);
      }
    }
  });
}

void ra_graph_free(ra_graph* g) {
  if (!g) return;
  {
    DeviceGuard dg(g->kv ? g->kv->device : 0, true);
    g->adj.reset();
  }
  ra_kv_release(g->kv);
  delete g;
}

uint64_t ra_graph_size(const ra_graph* g) { return g->n; }
uint64_t ra_graph_entry_point(const ra_graph* g) { return g->entry; }
uint32_t ra_graph_max_degree_bound(const ra_graph* g) { return g->max_degree; }
uint32_t ra_graph_default_ef(const ra_graph* g) { return g->default_ef; }
uint32_t ra_graph_degree(const ra_graph* g, uint64_t u) {
  g->host_mirror();
  return uint32_t(g->offsets[u + 1] - g->offsets[u]);
}
uint32_t ra_graph_neighbors(const ra_graph* g, uint64_t u, uint32_t* out, uint32_t cap) {
  const uint32_t deg = ra_graph_degree(g, u);
  std::copy_n(g->adjacency.begin() + g->offsets[u], std::min(deg, cap), out);
  return deg;
}
// reachable_count (index_oodgraph.cpp:417-433)
uint64_t ra_graph_reachable_count(const ra_graph* g) {
  g->host_mirror();
  std::vector<uint8_t> seen(g->n, 0);
  std::vector<uint32_t> stack{uint32_t(g->entry)};
  seen[g->entry] = 1;
  uint64_t count = 1;
  while (!stack.empty()) {
    const uint32_t u = stack.back();
    stack.pop_back();
    for (uint64_t j = g->offsets[u]; j < g->offsets[u + 1]; ++j) {
      const uint32_t v = g->adjacency[j];
      if (!seen[v]) {
        seen[v] = 1;
        ++count;
        stack.push_back(v);
      }
    }
  }
  return count;
}
uint64_t ra_graph_memory_bytes(const ra_graph* g) {
  return (g->n + 1) * 8 + g->n_edges * 4;
}
uint64_t ra_graph_device_bytes(const ra_graph* g) { return g->adj.bytes(); }

ra_status ra_graph_csr(const ra_graph* g, uint64_t* offsets, uint32_t* adjacency) {
  return guard([&] {
    if (!g) invalid("null graph");
    g->host_mirror();
    if (offsets) std::copy(g->offsets.begin(), g->offsets.end(), offsets);
    if (adjacency) std::copy(g->adjacency.begin(), g->adjacency.end(), adjacency);
  });
}

// ---- search ------------------------------------------------------------------------------
ra_status ra_graph_search_batch(ra_ctx* ctx, const ra_graph* const* graphs, uint32_t B,
                                const float* q, uint32_t q_dim, uint32_t k, int64_t ef,
                                const uint32_t* mask, uint64_t mask_n, uint32_t* ids,
                                float* scores, uint32_t* n_out, uint64_t* scanned,
                                uint8_t* truncated, uint32_t* expanded) {
  return guard([&] {
    check_ctx(ctx);
    if (B == 0) return;
    uint32_t max_n = 0, max_M = 0, n_bf16 = 0;
    std::vector<GraphDesc> desc(B);
    for (uint32_t b = 0; b < B; ++b) {
      const ra_graph* g = graphs[b];
      if (!g) invalid("null graph");
      n_bf16 += g->kv->bf16;
      if (q_dim != g->kv->d) invalid("query dimension mismatch");  // :359
      if (k < 1) invalid("k must be >= 1");                         // :360
      const uint64_t e = ef >= 0 ? uint64_t(ef) : g->default_ef;
      if (e < k) invalid("ef must be >= k");                        // :362
      desc[b] = GraphDesc{g->adj.p, g->kv->keys.p, g->kv->bf16 ? g->kv->keys16.p : nullptr,
                          g->entry, uint32_t(g->n), g->max_degree,
                          uint32_t(std::min<uint64_t>(e, 0xFFFFFFFFu)), 0};
      max_n = std::max<uint32_t>(max_n, uint32_t(g->n));
      max_M = std::max<uint32_t>(max_M, g->max_degree);
    }
    DeviceGuard dg(ctx->device);
    const uint64_t words = (uint64_t(max_n) + 31) / 32;
    const size_t desc_bytes = (B * sizeof(GraphDesc) + 255) & ~size_t(255);
    uint8_t* a = arena<uint8_t>(ctx->scratch_a, desc_bytes + words * 4 + 256);
    GraphDesc* d_desc = reinterpret_cast<GraphDesc*>(a);
    uint32_t* bits = reinterpret_cast<uint32_t*>(a + desc_bytes);
    RA_CUDA(cudaMemcpyAsync(d_desc, desc.data(), B * sizeof(GraphDesc), cudaMemcpyHostToDevice,
                            ctx->stream));
    if (mask_n) launch_mask_bitset(ctx->stream, mask, mask_n, bits, words);
    if (n_bf16 && n_bf16 != B) invalid("mixed f32 and bf16 key groups in one batch");
    SearchArgs sa{};
    sa.desc = d_desc;
    sa.q = q;
    sa.mask_bits = mask_n ? bits : nullptr;
    sa.B = B;
    sa.d = q_dim;
    sa.k = k;
    sa.max_M = max_M;
    sa.bf16 = n_bf16 == B;
    sa.ids = ids;
    sa.scores = scores;
    sa.scores64 = nullptr;
    sa.n_out = n_out;
    sa.scanned = scanned;
    sa.truncated = truncated;
    sa.expanded = expanded;
    const size_t sbytes = search_scratch_bytes(ctx, B, max_n, q_dim);
    uint8_t* scr = sbytes ? arena<uint8_t>(ctx->scratch_b, sbytes) : nullptr;
    launch_graph_search(ctx, sa, max_n, scr);
  });
}

ra_status ra_graph_search_host(ra_ctx* ctx, const ra_graph* g, const float* q, uint32_t q_dim,
                               uint32_t k, int64_t ef, const uint32_t* mask, uint64_t mask_n,
                               uint32_t* ids, float* scores, uint32_t* n_out, uint64_t* scanned,
                               uint8_t* truncated) {
  return guard([&] {
    check_ctx(ctx);
    if (!g) invalid("null graph");
    if (q_dim != g->kv->d) invalid("query dimension mismatch");  // :359 (checked first)
    DeviceGuard dg(ctx->device);
    const uint32_t kk = std::max<uint32_t>(k, 1);
    // one staging block: q | mask | ids | scores | n_out | scanned | truncated
    const size_t off_mask = (size_t(q_dim) * 4 + 255) & ~size_t(255);
    const size_t off_ids = off_mask + ((mask_n * 4 + 255) & ~size_t(255));
    const size_t off_sc = off_ids + ((size_t(kk) * 4 + 255) & ~size_t(255));
    const size_t off_n = off_sc + ((size_t(kk) * 4 + 255) & ~size_t(255));
    const size_t total = off_n + 256;
    uint8_t* d = arena<uint8_t>(ctx->scratch_c, total);
    cudaStream_t s = ctx->stream;
    RA_CUDA(cudaMemcpyAsync(d, q, size_t(q_dim) * 4, cudaMemcpyHostToDevice, s));
    if (mask_n) RA_CUDA(cudaMemcpyAsync(d + off_mask, mask, mask_n * 4, cudaMemcpyHostToDevice, s));
    uint32_t* d_n = reinterpret_cast<uint32_t*>(d + off_n);
    uint64_t* d_sc = reinterpret_cast<uint64_t*>(d + off_n + 8);
    uint8_t* d_tr = d + off_n + 16;
    const ra_graph* gs[1] = {g};
    const ra_status st = ra_graph_search_batch(
        ctx, gs, 1, reinterpret_cast<const float*>(d), q_dim, k, ef,
        mask_n ? reinterpret_cast<const uint32_t*>(d + off_mask) : nullptr, mask_n,
        reinterpret_cast<uint32_t*>(d + off_ids), reinterpret_cast<float*>(d + off_sc), d_n, d_sc,
        d_tr, nullptr);
    if (st != RA_OK) throw Error(st, g_last_error);
    uint32_t n = 0;
    RA_CUDA(cudaMemcpyAsync(&n, d_n, 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaMemcpyAsync(scanned, d_sc, 8, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaMemcpyAsync(truncated, d_tr, 1, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaMemcpyAsync(ids, d + off_ids, size_t(kk) * 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaMemcpyAsync(scores, d + off_sc, size_t(kk) * 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    *n_out = n;
  });
}

// ---- attention ------------------------------------------------------------------------------
ra_status ra_static_partition(uint64_t t, uint64_t s_init, uint64_t s_local,
                              uint32_t* static_ids, uint64_t* n_static, uint32_t* pool_ids,
                              uint64_t* n_pool) {
  return guard([&] {
    if (t > 0xFFFFFFFFull) invalid("context length exceeds id width");
    const uint64_t head_end = std::min(s_init, t);
    const uint64_t tail_begin = t > s_local ? std::max(t - s_local, head_end) : head_end;
    uint64_t ns = 0, np = 0;
    for (uint64_t i = 0; i < head_end; ++i, ++ns)
      if (static_ids) static_ids[ns] = uint32_t(i);
    for (uint64_t i = tail_begin; i < t; ++i, ++ns)
      if (static_ids) static_ids[ns] = uint32_t(i);
    for (uint64_t i = head_end; i < tail_begin; ++i, ++np)
      if (pool_ids) pool_ids[np] = uint32_t(i);
    *n_static = ns;
    *n_pool = np;
  });
}

static uint32_t read_flag(ra_ctx* ctx, uint32_t* d_flag) {
  uint32_t f = 0;
  RA_CUDA(cudaMemcpyAsync(&f, d_flag, 4, cudaMemcpyDeviceToHost, ctx->stream));
  RA_CUDA(cudaStreamSynchronize(ctx->stream));
  return f;
}

ra_status ra_partial_attention(ra_ctx* ctx, ra_kv* kv, uint32_t B, const float* q,
                               const uint32_t* idx, uint32_t m_stride, const uint32_t* m,
                               double* out, double* zmax, double* expsum) {
  return guard([&] {
    check_ctx(ctx);
    if (!kv) invalid("null kv");
    if (kv->values.n != kv->keys.n || !kv->values.p)
      invalid("keys and values must have equal n");
    if (B == 0) return;
    DeviceGuard dg(ctx->device);
    const size_t refs_bytes = (B * sizeof(KVRef) + 255) & ~size_t(255);
    uint8_t* a = arena<uint8_t>(ctx->scratch_a, refs_bytes + 256);
    KVRef* refs = reinterpret_cast<KVRef*>(a);
    uint32_t* flag = reinterpret_cast<uint32_t*>(a + refs_bytes);
    std::vector<KVRef> h(B, KVRef{kv->keys.p, kv->values.p, kv->n, nullptr, nullptr});
    RA_CUDA(cudaMemcpyAsync(refs, h.data(), B * sizeof(KVRef), cudaMemcpyHostToDevice,
                            ctx->stream));
    RA_CUDA(cudaMemsetAsync(flag, 0, 4, ctx->stream));
    const size_t zd = partial_scratch_doubles(B, m_stride ? m_stride : 1u << 30);
    double* z = nullptr;
    if (m_stride > 8192) z = arena<double>(ctx->scratch_c, zd);
    launch_partial_attention_ex(ctx->stream, refs, kv->d, B, q, idx, m_stride, m, nullptr, 0,
                                out, zmax, expsum, z, m_stride, nullptr, flag);
    if (read_flag(ctx, flag) & 1u) invalid("index out of range");
  });
}

// partial_attention on HOST buffers (attention.cpp:102-128): the rows named
// by idx are staged (gathered in idx order) and the device kernel computes
// the partial over them - the same arithmetic order as the reference.
ra_status ra_partial_attention_host(ra_ctx* ctx, const float* q, uint32_t q_dim,
                                    const float* keys, uint64_t n_keys, const float* values,
                                    uint64_t n_values, uint32_t d, const uint32_t* idx,
                                    uint64_t m, double* out, double* zmax, double* expsum) {
  return guard([&] {
    check_ctx(ctx);
    if (q_dim != d) invalid("query dimension mismatch");
    if (n_keys != n_values || !values) invalid("keys and values must have equal n");
    if (m == 0) invalid("empty index set");
    if (m > 0xFFFFFFFFull) invalid("too many indices");
    for (uint64_t i = 0; i < m; ++i)
      if (idx[i] >= n_keys) invalid("index out of range");
    DeviceGuard dg(ctx->device);
    // device layout: q f32[d] | K f32[m][d] | V f32[m][d] | ids u32[m] | cnt u32 | pad
    //                | out f64[d] | zmax | expsum | flag
    const size_t rowb = size_t(d) * 4;
    const size_t o_q = 0, o_k = (o_q + rowb + 15) & ~size_t(15);
    const size_t o_v = (o_k + m * rowb + 15) & ~size_t(15);
    const size_t o_i = (o_v + m * rowb + 15) & ~size_t(15);
    const size_t o_c = (o_i + m * 4 + 15) & ~size_t(15);
    const size_t o_o = (o_c + 16 + 15) & ~size_t(15);
    const size_t o_end = o_o + (size_t(d) + 2) * 8 + 16;
    std::vector<uint8_t> h(o_c + 16);
    std::memcpy(h.data() + o_q, q, rowb);
    for (uint64_t i = 0; i < m; ++i) {
      std::memcpy(h.data() + o_k + i * rowb, keys + size_t(idx[i]) * d, rowb);
      std::memcpy(h.data() + o_v + i * rowb, values + size_t(idx[i]) * d, rowb);
      const uint32_t j = uint32_t(i);
      std::memcpy(h.data() + o_i + i * 4, &j, 4);
    }
    const uint32_t cnt = uint32_t(m);
    std::memcpy(h.data() + o_c, &cnt, 4);
    uint8_t* dv = arena<uint8_t>(ctx->scratch_c, o_end + 256);
    RA_CUDA(cudaMemcpyAsync(dv, h.data(), h.size(), cudaMemcpyHostToDevice, ctx->stream));
    uint8_t* a = arena<uint8_t>(ctx->scratch_a, 256);
    KVRef* ref = reinterpret_cast<KVRef*>(a);
    uint32_t* flag = reinterpret_cast<uint32_t*>(a + 128);
    const KVRef hr{reinterpret_cast<const float*>(dv + o_k), reinterpret_cast<const float*>(dv + o_v),
                   m, nullptr, nullptr};
    RA_CUDA(cudaMemcpyAsync(ref, &hr, sizeof(KVRef), cudaMemcpyHostToDevice, ctx->stream));
    RA_CUDA(cudaMemsetAsync(flag, 0, 4, ctx->stream));
    double* dout = reinterpret_cast<double*>(dv + o_o);
    double* z = nullptr;
    if (m > 8192) z = arena<double>(ctx->scratch_b, partial_scratch_doubles(1, uint32_t(m)));
    launch_partial_attention_ex(ctx->stream, ref, d, 1, reinterpret_cast<const float*>(dv + o_q),
                                reinterpret_cast<const uint32_t*>(dv + o_i), uint32_t(m),
                                reinterpret_cast<const uint32_t*>(dv + o_c), nullptr, 0, dout,
                                dout + d, dout + d + 1, z, uint32_t(m), nullptr, flag);
    std::vector<double> r(size_t(d) + 2);
    RA_CUDA(cudaMemcpyAsync(r.data(), dout, r.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (read_flag(ctx, flag) & 1u) invalid("index out of range");
    std::memcpy(out, r.data(), size_t(d) * 8);
    *zmax = r[d];
    *expsum = r[size_t(d) + 1];
  });
}

// merge_gammas + merge of one partial pair on HOST buffers
// (attention.cpp:136-157); gw / go may be NULL.
ra_status ra_merge_host(ra_ctx* ctx, uint32_t d, const double* ow, double zw, double sw,
                        int w_empty, const double* oo, double zo, double so, int o_empty,
                        double* out, double* gw, double* go) {
  return guard([&] {
    check_ctx(ctx);
    DeviceGuard dg(ctx->device);
    // device: ow[d] | oo[d] | zw sw zo so | out[d] | gw go | flags u8[2] | err u32
    const size_t nd = size_t(d);
    std::vector<double> h(3 * nd + 6 + 2, 0.0);
    if (!w_empty) std::memcpy(h.data(), ow, nd * 8);
    if (!o_empty) std::memcpy(h.data() + nd, oo, nd * 8);
    h[2 * nd] = zw, h[2 * nd + 1] = sw, h[2 * nd + 2] = zo, h[2 * nd + 3] = so;
    uint8_t* fl = reinterpret_cast<uint8_t*>(h.data() + 3 * nd + 6);
    fl[0] = uint8_t(w_empty != 0), fl[1] = uint8_t(o_empty != 0);
    double* dv = arena<double>(ctx->scratch_c, h.size() + 2);
    uint32_t* flag = reinterpret_cast<uint32_t*>(dv + h.size());
    RA_CUDA(cudaMemcpyAsync(dv, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    RA_CUDA(cudaMemsetAsync(flag, 0, 4, ctx->stream));
    const uint8_t* dfl = reinterpret_cast<const uint8_t*>(dv + 3 * nd + 6);
    launch_merge(ctx->stream, 1, d, dv, dv + 2 * nd, dv + 2 * nd + 1, dfl, dv + nd,
                 dv + 2 * nd + 2, dv + 2 * nd + 3, dfl + 1, dv + 2 * nd + 4, dv + 3 * nd + 4,
                 dv + 3 * nd + 5, flag);
    std::vector<double> r(nd + 2);
    RA_CUDA(cudaMemcpyAsync(r.data(), dv + 2 * nd + 4, (nd + 2) * 8, cudaMemcpyDeviceToHost,
                            ctx->stream));
    if (read_flag(ctx, flag) & 2u) invalid("empty attention support");  // :138-139
    if (out) std::memcpy(out, r.data(), nd * 8);
    if (gw) *gw = r[nd];
    if (go) *go = r[nd + 1];
  });
}

ra_status ra_merge(ra_ctx* ctx, uint32_t B, uint32_t d, const double* ow, const double* zw,
                   const double* sw, const uint8_t* w_empty, const double* oo,
                   const double* zo, const double* so, const uint8_t* o_empty, double* out,
                   double* gw, double* go) {
  return guard([&] {
    check_ctx(ctx);
    DeviceGuard dg(ctx->device);
    uint32_t* flag = arena<uint32_t>(ctx->scratch_a, 1);
    RA_CUDA(cudaMemsetAsync(flag, 0, 4, ctx->stream));
    launch_merge(ctx->stream, B, d, ow, zw, sw, w_empty, oo, zo, so, o_empty, out, gw, go, flag);
    if (read_flag(ctx, flag) & 2u) invalid("empty attention support");  // :138-139
  });
}

}  // extern "C"

// ---- decode engine (engine.cpp:23-115) -----------------------------------------------
struct ra_engine {
  // CUDA graph of one whole step (H2D, kernels on both streams, D2H) per
  // (mode, buffer pointers); captured on the second call with the same
  // pointers, replayed after that. Opt-in (RA_ENGINE_GRAPH=1): the step is
  // one ~0.3 ms latency-bound search, launch overhead is a few microseconds,
  // and replaying measured no faster on B200.
  struct StepGraph {
    const void* key[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
  } sg[2];
  bool graphs_off = false;
  cudaStream_t cap_stream = nullptr;  // capture happens here (the legacy stream can't capture)
  ra_ctx* ctx = nullptr;
  uint32_t H = 0, G = 0, d = 0, k = 0;
  uint64_t t = 0, n_pool = 0, n_static = 0;
  ra_engine_config cfg{};
  std::vector<ra_kv*> groups;     // retained
  std::vector<ra_graph*> graphs;  // borrowed (caller keeps them alive)
  std::string step_error;         // deferred "ef must be >= k" (raised per step)
  DevBuf<GraphDesc> desc;
  DevBuf<KVRef> kvrefs;
  DevBuf<uint32_t> w_ids, w_bits, w_m, o_m;
  DevBuf<uint8_t> w_empty, o_empty;
  DevBuf<float> q;
  DevBuf<uint32_t> ids, n_out, expanded, flag;
  DevBuf<float> scores;
  DevBuf<double> scores64, ow, zw, sw, oo, zo, so, out;
  DevBuf<uint64_t> scanned;
  DevBuf<uint8_t> truncated;
  DevBuf<uint8_t> search_scratch;
  DevBuf<uint64_t> dbg;
  uint32_t max_n = 0, max_M = 0;
  // events bracketing the search kernel and the attention kernels of the
  // last step, recorded on the ctx stream (ra_engine_last_timing)
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  // fast attention path: W partials on a side stream overlapping the search
  bool fast_attn = false;
  // fused decode step: the search kernel also computes the W partials (idle
  // helpers) and the Omega partial + merge (its tail); one launch per step
  bool fused = false;
  uint32_t fa_nchunk = 0;
  DevBuf<const float*> hvals;  // [H] each head's V rows
  DevBuf<double> fa_chunk;     // [H][nchunk][d + 2]
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  DevBuf<KVRef> gkv;
  DevBuf<double> part;
  uint32_t hpg = 0;
};

extern "C" {

ra_status ra_engine_create(ra_ctx* ctx, ra_kv* const* groups, uint32_t n_groups,
                           ra_graph* const* head_graphs, uint32_t n_heads,
                           const ra_engine_config* cfg, ra_engine** out) {
  return guard([&] {
    check_ctx(ctx);
    if (n_heads == 0) invalid("no heads");
    if (cfg->top_k < 1) invalid("top_k must be >= 1");
    if (n_groups == 0 || n_heads % n_groups) invalid("n_heads must be divisible by n_kv_groups");
    const uint64_t t = groups[0]->n;
    if (t == 0) invalid("empty context");
    for (uint32_t gi = 0; gi < n_groups; ++gi)
      if (groups[gi]->n != t || groups[gi]->values.n != groups[gi]->keys.n)
        invalid("context length mismatch across heads");
    const uint32_t per = n_heads / n_groups;
    for (uint32_t h = 0; h < n_heads; ++h)
      if (!head_graphs[h] || head_graphs[h]->kv != groups[h / per])
        invalid("head graph is not built over its group's keys");
    for (uint32_t gi = 1; gi < n_groups; ++gi)
      if (groups[gi]->bf16 != groups[0]->bf16 || groups[gi]->bf16_attn != groups[0]->bf16_attn)
        invalid("mixed f32 and bf16 key groups");
    DeviceGuard dg(ctx->device);
    auto e = std::make_unique<ra_engine>();
    e->ctx = ctx;
    e->H = n_heads;
    e->G = n_groups;
    e->d = groups[0]->d;
    e->t = t;
    e->cfg = *cfg;
    for (uint32_t gi = 0; gi < n_groups; ++gi) {
      ra_kv_retain(groups[gi]);
      e->groups.push_back(groups[gi]);
    }
    e->graphs.assign(head_graphs, head_graphs + n_heads);
    uint64_t ns, np;
    if (ra_static_partition(t, cfg->s_init, cfg->s_local, nullptr, &ns, nullptr, &np))
      invalid(ra_last_error());
    std::vector<uint32_t> w(ns), pool(np);
    ra_static_partition(t, cfg->s_init, cfg->s_local, w.data(), &ns, pool.data(), &np);
    e->n_static = ns;
    e->n_pool = np;
    e->k = uint32_t(std::min<uint64_t>(cfg->top_k, np));
    const uint32_t H = n_heads, d = e->d, kk = std::max<uint32_t>(e->k, 1);
    std::vector<GraphDesc> desc(H);
    std::vector<KVRef> refs(H);
    for (uint32_t h = 0; h < H; ++h) {
      const ra_graph* g = head_graphs[h];
      const uint64_t ef = cfg->ef >= 0 ? uint64_t(cfg->ef) : g->default_ef;
      if (np > 0 && ef < e->k) e->step_error = "ef must be >= k";
      desc[h] = GraphDesc{g->adj.p, g->kv->keys.p, g->kv->bf16 ? g->kv->keys16.p : nullptr,
                          g->entry, uint32_t(g->n), g->max_degree,
                          uint32_t(std::min<uint64_t>(ef, 0xFFFFFFFFu)), 0};
      refs[h] = KVRef{g->kv->keys.p, g->kv->values.p, g->kv->n, g->kv->keys16.p,
                      g->kv->values16.p};
      e->max_n = std::max<uint32_t>(e->max_n, uint32_t(g->n));
      e->max_M = std::max<uint32_t>(e->max_M, g->max_degree);
    }
    auto up = [&](auto& buf, const auto& vec) {
      buf.alloc(std::max<size_t>(vec.size(), 1));
      if (!vec.empty())
        RA_CUDA(cudaMemcpy(buf.p, vec.data(), vec.size() * sizeof(vec[0]),
                           cudaMemcpyHostToDevice));
    };
    up(e->desc, desc);
    up(e->kvrefs, refs);
    std::vector<KVRef> grefs(n_groups);
    for (uint32_t gi = 0; gi < n_groups; ++gi)
      grefs[gi] = KVRef{groups[gi]->keys.p, groups[gi]->values.p, groups[gi]->n,
                        groups[gi]->keys16.p, groups[gi]->values16.p};
    up(e->gkv, grefs);
    e->hpg = per;
    e->fast_attn = engine_attention_supported(d);
    if (e->fast_attn)
      e->part.alloc(engine_attention_part_doubles(n_groups, per, uint32_t(ns), d));
    up(e->w_ids, w);
    up(e->w_m, std::vector<uint32_t>(H, uint32_t(ns)));
    up(e->w_empty, std::vector<uint8_t>(H, ns == 0));
    const uint64_t words = (t + 31) / 32;
    e->w_bits.alloc(words);
    launch_mask_bitset(ctx->stream, e->w_ids.p, ns, e->w_bits.p, words);
    e->q.alloc(size_t(H) * d);
    e->ids.alloc(size_t(H) * kk);
    e->scores.alloc(size_t(H) * kk);
    e->scores64.alloc(size_t(H) * kk);
    e->n_out.alloc(H);
    e->scanned.alloc(H);
    e->truncated.alloc(H);
    e->expanded.alloc(H);
    e->o_empty.alloc(H);
    e->dbg.alloc(size_t(H) * 12);
    RA_CUDA(cudaMemset(e->dbg.p, 0, size_t(H) * 96));
    e->flag.alloc(1);
    for (auto* b : {&e->ow, &e->oo, &e->out}) b->alloc(size_t(H) * d);
    for (auto* b : {&e->zw, &e->sw, &e->zo, &e->so}) b->alloc(H);
    {
      SearchArgs probe{};
      probe.B = H, probe.d = d, probe.max_M = e->max_M, probe.bf16 = e->groups[0]->bf16;
      static const bool fa_off = [] {
        const char* v = std::getenv("RA_FUSED_ATTN");
        return v && v[0] == '0';
      }();
      e->fused = !fa_off && e->fast_attn &&
                 !(e->groups[0]->bf16_attn && !e->groups[0]->bf16) &&  // (not attention-only bf16)
                 e->n_pool > 0 && search_fuses_attention(ctx, probe, e->max_n);
      if (e->fused) {
        const uint32_t rows = std::max<uint32_t>(e->max_M, 1);  // the kernel's tile rows
        e->fa_nchunk = uint32_t((ns + rows - 1) / rows);
        std::vector<const float*> hv(H);
        for (uint32_t h = 0; h < H; ++h) hv[h] = head_graphs[h]->kv->values.p;
        up(e->hvals, hv);
        e->fa_chunk.alloc(std::max<size_t>(size_t(H) * e->fa_nchunk * (d + 2), 1));
      }
    }
    const size_t sb = search_scratch_bytes(ctx, H, e->max_n, d);
    e->search_scratch.alloc(sb);
    for (auto& ev : e->ev) RA_CUDA(cudaEventCreate(&ev));
    RA_CUDA(cudaStreamCreateWithFlags(&e->aux, cudaStreamNonBlocking));
    RA_CUDA(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));
    RA_CUDA(cudaEventCreateWithFlags(&e->join, cudaEventDisableTiming));
    RA_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = e.release();
  });
}

void ra_engine_destroy(ra_engine* e) {
  if (!e) return;
  {
    DeviceGuard dg(e->ctx->device, true);
    cudaStreamSynchronize(e->ctx->stream);
    for (ra_kv* g : e->groups) ra_kv_release(g);
    for (auto& ev : e->ev)
      if (ev) cudaEventDestroy(ev);
    if (e->aux) cudaStreamDestroy(e->aux);
    if (e->fork) cudaEventDestroy(e->fork);
    if (e->join) cudaEventDestroy(e->join);
    for (auto& g : e->sg)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
  }
  delete e;
}

namespace {
// timing event: a real event-record node when the step is being captured
// into a CUDA graph (a plain record there would only be a dependency marker)
void record_timing(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  RA_CUDA(cudaStreamIsCapturing(s, &st));
  if (st == cudaStreamCaptureStatusActive)
    RA_CUDA(cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal));
  else
    RA_CUDA(cudaEventRecord(ev, s));
}
// run_head for every head (engine.cpp:69-101): search with Mask{W} ->
// partial over W -> partial over Omega (scores reused) -> merge.
// out_dev / ids_dev: where the attention output [H, d] f64 and the Omega
// ids [H, k] go (the caller's device buffers, or the engine's own)
void engine_enqueue(ra_engine* e, const float* q_dev, double* out_dev, uint32_t* ids_dev,
                    uint64_t* scanned_dev, uint32_t* ids_copy = nullptr) {
  ra_ctx* ctx = e->ctx;
  cudaStream_t s = ctx->stream;
  const uint32_t H = e->H, d = e->d;
  EngineAttn ea{};
  if (e->fused) {  // one launch: search + W partials + Omega partial + merge
    record_timing(e->ev[0], s);
    SearchArgs sa{};
    sa.desc = e->desc.p;
    sa.q = q_dev;
    sa.mask_bits = e->n_static ? e->w_bits.p : nullptr;
    sa.B = H;
    sa.d = d;
    sa.k = e->k;
    sa.max_M = e->max_M;
    sa.ids = ids_copy ? ids_copy : ids_dev;
    sa.scores = e->scores.p;
    sa.scores64 = e->scores64.p;
    sa.n_out = e->n_out.p;
    sa.scanned = scanned_dev;
    sa.scanned_own = scanned_dev == e->scanned.p ? nullptr : e->scanned.p;
    sa.truncated = e->truncated.p;
    sa.expanded = e->expanded.p;
    sa.dbg = e->dbg.p;
    sa.fa = {e->hvals.p, e->w_ids.p, uint32_t(e->n_static), e->fa_nchunk,
             std::max<uint32_t>(e->max_M, 1), 1.0 / std::sqrt(double(d)), out_dev,
             e->fa_chunk.p};
    launch_graph_search(ctx, sa, e->max_n, e->search_scratch.p);
    record_timing(e->ev[1], s);
    record_timing(e->ev[2], s);
    return;
  }
  if (e->fast_attn) {
    const uint32_t C = uint32_t((e->n_static + 63) / 64);
    ea = EngineAttn{e->gkv.p, e->kvrefs.p, q_dev, e->w_ids.p, uint32_t(e->n_static), e->G, H,
                    e->hpg, d, e->k, 1.0 / std::sqrt(double(d)), ids_dev, e->scores64.p,
                    e->n_out.p, e->part.p, e->part.p + size_t(e->G) * std::max(C, 1u) * e->hpg * d,
                    e->part.p + size_t(e->G) * std::max(C, 1u) * e->hpg * (d + 1), out_dev,
                    uint32_t(e->groups[0]->bf16_attn), ids_copy};
    // fork: the W partials depend only on q, so they run beside the search
    RA_CUDA(cudaEventRecord(e->fork, s));
    RA_CUDA(cudaStreamWaitEvent(e->aux, e->fork, 0));
    launch_engine_wpartial(e->aux, ea);
    RA_CUDA(cudaEventRecord(e->join, e->aux));
  }
  record_timing(e->ev[0], s);
  if (e->n_pool > 0) {
    SearchArgs sa{};
    sa.desc = e->desc.p;
    sa.q = q_dev;
    sa.mask_bits = e->n_static ? e->w_bits.p : nullptr;
    sa.B = H;
    sa.d = d;
    sa.k = e->k;
    sa.max_M = e->max_M;
    sa.bf16 = e->groups[0]->bf16;
    sa.ids = ids_dev;
    sa.scores = e->scores.p;
    sa.scores64 = e->scores64.p;
    sa.n_out = e->n_out.p;
    sa.scanned = scanned_dev;
    sa.scanned_own = scanned_dev == e->scanned.p ? nullptr : e->scanned.p;
    sa.truncated = e->truncated.p;
    sa.expanded = e->expanded.p;
    sa.dbg = e->dbg.p;
    launch_graph_search(ctx, sa, e->max_n, e->search_scratch.p);
  } else {
    RA_CUDA(cudaMemsetAsync(e->n_out.p, 0, H * 4, s));
    RA_CUDA(cudaMemsetAsync(scanned_dev, 0, H * 8, s));
    if (scanned_dev != e->scanned.p) RA_CUDA(cudaMemsetAsync(e->scanned.p, 0, H * 8, s));
    RA_CUDA(cudaMemsetAsync(e->expanded.p, 0, H * 4, s));
  }
  record_timing(e->ev[1], s);
  if (e->fast_attn) {
    RA_CUDA(cudaStreamWaitEvent(s, e->join, 0));
    launch_engine_omega_merge(s, ea);
    record_timing(e->ev[2], s);
    return;
  }
  launch_partial_attention_ex(s, e->kvrefs.p, d, H, q_dev, e->w_ids.p, 0, e->w_m.p, nullptr, 0,
                              e->ow.p, e->zw.p, e->sw.p, nullptr, 0, e->w_empty.p, e->flag.p);
  launch_partial_attention_ex(s, e->kvrefs.p, d, H, q_dev, ids_dev, e->k, e->n_out.p,
                              e->scores64.p, e->k, e->oo.p, e->zo.p, e->so.p, nullptr, 0,
                              e->o_empty.p, e->flag.p);
  launch_merge(s, H, d, e->ow.p, e->zw.p, e->sw.p, e->w_empty.p, e->oo.p, e->zo.p, e->so.p,
               e->o_empty.p, out_dev, nullptr, nullptr, e->flag.p);
  record_timing(e->ev[2], s);
}
}  // namespace

}  // extern "C"

namespace {
void step_device_ops(ra_engine* e, const float* q, double* out, uint32_t* omega,
                     uint64_t* scanned) {
  cudaStream_t s = e->ctx->stream;
  // out and omega are written in place by the kernels (no copies)
  engine_enqueue(e, q, out ? out : e->out.p, omega && e->k ? omega : e->ids.p,
                 scanned ? scanned : e->scanned.p);
  (void)s;
}

void step_host_ops(ra_engine* e, const float* q, double* out, uint32_t* omega,
                   uint64_t* scanned) {
  cudaStream_t s = e->ctx->stream;
  // pinned (page-locked, device-mapped) host buffers: the kernels read q
  // and write out / Omega / scanned across the bus themselves, so the step
  // has no separate copy operations; pageable buffers go through copies
  static const bool zc_off = std::getenv("RA_NO_ZERO_COPY") != nullptr;
  auto mapped = [](const void* p) -> void* {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
  };
  if (!zc_off) {
    void* qd = mapped(q);
    void* od = out ? mapped(out) : e->out.p;
    void* id = omega && e->k ? mapped(omega) : e->ids.p;
    void* sd = scanned ? mapped(scanned) : e->scanned.p;
    if (qd && od && id && sd && e->fast_attn) {
      // Omega ids stay in HBM for the attention; its kernel also writes
      // them to the caller's buffer
      engine_enqueue(e, static_cast<const float*>(qd), static_cast<double*>(od), e->ids.p,
                     static_cast<uint64_t*>(sd),
                     id == e->ids.p ? nullptr : static_cast<uint32_t*>(id));
      return;
    }
  }
  RA_CUDA(cudaMemcpyAsync(e->q.p, q, size_t(e->H) * e->d * 4, cudaMemcpyHostToDevice, s));
  engine_enqueue(e, e->q.p, e->out.p, e->ids.p, e->scanned.p);
  if (out) RA_CUDA(cudaMemcpyAsync(out, e->out.p, size_t(e->H) * e->d * 8, cudaMemcpyDeviceToHost, s));
  if (omega && e->k)
    RA_CUDA(cudaMemcpyAsync(omega, e->ids.p, size_t(e->H) * e->k * 4, cudaMemcpyDeviceToHost, s));
  if (scanned)
    RA_CUDA(cudaMemcpyAsync(scanned, e->scanned.p, size_t(e->H) * 8, cudaMemcpyDeviceToHost, s));
}

bool engine_graphs_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("RA_ENGINE_GRAPH");
    return v && v[0] == '1';
  }();
  return on;
}

bool pinned_or_device(const void* p) {
  if (!p) return true;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
         at.type == cudaMemoryTypeManaged;
}

// run `ops` through the step graph cache of slot `mode`
template <typename Ops>
void run_step(ra_engine* e, int mode, const void* k0, const void* k1, const void* k2,
              const void* k3, Ops&& ops) {
  static const bool env_off = !engine_graphs_enabled();
  cudaStream_t s = e->ctx->stream;
  auto& g = e->sg[mode];
  const void* key[5] = {k0, k1, k2, k3, s};
  const bool same = std::equal(key, key + 5, g.key);
  if (env_off || e->graphs_off || !(pinned_or_device(k1) && pinned_or_device(k2) &&
                                    pinned_or_device(k3) && pinned_or_device(k0))) {
    ops();
    return;
  }
  if (same && g.exec) {
    RA_CUDA(cudaGraphLaunch(g.exec, s));
    return;
  }
  if (!same) {
    std::copy(key, key + 5, g.key);
    g.seen = 0;
    if (g.exec) cudaGraphExecDestroy(g.exec), g.exec = nullptr;
  }
  if (++g.seen < 2) {  // first call with these buffers: eager (sets kernel attributes)
    ops();
    return;
  }
  // capture on the engine's private stream (ops read ctx->stream), launch on s
  cudaGraph_t graph = nullptr;
  bool ok = true;
  if (!e->cap_stream && cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    ok = false;
  if (ok) {
    RA_CUDA(cudaStreamSynchronize(s));  // the eager prefix (e.g. q staging) is done
    e->ctx->stream = e->cap_stream;
    if (cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      ok = false;
    } else {
      try {
        ops();
      } catch (...) {
        ok = false;
      }
      if (cudaStreamEndCapture(e->cap_stream, &graph) != cudaSuccess) ok = false;
      if (ok && cudaGraphInstantiate(&g.exec, graph, 0) != cudaSuccess) ok = false;
    }
    e->ctx->stream = s;
  }
  if (graph) cudaGraphDestroy(graph), graph = nullptr;
  if (!ok) {
    cudaGetLastError();
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    e->graphs_off = true;
    ops();
    return;
  }
  RA_CUDA(cudaGraphLaunch(g.exec, s));
}
}  // namespace

extern "C" {

ra_status ra_engine_step_device(ra_engine* e, const float* q, double* out, uint32_t* omega,
                                uint64_t* scanned) {
  return guard([&] {
    if (!e) invalid("null engine");
    if (!e->step_error.empty()) invalid(e->step_error);
    DeviceGuard dg(e->ctx->device);
    // q is staged into the engine's own buffer so the captured step does not
    // depend on the caller's (often per-step) query pointer
    if (!engine_graphs_enabled()) {
      step_device_ops(e, q, out, omega, scanned);
      return;
    }
    RA_CUDA(cudaMemcpyAsync(e->q.p, q, size_t(e->H) * e->d * 4, cudaMemcpyDeviceToDevice,
                            e->ctx->stream));
    run_step(e, 0, nullptr, out, omega, scanned,
             [&] { step_device_ops(e, e->q.p, out, omega, scanned); });
  });
}

ra_status ra_engine_step_host(ra_engine* e, const float* q, double* out, uint32_t* omega,
                              uint64_t* scanned) {
  return guard([&] {
    if (!e) invalid("null engine");
    if (!e->step_error.empty()) invalid(e->step_error);
    DeviceGuard dg(e->ctx->device);
    run_step(e, 1, q, out, omega, scanned, [&] { step_host_ops(e, q, out, omega, scanned); });
    RA_CUDA(cudaStreamSynchronize(e->ctx->stream));
  });
}

ra_status ra_engine_last_stats(ra_engine* e, uint64_t* total_scanned, uint64_t* total_expanded) {
  return guard([&] {
    if (!e) invalid("null engine");
    DeviceGuard dg(e->ctx->device);
    std::vector<uint64_t> sc(e->H);
    std::vector<uint32_t> ex(e->H);
    // the kernels also write scanned into the engine's own buffer, so this
    // never reads through the caller's (possibly freed) output buffer
    RA_CUDA(cudaMemcpyAsync(sc.data(), e->scanned.p, e->H * 8, cudaMemcpyDeviceToHost,
                            e->ctx->stream));
    RA_CUDA(cudaMemcpyAsync(ex.data(), e->expanded.p, e->H * 4, cudaMemcpyDeviceToHost, e->ctx->stream));
    RA_CUDA(cudaStreamSynchronize(e->ctx->stream));
    if (total_scanned) *total_scanned = std::accumulate(sc.begin(), sc.end(), uint64_t(0));
    if (total_expanded) *total_expanded = std::accumulate(ex.begin(), ex.end(), uint64_t(0));
  });
}

uint32_t ra_engine_k(const ra_engine* e) { return e ? e->k : 0u; }

uint32_t ra_engine_kernels_per_step(const ra_engine* e) {
  return !e ? 0u : e->fused ? 1u : e->fast_attn ? 3u : 4u;
}

ra_status ra_engine_last_timing(ra_engine* e, float* search_ms, float* attention_ms) {
  return guard([&] {
    if (!e) invalid("null engine");
    DeviceGuard dg(e->ctx->device);
    RA_CUDA(cudaEventSynchronize(e->ev[2]));
    if (search_ms) RA_CUDA(cudaEventElapsedTime(search_ms, e->ev[0], e->ev[1]));
    if (attention_ms) RA_CUDA(cudaEventElapsedTime(attention_ms, e->ev[1], e->ev[2]));
  });
}

// Search-kernel counters of the last step summed over heads: rounds,
// cycles in pre-expansion, cycles in commit, commits (profiling aid).
ra_status ra_engine_debug_counters(ra_engine* e, uint64_t* out12) {
  return guard([&] {
    if (!e) invalid("null engine");
    DeviceGuard dg(e->ctx->device);
    std::vector<uint64_t> h(size_t(e->H) * 12);
    RA_CUDA(cudaMemcpyAsync(h.data(), e->dbg.p, h.size() * 8, cudaMemcpyDeviceToHost, e->ctx->stream));
    RA_CUDA(cudaStreamSynchronize(e->ctx->stream));
    for (int j = 0; j < 12; ++j) out12[j] = 0;
    for (size_t i = 0; i < h.size(); ++i) out12[i % 12] += h[i];
  });
}

ra_status ra_engine_debug_counters_per_head(ra_engine* e, uint64_t* out) {
  return guard([&] {
    if (!e) invalid("null engine");
    DeviceGuard dg(e->ctx->device);
    RA_CUDA(cudaMemcpyAsync(out, e->dbg.p, size_t(e->H) * 96, cudaMemcpyDeviceToHost, e->ctx->stream));
    RA_CUDA(cudaStreamSynchronize(e->ctx->stream));
  });
}

}  // extern "C"
