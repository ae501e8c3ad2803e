// Shared internals of libra_b200.so (sm_100a). Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "ra_capi.h"

namespace ra {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kSentinel = 0xFFFFFFFFu;  // padded adjacency slot / "no id"

// ---- error plumbing: exceptions inside, ra_status at the ABI --------------
struct Error : std::runtime_error {
  ra_status code;
  Error(ra_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void invalid(const std::string& m) {
  throw Error(RA_ERR_INVALID_ARGUMENT, m);
}
[[noreturn]] inline void runtime(const std::string& m) { throw Error(RA_ERR_RUNTIME, m); }

void set_last_error(const std::string& m);

template <typename F>
ra_status guard(F&& f) {
  try {
    f();
    return RA_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return RA_ERR_RUNTIME;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return RA_ERR_RUNTIME;
  }
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(RA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                                 ":" + std::to_string(line) + ")");
}
#define RA_CUDA(x) ::ra::cuda_check((x), #x, __FILE__, __LINE__)
#define RA_LAUNCH_CHECK() ::ra::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// ---- device buffers ------------------------------------------------------------
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  // stream-ordered temporaries (alloc with a stream): cudaMallocAsync /
  // cudaFreeAsync from the device's default pool, which keeps freed blocks
  // (release threshold set at context creation), so a build's gigabyte-
  // sized scratch costs no cudaMalloc / cudaFree (device sync) per call.
  // Only for buffers that die before their stream does.
  cudaStream_t st = nullptr;
  bool pooled = false;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(size_t count, cudaStream_t s) { alloc(count, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), st(o.st), pooled(o.pooled) {
    o.p = nullptr, o.n = 0, o.pooled = false;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(st, o.st);
    std::swap(pooled, o.pooled);
    return *this;
  }
  ~DevBuf() { reset(); }
  void alloc(size_t count) {
    reset();
    if (count) RA_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void alloc(size_t count, cudaStream_t s) {
    reset();
    if (count) RA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    n = count, st = s, pooled = true;
  }
  // a long-lived buffer taken from the stream-ordered pool (no synchronous
  // cudaMalloc on the build path: those measured up to 135 ms at times),
  // released with cudaFree (valid for pool memory; it synchronizes)
  void alloc_lived(size_t count, cudaStream_t s) {
    reset();
    if (count) RA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    n = count;
  }
  // grow-only reallocation (contents not preserved)
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void reset() {
    if (p) {
      if (pooled) cudaFreeAsync(p, st);
      else cudaFree(p);
    }
    p = nullptr;
    n = 0;
    pooled = false;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Device-side view of one query head's graph (what the search kernel reads).
struct GraphDesc {
  const uint32_t* adj;  // [n][M], kSentinel-padded rows
  const float* keys;    // [n][d]
  const uint16_t* keys16;  // [n][d] bf16 copy (bf16 KV groups), else nullptr
  uint64_t entry;
  uint32_t n, M;
  uint32_t ef;          // resolved ef for this query
  uint32_t pad;
};

}  // namespace ra

// ---- handles -----------------------------------------------------------------
struct ra_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 0;
  int search_kernel = -1;  // K6 variant override (ra_ctx_set_search_kernel); -1 = env / auto
  // grow-only scratch arenas reused across calls (one call at a time per ctx)
  ra::DevBuf<uint8_t> scratch_a;
  ra::DevBuf<uint8_t> scratch_b;
  ra::DevBuf<uint8_t> scratch_c;
  // a side stream + fork / join events (created on first use): the build's
  // column mean runs there beside phases 1-3
  cudaStream_t side = nullptr;
  cudaEvent_t side_fork = nullptr, side_join = nullptr;
};

struct ra_kv {
  std::atomic<int> refs{1};
  int device = 0;
  uint64_t n = 0;
  uint32_t d = 0;
  ra::DevBuf<float> keys;    // n x d row-major (f32, the reference's VectorSet layout)
  ra::DevBuf<float> values;  // n x d row-major (may be empty)
  // bf16 KV groups (ra_kv_create_bf16): K and V also stored rounded to bf16
  // (RNE). bf16: the search reads bf16 key rows too, and the f32 arrays above
  // hold the same rounded values (builder, generic paths) - the reference's
  // results on the rounded inputs. bf16_attn only: the search keeps the exact
  // f32 keys (retrieved ids identical to f32), attention reads bf16 K/V.
  bool bf16 = false;
  bool bf16_attn = false;
  ra::DevBuf<uint16_t> keys16, values16;
};

struct ra_graph {
  ra_kv* kv = nullptr;  // retained
  uint64_t n = 0;
  uint32_t max_degree = 0;
  uint32_t default_ef = 128;
  uint64_t entry = 0;
  // device: fixed-stride adjacency, row u = adj[u*max_degree ...], padded
  // with kSentinel past degree(u): one coalesced load per expansion, no
  // offsets hop.
  ra::DevBuf<uint32_t> adj;
  uint64_t n_edges = 0;
  // host mirror (reference CSR) for accessors and OODG serialization: set by
  // deserialize; a GPU build leaves it empty and host_mirror() downloads the
  // device rows on first use (the build never waits for it)
  mutable std::vector<uint64_t> offsets;
  mutable std::vector<uint32_t> adjacency;
  mutable std::once_flag host_once;
  void host_mirror() const;
};

namespace ra {

struct DeviceGuard {
  int prev = -1;
  // no_throw: for destroy/release paths (possibly at process teardown, when
  // the runtime is already gone) - a failure there must not terminate
  explicit DeviceGuard(int dev, bool no_throw = false) {
    cudaGetDevice(&prev);
    if (prev != dev) {
      if (no_throw) {
        if (cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
      } else {
        RA_CUDA(cudaSetDevice(dev));
      }
    }
  }
  ~DeviceGuard() {
    int cur;
    if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Host CSR mirror -> fixed-stride device adjacency (capi.cu).
void graph_upload(ra_ctx* ctx, ra_graph* g);

// grow-only typed carve-outs from a ctx arena
template <typename T>
T* arena(DevBuf<uint8_t>& a, size_t count) {
  a.ensure(count * sizeof(T) + 256);
  return reinterpret_cast<T*>(a.p);
}

// ---- search (search.cu) --------------------------------------------------------
struct SearchArgs {
  const GraphDesc* desc;      // [B] device
  const float* q;             // [B][d]
  const uint32_t* mask_bits;  // bitset over ids, nullptr = no mask (shared by batch)
  uint32_t B, d, k;
  uint32_t max_M;             // max degree bound over the batch's graphs
  uint32_t* ids;              // [B][k]
  float* scores;              // [B][k]
  double* scores64;           // optional [B][k] exact f64 scores
  uint32_t* n_out;            // [B]
  uint64_t* scanned;          // [B]
  uint64_t* scanned_own;      // [B] optional second copy (engine-owned, read by last_stats)
  uint8_t* truncated;         // [B]
  uint32_t* expanded;         // optional [B]
  uint64_t* dbg;              // optional [B][4]: rounds, cycles A, cycles B, commits
  // HBM spill area used when a query outgrows its shared-memory list
  // (per query: max_n entries of f64 + u32 + u8) and the visited bitset
  // when it does not fit shared memory (per query: ceil(max_n/32) words).
  uint8_t* spill;
  uint32_t* vis_global;
  uint32_t flags;  // profiling switches (RA_PIPE_FLAGS): 1 = helpers idle
  uint32_t bf16;   // every desc[b].keys16 is set: score from the bf16 rows
  // fused decode attention (latency-mode pipe kernel, f32 groups): idle
  // helpers compute the W partials in chunks during the search, the CTA
  // computes the Omega partial and the merge after it. out == nullptr: off.
  struct FusedAttn {
    const float* const* values;  // [B] the head's V rows (n x d f32)
    const uint32_t* W;           // static ids, ascending
    uint32_t nW, nchunk;         // nchunk = ceil(nW / crows)
    uint32_t crows;              // W rows per chunk (<= 32 and <= the helpers' tile rows)
    double inv_sqrt_d;
    double* out;                 // [B][d] attention output
    double* chunk;               // scratch [B][nchunk][d + 2]: (out, max, expsum)
  } fa;
};

// Returns bytes of scratch needed for (B, max_n, d); then launches.
size_t search_scratch_bytes(const ra_ctx* ctx, uint32_t B, uint32_t max_n, uint32_t d);
void launch_graph_search(ra_ctx* ctx, SearchArgs a, uint32_t max_n, uint8_t* scratch);
// v5 pipelined kernel (search_pipe.cu); false when the shape is unsupported.
// mode: 0 = auto (latency / throughput by batch size), 1 = throughput, 2 = latency
size_t search_pipe_scratch_bytes(uint32_t B, uint32_t max_n);
bool launch_graph_search_pipe(ra_ctx* ctx, const SearchArgs& a, uint32_t max_n,
                              uint8_t* scratch, int mode);
// whether launch_graph_search will run a.fa (the fused attention) for this
// batch: latency-mode pipe kernel, f32 rows, supported shape
bool search_fuses_attention(const ra_ctx* ctx, const SearchArgs& a, uint32_t max_n);
// K6 variant by name (RA_SEARCH_KERNEL / ra_ctx_set_search_kernel); -1 = unknown
int search_variant_of(const char* name);
bool pipe_latency_supported(const ra_ctx* ctx, uint32_t d, uint32_t max_M, uint32_t max_n);

void launch_mask_bitset(cudaStream_t s, const uint32_t* mask, uint64_t mask_n, uint32_t* bits,
                        uint64_t words);

// ---- attention (attention.cu) --------------------------------------------------
size_t partial_scratch_doubles(uint32_t B, uint32_t max_m);
struct KVRef {
  const float* keys;
  const float* values;
  uint64_t n;
  const uint16_t* keys16;    // bf16 groups only
  const uint16_t* values16;
};
void launch_partial_attention_ex(cudaStream_t s, const KVRef* kvs, uint32_t d, uint32_t B, const float* q,
                                 const uint32_t* idx, uint32_t m_stride, const uint32_t* m,
                                 const double* scores64, uint32_t s_stride, double* out,
                                 double* zmax, double* expsum, double* zscratch,
                                 uint64_t z_stride, uint8_t* empty_out, uint32_t* err_flag);
void launch_merge(cudaStream_t s, uint32_t B, uint32_t d, const double* ow, const double* zw,
                  const double* sw, const uint8_t* w_empty, const double* oo,
                  const double* zo, const double* so, const uint8_t* o_empty, double* out,
                  double* gw, double* go, uint32_t* err_flag);

// engine fast path (attention.cu): W partial per (group, 64-row chunk) on a
// side stream (overlaps the search), then Omega partial + chunk fold + merge
// per head on the main stream after the search.
struct EngineAttn {
  const KVRef* gkv;   // [G] per group
  const KVRef* hkv;   // [H] per head
  const float* q;     // [H][d]
  const uint32_t* W;  // static ids
  uint32_t nW, G, H, hpg, d, k;
  double inv_sqrt_d;
  const uint32_t* ids;   // [H][k] omega
  const double* s64;     // [H][k] exact scores
  const uint32_t* n_out; // [H]
  double* part_out;      // [G][C][hpg][d]
  double* part_m;        // [G][C][hpg]
  double* part_s;
  double* out;           // [H][d]
  uint32_t bf16;         // K/V read from the groups' bf16 copies
  uint32_t* ids_out = nullptr;  // optional second home of the Omega ids (caller's buffer)
};
bool engine_attention_supported(uint32_t d);
size_t engine_attention_part_doubles(uint32_t G, uint32_t hpg, uint32_t nW, uint32_t d);
void launch_engine_wpartial(cudaStream_t st, const EngineAttn& a);
void launch_engine_omega_merge(cudaStream_t st, const EngineAttn& a);

// tensor-core kNN (knn_tc.cu)
bool knn_tc_supported(uint32_t d, uint64_t nq, uint32_t n, uint32_t kt);
uint32_t knn_tc(ra_ctx* ctx, const float* Q, uint64_t nq, const float* K, uint32_t n, uint32_t d,
                uint32_t kt, uint32_t* knn, DevBuf<uint32_t>& fail_rows, double* ms_gemm);

}  // namespace ra
