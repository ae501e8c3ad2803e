// Graph build on the GPU: B200 restatement of OODGraph::build
// (/root/reference/proj/src/index_oodgraph.cpp:89-355).
//
//   K0 k_norms        squared norms, in-order f64 (:101-102)
//   K1 k_knn          phase 1 exact query->key top-k_train (:104-128): tiled
//                     f64 products accumulated in dimension order (identical
//                     to the reference's f64 GEMM of f32-widened inputs),
//                     fused with a per-query threshold + candidate buffer so
//                     the nq x n score matrix never exists
//   K2 k_proposals    phase 2 rank-window edge proposals (:130-156); the
//                     global sort+unique runs on CUB radix sort
//   K3 k_prune        phase 3 occlusion prune, one warp per node (:162-202)
//   K4 entry point    medoid / max-norm argmin-argmax (:207-233)
//   K5 repair         phase 4 (:235-348) on the GPU: reachability by a
//                     work-queue sweep, pending / anchor lists by stream
//                     compaction, the nearest anchor as a tiled FP64 GEMM,
//                     (anchor, node) sort, one block per anchor group for the
//                     chained attachments; the host only reads the counts
// Every f64 reduction runs in the reference's order (through the
// sequential-order Eigen contract of oracle/shim), so adjacency, entry point
// and OODG blob are bit-identical to the oracle build.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cstring>
#include <memory>
#include <numeric>

#include "common.cuh"

#include <cstdlib>

namespace ra {
namespace {

__device__ __forceinline__ bool better(double sa, uint32_t ia, double sb, uint32_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// in-order f64 dot of two f32 rows (products exact, so fma == mul+add)
__device__ __forceinline__ double dot_rows(const float* __restrict__ a,
                                           const float* __restrict__ b, uint32_t d) {
  double acc = 0.0;
  if ((d & 3) == 0) {
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll 4
    for (uint32_t c = 0; c < d / 4; ++c) {
      const float4 x = __ldg(a4 + c), y = __ldg(b4 + c);
      acc = fma((double)x.x, (double)y.x, acc);
      acc = fma((double)x.y, (double)y.y, acc);
      acc = fma((double)x.z, (double)y.z, acc);
      acc = fma((double)x.w, (double)y.w, acc);
    }
  } else {
    for (uint32_t i = 0; i < d; ++i) acc = fma((double)__ldg(a + i), (double)__ldg(b + i), acc);
  }
  return acc;
}

// f32 dot with four partial sums (one per float4 lane component): a fast
// estimate whose error is at most (d / 4 + 3) * 2^-24 * sum |a_i b_i| <=
// (d / 4 + 3) * 2^-24 * |a| |b| (recursive fp32 FMA summation, Cauchy-Schwarz)
__device__ __forceinline__ float dot_f32_est(const float* __restrict__ a, const float* __restrict__ b,
                                             uint32_t d) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if ((d & 3) == 0) {
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll 8
    for (uint32_t c = 0; c < d / 4; ++c) {
      const float4 x = __ldg(a4 + c), y = __ldg(b4 + c);
      s0 = fmaf(x.x, y.x, s0);
      s1 = fmaf(x.y, y.y, s1);
      s2 = fmaf(x.z, y.z, s2);
      s3 = fmaf(x.w, y.w, s3);
    }
  } else {
    for (uint32_t i = 0; i < d; ++i) s0 = fmaf(__ldg(a + i), __ldg(b + i), s0);
  }
  return (s0 + s1) + (s2 + s3);
}

// ---- K0 -------------------------------------------------------------------------
__global__ void k_norms(const float* __restrict__ keys, uint32_t n, uint32_t d, double* norms) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) norms[i] = dot_rows(keys + size_t(i) * d, keys + size_t(i) * d, d);
}

// ---- K1 -------------------------------------------------------------------------
// CTA = 64 queries x (all keys in tiles of 64). Thread (ty, tx) owns queries
// ty + 16i and keys tx + 16j (i, j < 4); dims stream through shared memory in
// chunks of 32, widened to f64 once, so each accumulator is the reference's
// in-order f64 sum. After each key tile, scores strictly better than the
// query's running k-th best (theta) are appended to its HBM candidate buffer;
// a buffer about to overflow is compacted (bitonic sort, keep kt, theta =
// kt-th). Result: rows ranked (score desc, id asc) == TopKCollector order.
constexpr int KQ = 64, KK = 64, KDC = 32, KTHREADS = 256;

__device__ void warp_bitonic_desc(double* s, uint32_t* id, uint32_t n_pow2, uint32_t lane) {
  for (uint32_t k = 2; k <= n_pow2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < n_pow2; i += 32) {
        const uint32_t p = i ^ j;
        if (p > i) {
          const bool desc = (i & k) == 0;
          const double si = s[i], sp = s[p];
          const uint32_t ii = id[i], ip = id[p];
          const bool swap = desc ? better(sp, ip, si, ii) : better(si, ii, sp, ip);
          if (swap) {
            s[i] = sp, s[p] = si;
            id[i] = ip, id[p] = ii;
          }
        }
      }
      __syncwarp();
    }
  }
}

// sort buffer of query q (cnt entries) best-first, keep kt; returns new count
__device__ uint32_t compact_query(double* bs, uint32_t* bi, uint32_t cnt, uint32_t kt,
                                  uint32_t lane) {
  uint32_t p2 = 1;
  while (p2 < cnt) p2 <<= 1;
  for (uint32_t i = cnt + lane; i < p2; i += 32) {
    bs[i] = -DBL_MAX;
    bi[i] = kSentinel;
  }
  __syncwarp();
  warp_bitonic_desc(bs, bi, p2, lane);
  return cnt < kt ? cnt : kt;
}

__global__ void __launch_bounds__(KTHREADS)
    k_knn(const float* __restrict__ Q, uint64_t nq, const float* __restrict__ K, uint32_t n,
          uint32_t d, uint32_t kt, uint32_t cb, double* __restrict__ bufS,
          uint32_t* __restrict__ bufI, uint32_t* __restrict__ knn, unsigned long long* widen_ctr,
          double* __restrict__ knn_s = nullptr, uint32_t kchunk = 0) {
  // key split (few rows): block y scans keys [y * kchunk, +kchunk) into its
  // own buffers and writes that range's top kt (ids absolute, with scores)
  // at row y * nq + q; k_knn_merge then ranks the union
  const uint32_t kbeg = kchunk ? blockIdx.y * kchunk : 0;
  const uint32_t kend = kchunk ? min(n, kbeg + kchunk) : n;
  const uint64_t rbase = uint64_t(blockIdx.y) * nq;
  bufS += rbase * cb, bufI += rbase * cb, knn += rbase * kt;
  if (knn_s) knn_s += rbase * kt;
  __shared__ double Qs[KDC][KQ + 1];
  __shared__ double Ks[KDC][KK + 1];
  __shared__ double th_s[KQ];
  __shared__ uint32_t th_i[KQ];
  __shared__ uint32_t cnt[KQ];
  __shared__ int need_compact;
  const uint32_t tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const uint32_t lane = tid & 31, warp = tid >> 5;
  const uint64_t q0 = uint64_t(blockIdx.x) * KQ;
  if (tid < KQ) {
    th_s[tid] = -DBL_MAX;
    th_i[tid] = kSentinel;
    cnt[tid] = 0;
  }
  __syncthreads();

  for (uint32_t k0 = kbeg; k0 < kend; k0 += KK) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (uint32_t c0 = 0; c0 < d; c0 += KDC) {
      // stage 64 x 32 dims of Q and K, widened to f64, dimension-major
      for (uint32_t e = tid; e < KQ * KDC; e += KTHREADS) {
        const uint32_t r = e / KDC, c = e % KDC;
        const uint64_t qi = q0 + r;
        const uint32_t ki = k0 + r;
        Qs[c][r] = (qi < nq && c0 + c < d) ? (double)Q[qi * d + c0 + c] : 0.0;
        Ks[c][r] = (ki < kend && c0 + c < d) ? (double)K[size_t(ki) * d + c0 + c] : 0.0;
      }
      __syncthreads();
      const uint32_t cmax = min(KDC, d - c0);
      for (uint32_t c = 0; c < cmax; ++c) {
        double qv[4], kv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[i] = Qs[c][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) kv[j] = Ks[c][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(qv[i], kv[j], acc[i][j]);
      }
      __syncthreads();
    }
    // offer to per-query candidate buffers
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t ql = ty + 16 * i;
      if (q0 + ql >= nq) continue;
      const double ts = th_s[ql];
      const uint32_t ti = th_i[ql];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = k0 + tx + 16 * j;
        if (key < kend && better(acc[i][j], key, ts, ti)) {
          const uint32_t pos = atomicAdd(&cnt[ql], 1u);
          bufS[(q0 + ql) * cb + pos] = acc[i][j];
          bufI[(q0 + ql) * cb + pos] = key;
        }
      }
    }
    if (tid == 0) need_compact = 0;
    __syncthreads();
    if (tid < KQ && cnt[tid] + KK > cb) need_compact = 1;
    __syncthreads();
    if (need_compact) {
      __threadfence_block();
      for (uint32_t ql = warp; ql < KQ; ql += KTHREADS / 32) {
        if (q0 + ql >= nq || cnt[ql] + KK <= cb) continue;
        double* bs = bufS + (q0 + ql) * cb;
        uint32_t* bi = bufI + (q0 + ql) * cb;
        const uint32_t c = compact_query(bs, bi, cnt[ql], kt, lane);
        if (lane == 0) {
          cnt[ql] = c;
          if (c == kt) {
            th_s[ql] = bs[kt - 1];
            th_i[ql] = bi[kt - 1];
          }
        }
        if (lane == 0 && widen_ctr) atomicAdd(widen_ctr, 1ull);
      }
      __syncthreads();
    }
  }
  // final ranking
  __threadfence_block();
  __syncthreads();
  for (uint32_t ql = warp; ql < KQ; ql += KTHREADS / 32) {
    if (q0 + ql >= nq) continue;
    double* bs = bufS + (q0 + ql) * cb;
    uint32_t* bi = bufI + (q0 + ql) * cb;
    const uint32_t c = compact_query(bs, bi, cnt[ql], kt, lane);
    for (uint32_t r = lane; r < kt; r += 32) {  // r >= c only for a short key range
      knn[(q0 + ql) * kt + r] = r < c ? bi[r] : kSentinel;
      if (knn_s) knn_s[(q0 + ql) * kt + r] = r < c ? bs[r] : -DBL_MAX;
    }
  }
}

// union of the key-split partial lists of each row (C ranges x kt, exact
// scores) -> the row's top kt; warp per row, sorted in its bufS/bufI slot
__global__ void k_knn_merge(const uint32_t* __restrict__ pid, const double* __restrict__ ps,
                            uint32_t nq, uint32_t C, uint32_t kt, uint32_t cb,
                            double* __restrict__ bufS, uint32_t* __restrict__ bufI,
                            uint32_t* __restrict__ knn) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= nq) return;
  double* bs = bufS + size_t(row) * cb;
  uint32_t* bi = bufI + size_t(row) * cb;
  for (uint32_t e = lane; e < C * kt; e += 32) {
    const uint32_t c = e / kt, r = e % kt;
    bs[e] = ps[(size_t(c) * nq + row) * kt + r];
    bi[e] = pid[(size_t(c) * nq + row) * kt + r];
  }
  __syncwarp();
  compact_query(bs, bi, C * kt, kt, lane);
  for (uint32_t r = lane; r < kt; r += 32) knn[size_t(row) * kt + r] = bi[r];
}

// exact fallback rows (few): every key's in-order f64 score for each row,
// as (order-preserving key, id) pairs for a segmented radix sort (stable:
// equal scores keep ascending ids, the TopKCollector order)
__device__ __forceinline__ uint64_t okey64(double x) {
  const uint64_t u = __double_as_longlong(x + 0.0);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}
__global__ void k_exact_scores(const float* __restrict__ Q, const uint32_t* __restrict__ rows,
                               uint32_t nr, const float* __restrict__ K, uint32_t n, uint32_t d,
                               uint64_t* __restrict__ sk, uint32_t* __restrict__ sv) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= uint64_t(nr) * n) return;
  const uint32_t r = uint32_t(t / n), j = uint32_t(t % n);
  sk[t] = okey64(dot_rows(Q + size_t(rows[r]) * d, K + size_t(j) * d, d));
  if (sv) sv[t] = j;
}

// Block per exact-fallback row: radix-select the kt-th largest key of the
// row's n keys (8 bits per pass, warp-aggregated histogram), gather the keys
// >= it and bitonic-sort them by (key desc, id asc) in shared memory: the
// first kt are exactly the stable segmented sort's first kt. Rows with more
// than XCAP keys >= the kt-th (mass ties) are listed in ovf_rows (query ids)
// for the segmented sort.
constexpr uint32_t XT = 1024, XCAP = 2048;
__global__ void __launch_bounds__(XT)
    k_exact_topk(const uint64_t* __restrict__ sk, uint32_t n, uint32_t kt,
                 const uint32_t* __restrict__ rows, uint32_t* __restrict__ knn,
                 uint32_t* __restrict__ ovf_rows, uint32_t* __restrict__ n_ovf, uint32_t cap) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t ck[XCAP];
  __shared__ uint32_t ci[XCAP];
  __shared__ uint32_t s_digit, s_need, s_cnt;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint64_t* kr = sk + uint64_t(blockIdx.x) * n;
  uint64_t prefix = 0, pmask = 0;
  uint32_t need = kt;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (uint32_t b = tid; b < 256; b += XT) hist[b] = 0;
    __syncthreads();
    for (uint32_t i0 = 0; i0 < n; i0 += XT) {
      const uint32_t i = i0 + tid;
      const uint64_t k = i < n ? kr[i] : 0;
      const bool in = i < n && (k & pmask) == prefix;
      const uint32_t dg = in ? uint32_t(k >> shift) & 255u : 256u;
      const uint32_t peers = __match_any_sync(kFull, dg);
      if (in && lane == uint32_t(__ffs(peers) - 1)) atomicAdd(&hist[dg], uint32_t(__popc(peers)));
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int b = 255; b >= 0; --b) {
        if (acc + hist[b] >= need) {
          s_digit = uint32_t(b);
          s_need = need - acc;
          break;
        }
        acc += hist[b];
      }
    }
    __syncthreads();
    prefix |= uint64_t(s_digit) << shift;
    pmask |= 0xFFull << shift;
    need = s_need;
    __syncthreads();
  }
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (uint32_t i = tid; i < n; i += XT) {
    const uint64_t k = kr[i];
    if (k >= prefix) {
      const uint32_t at = atomicAdd(&s_cnt, 1u);
      if (at < XCAP) ck[at] = k, ci[at] = i;
    }
  }
  __syncthreads();
  const uint32_t cnt = s_cnt;
  if (cnt > cap) {
    if (tid == 0) ovf_rows[atomicAdd(n_ovf, 1u)] = rows[blockIdx.x];
    return;
  }
  uint32_t p2 = 1;
  while (p2 < cnt) p2 <<= 1;
  for (uint32_t i = cnt + tid; i < p2; i += XT) ck[i] = 0, ci[i] = 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t k = 2; k <= p2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < p2; i += XT) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const uint64_t ki = ck[i], kl = ck[l];
          const uint32_t ii = ci[i], il = ci[l];
          const bool l_first = kl > ki || (kl == ki && il < ii);
          const bool i_first = ki > kl || (ki == kl && ii < il);
          if ((i & k) == 0 ? l_first : i_first) {
            ck[i] = kl, ck[l] = ki;
            ci[i] = il, ci[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t j = tid; j < kt; j += XT) knn[uint64_t(rows[blockIdx.x]) * kt + j] = ci[j];
}
__global__ void k_take_top(const uint32_t* __restrict__ sv, uint32_t nr, uint32_t n, uint32_t kt,
                           const uint32_t* __restrict__ rows, uint32_t* __restrict__ knn) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= uint64_t(nr) * kt) return;
  const uint32_t r = uint32_t(t / kt), i = uint32_t(t % kt);
  knn[uint64_t(rows[r]) * kt + i] = sv[uint64_t(r) * n + i];
}
__global__ void k_seg_offsets(uint32_t nr, uint32_t n, int* off) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= nr) off[i] = int(i * n);
}

__global__ void k_gather_rows(const float* __restrict__ Q, uint32_t d,
                              const uint32_t* __restrict__ rows, uint32_t nr, float* out) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t < uint64_t(nr) * d) out[t] = Q[uint64_t(rows[t / d]) * d + t % d];
}
__global__ void k_scatter_knn(const uint32_t* __restrict__ kf, const uint32_t* __restrict__ rows,
                              uint32_t nr, uint32_t kt, uint32_t* knn) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t < uint64_t(nr) * kt) knn[uint64_t(rows[t / kt]) * kt + t % kt] = kf[t];
}

// ---- K2 -------------------------------------------------------------------------
// proposals of rank b (:142-148): count(b) = (lo > 0) + (b - lo)
__host__ __device__ inline uint32_t prop_lo(uint32_t b, uint32_t w) {
  return (w > 0 && b > w) ? b - w : 0;
}
__host__ __device__ inline uint32_t prop_count(uint32_t b, uint32_t w) {
  const uint32_t lo = prop_lo(b, w);
  return (lo > 0 ? 1u : 0u) + (b - lo);
}

// bits of an id in [0, n) (>= 1)
__host__ __device__ __forceinline__ uint32_t edge_bits(uint32_t n) {
  uint32_t b = 1;
  while (b < 32 && (uint64_t(n - 1) >> b) != 0) ++b;
  return b;
}

// proposals packed as (src << eb) | dst with eb = bits of n - 1, so the
// radix sort runs over 2 * eb key bits only
__global__ void k_proposals(const uint32_t* __restrict__ knn, uint64_t nq, uint32_t kt,
                            uint32_t w, const uint32_t* __restrict__ b_off, uint32_t per_row,
                            uint32_t eb, uint64_t* __restrict__ out) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= nq * (kt - 1)) return;
  const uint64_t qi = t / (kt - 1);
  const uint32_t b = uint32_t(t % (kt - 1)) + 1;
  const uint32_t* row = knn + qi * kt;
  const uint64_t u = row[b];
  uint64_t* o = out + qi * per_row + b_off[b];
  const uint32_t lo = prop_lo(b, w);
  if (lo > 0) *o++ = u << eb | row[0];
  for (uint32_t a = lo; a < b; ++a) *o++ = u << eb | row[a];
}

// Proposals deduplicated in an open-addressing set instead of a global
// sort + unique of every proposal (~30x duplicates at 128K: the same hub
// pairs are proposed by many queries). Slots hold a key or kHEmpty and go
// only from empty to a key, so a stale read can only show empty (then the
// CAS decides). A probe run past kHProbe sets *overflow and the caller
// takes the sort path. The surviving keys are compacted and sorted, which
// gives exactly the sorted unique list of the sort path.
constexpr unsigned long long kHEmpty = ~0ull;
constexpr int kHProbe = 128;

__global__ void k_proposals_hash(const uint32_t* __restrict__ knn, uint64_t nq, uint32_t kt,
                                 uint32_t w, uint32_t eb, unsigned long long* __restrict__ tab,
                                 uint32_t lg, uint32_t* overflow) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= nq * (kt - 1)) return;
  const uint64_t qi = t / (kt - 1);
  const uint32_t b = uint32_t(t % (kt - 1)) + 1;
  const uint32_t* row = knn + qi * kt;
  const uint64_t u = row[b];
  const uint64_t mask = (1ull << lg) - 1;
  auto insert = [&](uint32_t v) {
    const unsigned long long key = u << eb | v;
    uint64_t h = (key * 0x9E3779B97F4A7C15ull) >> (64 - lg);
    for (int pr = 0; pr < kHProbe; ++pr, h = (h + 1) & mask) {
      unsigned long long cur = tab[h];
      if (cur == kHEmpty) cur = atomicCAS(tab + h, kHEmpty, key);
      if (cur == kHEmpty || cur == key) return;
    }
    atomicOr(overflow, 1u);
  };
  const uint32_t lo = prop_lo(b, w);
  if (lo > 0) insert(row[0]);
  for (uint32_t a = lo; a < b; ++a) insert(row[a]);
}

struct HNotEmpty {
  __device__ bool operator()(unsigned long long k) const { return k != kHEmpty; }
};

__global__ void k_src_offsets(const uint64_t* __restrict__ edges, uint64_t ne, uint32_t n,
                              uint32_t eb, uint64_t* __restrict__ off) {
  const uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (u > n) return;
  const uint64_t key = u << eb;
  uint64_t lo = 0, hi = ne;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (edges[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  off[u] = lo;
}

// ---- K3 -------------------------------------------------------------------------
// Warp per node u. Candidates (m_uv, v) are formed with in-order f64 dots,
// sorted ascending (std::pair order), truncated to ef_construction, then
// the occlusion loop keeps v unless some kept w has m_vw < m_uv; lanes test
// all kept w of one candidate in parallel (the reference's early break does
// not change the outcome). Fill to the cap from the ordered list.
constexpr int PWARPS = 8;
constexpr uint32_t PCAP = 1024;  // candidates held in shared memory per warp

__device__ void warp_bitonic_asc(double* m, uint32_t* v, uint32_t n_pow2, uint32_t lane) {
  for (uint32_t k = 2; k <= n_pow2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < n_pow2; i += 32) {
        const uint32_t p = i ^ j;
        if (p > i) {
          const bool asc = (i & k) == 0;
          const double mi = m[i], mp = m[p];
          const uint32_t vi = v[i], vp = v[p];
          const bool p_less = mp < mi || (mp == mi && vp < vi);
          const bool i_less = mi < mp || (mi == mp && vi < vp);
          if (asc ? p_less : i_less) {
            m[i] = mp, m[p] = mi;
            v[i] = vp, v[p] = vi;
          }
        }
      }
      __syncwarp();
    }
  }
}

// prune work order: candidate count per node (keys for a descending sort);
// nodes without candidates get their empty row here and are counted out
__global__ void k_prune_order(const uint64_t* __restrict__ off, uint32_t n, uint32_t M,
                              uint32_t* key, uint32_t* val, uint32_t* adj, uint32_t* deg,
                              uint32_t* n_active) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const uint64_t c = off[u + 1] - off[u];
  key[u] = c > 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(c);
  val[u] = u;
  if (c) {
    atomicAdd(n_active, 1u);
  } else {
    deg[u] = 0;
    for (uint32_t j = 0; j < M; ++j) adj[size_t(u) * M + j] = 0xFFFFFFFFu;
  }
}

#ifdef RA_PRUNE_PROF
// (profiling aid) score+sort / occlusion / fill cycles, candidates tested,
// ballot rounds, pair tests, nodes that filled M, kept sum, exact tests
__device__ unsigned long long g_prune_prof[9];
#define PPROF(i, v) \
  do { if (lane == 0) atomicAdd(&g_prune_prof[i], (unsigned long long)(v)); } while (0)
#else
#define PPROF(i, v) do {} while (0)
#endif

__global__ void __launch_bounds__(PWARPS * 32)
    k_prune(const float* __restrict__ keys, uint32_t n, uint32_t d,
            const double* __restrict__ norms, const uint64_t* __restrict__ edges,
            const uint64_t* __restrict__ off, const uint32_t* __restrict__ nodes,
            uint32_t n_nodes, uint32_t M, uint32_t efc, int euclid, double* gm, uint32_t* gv,
            uint64_t g_stride, uint32_t* __restrict__ adj, uint32_t* __restrict__ deg,
            uint32_t* big_nodes, uint32_t* big_count, uint32_t* queue) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t wid = blockIdx.x * PWARPS + warp;
  const uint64_t dst_mask = (1ull << edge_bits(n)) - 1;  // (edges: src << eb | dst)
  const bool global_mode = gm != nullptr;
  double* sm = reinterpret_cast<double*>(smem) + size_t(warp) * PCAP;
  uint32_t* sv = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(smem) + PWARPS * PCAP) +
                 size_t(warp) * PCAP;
  uint32_t* kept = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(smem) + PWARPS * PCAP) +
                   PWARPS * PCAP + size_t(warp) * M;
  // queue != null: `nodes` is ordered by candidate count, descending, and
  // warps take the next node from queue[0] until queue[1] (largest first:
  // the hubs start at once and the small nodes fill in behind them)
  const uint32_t n_work = queue ? queue[1] : n_nodes;
  for (uint32_t it = 0;; ++it) {
    uint32_t idx = wid + it * gridDim.x * PWARPS;
    if (queue) {
      if (lane == 0) idx = atomicAdd(queue, 1u);
      idx = __shfl_sync(kFull, idx, 0);
    }
    if (idx >= n_work) break;
    const uint32_t u = nodes ? nodes[idx] : idx;
    const uint64_t c0 = off[u], c1 = off[u + 1];
    const uint32_t c = uint32_t(c1 - c0);
    if (c == 0) {
      if (lane == 0) deg[u] = 0;
      for (uint32_t j = lane; j < M; j += 32) adj[size_t(u) * M + j] = kSentinel;
      continue;
    }
    double* bm = sm;
    uint32_t* bv = sv;
#ifdef RA_PRUNE_PROF
    long long t0 = clock64();
    uint64_t n_tests = 0, n_rounds = 0, n_cand = 0;
#endif
    const float* ku = keys + size_t(u) * d;
    auto score = [&](uint32_t i, uint32_t at) {  // candidate i's m_uv into slot `at`
      const uint32_t v = uint32_t(edges[c0 + i] & dst_mask);
      const double ip = dot_rows(ku, keys + size_t(v) * d, d);
      bm[at] = euclid ? norms[u] + norms[v] - 2.0 * ip : -ip;
      bv[at] = v;
    };
    auto sort_first = [&](uint32_t total) {  // ascending (m, v) over [0, total)
      uint32_t p2 = 1;
      while (p2 < total) p2 <<= 1;
      for (uint32_t i = total + lane; i < p2; i += 32) {
        bm[i] = DBL_MAX;
        bv[i] = kSentinel;
      }
      __syncwarp();
      warp_bitonic_asc(bm, bv, p2, lane);
    };
    if (global_mode) {
      bm = gm + size_t(wid) * g_stride;
      bv = gv + size_t(wid) * g_stride;
    } else if (c > PCAP) {
      if (2 * efc > PCAP) {  // (very large ef_construction: the HBM pass)
        if (lane == 0) big_nodes[atomicAdd(big_count, 1u)] = u;
        continue;
      }
      // hub node: only the best efc candidates are ever read (:179), so
      // stream the candidates through shared memory in chunks, keeping the
      // best efc so far sorted in front of each chunk
      const uint32_t chunk = PCAP - efc;
      uint32_t r = 0;
      for (uint32_t s0 = 0; s0 < c; s0 += chunk) {
        const uint32_t cn = min(chunk, c - s0);
        for (uint32_t i = lane; i < cn; i += 32) score(s0 + i, r + i);
        __syncwarp();
        sort_first(r + cn);
        r = min(r + cn, efc);
        __syncwarp();
      }
    }
    if (global_mode || c <= PCAP) {
      for (uint32_t i = lane; i < c; i += 32) score(i, i);
      sort_first(c);
    }
    const uint32_t no = c < efc ? c : efc;
    uint32_t kn = 0;
#ifdef RA_PRUNE_PROF
    long long t1 = clock64();
    PPROF(0, t1 - t0);
#endif
    for (uint32_t i = 0; i < no && kn < M; ++i) {
      const uint32_t v = bv[i];
      const double m_uv = bm[i];
      bool occl = false;
#ifdef RA_PRUNE_PROF
      ++n_cand;
      n_tests += kn;
      n_rounds += kn ? 1 : 0;
#endif
      for (uint32_t j0 = 0; j0 < kn; j0 += 32) {
        const uint32_t j = j0 + lane;
        bool o = false;
        if (j < kn) {
          // decided by the fp32 estimate when it is clear of m_uv by more than
          // its error bound; the exact in-order f64 test otherwise
          const uint32_t w = kept[j];
          const float* kv_ = keys + size_t(v) * d;
          const float* kw_ = keys + size_t(w) * d;
          const double nv = norms[v], nw = norms[w];
          const float ipf = dot_f32_est(kv_, kw_, d);
          bool decided = false;
          if (isfinite(ipf)) {
            const double ipa = ipf;
            const double eps = double(d + 16) * 0x1p-24 * sqrt(nv * nw);
            const double ma = euclid ? nv + nw - 2.0 * ipa : -ipa;
            const double em = (euclid ? 2.0 * eps : eps) +
                              0x1p-50 * (nv + nw + 2.0 * fabs(ipa) + fabs(m_uv));
            if (ma + em < m_uv) o = true, decided = true;
            else if (ma - em > m_uv) decided = true;
          }
          if (!decided) {
#ifdef RA_PRUNE_PROF
            atomicAdd(&g_prune_prof[8], 1ull);
#endif
            const double ip = dot_rows(kv_, kw_, d);
            const double m_vw = euclid ? nv + nw - 2.0 * ip : -ip;
            o = m_vw < m_uv;
          }
        }
        if (__ballot_sync(kFull, o)) {
          occl = true;
          break;
        }
      }
      if (!occl) {
        if (lane == 0) kept[kn] = v;
        ++kn;
        __syncwarp();
      }
    }
#ifdef RA_PRUNE_PROF
    long long t2 = clock64();
    PPROF(1, t2 - t1);
    PPROF(3, n_cand);
    PPROF(4, n_rounds);
    PPROF(5, n_tests);
    PPROF(6, kn == M ? 1 : 0);
    PPROF(7, kn);
#endif
    // fill from the ordered list (:196-201)
    for (uint32_t i = 0; i < no && kn < M; ++i) {
      const uint32_t v = bv[i];
      bool found = false;
      for (uint32_t j0 = 0; j0 < kn; j0 += 32) {
        const uint32_t j = j0 + lane;
        if (__ballot_sync(kFull, j < kn && kept[j] == v)) {
          found = true;
          break;
        }
      }
      if (!found) {
        if (lane == 0) kept[kn] = v;
        ++kn;
        __syncwarp();
      }
    }
    for (uint32_t j = lane; j < M; j += 32) adj[size_t(u) * M + j] = j < kn ? kept[j] : kSentinel;
    if (lane == 0) deg[u] = kn;
    __syncwarp();
#ifdef RA_PRUNE_PROF
    PPROF(2, clock64() - t2);
#endif
  }
}

// ---- K4 -------------------------------------------------------------------------
// column mean, in row order per dimension (Eigen colwise().mean() as shimmed)
// Block = 32 columns; its 8 warps stage 128-row chunks of those columns in
// shared memory (double-buffered) while warp 0 runs the sequential f64 adds,
// so the dependent add chain, not the load latency, sets the pace.
__global__ void __launch_bounds__(256) k_colmean(const float* __restrict__ keys, uint32_t n,
                                                 uint32_t d, double* mean) {
  constexpr uint32_t CH = 128;
  __shared__ float tile[2][CH][33];
  const uint32_t c0 = blockIdx.x * 32, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t col = c0 + lane;
  const uint32_t nch = (n + CH - 1) / CH;
  auto stage = [&](uint32_t ch, uint32_t buf) {
    for (uint32_t r = warp; r < CH; r += 8) {
      const uint64_t row = uint64_t(ch) * CH + r;
      tile[buf][r][lane] = (row < n && col < d) ? __ldg(keys + row * d + col) : 0.f;
    }
  };
  double acc = 0.0;
  if (nch) stage(0, 0);
  __syncthreads();
  for (uint32_t ch = 0; ch < nch; ++ch) {
    const uint32_t buf = ch & 1u;
    if (ch + 1 < nch && warp != 0) stage(ch + 1, buf ^ 1u);
    if (warp == 0) {
      const uint32_t rows = min(CH, n - ch * CH);
      if (rows == CH) {
#pragma unroll 32
        for (uint32_t r = 0; r < CH; ++r) acc += (double)tile[buf][r][lane];
      } else {
        for (uint32_t r = 0; r < rows; ++r) acc += (double)tile[buf][r][lane];
      }
    }
    __syncthreads();
    if (ch + 1 < nch && warp == 0) {  // warp 0's share of the next chunk
      for (uint32_t r = 0; r < CH; r += 8) {
        const uint64_t row = uint64_t(ch + 1) * CH + r;
        tile[buf ^ 1u][r][lane] = (row < n && col < d) ? __ldg(keys + row * d + col) : 0.f;
      }
    }
    __syncthreads();
  }
  if (warp == 0 && col < d) mean[col] = acc / (double)n;
}

// per-node key for the entry argmin: medoid distance (:222-230) or -norm (:218-220)
__global__ void k_entry_key(const float* __restrict__ keys, uint32_t n, uint32_t d,
                            const double* __restrict__ mean, const double* __restrict__ norms,
                            const uint32_t* __restrict__ deg, int any_covered, int maxnorm,
                            unsigned long long* best) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  double key = DBL_MAX;
  if (u < n && (!any_covered || deg[u] > 0)) {
    if (maxnorm) {
      key = -norms[u];
    } else {
      double acc = 0.0;
      const float* r = keys + size_t(u) * d;
      for (uint32_t j = 0; j < d; ++j) {
        const double t = (double)r[j] - mean[j];
        acc = fma(t, t, acc);
      }
      key = acc;
    }
  }
  // (key asc, u asc) argmin via an order-preserving 64-bit encoding per block,
  // then a global min over (encoded key, u) pairs
  __shared__ double bk[256];
  __shared__ uint32_t bu[256];
  bk[threadIdx.x] = key;
  bu[threadIdx.x] = u < n ? u : kSentinel;
  __syncthreads();
  for (uint32_t s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double k2 = bk[threadIdx.x + s];
      const uint32_t u2 = bu[threadIdx.x + s];
      if (k2 < bk[threadIdx.x] || (k2 == bk[threadIdx.x] && u2 < bu[threadIdx.x])) {
        bk[threadIdx.x] = k2;
        bu[threadIdx.x] = u2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    best[2 * blockIdx.x] = __double_as_longlong(bk[0]);
    best[2 * blockIdx.x + 1] = bu[0];
  }
}

__global__ void k_any_covered(const uint32_t* deg, uint32_t n, uint32_t* flag) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n && deg[u] > 0) *flag = 1;
}

// ---- K5 helper: nearest anchor per pending node (:287-316) ------------------------
// The reference's a_norm - 2 * U.A^T + argmin as a tiled FP64 CUDA-core
// GEMM: a block holds 64 pending rows and, chunk by chunk, 64 anchor rows
// in shared memory widened to f64 (exact); each thread keeps a 4 x 4 block
// of in-order dot chains (16 independent chains, operands reused 4x), then
// the running (distance, anchor index) minimum per pending row, lower index
// first on ties (the reference's strict < over ascending anchors).
constexpr uint32_t NA_T = 64;  // pending rows and anchors per tile

// wide rows (the tiles would not fit shared memory): one warp per pending
// node, lanes stride the anchors
__global__ void __launch_bounds__(256)
    k_nearest_anchor_warp(const float* __restrict__ keys, uint32_t d,
                          const double* __restrict__ norms, const uint32_t* __restrict__ pending,
                          uint32_t np, const uint32_t* __restrict__ anchors, uint32_t na,
                          uint32_t* __restrict__ nearest) {
  const uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= np) return;
  const float* ku = keys + size_t(pending[i]) * d;
  double best = DBL_MAX;
  uint32_t bj = kSentinel;
  for (uint32_t j = lane; j < na; j += 32) {
    const double dist = norms[anchors[j]] - 2.0 * dot_rows(ku, keys + size_t(anchors[j]) * d, d);
    if (dist < best) best = dist, bj = j;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double b2 = __shfl_xor_sync(kFull, best, o);
    const uint32_t j2 = __shfl_xor_sync(kFull, bj, o);
    if (b2 < best || (b2 == best && j2 < bj)) best = b2, bj = j2;
  }
  if (lane == 0) nearest[i] = anchors[bj];
}

__global__ void __launch_bounds__(256)
    k_nearest_anchor(const float* __restrict__ keys, uint32_t d, const double* __restrict__ norms,
                     const uint32_t* __restrict__ pending, uint32_t np,
                     const uint32_t* __restrict__ anchors, uint32_t na,
                     uint32_t* __restrict__ nearest) {
  extern __shared__ double nsm[];
  const uint32_t ld = d + 1;  // odd row stride: conflict-free column reads
  double* P = nsm;            // [NA_T][ld]
  double* A = nsm + size_t(NA_T) * ld;
  double* red = A + size_t(NA_T) * ld;  // [NA_T][16] best distances
  uint32_t* redj = reinterpret_cast<uint32_t*>(red + NA_T * 16);
  const uint32_t tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const uint32_t p0 = blockIdx.x * NA_T;
  for (uint32_t t = threadIdx.x; t < NA_T * d; t += blockDim.x) {
    const uint32_t r = t / d, c = t % d;
    P[r * ld + c] = p0 + r < np ? (double)keys[size_t(pending[p0 + r]) * d + c] : 0.0;
  }
  double best[4];
  uint32_t bj[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) best[i] = DBL_MAX, bj[i] = kSentinel;
  for (uint32_t a0 = 0; a0 < na; a0 += NA_T) {
    __syncthreads();  // (previous chunk consumed; P staged on the first pass)
    for (uint32_t t = threadIdx.x; t < NA_T * d; t += blockDim.x) {
      const uint32_t r = t / d, c = t % d;
      A[r * ld + c] = a0 + r < na ? (double)keys[size_t(anchors[a0 + r]) * d + c] : 0.0;
    }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (uint32_t c = 0; c < d; ++c) {  // k order (the reference's in-order dot)
      double pv[4], av[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pv[i] = P[(ty + 16 * i) * ld + c];
#pragma unroll
      for (int j = 0; j < 4; ++j) av[j] = A[(tx + 16 * j) * ld + c];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(pv[i], av[j], acc[i][j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // ascending anchor index within this thread
      const uint32_t aj = a0 + tx + 16 * j;
      if (aj >= na) continue;
      const double an = norms[anchors[aj]];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double dist = an - 2.0 * acc[i][j];
        if (dist < best[i]) best[i] = dist, bj[i] = aj;
      }
    }
  }
  // argmin over the 16 threads sharing each pending row
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    red[(ty + 16 * i) * 16 + tx] = best[i];
    redj[(ty + 16 * i) * 16 + tx] = bj[i];
  }
  __syncthreads();
  if (threadIdx.x < NA_T && p0 + threadIdx.x < np) {
    double b = DBL_MAX;
    uint32_t j = kSentinel;
    for (uint32_t k = 0; k < 16; ++k) {
      const double b2 = red[threadIdx.x * 16 + k];
      const uint32_t j2 = redj[threadIdx.x * 16 + k];
      if (b2 < b || (b2 == b && j2 < j)) b = b2, j = j2;
    }
    nearest[p0 + threadIdx.x] = anchors[j];
  }
}

// ---- K5: reachability (the reference's DFS sweep :240-253 and, for the
// no-anchor case, its BFS depths :263-279; only the reached SET and the BFS
// depth matter, so a level-synchronous parallel BFS gives both) ---------------
// depth[] = 0xFFFFFFFF (unreached) on entry; cnt[3] = 0. Cooperative launch.
__global__ void __launch_bounds__(512)
    k_bfs(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ deg, uint32_t M,
          uint32_t entry, uint32_t* depth, uint32_t* qa, uint32_t* qb, uint32_t* cnt) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const uint64_t tid = grid.thread_rank(), nt = grid.size();
  if (tid == 0) {
    depth[entry] = 0;
    qa[0] = entry;
    cnt[0] = 1;
  }
  grid.sync();
  uint32_t* cur = qa;
  uint32_t* nxt = qb;
  // cnt[L % 3] = size of level L; cnt[(L + 1) % 3] was zeroed during level
  // L - 1; cnt[(L + 2) % 3] (level L - 1's, read by everyone) is zeroed now
  for (uint32_t level = 0;; ++level) {
    const uint32_t ncur = *reinterpret_cast<volatile uint32_t*>(cnt + level % 3);
    if (ncur == 0) break;
    if (tid == 0) cnt[(level + 2) % 3] = 0;
    for (uint64_t i = tid; i < uint64_t(ncur) * M; i += nt) {
      const uint32_t u = cur[i / M], e = uint32_t(i % M);
      if (e < deg[u]) {
        const uint32_t v = adj[size_t(u) * M + e];
        if (atomicCAS(depth + v, 0xFFFFFFFFu, level + 1) == 0xFFFFFFFFu)
          nxt[atomicAdd(cnt + (level + 1) % 3, 1u)] = v;
      }
    }
    grid.sync();
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
  }
}

// reachability only (the reference's DFS sweep, :240-253): a work queue
// instead of BFS levels (attachment chains make the graph thousands of levels
// deep). Each thread claims the next queue slot, waits for it to be published
// (q[] pre-filled with kSentinel), pushes the unmarked neighbours, and counts
// the node as processed; a thread whose slot is never published leaves once
// every published node is processed (processed == tail, read around it).
// mark[entry] = 1, q[0] = entry, ctr = {tail 1, head 0, processed 0} on entry.
__global__ void __launch_bounds__(256)
    k_reach(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ deg, uint32_t M,
            uint32_t n, uint32_t* mark, uint32_t* q, uint32_t* ctr) {
  volatile uint32_t* vq = q;
  volatile uint32_t* vc = ctr;
  for (;;) {
    const uint32_t i = atomicAdd(ctr + 1, 1u);
    uint32_t u;
    for (;;) {
      u = i < n ? vq[i] : 0xFFFFFFFFu;  // (claims run past n once everything is queued)
      if (u != kSentinel) break;
      const uint32_t t1 = vc[0];
      if (i < t1) continue;  // claimed slot published, store not visible yet
      const uint32_t pr = vc[2];
      if (pr == t1 && vc[0] == t1) return;  // nothing in flight: all reached
      __nanosleep(64);
    }
    const uint32_t dg = deg[u];
    for (uint32_t e = 0; e < dg; ++e) {
      const uint32_t v = adj[size_t(u) * M + e];
      if (atomicExch(mark + v, 1u) == 0u) {
        const uint32_t slot = atomicAdd(ctr, 1u);
        vq[slot] = v;
      }
    }
    __threadfence();
    atomicAdd(ctr + 2, 1u);
  }
}

__global__ void k_reach_init(uint32_t* mark, uint32_t* q, uint32_t* ctr, uint32_t entry) {
  mark[entry] = 1;
  q[0] = entry;
  ctr[0] = 1, ctr[1] = 0, ctr[2] = 0;
}

// flags for the round's lists (:256-262): pending = unreached, anchors =
// reached with spare degree
__global__ void k_repair_flags(const uint32_t* __restrict__ mark, const uint32_t* __restrict__ deg,
                               uint32_t n, uint32_t M, uint8_t* pend, uint8_t* anch) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const bool r = mark[u] != 0;
  pend[u] = !r;
  anch[u] = r && deg[u] < M;
}

// no anchor (:263-282): the deepest reached node (depth desc, id asc) drops
// its last edge and becomes the only anchor. One block.
__global__ void k_deepest_drop(const uint32_t* __restrict__ depth, uint32_t n, uint32_t M,
                               uint32_t* adj, uint32_t* deg, uint32_t* anchors) {
  __shared__ unsigned long long red[32];
  unsigned long long best = 0;  // (depth + 1) << 32 | ~id: max = deepest, then lowest id
  for (uint32_t u = threadIdx.x; u < n; u += blockDim.x) {
    const uint32_t dp = depth[u];
    if (dp != 0xFFFFFFFFu) {
      const unsigned long long key = (uint64_t(dp) + 1) << 32 | uint32_t(~u);
      if (key > best) best = key;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(kFull, best, o);
    if (x > best) best = x;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < blockDim.x / 32; ++w)
      if (red[w] > best) best = red[w];
    const uint32_t u = ~uint32_t(best);
    const uint32_t dg = deg[u] - 1;  // adj[deepest].pop_back()
    adj[size_t(u) * M + dg] = kSentinel;
    deg[u] = dg;
    anchors[0] = u;
  }
}

__global__ void k_pair_keys(const uint32_t* __restrict__ nearest,
                            const uint32_t* __restrict__ pending, uint32_t np, uint64_t* keys) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < np) keys[i] = (uint64_t(nearest[i]) << 32) | pending[i];
}

// the chained attachments (:320-345), one block per anchor group of the
// sorted (anchor, node) pairs; groups touch disjoint rows (their anchor and
// their own pending nodes). The group's node ids and degrees are staged in
// shared memory, so the sequential chain (each step depends on where the
// previous node went) runs on-chip; groups beyond kAttachCap nodes walk the
// global arrays. `deferred` counts the nodes left for the next round.
constexpr uint32_t kAttachCap = 6144;

__global__ void __launch_bounds__(256)
    k_attach(const uint64_t* __restrict__ keys, uint32_t np, uint32_t M, uint32_t* adj,
             uint32_t* deg, uint32_t* deferred) {
  __shared__ uint32_t s_id[kAttachCap];
  __shared__ uint16_t s_dg[kAttachCap];
  __shared__ uint32_t s_end;
  const uint32_t g0 = blockIdx.x;
  const uint32_t a = uint32_t(keys[g0] >> 32);
  if (g0 > 0 && uint32_t(keys[g0 - 1] >> 32) == a) return;  // not a group start
  // group end: the first index whose anchor differs
  if (threadIdx.x == 0) s_end = np;
  __syncthreads();
  for (uint32_t c = g0; c < np; c += blockDim.x) {
    const uint32_t i = c + threadIdx.x;
    if (i < np && uint32_t(keys[i] >> 32) != a) atomicMin(&s_end, i);
    __syncthreads();
    if (s_end != np) break;
  }
  const uint32_t L = s_end - g0;
  if (L <= kAttachCap && M < 65536u) {
    for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) {
      const uint32_t u = uint32_t(keys[g0 + j]);
      s_id[j] = u;
      s_dg[j] = uint16_t(deg[u]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t dA = deg[a], tj = 0xFFFFFFFFu, next_t = 0, i = 0;  // tj = max: t is the anchor
      for (; i < L; ++i) {
        uint32_t dt = tj == 0xFFFFFFFFu ? dA : s_dg[tj];
        bool def = false;
        while (dt >= M) {
          if (next_t >= i) {
            def = true;
            break;
          }
          tj = next_t++;
          dt = s_dg[tj];
        }
        if (def) break;
        const uint32_t u = s_id[i];
        adj[size_t(tj == 0xFFFFFFFFu ? a : s_id[tj]) * M + dt] = u;
        if (tj == 0xFFFFFFFFu) ++dA;
        else s_dg[tj] = uint16_t(dt + 1);
        if (s_dg[i] < M) tj = i;
      }
      deg[a] = dA;
      if (i < L) atomicAdd(deferred, L - i);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) deg[s_id[j]] = s_dg[j];
    return;
  }
  if (threadIdx.x != 0) return;
  uint32_t t = a, next_t = 0, i = g0;
  for (; i < s_end; ++i) {
    const uint32_t u = uint32_t(keys[i]);
    bool def = false;
    while (deg[t] >= M) {
      if (next_t >= i - g0) {  // attached so far = the group's nodes before i
        def = true;
        break;
      }
      t = uint32_t(keys[g0 + next_t++]);
    }
    if (def) break;
    adj[size_t(t) * M + deg[t]++] = u;
    if (deg[u] < M) t = u;
  }
  if (i < s_end) atomicAdd(deferred, s_end - i);
}

struct Timer {
  cudaStream_t s;
  cudaEvent_t a, b;
  explicit Timer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double peek() {  // ms since the last lap, without resetting
    cudaEvent_t c;
    cudaEventCreate(&c);
    cudaEventRecord(c, s);
    cudaEventSynchronize(c);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, c);
    cudaEventDestroy(c);
    return ms;
  }
  double lap() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::swap(a, b);
    return ms;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// FlatIndex: drop masked ids from each exact top-(k + |mask|) row, keep k
__global__ void k_flat_pick(const uint32_t* __restrict__ ids, const double* __restrict__ sc,
                            uint32_t B, uint32_t kt, uint32_t k, const uint32_t* __restrict__ bits,
                            uint32_t* out_ids, float* out_sc, uint64_t* scanned, uint64_t nscan) {
  const uint32_t b = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (b >= B) return;
  uint32_t w = 0;
  for (uint32_t c0 = 0; c0 < kt && w < k; c0 += 32) {
    const uint32_t i = c0 + lane;
    const uint32_t v = i < kt ? ids[size_t(b) * kt + i] : kSentinel;
    const bool keep = v != kSentinel && !(bits && ((bits[v >> 5] >> (v & 31)) & 1u));
    const uint32_t m = __ballot_sync(kFull, keep);
    const uint32_t o = w + __popc(m & ((1u << lane) - 1u));
    if (keep && o < k) {
      out_ids[size_t(b) * k + o] = v;
      out_sc[size_t(b) * k + o] = float(sc[size_t(b) * kt + i]);
    }
    w += __popc(m);
  }
  if (lane == 0) scanned[b] = nscan;
}

}  // namespace

// phase 4 (:235-348) on the device rows (row u = adj[u*M .. u*M+deg[u]),
// kSentinel past it; appends stay within M by construction)
static void repair(ra_ctx* ctx, ra_kv* kv, const double* norms_dev, uint64_t entry,
                   uint32_t M, uint32_t* adj, uint32_t* deg, ra_build_stats* st) {
  const uint32_t n = uint32_t(kv->n), d = kv->d;
  cudaStream_t s = ctx->stream;
  static const bool trace = std::getenv("RA_REPAIR_TRACE") != nullptr;
  DevBuf<uint32_t> depth(n, s), qa(n, s), qb(n, s), cnt(3, s), lists(2 * size_t(n), s),
      counts(2, s), nearest(n, s);
  DevBuf<uint8_t> fl(2 * size_t(n), s);
  DevBuf<uint64_t> keys(n, s), keys2(n, s);
  int bps = 0;
  RA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_bfs, 512, 0));
  const uint32_t bfs_grid = uint32_t(std::max(1, bps) * ctx->num_sms);
  size_t tb_sel = 0, tb_sort = 0;
  cub::CountingInputIterator<uint32_t> ids(0);
  cub::DeviceSelect::Flagged(nullptr, tb_sel, ids, fl.p, lists.p, counts.p, n, s);
  cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, keys.p, keys2.p, int64_t(n), 0, 64, s);
  DevBuf<uint8_t> tmp(std::max(tb_sel, tb_sort), s);
  for (uint32_t round = 0;; ++round) {
    if (round > n) runtime("graph repair did not converge");
    const auto t0 = std::chrono::steady_clock::now();
    // the sweep: reached set (mark in depth[], q in qa[])
    RA_CUDA(cudaMemsetAsync(depth.p, 0, size_t(n) * 4, s));
    RA_CUDA(cudaMemsetAsync(qa.p, 0xFF, size_t(n) * 4, s));
    k_reach_init<<<1, 1, 0, s>>>(depth.p, qa.p, cnt.p, uint32_t(entry));
    k_reach<<<ctx->num_sms * 4, 256, 0, s>>>(adj, deg, M, n, depth.p, qa.p, cnt.p);
    k_repair_flags<<<(n + 255) / 256, 256, 0, s>>>(depth.p, deg, n, M, fl.p, fl.p + n);
    size_t tb = tmp.n;
    RA_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, ids, fl.p, lists.p, counts.p, n, s));
    tb = tmp.n;
    RA_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, ids, fl.p + n, lists.p + n, counts.p + 1, n, s));
    uint32_t h[2] = {0, 0};
    RA_CUDA(cudaMemcpyAsync(h, counts.p, 8, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    const uint32_t np = h[0];
    uint32_t na = h[1];
    if (trace)
      fprintf(stderr, "repair: round %u sweep+lists %.2f ms\n", round,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
    if (np == 0) break;
    st->repair_rounds++;
    st->repaired_nodes += np;
    uint32_t* pending = lists.p;
    uint32_t* anchors = lists.p + n;
    bool dropped = false;
    if (na == 0) {  // (rare) BFS depths for the deepest reached node
      dropped = true;
      RA_CUDA(cudaMemsetAsync(depth.p, 0xFF, size_t(n) * 4, s));
      RA_CUDA(cudaMemsetAsync(cnt.p, 0, 12, s));
      uint32_t e32 = uint32_t(entry);
      uint32_t* ap = adj;
      uint32_t* dp = deg;
      void* args[] = {&ap, &dp, &M, &e32, &depth.p, &qa.p, &qb.p, &cnt.p};
      RA_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_bfs), dim3(bfs_grid),
                                          dim3(512), args, 0, s));
      k_deepest_drop<<<1, 1024, 0, s>>>(depth.p, n, M, adj, deg, anchors);
      na = 1;
    }
    auto tlap = [&](const char* what) {
      if (!trace) return;
      RA_CUDA(cudaStreamSynchronize(s));
      fprintf(stderr, "repair:   %s at %.2f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
    };
    tlap("lists");
    {
      const size_t sm = (2 * size_t(NA_T) * (d + 1) + NA_T * 16) * 8 + NA_T * 16 * 4;
      const size_t budget = ctx->smem_optin ? ctx->smem_optin : 227 * 1024;
      if (sm <= budget) {
        RA_CUDA(cudaFuncSetAttribute(k_nearest_anchor,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k_nearest_anchor<<<(np + NA_T - 1) / NA_T, 256, sm, s>>>(kv->keys.p, d, norms_dev,
                                                                 pending, np, anchors, na,
                                                                 nearest.p);
      } else {
        k_nearest_anchor_warp<<<(np + 7) / 8, 256, 0, s>>>(kv->keys.p, d, norms_dev, pending, np,
                                                           anchors, na, nearest.p);
      }
      RA_LAUNCH_CHECK();
    }
    tlap("nearest");
    k_pair_keys<<<(np + 255) / 256, 256, 0, s>>>(nearest.p, pending, np, keys.p);
    tb = tmp.n;
    RA_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, keys2.p, int64_t(np), 0, 64, s));
    tlap("sort");
    RA_CUDA(cudaMemsetAsync(cnt.p, 0, 4, s));
    k_attach<<<np, 256, 0, s>>>(keys2.p, np, M, adj, deg, cnt.p);
    RA_LAUNCH_CHECK();
    // every pending node attached beneath a reached one (and no edge dropped):
    // all nodes are reached now, the reference's next sweep finds none pending
    uint32_t ndef = 0;
    RA_CUDA(cudaMemcpyAsync(&ndef, cnt.p, 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    if (trace) {
      RA_CUDA(cudaStreamSynchronize(s));
      fprintf(stderr, "repair: round %u pending %u anchors %u deferred %u  %.2f ms\n", round, np,
              na, ndef,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
    }
    if (ndef == 0 && !dropped) break;
  }
}

}  // namespace ra

using namespace ra;

extern "C" ra_status ra_graph_build(ra_ctx* ctx, ra_kv* kv, const float* train_q, uint64_t nq,
                                    uint32_t q_dim, int on_device, const ra_build_params* p,
                                    ra_build_stats* stats, ra_graph** out) {
  return guard([&] {
    if (!ctx) invalid("null context");
    // ctor validation, same order and texts (index_oodgraph.cpp:71-79)
    if (!kv || kv->n == 0) invalid("empty keys");
    if (kv->n > 0xFFFFFFFFull) invalid("too many keys");
    if (p->k_train < 1) invalid("k_train must be >= 1");
    if (p->max_degree < 1) invalid("max_degree must be >= 1");
    if (p->ef_construction < 1) invalid("ef_construction must be >= 1");
    if (nq > 0 && q_dim != kv->d) invalid("query dimension mismatch");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->stream;
    ra_build_stats st{};
    const uint32_t n = uint32_t(kv->n), d = kv->d, M = p->max_degree;
    const float* K = kv->keys.p;
    Timer tm(s);

    DevBuf<double> norms(n, s);
    k_norms<<<(n + 255) / 256, 256, 0, s>>>(K, n, d, norms.p);
    RA_LAUNCH_CHECK();
    // the medoid's column mean (a long dependent add chain per column, on 4
    // SMs) runs on the side stream beside phases 1-3; joined at the entry
    DevBuf<double> mean(d, s);
    if (!p->entry_maxnorm) {
      if (!ctx->side) {
        RA_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        RA_CUDA(cudaEventCreateWithFlags(&ctx->side_fork, cudaEventDisableTiming));
        RA_CUDA(cudaEventCreateWithFlags(&ctx->side_join, cudaEventDisableTiming));
      }
      RA_CUDA(cudaEventRecord(ctx->side_fork, s));
      RA_CUDA(cudaStreamWaitEvent(ctx->side, ctx->side_fork, 0));
      k_colmean<<<(d + 31) / 32, 256, 0, ctx->side>>>(K, n, d, mean.p);
      RA_LAUNCH_CHECK();
      RA_CUDA(cudaEventRecord(ctx->side_join, ctx->side));
    }

    // ---- phase 1 ----
    const uint32_t kt = std::min<uint64_t>(p->k_train, n);
    DevBuf<float> tq_own;
    const float* TQ = train_q;
    if (nq && !on_device) {
      tq_own.alloc(size_t(nq) * d, s);
      RA_CUDA(cudaMemcpyAsync(tq_own.p, train_q, size_t(nq) * d * 4, cudaMemcpyHostToDevice, s));
      TQ = tq_own.p;
    }
    DevBuf<uint32_t> knn(std::max<size_t>(size_t(nq) * kt, 1), s);
    const char* force_exact = std::getenv("RA_KNN_EXACT");
    const bool use_tc = nq && !(force_exact && force_exact[0] == '1') &&
                        knn_tc_supported(d, nq, n, kt);
    if (use_tc) {
      // tensor-core filter + exact rescoring; certificate failures -> exact path
      DevBuf<uint32_t> fail;
      double ms_gemm = 0;
      const uint32_t nf = knn_tc(ctx, TQ, nq, K, n, d, kt, knn.p, fail, &ms_gemm);
      st.ms_knn_tensor = ms_gemm;
      st.knn_rows = nq;
      st.knn_rows_widened = nf;
      if (nf) {
        // rows the certificate could not vouch for: exact in-order scores of
        // every key, then the row's top kt by a block radix select +
        // shared-memory sort (k_exact_topk); rows with mass ties past its
        // capacity take a stable segmented sort (score desc, id asc). Batched
        // so the score buffers stay bounded.
        const uint32_t per = std::max<uint32_t>(1, uint32_t((256ull << 20) / (24ull * n)));
        auto segmented = [&](const uint32_t* ids, uint32_t cnt_rows) {
          for (uint32_t r0 = 0; r0 < cnt_rows; r0 += per) {
            const uint32_t nr = std::min(per, cnt_rows - r0);
            const uint64_t tot = uint64_t(nr) * n;
            DevBuf<uint64_t> k1(tot, s), k2(tot, s);
            DevBuf<uint32_t> v1(tot, s), v2(tot, s);
            DevBuf<int> off(nr + 1, s);
            k_exact_scores<<<uint32_t((tot + 255) / 256), 256, 0, s>>>(TQ, ids + r0, nr, K, n, d,
                                                                       k1.p, v1.p);
            k_seg_offsets<<<(nr + 1 + 255) / 256, 256, 0, s>>>(nr, n, off.p);
            size_t tb = 0;
            cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, tb, k1.p, k2.p, v1.p, v2.p,
                                                               int64_t(tot), int64_t(nr), off.p,
                                                               off.p + 1, 0, 64, s);
            DevBuf<uint8_t> tmp(tb, s);
            RA_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(
                tmp.p, tb, k1.p, k2.p, v1.p, v2.p, int64_t(tot), int64_t(nr), off.p, off.p + 1, 0,
                64, s));
            k_take_top<<<uint32_t((uint64_t(nr) * kt + 255) / 256), 256, 0, s>>>(v2.p, nr, n, kt,
                                                                                 ids + r0, knn.p);
            RA_LAUNCH_CHECK();
          }
        };
        if (std::getenv("RA_KNN_SEGSORT")) {
          segmented(fail.p, nf);
        } else {
          DevBuf<uint32_t> ovf(nf, s), novf(1, s);
          RA_CUDA(cudaMemsetAsync(novf.p, 0, 4, s));
          const uint32_t per_x = std::max<uint32_t>(1, uint32_t((512ull << 20) / (8ull * n)));
          uint32_t xcap = XCAP;
          if (const char* e = std::getenv("RA_KNN_TOPK_CAP"))  // (tests: force the sort path)
            xcap = std::min<uint32_t>(XCAP, uint32_t(std::atoi(e)));
          for (uint32_t r0 = 0; r0 < nf; r0 += per_x) {
            const uint32_t nr = std::min(per_x, nf - r0);
            const uint64_t tot = uint64_t(nr) * n;
            DevBuf<uint64_t> k1(tot, s);
            k_exact_scores<<<uint32_t((tot + 255) / 256), 256, 0, s>>>(TQ, fail.p + r0, nr, K, n, d,
                                                                       k1.p, nullptr);
            k_exact_topk<<<nr, XT, 0, s>>>(k1.p, n, kt, fail.p + r0, knn.p, ovf.p, novf.p, xcap);
            RA_LAUNCH_CHECK();
          }
          uint32_t h_novf = 0;
          RA_CUDA(cudaMemcpyAsync(&h_novf, novf.p, 4, cudaMemcpyDeviceToHost, s));
          RA_CUDA(cudaStreamSynchronize(s));
          if (h_novf) segmented(ovf.p, h_novf);
        }
        if (std::getenv("RA_KNN_TRACE")) {
          RA_CUDA(cudaStreamSynchronize(s));
          fprintf(stderr, "knn: exact fallback for %u rows done at %.2f ms\n", nf, tm.peek());
        }
      }
    } else if (nq) {
      uint32_t cb = 1;
      while (cb < 2 * kt + KK) cb <<= 1;
      const uint64_t chunk = std::min<uint64_t>(nq, std::max<uint64_t>(KQ, (1ull << 30) / (cb * 12ull)) / KQ * KQ);
      DevBuf<double> bs(size_t(chunk) * cb, s);
      DevBuf<uint32_t> bi(size_t(chunk) * cb, s);
      DevBuf<unsigned long long> ctr(1, s);
      RA_CUDA(cudaMemsetAsync(ctr.p, 0, 8, s));
      for (uint64_t c0 = 0; c0 < nq; c0 += chunk) {
        const uint64_t cn = std::min<uint64_t>(chunk, nq - c0);
        k_knn<<<uint32_t((cn + KQ - 1) / KQ), KTHREADS, 0, s>>>(
            TQ + c0 * d, cn, K, n, d, kt, cb, bs.p, bi.p, knn.p + c0 * kt, ctr.p);
        RA_LAUNCH_CHECK();
      }
      unsigned long long w = 0;
      RA_CUDA(cudaMemcpyAsync(&w, ctr.p, 8, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaStreamSynchronize(s));
      st.knn_rows = nq;
      st.knn_rows_widened = w;  // compaction passes (diagnostic)
    }
    st.ms_knn = tm.lap();

    // ---- phase 2 ----
    std::vector<uint32_t> b_off(std::max<uint32_t>(kt, 1) + 1, 0);
    for (uint32_t b = 1; b < kt; ++b) b_off[b + 1] = b_off[b] + prop_count(b, p->edge_window);
    const uint32_t per_row = kt > 1 ? b_off[kt] : 0;
    const uint64_t total = uint64_t(nq) * per_row;
    DevBuf<uint64_t> edges, edges2;
    uint64_t ne = 0;
    const int end_bit = int(2 * edge_bits(n));
    bool hashed = false;
    if (total && !std::getenv("RA_EDGES_SORT")) {
      // dedup set sized for ~128 distinct proposals per key (the bench
      // shape's heads have 2-7M distinct pairs at 128K: load <= ~0.4), capped
      // by the proposal count; on overflow it is rebuilt 4x larger once
      uint32_t lg = 10;
      while (lg < 40 && (1ull << lg) < std::min<uint64_t>(2 * total, uint64_t(n) * 128)) ++lg;
      if (const char* e = std::getenv("RA_EDGES_HASH_LG"))  // (tests: force the overflow path)
        lg = std::max(4, std::min(40, std::atoi(e)));
      for (int attempt = 0; !hashed; ++attempt) {
        DevBuf<unsigned long long> tab(1ull << lg, s);
        DevBuf<uint32_t> ovf(1, s);
        RA_CUDA(cudaMemsetAsync(tab.p, 0xFF, (1ull << lg) * 8, s));
        RA_CUDA(cudaMemsetAsync(ovf.p, 0, 4, s));
        const uint64_t threads = uint64_t(nq) * (kt - 1);
        k_proposals_hash<<<uint32_t((threads + 255) / 256), 256, 0, s>>>(
            knn.p, nq, kt, p->edge_window, edge_bits(n), tab.p, lg, ovf.p);
        RA_LAUNCH_CHECK();
        edges2.alloc(1ull << lg, s);
        DevBuf<uint64_t> nsel(1, s);
        size_t tb = 0;
        cub::DeviceSelect::If(nullptr, tb, reinterpret_cast<uint64_t*>(tab.p), edges2.p, nsel.p,
                              int64_t(1ull << lg), HNotEmpty(), s);
        DevBuf<uint8_t> tmp(tb, s);
        RA_CUDA(cub::DeviceSelect::If(tmp.p, tb, reinterpret_cast<uint64_t*>(tab.p), edges2.p,
                                      nsel.p, int64_t(1ull << lg), HNotEmpty(), s));
        uint32_t h_ovf = 0;
        RA_CUDA(cudaMemcpyAsync(&ne, nsel.p, 8, cudaMemcpyDeviceToHost, s));
        RA_CUDA(cudaMemcpyAsync(&h_ovf, ovf.p, 4, cudaMemcpyDeviceToHost, s));
        RA_CUDA(cudaStreamSynchronize(s));
        if (std::getenv("RA_PRUNE_TRACE"))
          fprintf(stderr, "edges: %llu proposals, set 2^%u slots, %llu distinct%s\n",
                  (unsigned long long)total, lg, (unsigned long long)ne, h_ovf ? " (overflow)" : "");
        if (!h_ovf) {
          hashed = true;
          tab.reset();
          edges.alloc(std::max<uint64_t>(ne, 1), s);
          if (ne) {
            size_t tb2 = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tb2, edges2.p, edges.p, (int64_t)ne, 0, end_bit,
                                           s);
            DevBuf<uint8_t> tmp2(tb2, s);
            RA_CUDA(cub::DeviceRadixSort::SortKeys(tmp2.p, tb2, edges2.p, edges.p, (int64_t)ne, 0,
                                                   end_bit, s));
          }
        } else {
          ne = 0;
          edges2.reset();
          if (attempt >= 1 || (1ull << (lg + 2)) > 2 * total || lg + 2 > 36) break;
          lg += 2;
        }
      }
    }
    if (total && !hashed) {
      edges.alloc(std::max<uint64_t>(total, 1), s);
      edges2.alloc(std::max<uint64_t>(total, 1), s);
      DevBuf<uint32_t> d_boff(b_off.size(), s);
      RA_CUDA(cudaMemcpyAsync(d_boff.p, b_off.data(), b_off.size() * 4, cudaMemcpyHostToDevice, s));
      const uint64_t threads = uint64_t(nq) * (kt - 1);
      k_proposals<<<uint32_t((threads + 255) / 256), 256, 0, s>>>(
          knn.p, nq, kt, p->edge_window, d_boff.p, per_row, edge_bits(n), edges.p);
      RA_LAUNCH_CHECK();
      size_t tb = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, tb, edges.p, edges2.p, (int64_t)total, 0, end_bit, s);
      DevBuf<uint8_t> tmp(tb, s);
      RA_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, edges.p, edges2.p, (int64_t)total, 0,
                                             end_bit, s));
      DevBuf<uint64_t> nsel(1, s);
      size_t tb2 = 0;
      cub::DeviceSelect::Unique(nullptr, tb2, edges2.p, edges.p, nsel.p, (int64_t)total, s);
      DevBuf<uint8_t> tmp2(tb2, s);
      RA_CUDA(cub::DeviceSelect::Unique(tmp2.p, tb2, edges2.p, edges.p, nsel.p, (int64_t)total, s));
      RA_CUDA(cudaMemcpyAsync(&ne, nsel.p, 8, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaStreamSynchronize(s));
    }
    if (!total) edges.alloc(1, s);
    edges2.reset();
    st.candidate_edges = ne;
    DevBuf<uint64_t> off(size_t(n) + 1, s);
    k_src_offsets<<<(n + 1 + 255) / 256, 256, 0, s>>>(edges.p, ne, n, edge_bits(n), off.p);
    RA_LAUNCH_CHECK();
    st.ms_edges = tm.lap();

    // ---- phase 3 ----
    auto g = std::make_unique<ra_graph>();
    g->n = n;
    g->max_degree = M;
    g->default_ef = p->default_ef;
    const auto ta0 = std::chrono::steady_clock::now();
    g->adj.alloc_lived(size_t(n) * M, s);
    DevBuf<uint32_t> deg(n, s), big(n, s), big_cnt(1, s);
    const double alloc_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta0).count();
    RA_CUDA(cudaMemsetAsync(big_cnt.p, 0, 4, s));
    const size_t psmem = PWARPS * (PCAP * 12 + size_t(M) * 4);
    RA_CUDA(cudaFuncSetAttribute(k_prune, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
    const uint32_t pgrid = std::min<uint32_t>((n + PWARPS - 1) / PWARPS, ctx->num_sms * 8);
    static const bool ptrace = std::getenv("RA_PRUNE_TRACE") != nullptr;
    if (ptrace) {  // candidate-count profile (profiling aid)
      std::vector<uint64_t> h(size_t(n) + 1);
      RA_CUDA(cudaMemcpyAsync(h.data(), off.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaStreamSynchronize(s));
      uint64_t mx = 0, big = 0, sum_big = 0;
      for (uint32_t u = 0; u < n; ++u) {
        const uint64_t c = h[u + 1] - h[u];
        mx = std::max(mx, c);
        if (c > PCAP) ++big, sum_big += c;
      }
      fprintf(stderr, "prune: candidates %llu, max per node %llu, nodes > %u: %llu (%llu candidates)\n",
              (unsigned long long)h[n], (unsigned long long)mx, PCAP, (unsigned long long)big,
              (unsigned long long)sum_big);
    }
    Timer ptm(s);
    {
      // largest-first dynamic schedule: nodes sorted by candidate count
      // (descending), one resident wave of warps pulling from a counter
      DevBuf<uint32_t> k1(n, s), k2(n, s), v1(n, s), order(n, s), queue(2, s);
      RA_CUDA(cudaMemsetAsync(queue.p, 0, 8, s));
      k_prune_order<<<(n + 255) / 256, 256, 0, s>>>(off.p, n, M, k1.p, v1.p, g->adj.p, deg.p,
                                                    queue.p + 1);
      RA_LAUNCH_CHECK();
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, k1.p, k2.p, v1.p, order.p, int64_t(n), 0,
                                                32, s);
      DevBuf<uint8_t> tmp(tb, s);
      RA_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, k1.p, k2.p, v1.p, order.p,
                                                        int64_t(n), 0, 32, s));
      int per_sm = 0;
      RA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_prune, PWARPS * 32, psmem));
      const uint32_t qgrid = std::max<uint32_t>(1, std::min<uint32_t>(
                                                       pgrid, uint32_t(std::max(per_sm, 1)) * ctx->num_sms));
      k_prune<<<qgrid, PWARPS * 32, psmem, s>>>(K, n, d, norms.p, edges.p, off.p, order.p, n, M,
                                               p->ef_construction, !p->prune_inner_product, nullptr,
                                               nullptr, 0, g->adj.p, deg.p, big.p, big_cnt.p,
                                               queue.p);
      RA_LAUNCH_CHECK();
    }
    uint32_t nbig = 0;
    RA_CUDA(cudaMemcpyAsync(&nbig, big_cnt.p, 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    if (nbig) {
      // hub nodes with more candidates than shared memory holds: HBM buffers
      std::vector<uint64_t> h_off(size_t(n) + 1);
      RA_CUDA(cudaMemcpyAsync(h_off.data(), off.p, h_off.size() * 8, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaStreamSynchronize(s));
      uint64_t maxc = 0;
      for (uint32_t u = 0; u < n; ++u) maxc = std::max(maxc, h_off[u + 1] - h_off[u]);
      uint64_t p2 = 1;
      while (p2 < maxc) p2 <<= 1;
      const uint32_t gwarps = std::min<uint32_t>(nbig, 1024);
      const uint32_t ggrid = (gwarps + PWARPS - 1) / PWARPS;
      DevBuf<double> gm(size_t(ggrid) * PWARPS * p2, s);
      DevBuf<uint32_t> gv(size_t(ggrid) * PWARPS * p2, s);
      k_prune<<<ggrid, PWARPS * 32, psmem, s>>>(K, n, d, norms.p, edges.p, off.p, big.p, nbig, M,
                                               p->ef_construction, !p->prune_inner_product, gm.p,
                                               gv.p, p2, g->adj.p, deg.p, nullptr, nullptr, nullptr);
      RA_LAUNCH_CHECK();
    }
    edges.reset();
    if (ptrace)
      fprintf(stderr, "prune: %.2f ms (second pass nodes %u), allocations %.2f ms\n", ptm.lap(), nbig,
              alloc_ms);
#ifdef RA_PRUNE_PROF
    {
      unsigned long long pp[9];
      RA_CUDA(cudaMemcpyFromSymbol(pp, g_prune_prof, sizeof(pp)));
      fprintf(stderr,
              "prune prof (per node): score+sort %.0f occl %.0f fill %.0f cycles; tested %.1f rounds "
              "%.1f pairs %.1f; filled M %.3f kept %.1f exact %.2f\n",
              pp[0] / double(n), pp[1] / double(n), pp[2] / double(n), pp[3] / double(n),
              pp[4] / double(n), pp[5] / double(n), pp[6] / double(n), pp[7] / double(n),
              pp[8] / double(n));
      const unsigned long long z[9] = {};
      RA_CUDA(cudaMemcpyToSymbol(g_prune_prof, z, sizeof(z)));
    }
#endif
    st.ms_prune = tm.lap();

    // ---- entry point ----
    DevBuf<uint32_t> covered(1, s);
    RA_CUDA(cudaMemsetAsync(covered.p, 0, 4, s));
    k_any_covered<<<(n + 255) / 256, 256, 0, s>>>(deg.p, n, covered.p);
    if (!p->entry_maxnorm) RA_CUDA(cudaStreamWaitEvent(s, ctx->side_join, 0));
    uint32_t any = 0;
    RA_CUDA(cudaMemcpyAsync(&any, covered.p, 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    const uint32_t eblocks = (n + 255) / 256;
    DevBuf<unsigned long long> best(2 * eblocks, s);
    k_entry_key<<<eblocks, 256, 0, s>>>(K, n, d, mean.p, norms.p, deg.p, any, p->entry_maxnorm,
                                        best.p);
    RA_LAUNCH_CHECK();
    std::vector<unsigned long long> hb(2 * eblocks);
    RA_CUDA(cudaMemcpyAsync(hb.data(), best.p, hb.size() * 8, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    double bk = DBL_MAX;
    uint32_t bu = kSentinel;
    for (uint32_t b = 0; b < eblocks; ++b) {
      double k2;
      std::memcpy(&k2, &hb[2 * b], 8);
      const uint32_t u2 = uint32_t(hb[2 * b + 1]);
      if (k2 < bk || (k2 == bk && u2 < bu)) bk = k2, bu = u2;
    }
    g->entry = bu;
    st.ms_entry = tm.lap();

    // ---- phase 4 on the device; the host CSR mirror is built on first use ----
    repair(ctx, kv, norms.p, g->entry, M, g->adj.p, deg.p, &st);
    {
      DevBuf<unsigned long long> esum(1, s);
      size_t tb = 0;
      cub::DeviceReduce::Sum(nullptr, tb, deg.p, esum.p, n, s);
      DevBuf<uint8_t> tmp(tb, s);
      RA_CUDA(cub::DeviceReduce::Sum(tmp.p, tb, deg.p, esum.p, n, s));
      unsigned long long e = 0;
      RA_CUDA(cudaMemcpyAsync(&e, esum.p, 8, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaStreamSynchronize(s));
      g->n_edges = e;
    }
    st.ms_repair = tm.lap();

    ra_kv_retain(kv);
    g->kv = kv;
    if (stats) *stats = st;
    *out = g.release();
  });
}

// FlatIndex::search (index_flat.cpp:22-43) for B queries on the device:
// exact in-order f64 scores of every key and the (score desc, id asc) top
// k + |mask| by the K1 exact kernel, then masked ids are dropped. Mask ids
// must be sorted and unique (the reference's Mask contract, index.hpp:16-26).
extern "C" ra_status ra_flat_search_batch(ra_ctx* ctx, ra_kv* kv, uint32_t B, const float* q,
                                          uint32_t k, const uint32_t* mask, uint64_t mask_n,
                                          uint32_t* ids, float* scores, uint64_t* scanned) {
  using namespace ra;
  return guard([&] {
    if (!ctx) invalid("null context");
    if (!kv || kv->n == 0) invalid("empty keys");
    const uint64_t n = kv->n;
    if (n < mask_n || k < 1 || k > n - mask_n) invalid("k out of range after masking");
    if (B == 0) return;
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->stream;
    const uint32_t d = kv->d;
    const uint32_t kt = uint32_t(std::min<uint64_t>(n, uint64_t(k) + mask_n));
    DevBuf<uint32_t> bits;
    if (mask_n) {
      const uint64_t words = (n + 31) / 32;
      bits.alloc(words, s);
      launch_mask_bitset(s, mask, mask_n, bits.p, words);
    }
    uint32_t cb = 1;
    while (cb < 2 * kt + KK) cb <<= 1;
    const uint64_t chunk = std::min<uint64_t>(
        B, std::max<uint64_t>(KQ, (1ull << 30) / (uint64_t(cb) * 12ull)) / KQ * KQ);
    DevBuf<double> bs(size_t((chunk + KQ - 1) / KQ * KQ) * cb, s);
    DevBuf<uint32_t> bi(size_t((chunk + KQ - 1) / KQ * KQ) * cb, s);
    DevBuf<uint32_t> tk(size_t(chunk) * kt, s);
    DevBuf<double> ts(size_t(chunk) * kt, s);
    for (uint64_t c0 = 0; c0 < B; c0 += chunk) {
      const uint32_t cn = uint32_t(std::min<uint64_t>(chunk, B - c0));
      k_knn<<<(cn + KQ - 1) / KQ, KTHREADS, 0, s>>>(q + c0 * d, cn, kv->keys.p, uint32_t(n), d, kt,
                                                    cb, bs.p, bi.p, tk.p, nullptr, ts.p);
      k_flat_pick<<<(cn + 7) / 8, 256, 0, s>>>(tk.p, ts.p, cn, kt, k, mask_n ? bits.p : nullptr,
                                              ids + c0 * k, scores + c0 * k, scanned + c0,
                                              n - mask_n);
      RA_LAUNCH_CHECK();
    }
    RA_CUDA(cudaStreamSynchronize(s));
  });
}
