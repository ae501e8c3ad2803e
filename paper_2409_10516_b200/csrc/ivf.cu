// IVF index on the GPU (/root/reference/proj/src/index_ivf.cpp): k-means++
// seeding + Lloyd iterations over the keys, inner-product centroid ranking
// and exact scans of the nprobe nearest lists. A contrast baseline (§8 f3),
// not on the decode path.
//
// Arithmetic follows the reference's Eigen expressions as evaluated in
// index order with fused multiply-adds (the oracle's Eigen restatement,
// oracle/shim/Eigen/Dense): squared norms and the point x centroid product
// are fma chains over dimensions from 0.0, cluster sums add members in
// increasing id order, means divide elementwise. The sequential, RNG-driven
// parts of k-means++ (the cumulative-weight pick) and the rare empty-cluster
// reseed run on the host over device-computed vectors.
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"

struct ra_ivf {
  ra_kv* kv = nullptr;  // retained
  uint32_t nlist = 0, default_nprobe = 1, d = 0;
  uint64_t n = 0;
  ra::DevBuf<float> cent;       // nlist x d (f32, as the reference stores them)
  ra::DevBuf<uint32_t> offsets; // nlist + 1
  ra::DevBuf<uint32_t> ids;     // n, ascending within each list
  std::vector<uint32_t> h_offsets, h_ids;
  std::vector<float> h_cent;
};

namespace ra {
namespace {

// splitmix64 / Rng (util.hpp:13-45)
struct Rng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return double(next() >> 11) * 0x1.0p-53; }
  uint64_t uniform_index(uint64_t n) { return uint64_t(uniform() * double(n)) % n; }
};

// d2[i] = ||x_i - c||^2 (fma chain over dims), or min(d2[i], that)
__global__ void k_d2(const float* __restrict__ K, uint64_t n, uint32_t d,
                     const double* __restrict__ c, double* __restrict__ d2, int first) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const float* x = K + i * d;
  double acc = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    const double v = (double)x[j] - c[j];
    acc = fma(v, v, acc);
  }
  d2[i] = first ? acc : (acc < d2[i] ? acc : d2[i]);  // cwiseMin
}

// csq[c] = ||cent_c||^2
__global__ void k_csq(const double* __restrict__ cent, uint32_t nlist, uint32_t d, double* csq) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nlist) return;
  double acc = 0.0;
  for (uint32_t j = 0; j < d; ++j) acc = fma(cent[size_t(c) * d + j], cent[size_t(c) * d + j], acc);
  csq[c] = acc;
}

// assignment: argmin_c csq[c] - 2 sim(i, c), sim an fma chain over dims
// (x * cent^T), strict < (ties to the lower centroid). CTA = 128 points,
// rows staged in shared memory, centroids broadcast from L1.
constexpr uint32_t kAP = 128;
__global__ void __launch_bounds__(kAP) k_assign(const float* __restrict__ K, uint64_t n,
                                                uint32_t d, const double* __restrict__ cent,
                                                const double* __restrict__ csq, uint32_t nlist,
                                                uint32_t* __restrict__ assign) {
  extern __shared__ float xs[];  // [kAP][d + 1]
  const uint64_t i0 = uint64_t(blockIdx.x) * kAP;
  for (uint32_t e = threadIdx.x; e < kAP * d; e += kAP) {
    const uint32_t r = e / d, j = e % d;
    xs[r * (d + 1) + j] = i0 + r < n ? K[(i0 + r) * d + j] : 0.f;
  }
  __syncthreads();
  const uint64_t i = i0 + threadIdx.x;
  if (i >= n) return;
  const float* x = xs + threadIdx.x * (d + 1);
  double best = INFINITY;
  uint32_t best_c = 0;
  uint32_t c = 0;
  for (; c + 4 <= nlist; c += 4) {  // four independent chains
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double* c0 = cent + size_t(c) * d;
    for (uint32_t j = 0; j < d; ++j) {
      const double xj = (double)x[j];
      a0 = fma(xj, __ldg(c0 + j), a0);
      a1 = fma(xj, __ldg(c0 + d + j), a1);
      a2 = fma(xj, __ldg(c0 + 2 * d + j), a2);
      a3 = fma(xj, __ldg(c0 + 3 * d + j), a3);
    }
    const double dist[4] = {csq[c] - 2.0 * a0, csq[c + 1] - 2.0 * a1, csq[c + 2] - 2.0 * a2,
                            csq[c + 3] - 2.0 * a3};
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (dist[t] < best) best = dist[t], best_c = c + t;
  }
  for (; c < nlist; ++c) {
    double a = 0.0;
    for (uint32_t j = 0; j < d; ++j) a = fma((double)x[j], __ldg(cent + size_t(c) * d + j), a);
    const double dist = csq[c] - 2.0 * a;
    if (dist < best) best = dist, best_c = c;
  }
  assign[i] = best_c;
}

__global__ void k_iota(uint32_t* v, uint64_t n) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = uint32_t(i);
}

// list offsets from the (stably) sorted assignment keys
__global__ void k_offsets(const uint32_t* __restrict__ skey, uint64_t n, uint32_t nlist,
                          uint32_t* __restrict__ off) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nlist) return;
  uint64_t lo = 0, hi = n;  // first position with key >= c
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (skey[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  off[c] = uint32_t(lo);
}

// sums of each cluster in increasing id order (sums.row(assign[i]) += x.row(i))
__global__ void k_sums(const float* __restrict__ K, uint32_t d, const uint32_t* __restrict__ off,
                       const uint32_t* __restrict__ ids, uint32_t nlist,
                       double* __restrict__ sums) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= uint64_t(nlist) * d) return;
  const uint32_t c = uint32_t(t / d), j = uint32_t(t % d);
  double acc = 0.0;
  for (uint32_t p = off[c]; p < off[c + 1]; ++p) acc += (double)K[size_t(ids[p]) * d + j];
  sums[t] = acc;
}

// ---- search: CTA per query ----------------------------------------------------
__device__ __forceinline__ bool better_sid(double sa, uint32_t ia, double sb, uint32_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

struct IvfSearchArgs {
  const float* keys;
  const float* cent;
  const uint32_t* off;
  const uint32_t* ids;
  const float* q;
  const uint32_t* mask_bits;
  uint32_t d, nlist, nprobe, k, B;
  uint32_t cap;        // candidate capacity per query (pow2)
  double* sc_s;        // [B][cap] scratch scores
  uint32_t* sc_i;      // [B][cap] scratch ids
  double* rk_s;        // [B][nlist_p2] centroid ranking scratch
  uint32_t* rk_i;
  uint32_t nlist_p2;
  uint32_t* out_ids;
  float* out_sc;
  uint32_t* n_out;
  uint64_t* scanned;
  uint8_t* truncated;
};

template <typename KeyF>
__device__ void cta_bitonic(double* s, uint32_t* id, uint32_t n_pow2, KeyF better) {
  for (uint32_t kk = 2; kk <= n_pow2; kk <<= 1)
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n_pow2; i += blockDim.x) {
        const uint32_t p = i ^ j;
        if (p > i) {
          const bool desc = (i & kk) == 0;
          const double a = s[i], c = s[p];
          const uint32_t ia = id[i], ic = id[p];
          if (desc ? better(c, ic, a, ia) : better(a, ia, c, ic)) {
            s[i] = c, s[p] = a;
            id[i] = ic, id[p] = ia;
          }
        }
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_ivf_search(IvfSearchArgs a) {
  const uint32_t b = blockIdx.x, d = a.d;
  __shared__ uint32_t sh_cnt;
  const float* q = a.q + size_t(b) * d;
  double* rs = a.rk_s + size_t(b) * a.nlist_p2;
  uint32_t* ri = a.rk_i + size_t(b) * a.nlist_p2;
  // rank centroids by inner product (dot_f64: exact products, in-order sum),
  // ties toward the lower centroid: sort (dot desc, c asc)
  for (uint32_t c = threadIdx.x; c < a.nlist_p2; c += blockDim.x) {
    if (c < a.nlist) {
      double acc = 0.0;
      const float* cr = a.cent + size_t(c) * d;
      for (uint32_t j = 0; j < d; ++j) acc += double(q[j]) * double(cr[j]);
      rs[c] = acc, ri[c] = c;
    } else {
      rs[c] = -DBL_MAX, ri[c] = kSentinel;
    }
  }
  if (threadIdx.x == 0) sh_cnt = 0;
  __syncthreads();
  cta_bitonic(rs, ri, a.nlist_p2, better_sid);
  // scan the nprobe lists: exact scores of unmasked members
  double* cs = a.sc_s + size_t(b) * a.cap;
  uint32_t* ci = a.sc_i + size_t(b) * a.cap;
  for (uint32_t p = 0; p < a.nprobe; ++p) {
    const uint32_t c = ri[p];
    const uint32_t o0 = a.off[c], o1 = a.off[c + 1];
    for (uint32_t t = o0 + threadIdx.x; t < o1; t += blockDim.x) {
      const uint32_t id = a.ids[t];
      if (a.mask_bits && ((a.mask_bits[id >> 5] >> (id & 31)) & 1u)) continue;
      double acc = 0.0;
      const float* kr = a.keys + size_t(id) * d;
      for (uint32_t j = 0; j < d; ++j) acc += double(q[j]) * double(__ldg(kr + j));
      const uint32_t slot = atomicAdd(&sh_cnt, 1u);
      cs[slot] = acc, ci[slot] = id;
    }
  }
  __syncthreads();
  const uint32_t cnt = sh_cnt;
  uint32_t p2 = 1;
  while (p2 < cnt) p2 <<= 1;
  for (uint32_t i = cnt + threadIdx.x; i < p2; i += blockDim.x) cs[i] = -DBL_MAX, ci[i] = kSentinel;
  __syncthreads();
  cta_bitonic(cs, ci, p2, better_sid);
  const uint32_t take = cnt < a.k ? cnt : a.k;
  for (uint32_t r = threadIdx.x; r < a.k; r += blockDim.x) {
    a.out_ids[size_t(b) * a.k + r] = r < take ? ci[r] : kSentinel;
    a.out_sc[size_t(b) * a.k + r] = r < take ? float(cs[r]) : __int_as_float(0x7fc00000);
  }
  if (threadIdx.x == 0) {
    a.n_out[b] = take;
    a.scanned[b] = cnt;
    a.truncated[b] = take < a.k;
  }
}

uint32_t pow2_ge(uint64_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace
}  // namespace ra

using namespace ra;

extern "C" {

ra_status ra_ivf_build(ra_ctx* ctx, ra_kv* kv, uint32_t nlist_param, uint64_t seed,
                       uint32_t iters, uint32_t default_nprobe, ra_ivf** out) {
  return guard([&] {
    if (!ctx) invalid("null context");
    if (!kv || kv->n == 0) invalid("empty keys");  // index_ivf.cpp:60
    const uint64_t n = kv->n;
    const uint32_t d = kv->d;
    const uint32_t nlist =
        nlist_param == 0 ? uint32_t(std::ceil(std::sqrt(double(n)))) : nlist_param;
    if (nlist < 1 || nlist > n) invalid("nlist out of range");
    if (n > 0xFFFFFFFFull) invalid("too many keys");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->stream;
    const float* K = kv->keys.p;
    auto ivf = std::make_unique<ra_ivf>();
    ivf->nlist = nlist;
    ivf->default_nprobe = std::clamp<uint32_t>(default_nprobe, 1, nlist);
    ivf->d = d;
    ivf->n = n;
    // host copy of the keys' rows is needed for seeding and reseeds only
    std::vector<float> hx(size_t(n) * d);
    RA_CUDA(cudaMemcpyAsync(hx.data(), K, hx.size() * 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    // ---- k-means++ (index_ivf.cpp:24-52) ----
    Rng rng{seed};
    std::vector<double> cent(size_t(nlist) * d);
    auto set_row = [&](uint32_t c, uint64_t i) {
      for (uint32_t j = 0; j < d; ++j) cent[size_t(c) * d + j] = double(hx[i * d + j]);
    };
    set_row(0, rng.uniform_index(n));
    DevBuf<double> dc(d), d2(n);
    std::vector<double> hd2(n);
    RA_CUDA(cudaMemcpyAsync(dc.p, cent.data(), d * 8, cudaMemcpyHostToDevice, s));
    const uint32_t gb = uint32_t((n + 255) / 256);
    k_d2<<<gb, 256, 0, s>>>(K, n, d, dc.p, d2.p, 1);
    RA_LAUNCH_CHECK();
    for (uint32_t c = 1; c < nlist; ++c) {
      RA_CUDA(cudaMemcpyAsync(hd2.data(), d2.p, n * 8, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaStreamSynchronize(s));
      double total = 0.0;
      for (uint64_t i = 0; i < n; ++i) total += hd2[i];
      uint64_t pick = 0;
      if (total > 0) {
        const double target = (1.0 - rng.uniform()) * total;
        double run = 0;
        pick = n - 1;
        for (uint64_t i = 0; i < n; ++i) {
          run += hd2[i];
          if (run >= target) {
            pick = i;
            break;
          }
        }
      } else {
        pick = c % uint32_t(n);
      }
      set_row(c, pick);
      RA_CUDA(cudaMemcpyAsync(dc.p, cent.data() + size_t(c) * d, d * 8, cudaMemcpyHostToDevice, s));
      k_d2<<<gb, 256, 0, s>>>(K, n, d, dc.p, d2.p, 0);
      RA_LAUNCH_CHECK();
    }
    // ---- Lloyd (index_ivf.cpp:74-125) ----
    DevBuf<double> dcent(size_t(nlist) * d), csq(nlist), sums(size_t(nlist) * d);
    DevBuf<uint32_t> assign(n), skey(n), iota(n), sids(n), off(nlist + 1);
    k_iota<<<gb, 256, 0, s>>>(iota.p, n);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, assign.p, skey.p, iota.p, sids.p, int(n),
                                    0, 32, s);
    DevBuf<uint8_t> tmp(tmp_bytes + 16);
    int end_bit = 1;
    while ((1u << end_bit) <= nlist) ++end_bit;
    const size_t smem = size_t(kAP) * (d + 1) * 4;
    RA_CUDA(cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    auto assign_and_lists = [&]() {
      RA_CUDA(cudaMemcpyAsync(dcent.p, cent.data(), cent.size() * 8, cudaMemcpyHostToDevice, s));
      k_csq<<<(nlist + 127) / 128, 128, 0, s>>>(dcent.p, nlist, d, csq.p);
      k_assign<<<uint32_t((n + kAP - 1) / kAP), kAP, smem, s>>>(K, n, d, dcent.p, csq.p, nlist,
                                                                assign.p);
      // stable sort by cluster keeps ids ascending within each list
      cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, assign.p, skey.p, iota.p, sids.p, int(n),
                                      0, end_bit, s);
      k_offsets<<<(nlist + 1 + 127) / 128, 128, 0, s>>>(skey.p, n, nlist, off.p);
      RA_LAUNCH_CHECK();
    };
    std::vector<uint32_t> h_off(nlist + 1), h_assign;
    std::vector<double> h_sums(size_t(nlist) * d);
    for (uint32_t it = 0; it < iters; ++it) {
      assign_and_lists();
      k_sums<<<uint32_t((uint64_t(nlist) * d + 255) / 256), 256, 0, s>>>(K, d, off.p, sids.p,
                                                                        nlist, sums.p);
      RA_LAUNCH_CHECK();
      RA_CUDA(cudaMemcpyAsync(h_off.data(), off.p, (nlist + 1) * 4, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaMemcpyAsync(h_sums.data(), sums.p, h_sums.size() * 8, cudaMemcpyDeviceToHost, s));
      RA_CUDA(cudaStreamSynchronize(s));
      std::vector<uint64_t> count(nlist);
      for (uint32_t c = 0; c < nlist; ++c) count[c] = h_off[c + 1] - h_off[c];
      // reseed empty clusters from the largest cluster's farthest member (:96-118)
      bool reseeded = false;
      for (uint32_t c = 0; c < nlist; ++c) {
        if (count[c] != 0) continue;
        if (!reseeded) {
          h_assign.resize(n);
          RA_CUDA(cudaMemcpyAsync(h_assign.data(), assign.p, n * 4, cudaMemcpyDeviceToHost, s));
          RA_CUDA(cudaStreamSynchronize(s));
          reseeded = true;
        }
        const uint32_t largest =
            uint32_t(std::max_element(count.begin(), count.end()) - count.begin());
        if (count[largest] <= 1) break;
        std::vector<double> mean(d);
        for (uint32_t j = 0; j < d; ++j)
          mean[j] = h_sums[size_t(largest) * d + j] / double(count[largest]);
        double far_d = -1.0;
        uint64_t far_i = 0;
        for (uint64_t i = 0; i < n; ++i) {
          if (h_assign[i] != largest) continue;
          double acc = 0.0;
          for (uint32_t j = 0; j < d; ++j) {
            const double v = double(hx[i * d + j]) - mean[j];
            acc = std::fma(v, v, acc);
          }
          if (acc > far_d) far_d = acc, far_i = i;
        }
        for (uint32_t j = 0; j < d; ++j) {
          h_sums[size_t(largest) * d + j] -= double(hx[far_i * d + j]);
          h_sums[size_t(c) * d + j] = double(hx[far_i * d + j]);
        }
        count[largest]--;
        count[c] = 1;
        h_assign[far_i] = c;
      }
      for (uint32_t c = 0; c < nlist; ++c)
        if (count[c] > 0)
          for (uint32_t j = 0; j < d; ++j)
            cent[size_t(c) * d + j] = h_sums[size_t(c) * d + j] / double(count[c]);
    }
    // final assignment under the final centroids (:128-145)
    assign_and_lists();
    ivf->h_cent.resize(size_t(nlist) * d);
    for (size_t e = 0; e < cent.size(); ++e) ivf->h_cent[e] = float(cent[e]);
    ivf->cent.alloc(ivf->h_cent.size());
    ivf->offsets.alloc(nlist + 1);
    ivf->ids.alloc(n);
    RA_CUDA(cudaMemcpyAsync(ivf->cent.p, ivf->h_cent.data(), ivf->h_cent.size() * 4,
                            cudaMemcpyHostToDevice, s));
    RA_CUDA(cudaMemcpyAsync(ivf->offsets.p, off.p, (nlist + 1) * 4, cudaMemcpyDeviceToDevice, s));
    RA_CUDA(cudaMemcpyAsync(ivf->ids.p, sids.p, n * 4, cudaMemcpyDeviceToDevice, s));
    ivf->h_offsets.resize(nlist + 1);
    ivf->h_ids.resize(n);
    RA_CUDA(cudaMemcpyAsync(ivf->h_offsets.data(), off.p, (nlist + 1) * 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaMemcpyAsync(ivf->h_ids.data(), sids.p, n * 4, cudaMemcpyDeviceToHost, s));
    RA_CUDA(cudaStreamSynchronize(s));
    ra_kv_retain(kv);
    ivf->kv = kv;
    *out = ivf.release();
  });
}

void ra_ivf_free(ra_ivf* ivf) {
  if (!ivf) return;
  DeviceGuard dg(ivf->kv ? ivf->kv->device : 0, true);
  ra_kv* kv = ivf->kv;
  delete ivf;
  ra_kv_release(kv);
}

uint32_t ra_ivf_nlist(const ra_ivf* ivf) { return ivf ? ivf->nlist : 0; }
uint32_t ra_ivf_default_nprobe(const ra_ivf* ivf) { return ivf ? ivf->default_nprobe : 0; }

// host copies: centroids (nlist x d f32), list offsets (nlist + 1) and ids (n)
ra_status ra_ivf_export(const ra_ivf* ivf, float* centroids, uint32_t* offsets, uint32_t* ids) {
  return guard([&] {
    if (!ivf) invalid("null index");
    if (centroids) std::memcpy(centroids, ivf->h_cent.data(), ivf->h_cent.size() * 4);
    if (offsets) std::memcpy(offsets, ivf->h_offsets.data(), ivf->h_offsets.size() * 4);
    if (ids) std::memcpy(ids, ivf->h_ids.data(), ivf->h_ids.size() * 4);
  });
}

uint64_t ra_ivf_memory_bytes(const ra_ivf* ivf) {  // index_ivf.cpp:183-187
  return ivf ? uint64_t(ivf->h_cent.size()) * 4 + ivf->n * 4 : 0;
}

// IVFIndex::search (index_ivf.cpp:153-181) for B queries (device pointers).
ra_status ra_ivf_search_batch(ra_ctx* ctx, const ra_ivf* ivf, uint32_t B, const float* q,
                              uint32_t q_dim, uint32_t k, int64_t nprobe, const uint32_t* mask,
                              uint64_t mask_n, uint32_t* ids, float* scores, uint32_t* n_out,
                              uint64_t* scanned, uint8_t* truncated) {
  return guard([&] {
    if (!ctx) invalid("null context");
    if (!ivf) invalid("null index");
    if (q_dim != ivf->d) invalid("query dimension mismatch");
    const int64_t np = nprobe >= 0 ? nprobe : int64_t(ivf->default_nprobe);
    if (np < 1 || np > int64_t(ivf->nlist)) invalid("nprobe out of range");
    if (k < 1) invalid("k out of range");
    if (B == 0) return;
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->stream;
    uint32_t max_len = 0;  // upper bound of candidates: the np largest lists
    {
      std::vector<uint32_t> lens(ivf->nlist);
      for (uint32_t c = 0; c < ivf->nlist; ++c) lens[c] = ivf->h_offsets[c + 1] - ivf->h_offsets[c];
      std::partial_sort(lens.begin(), lens.begin() + np, lens.end(), std::greater<uint32_t>());
      uint64_t sum = 0;
      for (int64_t p = 0; p < np; ++p) sum += lens[p];
      max_len = uint32_t(std::max<uint64_t>(sum, 1));
    }
    IvfSearchArgs a{};
    a.keys = ivf->kv->keys.p;
    a.cent = ivf->cent.p;
    a.off = ivf->offsets.p;
    a.ids = ivf->ids.p;
    a.q = q;
    a.d = ivf->d;
    a.nlist = ivf->nlist;
    a.nprobe = uint32_t(np);
    a.k = k;
    a.B = B;
    a.cap = pow2_ge(max_len);
    a.nlist_p2 = pow2_ge(ivf->nlist);
    const uint64_t words = (ivf->n + 31) / 32;
    DevBuf<uint32_t> bits;
    if (mask_n) {
      bits.alloc(words);
      launch_mask_bitset(s, mask, mask_n, bits.p, words);
      a.mask_bits = bits.p;
    }
    DevBuf<double> scs(size_t(B) * a.cap), rks(size_t(B) * a.nlist_p2);
    DevBuf<uint32_t> sci(size_t(B) * a.cap), rki(size_t(B) * a.nlist_p2);
    a.sc_s = scs.p, a.sc_i = sci.p, a.rk_s = rks.p, a.rk_i = rki.p;
    a.out_ids = ids, a.out_sc = scores, a.n_out = n_out, a.scanned = scanned,
    a.truncated = truncated;
    k_ivf_search<<<B, 256, 0, s>>>(a);
    RA_LAUNCH_CHECK();
    RA_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
