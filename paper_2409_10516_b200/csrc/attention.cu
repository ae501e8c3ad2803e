// K7 sparse attention + LSE merge (/root/reference/proj/src/attention.cpp:102-157).
//
// partial_attention: one CTA per query row. z_i is the reference's exact
// in-order f64 dot (one lane per index, as dot_f64) times 1/sqrt(d), or the
// caller's exact search score when supplied (the Omega side reuses the
// graph search's scores, so its keys are never re-read). Thread j then
// accumulates out[j] and expsum over indices in the reference's order, so
// the only deviation from the CPU result is the device exp() (<= 1 ulp).
#include <cfloat>

#include "common.cuh"
#include "tma.cuh"

namespace ra {
namespace {

constexpr int kThreads = 128;
constexpr uint32_t kSmemZ = 8192;  // z values kept in shared memory (else HBM)

template <int D>
__device__ __forceinline__ double exact_dot_f(const float* __restrict__ q,
                                              const float* __restrict__ k, uint32_t d) {
  double acc = 0.0;
  if constexpr (D > 0) {
    const float4* k4 = reinterpret_cast<const float4*>(k);
    const float4* q4 = reinterpret_cast<const float4*>(q);
#pragma unroll 8
    for (int c = 0; c < D / 4; ++c) {
      const float4 kv = __ldg(k4 + c), qv = q4[c];
      acc = fma((double)qv.x, (double)kv.x, acc);
      acc = fma((double)qv.y, (double)kv.y, acc);
      acc = fma((double)qv.z, (double)kv.z, acc);
      acc = fma((double)qv.w, (double)kv.w, acc);
    }
  } else {
    for (uint32_t i = 0; i < d; ++i) acc = fma((double)q[i], (double)__ldg(k + i), acc);
  }
  return acc;
}

__device__ double block_max(double v, double* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  v = -DBL_MAX;
  for (int i = 0; i < kThreads / 32; ++i) v = fmax(v, red[i]);
  return v;
}

template <int D>
__global__ void __launch_bounds__(kThreads)
    k_partial(const KVRef* __restrict__ kvs, uint32_t d, const float* __restrict__ q, const uint32_t* __restrict__ idx,
              uint32_t m_stride, const uint32_t* __restrict__ m_arr, const double* scores64,
              uint32_t s_stride, double inv_sqrt_d, double* out, double* zmax_out,
              double* expsum_out, double* zscratch, uint64_t z_stride, uint8_t* empty_out,
              uint32_t* err_flag) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* red = reinterpret_cast<double*>(smem);
  float* qs = reinterpret_cast<float*>(red + kThreads / 32);
  double* zs = reinterpret_cast<double*>(qs + ((d + 3) & ~3u));
  const uint32_t b = blockIdx.x;
  const float* __restrict__ keys = kvs[b].keys;
  const float* __restrict__ values = kvs[b].values;
  const uint64_t n = kvs[b].n;
  const uint32_t m = m_arr[b];
  if (empty_out && threadIdx.x == 0) empty_out[b] = m == 0;
  const uint32_t* ix = idx + size_t(b) * m_stride;
  if (m == 0) {  // empty_partial (attention.cpp:130-134)
    for (uint32_t j = threadIdx.x; j < d; j += kThreads) out[size_t(b) * d + j] = 0.0;
    if (threadIdx.x == 0) zmax_out[b] = 0.0, expsum_out[b] = 0.0;
    return;
  }
  double* z = m <= kSmemZ ? zs : zscratch + size_t(b) * z_stride;
  for (uint32_t j = threadIdx.x; j < d; j += kThreads) qs[j] = q[size_t(b) * d + j];
  __syncthreads();

  double zmax = -DBL_MAX;
  for (uint32_t i = threadIdx.x; i < m; i += kThreads) {
    const uint32_t id = ix[i];
    double zi;
    if (id >= n) {
      atomicOr(err_flag, 1u);
      zi = -DBL_MAX;
    } else if (scores64) {
      zi = scores64[size_t(b) * s_stride + i] * inv_sqrt_d;
    } else {
      zi = exact_dot_f<D>(qs, keys + size_t(id) * d, d) * inv_sqrt_d;
    }
    z[i] = zi;
    zmax = fmax(zmax, zi);
  }
  zmax = block_max(zmax, red);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < m; i += kThreads) z[i] = exp(z[i] - zmax);
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < d; j += kThreads) {
    double acc = 0.0, es = 0.0;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t id = ix[i];
      if (id >= n) continue;
      const double e = z[i];
      es += e;
      acc += e * (double)__ldg(values + size_t(id) * d + j);
    }
    out[size_t(b) * d + j] = acc / es;
    if (j == 0) {
      zmax_out[b] = zmax;
      expsum_out[b] = es;
    }
  }
}

// merge_gammas + merge (attention.cpp:136-157), one thread per (row, j)
__global__ void k_merge(uint32_t B, uint32_t d, const double* ow, const double* zw,
                        const double* sw, const uint8_t* w_empty, const double* oo,
                        const double* zo, const double* so, const uint8_t* o_empty,
                        double* out, double* gw_out, double* go_out, uint32_t* err_flag) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= uint64_t(B) * d) return;
  const uint32_t b = uint32_t(t / d), j = uint32_t(t % d);
  const bool we = w_empty && w_empty[b], oe = o_empty && o_empty[b];
  double gw, go;
  if (we && oe) {
    if (j == 0) atomicOr(err_flag, 2u);
    return;
  }
  if (we) {
    gw = 0.0, go = 1.0;
  } else if (oe) {
    gw = 1.0, go = 0.0;
  } else {
    const double zref = fmax(zw[b], zo[b]);
    const double ew = exp(zw[b] - zref) * sw[b];
    const double eo = exp(zo[b] - zref) * so[b];
    const double denom = ew + eo;
    gw = ew / denom;
    go = eo / denom;
  }
  double r;
  if (we)
    r = oo[t];
  else if (oe)
    r = ow[t];
  else
    r = gw * ow[t] + go * oo[t];
  out[t] = r;
  if (j == 0) {
    if (gw_out) gw_out[b] = gw;
    if (go_out) go_out[b] = go;
  }
}

// ---- engine path: W partial per (KV group, chunk of W) --------------------------
// The static set W is shared by the hpg query heads of a group, so each W
// key/value row is read from HBM once per group (TMA bulk copies into shared
// memory) and scored against all hpg queries. Each chunk emits an
// unnormalised partial (sum e*v, chunk max, sum e); k_omega_merge folds the
// chunks with the same log-sum-exp rescaling merge() uses.
constexpr uint32_t kWC = 64;  // W rows per CTA

// K/V element access for f32 or bf16 groups (bf16 -> f32 -> f64 is exact)
__device__ __forceinline__ double elem(const float* p, uint32_t i) { return (double)p[i]; }
__device__ __forceinline__ double elem(const uint16_t* p, uint32_t i) {
  return (double)__uint_as_float(uint32_t(p[i]) << 16);
}
template <typename T> __device__ __forceinline__ const T* kv_keys(const KVRef& r);
template <> __device__ __forceinline__ const float* kv_keys<float>(const KVRef& r) { return r.keys; }
template <> __device__ __forceinline__ const uint16_t* kv_keys<uint16_t>(const KVRef& r) {
  return r.keys16;
}
template <typename T> __device__ __forceinline__ const T* kv_vals(const KVRef& r);
template <> __device__ __forceinline__ const float* kv_vals<float>(const KVRef& r) { return r.values; }
template <> __device__ __forceinline__ const uint16_t* kv_vals<uint16_t>(const KVRef& r) {
  return r.values16;
}
// tile row stride in elements: rows stay 16-B aligned for the TMA copies
template <typename T> constexpr uint32_t kpad() { return 16 / sizeof(T); }

// in-order f64 dot of q (f64) with a staged key row
template <int D>
__device__ __forceinline__ double tile_dot(const double* qh, const float* row) {
  double acc = 0.0;
  const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll 8
  for (int cc = 0; cc < D / 4; ++cc) {
    const float4 kv = r4[cc];
    acc = fma(qh[4 * cc + 0], (double)kv.x, acc);
    acc = fma(qh[4 * cc + 1], (double)kv.y, acc);
    acc = fma(qh[4 * cc + 2], (double)kv.z, acc);
    acc = fma(qh[4 * cc + 3], (double)kv.w, acc);
  }
  return acc;
}
template <int D>
__device__ __forceinline__ double tile_dot(const double* qh, const uint16_t* row) {
  double acc = 0.0;
  const uint4* r4 = reinterpret_cast<const uint4*>(row);
#pragma unroll 4
  for (int cc = 0; cc < D / 8; ++cc) {
    const uint4 w = r4[cc];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      acc = fma(qh[8 * cc + 2 * t], (double)__uint_as_float(ws[t] << 16), acc);
      acc = fma(qh[8 * cc + 2 * t + 1], (double)__uint_as_float(ws[t] & 0xFFFF0000u), acc);
    }
  }
  return acc;
}

template <int D, typename T>
__global__ void __launch_bounds__(256)
    k_wpartial(const KVRef* __restrict__ gkv, const float* __restrict__ q,
               const uint32_t* __restrict__ W, uint32_t nW, uint32_t hpg, double inv_sqrt_d,
               double* __restrict__ part_out, double* __restrict__ part_m,
               double* __restrict__ part_s) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t c = blockIdx.x, g = blockIdx.y, C = gridDim.x;
  const uint32_t tid = threadIdx.x;
  const uint32_t i0 = c * kWC, rows = min(kWC, nW - i0);
  constexpr uint32_t KS = D + kpad<T>();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  T* Kt = reinterpret_cast<T*>(smem + 16);                          // [kWC][KS]
  T* Vt = Kt + kWC * KS;                                            // [kWC][D]
  double* qs = reinterpret_cast<double*>(Vt + kWC * D);             // [hpg][D]
  double* z = qs + size_t(hpg) * D;                                 // [hpg][kWC]
  const T* K = kv_keys<T>(gkv[g]);
  const T* V = kv_vals<T>(gkv[g]);
  if (tid == 0) {
    mbar_init(bar);
    mbar_arrive_expect_tx(bar, rows * D * uint32_t(2 * sizeof(T)));
  }
  __syncthreads();
  if (tid < rows) {
    const uint32_t id = W[i0 + tid];
    bulk_g2s(Kt + tid * KS, K + size_t(id) * D, D * uint32_t(sizeof(T)), bar);
    bulk_g2s(Vt + tid * D, V + size_t(id) * D, D * uint32_t(sizeof(T)), bar);
  }
  for (uint32_t e = tid; e < hpg * D; e += blockDim.x)
    qs[e] = (double)q[size_t(g) * hpg * D + e];
  __syncthreads();
  mbar_wait(bar, 0);
  for (uint32_t t = tid; t < hpg * kWC; t += blockDim.x) {
    const uint32_t h = t / kWC, i = t % kWC;
    double acc = -DBL_MAX;
    if (i < rows) acc = tile_dot<D>(qs + h * D, Kt + i * KS) * inv_sqrt_d;
    z[h * kWC + i] = acc;
  }
  __syncthreads();
  // per head: chunk max, e = exp(z - max), sum e (warp h handles head h)
  const uint32_t warp = tid >> 5, lane = tid & 31;
  for (uint32_t h = warp; h < hpg; h += blockDim.x / 32) {
    double m = -DBL_MAX;
    for (uint32_t i = lane; i < rows; i += 32) m = fmax(m, z[h * kWC + i]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
    double s = 0.0;
    for (uint32_t i = lane; i < rows; i += 32) {
      const double e = exp(z[h * kWC + i] - m);
      z[h * kWC + i] = e;
      s += e;
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) {
      part_m[(size_t(g) * C + c) * hpg + h] = m;
      part_s[(size_t(g) * C + c) * hpg + h] = s;
    }
  }
  __syncthreads();
  for (uint32_t t = tid; t < hpg * D; t += blockDim.x) {
    const uint32_t h = t / D, j = t % D;
    double acc = 0.0;
    for (uint32_t i = 0; i < rows; ++i) acc = fma(z[h * kWC + i], elem(Vt, i * D + j), acc);
    part_out[((size_t(g) * C + c) * hpg + h) * D + j] = acc;
  }
}

// ---- engine path: Omega partial (search scores reused) + merge per head --------
template <int D, typename T>
__global__ void __launch_bounds__(128)
    k_omega_merge(const KVRef* __restrict__ hkv, const uint32_t* __restrict__ ids,
                  const double* __restrict__ s64, const uint32_t* __restrict__ n_out,
                  uint32_t k, uint32_t hpg, uint32_t C, uint32_t nW, double inv_sqrt_d,
                  const double* __restrict__ part_out, const double* __restrict__ part_m,
                  const double* __restrict__ part_s, double* __restrict__ out, uint32_t TR,
                  uint32_t* __restrict__ ids_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t h = blockIdx.x, g = h / hpg, hl = h % hpg, tid = threadIdx.x;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  T* Vt = reinterpret_cast<T*>(smem + 16);                          // [TR][D]
  double* e = reinterpret_cast<double*>(Vt + size_t(TR) * D);       // [TR]
  double* wx = e + TR;                                              // [C] chunk weights
  __shared__ double red[4];
  const uint32_t m = n_out[h];
  const T* V = kv_vals<T>(hkv[h]);
  // the first Omega tile's V rows are requested before anything else, so
  // the copies overlap the max / W-fold arithmetic below
  uint32_t rows = min(TR, m);
  if (tid == 0) {
    mbar_init(bar);
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, rows * D * uint32_t(sizeof(T)));
  }
  __syncthreads();
  for (uint32_t i = tid; i < rows; i += blockDim.x)
    bulk_g2s(Vt + size_t(i) * D, V + size_t(ids[size_t(h) * k + i]) * D, D * uint32_t(sizeof(T)),
             bar);
  if (ids_out)
    for (uint32_t i = tid; i < k; i += blockDim.x) ids_out[size_t(h) * k + i] = ids[size_t(h) * k + i];
  // Omega max (scores are exact f64 search scores; z = s / sqrt(d))
  double zo = -DBL_MAX;
  for (uint32_t i = tid; i < m; i += blockDim.x) zo = fmax(zo, s64[size_t(h) * k + i] * inv_sqrt_d);
  for (int o = 16; o; o >>= 1) zo = fmax(zo, __shfl_xor_sync(kFull, zo, o));
  if ((tid & 31) == 0) red[tid >> 5] = zo;
  // W chunk maxima -> smem (one load per chunk)
  for (uint32_t c = tid; c < C; c += blockDim.x) wx[c] = part_m[(size_t(g) * C + c) * hpg + hl];
  __syncthreads();
  zo = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
  double zw = -DBL_MAX;
  for (uint32_t c = 0; c < C; ++c) zw = fmax(zw, wx[c]);
  __syncthreads();  // every thread has read the maxima
  for (uint32_t c = tid; c < C; c += blockDim.x) wx[c] = exp(wx[c] - zw);
  for (uint32_t i = tid; i < rows; i += blockDim.x) e[i] = exp(s64[size_t(h) * k + i] * inv_sqrt_d - zo);
  __syncthreads();
  double sw = 0.0;
  for (uint32_t c = 0; c < C; ++c) sw += wx[c] * part_s[(size_t(g) * C + c) * hpg + hl];
  double acc[(D + 127) / 128] = {};
  double so = 0.0;
  uint32_t phase = 0;
  for (uint32_t t0 = 0; t0 < m; t0 += TR) {
    if (t0) {  // further tiles (k > TR only)
      rows = min(TR, m - t0);
      __syncthreads();  // previous tile fully consumed
      fence_proxy_async();  // each issuing thread orders the reads before its copies
      if (tid == 0) mbar_arrive_expect_tx(bar, rows * D * uint32_t(sizeof(T)));
      __syncthreads();
      for (uint32_t i = tid; i < rows; i += blockDim.x) {
        bulk_g2s(Vt + size_t(i) * D, V + size_t(ids[size_t(h) * k + t0 + i]) * D,
                 D * uint32_t(sizeof(T)), bar);
        e[i] = exp(s64[size_t(h) * k + t0 + i] * inv_sqrt_d - zo);
      }
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    __syncthreads();
    for (uint32_t i = 0; i < rows; ++i) {
      const double ei = e[i];
      so += ei;
#pragma unroll
      for (uint32_t r = 0; r < (D + 127) / 128; ++r) {
        const uint32_t j = tid + r * 128;
        if (j < D) acc[r] = fma(ei, elem(Vt, i * D + j), acc[r]);
      }
    }
  }
  // W partial: fold the chunks (log-sum-exp), then merge() with Omega
  const bool we = nW == 0, oe = m == 0;
  double gw = 1.0, go = 0.0;
  if (we) {
    gw = 0.0, go = 1.0;
  } else if (!oe) {
    const double zref = fmax(zw, zo);
    const double ew = exp(zw - zref) * sw, eo = exp(zo - zref) * so;
    gw = ew / (ew + eo);
    go = eo / (ew + eo);
  }
#pragma unroll
  for (uint32_t r = 0; r < (D + 127) / 128; ++r) {
    const uint32_t j = tid + r * 128;
    if (j >= D) continue;
    double ow = 0.0;
    if (!we) {
      for (uint32_t c = 0; c < C; ++c)
        ow += wx[c] * part_out[((size_t(g) * C + c) * hpg + hl) * D + j];
      ow /= sw;
    }
    const double oo = oe ? 0.0 : acc[r] / so;
    out[size_t(h) * D + j] = we ? oo : (oe ? ow : gw * ow + go * oo);
  }
}

template <int D, typename T>
void launch_engine_attention_d(cudaStream_t st, const EngineAttn& a, int part) {
  const uint32_t C = (a.nW + kWC - 1) / kWC;
  if (part == 0) {
    if (!C) return;
    const size_t smem_w = 16 + kWC * (D + kpad<T>()) * sizeof(T) + kWC * D * sizeof(T) +
                          size_t(a.hpg) * D * 8 + size_t(a.hpg) * kWC * 8;
    RA_CUDA(cudaFuncSetAttribute(k_wpartial<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_w));
    k_wpartial<D, T><<<dim3(C, a.G), 256, smem_w, st>>>(a.gkv, a.q, a.W, a.nW, a.hpg,
                                                         a.inv_sqrt_d, a.part_out, a.part_m,
                                                         a.part_s);
    RA_LAUNCH_CHECK();
    return;
  }
  // one Omega tile for k up to ~180 rows (the whole top-k in one TMA round)
  const uint32_t TR = std::min<uint32_t>(std::max<uint32_t>(a.k, 1),
                                         uint32_t((150u << 10) / (D * sizeof(T) + 8)));
  const size_t smem_o = 16 + size_t(TR) * D * sizeof(T) + size_t(TR) * 8 + size_t(C) * 8;
  RA_CUDA(cudaFuncSetAttribute(k_omega_merge<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem_o));
  k_omega_merge<D, T><<<a.H, 128, smem_o, st>>>(a.hkv, a.ids, a.s64, a.n_out, a.k, a.hpg, C,
                                                a.nW, a.inv_sqrt_d, a.part_out, a.part_m,
                                                a.part_s, a.out, TR, a.ids_out);
  RA_LAUNCH_CHECK();
}

}  // namespace

size_t partial_scratch_doubles(uint32_t B, uint32_t max_m) {
  return max_m > kSmemZ ? size_t(B) * max_m : 0;
}

void launch_partial_attention_ex(cudaStream_t s, const KVRef* kvs, uint32_t d, uint32_t B, const float* q,
                                 const uint32_t* idx, uint32_t m_stride, const uint32_t* m,
                                 const double* scores64, uint32_t s_stride, double* out,
                                 double* zmax, double* expsum, double* zscratch,
                                 uint64_t z_stride, uint8_t* empty_out, uint32_t* err_flag) {
  if (!B) return;
  const double inv_sqrt_d = 1.0 / sqrt(double(d));
  const size_t smem = (kThreads / 32) * 8 + ((d + 3) & ~3u) * 4 + size_t(kSmemZ) * 8;
  auto go = [&](auto kern) {
    RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<B, kThreads, smem, s>>>(kvs, d, q, idx, m_stride, m, scores64, s_stride,
                                   inv_sqrt_d, out, zmax, expsum, zscratch, z_stride, empty_out, err_flag);
    RA_LAUNCH_CHECK();
  };
  if (d == 128)
    go(k_partial<128>);
  else if (d % 4 == 0 && d == 64)
    go(k_partial<64>);
  else
    go(k_partial<0>);
}

void launch_merge(cudaStream_t s, uint32_t B, uint32_t d, const double* ow, const double* zw,
                  const double* sw, const uint8_t* w_empty, const double* oo,
                  const double* zo, const double* so, const uint8_t* o_empty, double* out,
                  double* gw, double* go, uint32_t* err_flag) {
  const uint64_t total = uint64_t(B) * d;
  if (!total) return;
  k_merge<<<uint32_t((total + 255) / 256), 256, 0, s>>>(B, d, ow, zw, sw, w_empty, oo, zo, so,
                                                         o_empty, out, gw, go, err_flag);
  RA_LAUNCH_CHECK();
}

bool engine_attention_supported(uint32_t d) { return d == 128 || d == 64 || d == 32; }

size_t engine_attention_part_doubles(uint32_t G, uint32_t hpg, uint32_t nW, uint32_t d) {
  const uint32_t C = (nW + kWC - 1) / kWC;
  return size_t(G) * std::max<uint32_t>(C, 1) * hpg * (d + 2);
}

template <typename T>
static void engine_attention_t(cudaStream_t st, const EngineAttn& a, int part) {
  switch (a.d) {
    case 128: launch_engine_attention_d<128, T>(st, a, part); break;
    case 64: launch_engine_attention_d<64, T>(st, a, part); break;
    case 32: launch_engine_attention_d<32, T>(st, a, part); break;
    default: throw Error(RA_ERR_RUNTIME, "engine attention: unsupported head dim");
  }
}
static void engine_attention(cudaStream_t st, const EngineAttn& a, int part) {
  if (a.bf16) engine_attention_t<uint16_t>(st, a, part);
  else engine_attention_t<float>(st, a, part);
}
void launch_engine_wpartial(cudaStream_t st, const EngineAttn& a) { engine_attention(st, a, 0); }
void launch_engine_omega_merge(cudaStream_t st, const EngineAttn& a) {
  engine_attention(st, a, 1);
}

}  // namespace ra
