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

}  // namespace ra
