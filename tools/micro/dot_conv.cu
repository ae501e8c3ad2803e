// microbenchmark (profiling aid): the search's in-order f64 dot of an f32
// row against an f64 query, per element cycles for W warps per SM, with
// (a) F2F.F64.F32 conversions, (b) integer-op conversions (normal values),
// (c) rows already in f64 (no conversion: the DFMA chain alone)
#include <cstdint>
#include <cstdio>
constexpr int D = 128;
__device__ __forceinline__ double cvt_int(float f) {
  const uint32_t b = __float_as_uint(f);
  const uint32_t hi = ((((b & 0x7FFFFFFFu) >> 3) + 0x38000000u) | (b & 0x80000000u));
  return __hiloint2double(int(hi), int(b << 29));
}
// the search kernel's software-pipelined row dot (search_pipe.cu row_dot)
__device__ __forceinline__ double row_dot_pipe(const double* __restrict__ qd,
                                               const float* __restrict__ row) {
  const double2* q2 = reinterpret_cast<const double2*>(qd);
  const float4* r4 = reinterpret_cast<const float4*>(row);
  constexpr int NC = D / 8;
  double2 qa[4], qb[4];
  float4 ra[2], rb[2];
  auto load = [&](int c, double2 (&q)[4], float4 (&r)[2]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = q2[4 * c + j];
    r[0] = r4[2 * c];
    r[1] = r4[2 * c + 1];
  };
  double acc = 0.0;
  auto fma8 = [&](const double2 (&q)[4], const float4 (&r)[2]) {
    acc = fma(q[0].x, (double)r[0].x, acc);
    acc = fma(q[0].y, (double)r[0].y, acc);
    acc = fma(q[1].x, (double)r[0].z, acc);
    acc = fma(q[1].y, (double)r[0].w, acc);
    acc = fma(q[2].x, (double)r[1].x, acc);
    acc = fma(q[2].y, (double)r[1].y, acc);
    acc = fma(q[3].x, (double)r[1].z, acc);
    acc = fma(q[3].y, (double)r[1].w, acc);
  };
  load(0, qa, ra);
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    if (c + 1 < NC) load(c + 1, qb, rb);
    fma8(qa, ra);
    if (c + 2 < NC) load(c + 2, qa, ra);
    if (c + 1 < NC) fma8(qb, rb);
  }
  return acc;
}

template <int MODE>
__global__ void dotk(const float* rows, const double* rowsd, const double* q, int reps,
                     double* out, long long* cyc) {
  __shared__ double qs[D];
  __shared__ float rs[32][D + 4];
  __shared__ double rd[MODE == 2 ? 16 : 1][MODE == 2 ? D + 2 : 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < D; i += blockDim.x) qs[i] = q[i];
  for (int i = threadIdx.x; i < 32 * D; i += blockDim.x)
    rs[i / D][i % D] = rows[i];
  if (MODE == 2)
    for (int i = threadIdx.x; i < 16 * D; i += blockDim.x)
      rd[i / D][i % D] = rowsd[i];
  __syncthreads();
  const float* row = rs[lane];
  const double* rowd = MODE == 2 ? rd[lane % 16] : nullptr;
  double acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE == 3) {
      acc += row_dot_pipe(qs, row);
      continue;
    }
#pragma unroll 8
    for (int i = 0; i < D; ++i) {
      double k;
      if (MODE == 0) k = (double)row[i];
      else if (MODE == 1) k = cvt_int(row[i]);
      else k = rowd[i];
      acc = fma(qs[i], k, acc);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* rows;
  double *rowsd, *q, *out;
  long long* cyc;
  cudaMalloc(&rows, 32 * 16 * D * 4);
  cudaMalloc(&rowsd, 32 * 16 * D * 8);
  cudaMalloc(&q, D * 8);
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 8);
  cudaMemset(rows, 0, 32 * 16 * D * 4);
  cudaMemset(rowsd, 0, 32 * 16 * D * 8);
  cudaMemset(q, 0, D * 8);
  const int reps = 64;
  for (int wps : {1, 2, 4, 8, 16}) {
    long long h[4];
    for (int mode = 0; mode < 4; ++mode) {
      if (mode == 0) dotk<0><<<148, 32 * wps>>>(rows, rowsd, q, reps, out, cyc);
      if (mode == 1) dotk<1><<<148, 32 * wps>>>(rows, rowsd, q, reps, out, cyc);
      if (mode == 2) dotk<2><<<148, 32 * wps>>>(rows, rowsd, q, reps, out, cyc);
      if (mode == 3) dotk<3><<<148, 32 * wps>>>(rows, rowsd, q, reps, out, cyc);
      cudaMemcpy(&h[mode], cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("warps/SM %2d: cycles per element  F2F %.2f  int-cvt %.2f  f64 rows %.2f  pipelined %.2f\n",
           wps, double(h[0]) / (reps * D), double(h[1]) / (reps * D), double(h[2]) / (reps * D),
           double(h[3]) / (reps * D));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
