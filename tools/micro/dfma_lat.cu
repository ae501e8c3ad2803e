// microbenchmark: dependent DFMA / DADD / FFMA chain latency and
// L2/HBM dependent-load latency on this GPU (profiling aid)
#include <cstdio>
#include <cstdint>
__global__ void chain(double* out, const double* in, int n, long long* cyc) {
  double a = in[threadIdx.x], b = in[threadIdx.x + 32], acc = in[threadIdx.x + 64];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc = fma(a, b, acc);
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chainf(float* out, const float* in, int n, long long* cyc) {
  float a = in[threadIdx.x], b = in[threadIdx.x + 32], acc = in[threadIdx.x + 64];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc = fmaf(a, b, acc);
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chase(const uint32_t* next, int n, uint32_t* out, long long* cyc) {
  uint32_t p = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = t1 - t0;
}
int main() {
  double *din, *dout; float *fin, *fout; long long* cyc; long long h;
  cudaMalloc(&din, 1024); cudaMalloc(&dout, 1024); cudaMalloc(&fin, 1024); cudaMalloc(&fout, 1024);
  cudaMalloc(&cyc, 8);
  cudaMemset(din, 0, 1024); cudaMemset(fin, 0, 1024);
  int n = 4096;
  for (int w = 1; w <= 32; w *= 2) {
    chain<<<1, 32 * w>>>(dout, din, n, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent chain, %d warps/SM: %.2f cyc per op\n", w, double(h) / (n * 16));
  }
  chainf<<<1, 32>>>(fout, fin, n, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent chain: %.2f cyc per op\n", double(h) / (n * 16));
  // pointer chase: big (HBM) and small (L2) footprints, random permutation
  for (size_t elems : {size_t(1) << 28, size_t(1) << 20}) {
    uint32_t* hn = new uint32_t[elems];
    for (size_t i = 0; i < elems; ++i) hn[i] = 0;
    uint64_t x = 88172645463325252ull; size_t cur = 0;
    // random cycle over a strided subset (stride 64 elems = 256 B)
    size_t m = elems / 64;
    uint32_t* perm = new uint32_t[m];
    for (size_t i = 0; i < m; ++i) perm[i] = uint32_t(i);
    for (size_t i = m - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; size_t j = x % (i + 1); uint32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t; }
    for (size_t i = 0; i < m; ++i) { hn[cur] = perm[i] * 64; cur = perm[i] * 64; }
    uint32_t* dn; uint32_t* o; cudaMalloc(&dn, elems * 4); cudaMalloc(&o, 4);
    cudaMemcpy(dn, hn, elems * 4, cudaMemcpyHostToDevice);
    int steps = 20000;
    chase<<<1, 1>>>(dn, steps, o, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent load latency, footprint %zu MiB: %.1f cyc\n", elems * 4 >> 20, double(h) / steps);
    cudaFree(dn); cudaFree(o); delete[] hn; delete[] perm;
  }
  return 0;
}
