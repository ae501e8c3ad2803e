// microbenchmark: dependent-chain latency of warp collectives and smem ops
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out, long long* cyc, int n) {
  __shared__ uint32_t sm[1024];
  __shared__ unsigned long long s64[64];
  const uint32_t lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
  if (lane < 64) s64[lane] = lane;
  __syncwarp();
  uint32_t x = lane, acc = 0;
  long long t0, t1;
  // SHFL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (x + 1) & 31);
  t1 = clock64(); if (lane == 0) cyc[0] = t1 - t0; acc += x;
  // ballot chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __ballot_sync(0xffffffffu, (x >> (lane & 7)) & 1) + lane;
  t1 = clock64(); if (lane == 0) cyc[1] = t1 - t0; acc += x;
  // REDUX chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __reduce_max_sync(0xffffffffu, x + lane) & 1023;
  t1 = clock64(); if (lane == 0) cyc[2] = t1 - t0; acc += x;
  // LDS chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sm[x & 1023];
  t1 = clock64(); if (lane == 0) cyc[3] = t1 - t0; acc += x;
  // IADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 3 + lane;
  t1 = clock64(); if (lane == 0) cyc[4] = t1 - t0; acc += x;
  // u64 compare+select chain
  unsigned long long y = lane, z = 12345;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { y = (y > z) ? y - z : y + (z ^ lane); }
  t1 = clock64(); if (lane == 0) cyc[5] = t1 - t0; acc += uint32_t(y);
  // atomicCAS smem 64 chain (lane 0)
  t0 = clock64();
  if (lane == 0) for (int i = 0; i < n; ++i) y = atomicCAS(&s64[y & 63], y, y + 1) + 1;
  __syncwarp();
  t1 = clock64(); if (lane == 0) cyc[6] = t1 - t0; acc += uint32_t(y);
  // shfl of u64
  y = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = __shfl_sync(0xffffffffu, y, (uint32_t(y) + 1) & 31) + 1;
  t1 = clock64(); if (lane == 0) cyc[7] = t1 - t0; acc += uint32_t(y);
  // match_any chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __match_any_sync(0xffffffffu, x & 3) + lane;
  t1 = clock64(); if (lane == 0) cyc[8] = t1 - t0; acc += x;
  // clock64 back to back
  t0 = clock64();
  long long tt = 0;
  for (int i = 0; i < n; ++i) tt += clock64();
  t1 = clock64(); if (lane == 0) cyc[9] = t1 - t0; acc += uint32_t(tt);
  out[lane] = acc;
}
int main() {
  uint32_t* o; long long* c; long long h[10];
  cudaMalloc(&o, 128); cudaMalloc(&c, 80);
  const int n = 1000;
  k<<<1, 32>>>(o, c, n);
  k<<<1, 32>>>(o, c, n);
  cudaMemcpy(h, c, 80, cudaMemcpyDeviceToHost);
  const char* names[10] = {"SHFL", "BALLOT(+dep)", "REDUX.MAX", "LDS", "IMAD", "u64 cmp+sel", "ATOMS.CAS.64 (1 lane)", "SHFL u64", "MATCH.ANY", "CS2R clock"};
  for (int i = 0; i < 10; ++i) printf("%-24s %.1f cyc/op\n", names[i], double(h[i]) / n);
  return 0;
}
