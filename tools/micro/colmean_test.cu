#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
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


int main() {
  for (uint32_t n : {2048u, 1000u, 131072u, 300u}) for (uint32_t d : {32u, 128u, 16u}) {
    std::vector<float> h(size_t(n) * d);
    std::mt19937 g(n * 7 + d);
    std::normal_distribution<float> N;
    for (auto& x : h) x = N(g);
    float* dk; double* dm;
    cudaMalloc(&dk, h.size() * 4); cudaMalloc(&dm, d * 8);
    cudaMemcpy(dk, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    k_colmean<<<(d + 31) / 32, 256>>>(dk, n, d, dm);
    printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<double> m(d);
    cudaMemcpy(m.data(), dm, d * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (uint32_t j = 0; j < d; ++j) {
      double acc = 0.0;
      for (uint32_t i = 0; i < n; ++i) acc += (double)h[size_t(i) * d + j];
      if (acc / n != m[j]) { if (bad < 3) printf("n=%u d=%u col %u: %.17g vs %.17g\n", n, d, j, acc / n, m[j]); ++bad; }
    }
    printf("n=%u d=%u bad=%d\n", n, d, bad);
    cudaFree(dk); cudaFree(dm);
  }
}
