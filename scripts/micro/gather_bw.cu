// Microbenchmark (development tool): throughput of 128-byte row gathers by a
// random index vs. sequential rows, the access pattern of k_var's c2v reads.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int U>
__global__ void gather(const float* __restrict__ src, const int* __restrict__ idx, float* __restrict__ dst, int rows) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long r0 = w0 * U; r0 < rows; r0 += nw * U) {
    float v[U];
    int id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) id[u] = (r0 + u < rows) ? __ldg(&idx[r0 + u]) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (r0 + u < rows) ? __ldcs(&src[static_cast<size_t>(id[u]) * 32 + lane]) : 0.f;
    float acc = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
    if (r0 < rows) dst[(r0 / U) * 32 + lane] = acc;  // 1/U of the rows written (reduction)
  }
}

int main() {
  const int rows = 6'000'000;  // 768 MB
  float *src, *dst;
  int *idx_r, *idx_s;
  cudaMalloc(&src, size_t(rows) * 128);
  cudaMalloc(&dst, size_t(rows) * 128);
  cudaMalloc(&idx_r, size_t(rows) * 4);
  cudaMalloc(&idx_s, size_t(rows) * 4);
  cudaMemset(src, 0, size_t(rows) * 128);
  std::vector<int> h(rows);
  for (int i = 0; i < rows; ++i) h[i] = i;
  cudaMemcpy(idx_s, h.data(), size_t(rows) * 4, cudaMemcpyHostToDevice);
  std::mt19937 rng(1);
  std::shuffle(h.begin(), h.end(), rng);
  cudaMemcpy(idx_r, h.data(), size_t(rows) * 4, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int pass = 0; pass < 2; ++pass) {
    const int* idx = pass ? idx_r : idx_s;
    for (int blocks_per_sm : {4, 8, 16}) {
      const int grid = sms * blocks_per_sm;
      for (int it = 0; it < 2; ++it) gather<8><<<grid, 256>>>(src, idx, dst, rows);
      cudaEventRecord(a);
      const int reps = 10;
      for (int it = 0; it < reps; ++it) gather<8><<<grid, 256>>>(src, idx, dst, rows);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = double(rows) * (128 + 4 + 128.0 / 8);
      printf("%s grid=%d*sms: %.1f GB/s (rows %.1f GB/s)\n", pass ? "random" : "seq   ", blocks_per_sm,
             bytes * reps / ms / 1e6, double(rows) * 128 * reps / ms / 1e6);
    }
  }
  return 0;
}
