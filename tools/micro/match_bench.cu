// Microbenchmark: warp peer detection for a 6-bit digit -- __match_any_sync vs 6 ballots.
#include <cstdio>
#include <cstdint>
__global__ void k_match(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x], acc = 0;
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = (x >> (i & 7)) & 63u;
    acc += __match_any_sync(0xffffffffu, d);
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_ballot(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x], acc = 0;
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = (x >> (i & 7)) & 63u;
    uint32_t pm = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      pm &= bit ? bal : ~bal;
    }
    acc += pm;
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  const int blocks = 148 * 4, threads = 512, iters = 4096;
  uint32_t *in, *out;
  cudaMalloc(&in, 4 * blocks * threads);
  cudaMalloc(&out, 4 * blocks * threads);
  cudaMemset(in, 7, 4 * blocks * threads);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a);
    k_match<<<blocks, threads>>>(in, out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double warps = (double)blocks * threads / 32 * iters;
    printf("match_any: %.3f ms, %.2f G warp-ops/s\n", ms, warps / ms / 1e6);
    cudaEventRecord(a);
    k_ballot<<<blocks, threads>>>(in, out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("6 ballots: %.3f ms, %.2f G warp-ops/s\n", ms, warps / ms / 1e6);
  }
  return 0;
}
