// Microbenchmark: global RED.AND throughput on random words of a bitmask of
// R bytes (the large-prime strikes of k_large_strike land like this), and the
// same with a few ALU instructions of address work per RED.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t xs(uint32_t x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

__global__ void k_red(uint32_t* m, uint32_t words, int iters, int sorted) {
  uint32_t r = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int k = 0; k < iters; ++k) {
    r = xs(r);
    uint32_t w = sorted ? ((blockIdx.x * 977u + k * 131u) * 32u + (threadIdx.x & 31)) % words : r % words;
    atomicAnd(m + w, ~(1u << (r >> 27)));
  }
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const size_t maxb = 256ull << 20;
  uint32_t* m;
  cudaMalloc(&m, maxb);
  cudaMemset(m, 0xFF, maxb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t sizes[] = {4ull << 20, 16ull << 20, 33ull << 20, 67ull << 20, 100ull << 20, 134ull << 20, 200ull << 20};
  for (int sorted = 0; sorted < 2; ++sorted)
    for (size_t R : sizes) {
      const uint32_t words = (uint32_t)(R / 4);
      const int grid = sms * 8, thr = 256, iters = 512;
      k_red<<<grid, thr>>>(m, words, 16, sorted);
      cudaEventRecord(a);
      k_red<<<grid, thr>>>(m, words, iters, sorted);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)grid * thr * iters;
      printf("%s R=%4zu MB  %7.3f ms  %.3e RED/s  %.3f RED/clk/SM (max clock %.2f GHz)\n",
             sorted ? "coalesced" : "random   ", R >> 20, ms, ops / ms * 1e3, ops / (ms * 1e-3) / (sms * clk * 1e3), clk / 1e6);
    }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
