// Microbenchmark: throughput of the "strike" primitives a GPU sieve can use.
//  (1) atomicAnd on random 32-bit words of a shared-memory bit tile
//  (2) plain byte store of 0 to random bytes of a shared-memory byte tile
//  (3) "lanes-as-primes" byte strike loops (realistic sieve pattern)
//  (4) atomicAnd (RED) on random words of a 32 MB global bitmask
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t xs(uint32_t x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

template <int WORDS>
__global__ void k_smem_atom(int iters, uint32_t* sink) {
  extern __shared__ uint32_t t[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) t[i] = ~0u;
  __syncthreads();
  uint32_t r = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
  for (int k = 0; k < iters; ++k) {
    r = xs(r);
    atomicAnd(&t[r % WORDS], ~(1u << (r >> 27)));
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = t[blockIdx.x % WORDS];
}

template <int BYTES>
__global__ void k_smem_byte(int iters, uint32_t* sink) {
  extern __shared__ uint8_t b[];
  for (int i = threadIdx.x; i < BYTES; i += blockDim.x) b[i] = 1;
  __syncthreads();
  uint32_t r = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
  for (int k = 0; k < iters; ++k) {
    r = xs(r);
    b[r % BYTES] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = b[blockIdx.x % BYTES];
}

// each thread owns primes p = P0 + 2*(tid + k*blockDim) and strikes all multiples in the tile
template <int BYTES>
__global__ void k_smem_byte_sieve(int reps, uint32_t P0, uint32_t* sink, unsigned long long* strikes) {
  extern __shared__ uint8_t b[];
  unsigned long long cnt = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x * 16; i < BYTES; i += blockDim.x * 16) *(uint4*)(b + i) = make_uint4(0x01010101u,0x01010101u,0x01010101u,0x01010101u);
    __syncthreads();
    #pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      uint32_t p = P0 + 2 * (threadIdx.x + k * blockDim.x);
      uint32_t o = (p * 7u + rep) % p;
      #pragma unroll 4
      for (; o < BYTES; o += p) { b[o] = 0; ++cnt; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = b[blockIdx.x % BYTES];
  atomicAdd(strikes, cnt);
}

__global__ void k_global_red(int iters, uint32_t* g, uint32_t words) {
  uint32_t r = 0x9e3779b9u * (threadIdx.x + 1 + blockIdx.x * blockDim.x);
  for (int k = 0; k < iters; ++k) {
    r = xs(r);
    atomicAnd(&g[r % words], ~(1u << (r >> 27)));
  }
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d clock=%d MHz smem/block optin=%zu\n", prop.name, sms, clk_khz/1000, prop.sharedMemPerBlockOptin);
  uint32_t* sink; cudaMalloc(&sink, 1 << 20);
  unsigned long long* dstrikes; cudaMalloc(&dstrikes, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const double ghz = clk_khz / 1e6;
  auto report = [&](const char* name, double ops, float ms) {
    double rate = ops / (ms * 1e-3);
    printf("%-40s %8.3f ms  %10.3e ops/s  %6.2f ops/clk/SM (at %.2f GHz)\n", name, ms, rate, rate / (sms * ghz * 1e9), ghz);
  };
  for (int threads : {256, 512, 1024}) {
    const int W = 32768; // 128 KB tile
    auto k = k_smem_atom<W>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 4);
    int iters = 4096; int grid = sms * 1;
    k<<<grid, threads, W * 4>>>(16, sink);
    cudaEventRecord(e0); k<<<grid, threads, W * 4>>>(iters, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    char nm[64]; snprintf(nm, 64, "smem atomicAnd 128KB thr=%d", threads);
    report(nm, (double)grid * threads * iters, ms);
  }
  for (int threads : {256, 512, 1024}) {
    const int B = 98304;
    auto k = k_smem_byte<B>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, B);
    int iters = 4096; int grid = sms * 2;
    k<<<grid, threads, B>>>(16, sink);
    cudaEventRecord(e0); k<<<grid, threads, B>>>(iters, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    char nm[64]; snprintf(nm, 64, "smem byte store 96KB x2 thr=%d", threads);
    report(nm, (double)grid * threads * iters, ms);
  }
  for (uint32_t P0 : {1025u, 4097u, 16385u}) {
    const int B = 65536;
    auto k = k_smem_byte_sieve<B>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, B);
    int grid = sms * 3, threads = 512, reps = 64;
    cudaMemset(dstrikes, 0, 8);
    k<<<grid, threads, B>>>(2, P0, sink, dstrikes);
    cudaMemset(dstrikes, 0, 8);
    cudaEventRecord(e0); k<<<grid, threads, B>>>(reps, P0, sink, dstrikes); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long st; cudaMemcpy(&st, dstrikes, 8, cudaMemcpyDeviceToHost);
    char nm[64]; snprintf(nm, 64, "byte sieve loop 64KB x3 P0=%u", P0);
    report(nm, (double)st, ms);
  }
  {
    uint32_t words = 8u << 20; // 32 MB
    uint32_t* g; cudaMalloc(&g, words * 4ull); cudaMemset(g, 0xff, words * 4ull);
    int iters = 256, grid = sms * 8, threads = 512;
    k_global_red<<<grid, threads>>>(4, g, words);
    cudaEventRecord(e0); k_global_red<<<grid, threads>>>(iters, g, words); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("global atomicAnd (RED) 32MB", (double)grid * threads * iters, ms);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
