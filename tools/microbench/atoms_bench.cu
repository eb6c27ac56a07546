// Microbenchmark: shared-memory atomic (ATOMS / RED.S) throughput on B200.
// Measures updates/s for random-address u32 increments into a privatised table,
// the primitive the A/E builders are bound by. Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int TABLE_WORDS, int MODE>
__global__ void __launch_bounds__(1024, 1) k_atoms(int iters, uint32_t* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < TABLE_WORDS; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t base = s;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      uint32_t a;
      if (MODE == 0) a = (base >> (u & 7)) ^ (u * 0x9e37u);                 // random
      else if (MODE == 1) a = threadIdx.x + u * 1024u;                       // conflict-free
      else a = ((base >> 5) & 0x3f) * 64 + u;                                // skewed rows
      atomicAdd(&tab[a & (TABLE_WORDS - 1)], 1u);
    }
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < TABLE_WORDS; i += blockDim.x) acc += tab[i];
  atomicAdd(out, acc);
}

template <int TW, int MODE>
void run(const char* name, int blocks, int threads) {
  uint32_t* d; cudaMalloc(&d, 4);
  auto kern = k_atoms<TW, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TW * 4);
  int iters = 2000;
  kern<<<blocks, threads, TW * 4>>>(10, d);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, threads, TW * 4>>>(iters, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ups = double(blocks) * threads * iters * 16 / (ms * 1e-3);
  printf("%-28s blocks=%d threads=%d table=%dKB  %.3f ms  %.3f T updates/s  err=%s\n", name, blocks,
         threads, TW * 4 / 1024, ms, ups / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<32768, 0>("random 128KB", sms, 1024);
  run<32768, 1>("conflict-free 128KB", sms, 1024);
  run<32768, 2>("skewed 128KB", sms, 1024);
  run<16384, 0>("random 64KB x2/SM", 2 * sms, 1024);
  run<8192, 0>("random 32KB x4/SM", 4 * sms, 512);
  run<1024, 0>("random 4KB", 8 * sms, 256);
  return 0;
}
