// Microbenchmark: alternative E-counting resources on B200 (round 2).  Not product code.
//  1. legacy warp-level tensor MMAs (mma.sync): b1 AND+POPC m16n8k256, s4 m16n8k64, s8 m16n8k32
//     -- the binary form would count transitions from bit-packed multi-hot tiles;
//  2. L2 reductions (RED.E.ADD u32) at random addresses in an L2-resident 16 MB table;
//  3. shared-memory atomics with a share of the warps issuing L2 reductions (do the two add up?).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// MODE 0 = b1 and.popc m16n8k256, 1 = s4 m16n8k64, 2 = s8 m16n8k32; NACC independent accumulators
template <int MODE, int NACC>
__global__ void k_mma(int iters, int* out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = hash32(threadIdx.x * 7 + i);
  for (int i = 0; i < 2; ++i) b[i] = hash32(threadIdx.x * 13 + i + 100);
  int c[NACC][4];
  for (int n = 0; n < NACC; ++n)
    for (int i = 0; i < 4; ++i) c[n][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n) {
      if (MODE == 0)
        asm volatile(
            "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(c[n][0]), "+r"(c[n][1]), "+r"(c[n][2]), "+r"(c[n][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else if (MODE == 1)
        asm volatile(
            "mma.sync.aligned.m16n8k64.row.col.s32.s4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(c[n][0]), "+r"(c[n][1]), "+r"(c[n][2]), "+r"(c[n][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(c[n][0]), "+r"(c[n][1]), "+r"(c[n][2]), "+r"(c[n][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  int s = 0;
  for (int n = 0; n < NACC; ++n)
    for (int i = 0; i < 4; ++i) s += c[n][i];
  if (s == 0x7fffffff) *out = s;
}

template <int MODE, int NACC>
void run_mma(const char* name, int blocks, int threads) {
  int* d;
  cudaMalloc(&d, 4);
  const int iters = 4000;
  k_mma<MODE, NACC><<<blocks, threads>>>(10, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mma<MODE, NACC><<<blocks, threads>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double macs_per = MODE == 0 ? 16.0 * 8 * 256 : MODE == 1 ? 16.0 * 8 * 64 : 16.0 * 8 * 32;
  const double n_mma = double(blocks) * (threads / 32) * iters * NACC;
  printf("%-34s blocks=%d threads=%d acc=%d %.3f ms  %.1f T MAC/s  (%.0f MAC/clk/SM at 1.965 GHz)  err=%s\n", name,
         blocks, threads, NACC, ms, n_mma * macs_per / (ms * 1e-3) / 1e12,
         n_mma * macs_per / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

// global reductions into a TABLE-word u32 table (L2 resident), random addresses
__global__ void k_red(int iters, uint32_t* tab, uint32_t mask) {
  uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint32_t a = hash32(s + u) & mask;
      asm volatile("red.global.add.u32 [%0], 1;" ::"l"(tab + a) : "memory");
    }
  }
}

// shared random atomics in all warps except the last GW warps of each CTA, which issue global
// reductions; reports both rates
__global__ void __launch_bounds__(1024, 1) k_mixed(int iters, int gw, uint32_t* gtab, uint32_t gmask, uint32_t* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const bool glob = warp >= 32 - gw;
  uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t base = s;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      uint32_t a = (base >> (u & 7)) ^ (u * 0x9e37u);
      if (glob) {
        asm volatile("red.global.add.u32 [%0], 1;" ::"l"(gtab + (hash32(a + it) & gmask)) : "memory");
      } else {
        atomicAdd(&tab[a & 32767], 1u);
      }
    }
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) acc += tab[i];
  atomicAdd(out, acc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_mma<0, 4>("b1 and.popc m16n8k256", sms, 512);
  run_mma<0, 8>("b1 and.popc m16n8k256", sms, 1024);
  run_mma<0, 8>("b1 and.popc m16n8k256 x2/SM", 2 * sms, 512);
  run_mma<1, 8>("s4 m16n8k64", sms, 1024);
  run_mma<2, 8>("s8 m16n8k32", sms, 1024);

  const uint32_t words = 1u << 22;  // 16 MB
  uint32_t* gt;
  cudaMalloc(&gt, words * 4);
  cudaMemset(gt, 0, words * 4);
  uint32_t* d;
  cudaMalloc(&d, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int tpb : {256, 1024}) {
    const int blocks = sms * (2048 / tpb), iters = 400;
    k_red<<<blocks, tpb>>>(4, gt, words - 1);
    cudaEventRecord(e0);
    k_red<<<blocks, tpb>>>(iters, gt, words - 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("red.global.add.u32 random 16MB      blocks=%d threads=%d %.3f ms  %.3f T updates/s  err=%s\n", blocks, tpb, ms,
           double(blocks) * tpb * iters * 16 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
  for (int gw : {0, 2, 4, 8}) {
    const int iters = 2000;
    k_mixed<<<sms, 1024, 32768 * 4>>>(10, gw, gt, words - 1, d);
    cudaEventRecord(e0);
    k_mixed<<<sms, 1024, 32768 * 4>>>(iters, gw, gt, words - 1, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tot = double(sms) * 1024 * iters * 16;
    printf("mixed: %2d of 32 warps on L2         %.3f ms  total %.3f T updates/s (shared %.3f + L2 %.3f)  err=%s\n", gw,
           ms, tot / (ms * 1e-3) / 1e12, tot * (32 - gw) / 32 / (ms * 1e-3) / 1e12, tot * gw / 32 / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
