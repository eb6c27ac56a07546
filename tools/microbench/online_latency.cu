// Per-call latency of gimbal_online_iteration from C (no Python), next to the floors it sits on:
// an empty kernel launched and waited for with cudaStreamSynchronize, and an empty kernel that
// stores a sequence number into mapped pinned memory which the host polls.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include tools/microbench/online_latency.cu \
//        -o tools/microbench/online_latency -L paper_2602_21626_b200/lib -lgimbal_gpu -Xlinker -rpath=$PWD/paper_2602_21626_b200/lib
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "gimbal_gpu.h"

__global__ void empty_kernel() {}
__global__ void seq_kernel(volatile unsigned long long* out, unsigned long long s) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    *out = s;
  }
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 2000;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int i = 0; i < 100; ++i) empty_kernel<<<1, 32, 0, s>>>();
  cudaStreamSynchronize(s);
  double t0 = now_us();
  for (int i = 0; i < iters; ++i) {
    empty_kernel<<<1, 32, 0, s>>>();
    cudaStreamSynchronize(s);
  }
  printf("{\"what\": \"empty kernel + cudaStreamSynchronize\", \"us\": %.2f}\n", (now_us() - t0) / iters);
  unsigned long long* h = nullptr;
  unsigned long long* d = nullptr;
  cudaHostAlloc(&h, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&d, h, 0);
  *h = 0;
  t0 = now_us();
  for (int i = 1; i <= iters; ++i) {
    seq_kernel<<<1, 32, 0, s>>>(d, (unsigned long long)i);
    while (*(volatile unsigned long long*)h != (unsigned long long)i) {
    }
  }
  printf("{\"what\": \"kernel storing a sequence number to pinned memory, host poll\", \"us\": %.2f}\n",
         (now_us() - t0) / iters);
  cudaStreamSynchronize(s);

  struct Shape {
    const char* name;
    int L, ne, k, g;
  } shapes[] = {{"sim-test", 6, 16, 4, 4}, {"mixtral", 32, 8, 2, 8}, {"dsv2lite", 26, 64, 6, 8}, {"dsv3", 58, 256, 8, 8}};
  std::mt19937 rng(1);
  for (const Shape& sh : shapes) {
    for (int n : {64, 4096}) {
      gimbal_topology topo{sh.L, sh.ne, sh.k, sh.g};
      gimbal_stats_t w;
      gimbal_online_t o;
      if (gimbal_stats_create(&topo, 0, &w) || gimbal_online_create(w, &o)) {
        printf("create failed: %s\n", gimbal_last_error());
        return 1;
      }
      const int64_t m = (int64_t)sh.L * sh.ne;
      std::vector<int32_t> assign((size_t)m);
      for (int64_t f = 0; f < m; ++f) assign[(size_t)f] = (int32_t)((f % sh.ne) / (sh.ne / sh.g));
      gimbal_online_set_placement(o, assign.data(), m);
      std::vector<uint8_t> ids((size_t)n * sh.L * sh.k);
      for (int t = 0; t < n * sh.L; ++t)  // k distinct ids per token-layer
        for (int a = 0; a < sh.k; ++a) ids[(size_t)t * sh.k + a] = (uint8_t)((rng() % (sh.ne / sh.k)) * sh.k + a);
      double ex;
      int64_t cr;
      for (int i = 0; i < 20; ++i) gimbal_online_iteration(o, ids.data(), 1, n, &ex, &cr);
      t0 = now_us();
      for (int i = 0; i < iters; ++i)
        if (gimbal_online_iteration(o, ids.data(), 1, n, &ex, &cr)) {
          printf("iteration failed: %s\n", gimbal_last_error());
          return 1;
        }
      printf("{\"what\": \"gimbal_online_iteration\", \"shape\": \"%s\", \"tokens\": %d, \"us\": %.2f}\n", sh.name, n,
             (now_us() - t0) / iters);
      std::vector<int32_t> ids32(ids.begin(), ids.end());  // RoutedStream::choices as the engine passes them
      t0 = now_us();
      for (int i = 0; i < iters; ++i)
        if (gimbal_online_iteration(o, ids32.data(), 4, n, &ex, &cr)) {
          printf("iteration failed: %s\n", gimbal_last_error());
          return 1;
        }
      printf("{\"what\": \"gimbal_online_iteration, int32 ids\", \"shape\": \"%s\", \"tokens\": %d, \"us\": %.2f}\n",
             sh.name, n, (now_us() - t0) / iters);
      gimbal_online_destroy(o);
      gimbal_stats_destroy(w);
    }
  }
  return 0;
}
