// Trace-side kernels on sm_100a: comm_cost over a routed trace, and the synthetic routing-trace
// generator.
//
// comm_cost (/root/reference/proj/src/moe.cpp:241-267): sum over tokens, consecutive layer pairs
// and all top_k x top_k slot pairings of [P(f(l,j)) != P(f(l+1,k))].  Per token and layer pair
// this equals k^2 - sum_p c_l(p) c_{l+1}(p) with c_l(p) the number of the token's layer-l slots
// placed on GPU p; the kernel evaluates the k^2 comparisons directly (registers only, no atomics
// until the per-CTA total).
//
// Generator: RoutingModel semantics (moe.cpp:43-153) with a counter-based integer stream so that
// any token range is reproducible and bit-exact against the CPU twin go_generate_trace
// (oracle/gimbal_oracle.c).  Mixture sampling with rejection of already-chosen experts draws
// from the renormalised residual weights, i.e. top_k draws without replacement.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"

namespace gimbal_gpu {

namespace {

template <typename IdT>
__global__ void __launch_bounds__(256)
    comm_cost_kernel(int L, int ne, int K, const IdT* __restrict__ ids, int64_t T,
                     const int32_t* __restrict__ assign, unsigned long long* __restrict__ out,
                     uint32_t* __restrict__ flags) {
  extern __shared__ uint8_t gpu_of[];  // m entries (g <= 255 checked by the host)
  const int m = L * ne;
  for (int i = threadIdx.x; i < m; i += blockDim.x) gpu_of[i] = (uint8_t)assign[i];
  __syncthreads();
  unsigned long long crossings = 0;
  bool bad = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const IdT* row = ids + t * (int64_t)L * K;
    uint8_t cur[32], nxt[32];
    for (int a = 0; a < K; ++a) {
      const uint32_t e = (uint32_t)row[a];
      if (e >= (uint32_t)ne) bad = true;
      cur[a] = gpu_of[min(e, (uint32_t)ne - 1)];
    }
    for (int l = 0; l + 1 < L; ++l) {
      for (int b = 0; b < K; ++b) {
        const uint32_t e = (uint32_t)row[(int64_t)(l + 1) * K + b];
        if (e >= (uint32_t)ne) bad = true;
        nxt[b] = gpu_of[(l + 1) * ne + min(e, (uint32_t)ne - 1)];
      }
      for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) crossings += (cur[a] != nxt[b]);
      for (int b = 0; b < K; ++b) cur[b] = nxt[b];
    }
  }
  if (bad) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) crossings += __shfl_xor_sync(0xffffffffu, crossings, o);
  __shared__ unsigned long long part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = crossings;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
    if (s) atomicAdd(out, s);
  }
}

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ int pick_base(const uint32_t* cdf, int ne, uint32_t u) {
  int lo = 0, hi = ne - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (u < cdf[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// One thread per token; the per-layer base CDFs live in shared memory when they fit.
__global__ void __launch_bounds__(256)
    generate_trace_kernel(int L, int ne, int K, const uint32_t* __restrict__ cdf_g,
                          uint64_t thr_base, uint64_t thr_unif, uint64_t seed, int64_t t0,
                          int64_t T, uint8_t* __restrict__ out, int cdf_in_smem) {
  extern __shared__ uint32_t cdf_s[];
  if (cdf_in_smem) {
    for (int i = threadIdx.x; i < L * ne; i += blockDim.x) cdf_s[i] = cdf_g[i];
    __syncthreads();
  }
  const uint32_t* cdf = cdf_in_smem ? cdf_s : cdf_g;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t tok = (uint64_t)(t0 + t);
    uint64_t ctr = splitmix(seed ^ splitmix(tok));
    uint8_t prev[64], cur[64];
    uint8_t* dst = out + t * (int64_t)L * K;
    for (int l = 0; l < L; ++l) {
      uint64_t chosen[4] = {0, 0, 0, 0};
      for (int a = 0; a < K; ++a) {
        int pick = -1;
        for (int tries = 0; tries < 64 && pick < 0; ++tries) {
          ctr = splitmix(ctr);
          const uint32_t u1 = (uint32_t)(ctr >> 32), u2 = (uint32_t)ctr;
          int e;
          if (l == 0 || u1 < thr_base) e = pick_base(cdf + l * ne, ne, u2);
          else if (u1 < thr_unif) e = (int)(((uint64_t)u2 * (uint64_t)ne) >> 32);
          else e = (prev[((uint64_t)u2 * (uint64_t)K) >> 32] + 1) % ne;
          if (!((chosen[e >> 6] >> (e & 63)) & 1ULL)) pick = e;
        }
        if (pick < 0) {
          pick = 0;
          while ((chosen[pick >> 6] >> (pick & 63)) & 1ULL) ++pick;
        }
        chosen[pick >> 6] |= 1ULL << (pick & 63);
        cur[a] = (uint8_t)pick;
      }
      for (int a = 0; a < K; ++a) {
        dst[l * K + a] = cur[a];
        prev[a] = cur[a];
      }
    }
  }
}

}  // namespace

cudaError_t launch_comm_cost(int L, int ne, int k, const void* ids, int id_bytes, int64_t T,
                             const int32_t* assign, unsigned long long* out, uint32_t* flags,
                             cudaStream_t s) {
  if (T <= 0 || L < 2) return cudaSuccess;
  const size_t smem = (size_t)L * ne;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(8 * 148, (T + 255) / 256));
  if (id_bytes == 1) {
    cudaError_t e = cudaFuncSetAttribute(comm_cost_kernel<uint8_t>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    comm_cost_kernel<uint8_t><<<grid, 256, smem, s>>>(L, ne, k, static_cast<const uint8_t*>(ids), T,
                                                      assign, out, flags);
  } else {
    cudaError_t e = cudaFuncSetAttribute(comm_cost_kernel<int32_t>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    comm_cost_kernel<int32_t><<<grid, 256, smem, s>>>(L, ne, k, static_cast<const int32_t*>(ids), T,
                                                      assign, out, flags);
  }
  return cudaGetLastError();
}

cudaError_t launch_generate_trace(int L, int ne, int k, const uint32_t* cdf, uint64_t thr_base,
                                  uint64_t thr_unif, uint64_t seed, int64_t t0, int64_t T,
                                  uint8_t* out, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const size_t smem = (size_t)L * ne * 4;
  const int in_smem = smem <= 160 * 1024 ? 1 : 0;
  if (in_smem) {
    cudaError_t e = cudaFuncSetAttribute(generate_trace_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(16 * 148, (T + 255) / 256));
  generate_trace_kernel<<<grid, 256, in_smem ? smem : 0, s>>>(L, ne, k, cdf, thr_base, thr_unif,
                                                              seed, t0, T, out, in_smem);
  return cudaGetLastError();
}

}  // namespace gimbal_gpu
