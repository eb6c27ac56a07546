// Transition counting for small expert counts (Mixtral class: 8 experts, top-2) straight from the
// token-major uint8 trace: the whole E tensor ((L-1) x n_e x n_e u32, 7.9 KB at 32 layers x 8
// experts) lives in every CTA's shared memory, so one pass over the trace counts every layer pair
// with no transposition kernel and no per-pair units (moe.cpp:169-191: each of the k x k slot
// pairings of every layer pair is one increment, multiplicity included).
//
// Each CTA stages a block of token rows (L * k bytes each) with 16-byte coalesced loads into a
// padded shared buffer (row stride = row bytes + 4, so the per-thread reads of its own row are
// bank-conflict free), then every thread walks its token's layers and issues the k^2 increments
// per pair as shared atomics.  Ids are range-checked per token-layer (an out-of-range id flags
// the call and leaves that token-layer's pairings out).  At the end the CTA adds its non-zero
// cells to the u64 E with global atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kSmallThreads = 256;
constexpr int kSmallMaxTable = 48 * 1024;  // bytes of u32 cells per CTA (several CTAs per SM)

template <int K>
__global__ void __launch_bounds__(kSmallThreads)
    count_small_tm_kernel(int L, int ne, const uint8_t* __restrict__ trace, int64_t T, int row_bytes,
                          int stride, unsigned long long* __restrict__ E, uint32_t* __restrict__ flags) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int cells = (L - 1) * ne * ne;
  uint32_t* tab = reinterpret_cast<uint32_t*>(sm);
  uint8_t* rows = sm + ((cells * 4 + 15) & ~15);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) tab[i] = 0u;
  bool bad = false;
  const bool vec = (row_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(trace) & 15) == 0;
  for (int64_t t0 = (int64_t)blockIdx.x * kSmallThreads; t0 < T; t0 += (int64_t)gridDim.x * kSmallThreads) {
    const int n = (int)min((int64_t)kSmallThreads, T - t0);
    __syncthreads();  // the previous block's rows are consumed (and the table is zeroed)
    const uint8_t* src = trace + t0 * row_bytes;
    if (vec) {
      const int q = row_bytes >> 4;  // 16-byte words per row
      for (int i = threadIdx.x; i < n * q; i += blockDim.x) {
        const int r = i / q, w = i - r * q;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + i);
        uint32_t* d = reinterpret_cast<uint32_t*>(rows + r * stride + w * 16);
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
      }
    } else {
      for (int i = threadIdx.x; i < n * row_bytes; i += blockDim.x) {
        const int r = i / row_bytes;
        rows[r * stride + (i - r * row_bytes)] = __ldg(src + i);
      }
    }
    __syncthreads();
    if (threadIdx.x < n) {
      const uint8_t* row = rows + threadIdx.x * stride;
      uint32_t cur[K];
      bool ok_cur = true;
#pragma unroll
      for (int a = 0; a < K; ++a) {
        cur[a] = row[a];
        ok_cur &= cur[a] < (uint32_t)ne;
      }
      bad |= !ok_cur;
      for (int l = 0; l + 1 < L; ++l) {
        uint32_t nxt[K];
        bool ok_nxt = true;
#pragma unroll
        for (int b = 0; b < K; ++b) {
          nxt[b] = row[(l + 1) * K + b];
          ok_nxt &= nxt[b] < (uint32_t)ne;
        }
        bad |= !ok_nxt;
        if (ok_cur && ok_nxt) {
          uint32_t* El = tab + l * ne * ne;
#pragma unroll
          for (int a = 0; a < K; ++a)
#pragma unroll
            for (int b = 0; b < K; ++b) atomicAdd(El + cur[a] * ne + nxt[b], 1u);
        }
#pragma unroll
        for (int b = 0; b < K; ++b) cur[b] = nxt[b];
        ok_cur = ok_nxt;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cells; i += blockDim.x)
    if (tab[i]) atomicAdd(E + i, (unsigned long long)tab[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
}

size_t small_smem(int L, int ne, int k) {
  const size_t table = ((size_t)(L - 1) * ne * ne * 4 + 15) & ~(size_t)15;
  return table + (size_t)kSmallThreads * ((size_t)L * k + 4);
}

}  // namespace

bool small_count_supported(int L, int ne, int k, int id_bytes, int64_t T) {
  if (id_bytes != 1 || L < 2 || k < 1 || k > 8 || ne > 256) return false;
  if ((size_t)(L - 1) * ne * ne * 4 > (size_t)kSmallMaxTable) return false;
  if (small_smem(L, ne, k) > 96 * 1024) return false;
  // every CTA's u32 cells stay exact: at most tokens-per-CTA x k^2 increments each
  return T < ((int64_t)1 << 40);
}

cudaError_t launch_count_small(int L, int ne, int k, int sms, const uint8_t* trace, int64_t T,
                               unsigned long long* E, uint32_t* flags, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const size_t smem = small_smem(L, ne, k);
  const int per_sm = std::max(1, std::min(8, (int)((200 * 1024) / smem)));
  int64_t grid = std::min<int64_t>((int64_t)per_sm * sms, (T + kSmallThreads - 1) / kSmallThreads);
  // u32 cells: tokens per CTA x k^2 < 2^32
  const int64_t min_grid = T * k * k / ((int64_t)1 << 31) + 1;
  grid = std::max<int64_t>(grid, std::min<int64_t>(min_grid, (T + kSmallThreads - 1) / kSmallThreads));
  const int row_bytes = L * k;
  const int stride = row_bytes + 4;
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, kSmallThreads, smem, s>>>(L, ne, trace, T, row_bytes, stride, E, flags);
    return cudaGetLastError();
  };
  switch (k) {
    case 1: return go(count_small_tm_kernel<1>);
    case 2: return go(count_small_tm_kernel<2>);
    case 3: return go(count_small_tm_kernel<3>);
    case 4: return go(count_small_tm_kernel<4>);
    case 5: return go(count_small_tm_kernel<5>);
    case 6: return go(count_small_tm_kernel<6>);
    case 7: return go(count_small_tm_kernel<7>);
    case 8: return go(count_small_tm_kernel<8>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gimbal_gpu
