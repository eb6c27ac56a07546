// Routing-trace statistics on sm_100a: the layer-pair transition tensor E (and from it the
// activation histogram A and the aggregate W).
//
// Reference semantics (/root/reference/proj/src/moe.cpp):
//   add_token   :169-191  A(l,e) += 1 per id; E_l(j,k) += 1 for every (j in slots_l,
//                         k in slots_{l+1}) pairing, with multiplicity
//   affinity    :199-205  W = sum_l E_l
//   flat forms  :207-231
//
// Design:
//  * Only E is counted.  A is derived exactly: every token has exactly top_k ids in layer l+1,
//    so sum_k E_l(j,k) = top_k * A_l(j) for l < L-1 and sum_j E_{L-2}(j,k) = top_k * A_{L-1}(k).
//    (L == 1 has no pairs; A is counted directly.)
//  * Counting is privatised in shared memory as u32 counters: one CTA work unit owns
//    `pairs_per_group` consecutive layer pairs x `rows_per_part` rows j of E (<= ~200 KB), scans a
//    contiguous token chunk of the trace and increments with shared atomics (ATOMS.POPC.INC,
//    which aggregates equal addresses within a warp), then flushes non-zero counters once to
//    the u64 tensor in HBM with one global atomic each.  The binding resource is the shared
//    atomic unit (one bank wavefront per cycle per SM; profiles/ATOMS_microbench.md), not HBM.
//  * Work units are ordered chunk-major, so the CTAs working on different layer pairs of the
//    same token chunk read the same trace rows while they are resident in the 126 MB L2.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"

namespace gimbal_gpu {

namespace {

struct CountParams {
  int L, ne, k;
  int P, R;            // pairs per group, rows per part
  uint32_t swz;        // column XOR swizzle mask (row j stores column k at k ^ (j & swz))
  int n_groups, n_parts;
  int64_t n_units;
  int64_t chunk_tokens;
  int64_t T;
};

// Loads the K ids of one layer of one token as unsigned values, with the widest aligned vector
// access the layout allows (the trace is token-major, L*K ids per token).
template <typename IdT, int K>
__device__ __forceinline__ void load_layer(const IdT* __restrict__ p, uint32_t (&out)[K]) {
  constexpr int BYTES = K * (int)sizeof(IdT);
  if constexpr (sizeof(IdT) == 1 && BYTES % 8 == 0) {
#pragma unroll
    for (int v = 0; v < BYTES / 8; ++v) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(p) + v);
#pragma unroll
      for (int b = 0; b < 4; ++b) out[v * 8 + b] = (w.x >> (8 * b)) & 0xffu;
#pragma unroll
      for (int b = 0; b < 4; ++b) out[v * 8 + 4 + b] = (w.y >> (8 * b)) & 0xffu;
    }
  } else if constexpr (sizeof(IdT) == 1 && BYTES % 4 == 0) {
#pragma unroll
    for (int v = 0; v < BYTES / 4; ++v) {
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(p) + v);
#pragma unroll
      for (int b = 0; b < 4; ++b) out[v * 4 + b] = (w >> (8 * b)) & 0xffu;
    }
  } else if constexpr (sizeof(IdT) == 1 && BYTES % 2 == 0) {
#pragma unroll
    for (int v = 0; v < BYTES / 2; ++v) {
      const uint32_t w = __ldg(reinterpret_cast<const uint16_t*>(p) + v);
      out[v * 2] = w & 0xffu;
      out[v * 2 + 1] = (w >> 8) & 0xffu;
    }
  } else {
#pragma unroll
    for (int b = 0; b < K; ++b) out[b] = static_cast<uint32_t>(__ldg(p + b));
  }
}

template <typename IdT, int K>
__global__ void __launch_bounds__(1024, 1)
    count_pairs_kernel(CountParams prm, const IdT* __restrict__ ids,
                       unsigned long long* __restrict__ E, uint32_t* __restrict__ flags) {
  extern __shared__ uint32_t cnt[];
  const int ne = prm.ne;
  const int64_t stride = (int64_t)prm.L * K;
  const int units_per_chunk = prm.n_groups * prm.n_parts;
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int64_t chunk = unit / units_per_chunk;
    const int rem = (int)(unit % units_per_chunk);
    const int group = rem / prm.n_parts;
    const int part = rem % prm.n_parts;
    const int l0 = group * prm.P;
    const int l1 = min(l0 + prm.P, prm.L - 1);
    const int j0 = part * prm.R;
    const int jR = min(prm.R, ne - j0);
    const int words = (l1 - l0) * prm.R * ne;
    for (int w = threadIdx.x; w < words; w += blockDim.x) cnt[w] = 0u;
    __syncthreads();

    const int64_t t_begin = chunk * prm.chunk_tokens;
    const int64_t t_end = min(prm.T, t_begin + prm.chunk_tokens);
    bool bad = false;
    for (int64_t t = t_begin + threadIdx.x; t < t_end; t += blockDim.x) {
      const IdT* row = ids + t * stride;
      uint32_t cur[K], nxt[K];
      load_layer<IdT, K>(row + (int64_t)l0 * K, cur);
      uint32_t chk = 0;
#pragma unroll
      for (int a = 0; a < K; ++a) chk |= (cur[a] >= (uint32_t)ne);
      if (chk) {
        bad = true;
        continue;
      }
      for (int l = l0; l < l1; ++l) {
        load_layer<IdT, K>(row + (int64_t)(l + 1) * K, nxt);
        uint32_t c2 = 0;
#pragma unroll
        for (int b = 0; b < K; ++b) c2 |= (nxt[b] >= (uint32_t)ne);
        if (c2) {
          bad = true;
          break;
        }
        uint32_t* blk = cnt + (l - l0) * prm.R * ne;
#pragma unroll
        for (int a = 0; a < K; ++a) {
          const uint32_t j = cur[a] - (uint32_t)j0;
          if (j < (uint32_t)jR) {
            uint32_t* rowp = blk + j * ne;
            const uint32_t sw = j & prm.swz;
#pragma unroll
            for (int b = 0; b < K; ++b) atomicAdd(rowp + (nxt[b] ^ sw), 1u);
          }
        }
#pragma unroll
        for (int a = 0; a < K; ++a) cur[a] = nxt[a];
      }
    }
    if (bad) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
    __syncthreads();
    const int rows_ne = prm.R * ne;
    for (int w = threadIdx.x; w < words; w += blockDim.x) {
      const uint32_t v = cnt[w];
      if (v == 0u) continue;
      const int pr = w / rows_ne;
      const int r = w - pr * rows_ne;
      const int j = r / ne;
      const int kk = (r - j * ne) ^ (j & prm.swz);
      atomicAdd(E + ((int64_t)(l0 + pr) * ne + (j0 + j)) * ne + kk, (unsigned long long)v);
    }
    __syncthreads();
  }
}

// Generic top_k (runtime k <= 32) fallback with byte/word loads.
template <typename IdT>
__global__ void __launch_bounds__(1024, 1)
    count_pairs_generic_kernel(CountParams prm, const IdT* __restrict__ ids,
                               unsigned long long* __restrict__ E, uint32_t* __restrict__ flags) {
  extern __shared__ uint32_t cnt[];
  const int ne = prm.ne, K = prm.k;
  const int64_t stride = (int64_t)prm.L * K;
  const int units_per_chunk = prm.n_groups * prm.n_parts;
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int64_t chunk = unit / units_per_chunk;
    const int rem = (int)(unit % units_per_chunk);
    const int group = rem / prm.n_parts;
    const int part = rem % prm.n_parts;
    const int l0 = group * prm.P;
    const int l1 = min(l0 + prm.P, prm.L - 1);
    const int j0 = part * prm.R;
    const int jR = min(prm.R, ne - j0);
    const int words = (l1 - l0) * prm.R * ne;
    for (int w = threadIdx.x; w < words; w += blockDim.x) cnt[w] = 0u;
    __syncthreads();
    const int64_t t_begin = chunk * prm.chunk_tokens;
    const int64_t t_end = min(prm.T, t_begin + prm.chunk_tokens);
    bool bad = false;
    for (int64_t t = t_begin + threadIdx.x; t < t_end; t += blockDim.x) {
      const IdT* row = ids + t * stride;
      bool tok_bad = false;
      for (int l = l0; l <= l1 && !tok_bad; ++l)
        for (int a = 0; a < K; ++a)
          if ((uint32_t)row[(int64_t)l * K + a] >= (uint32_t)ne) tok_bad = true;
      if (tok_bad) {
        bad = true;
        continue;
      }
      for (int l = l0; l < l1; ++l) {
        uint32_t* blk = cnt + (l - l0) * prm.R * ne;
        for (int a = 0; a < K; ++a) {
          const uint32_t j = (uint32_t)row[(int64_t)l * K + a] - (uint32_t)j0;
          if (j >= (uint32_t)jR) continue;
          for (int b = 0; b < K; ++b)
            atomicAdd(blk + j * ne + ((uint32_t)row[(int64_t)(l + 1) * K + b] ^ (j & prm.swz)), 1u);
        }
      }
    }
    if (bad) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
    __syncthreads();
    const int rows_ne = prm.R * ne;
    for (int w = threadIdx.x; w < words; w += blockDim.x) {
      const uint32_t v = cnt[w];
      if (v == 0u) continue;
      const int pr = w / rows_ne;
      const int r = w - pr * rows_ne;
      const int j = r / ne;
      const int kk = (r - j * ne) ^ (j & prm.swz);
      atomicAdd(E + ((int64_t)(l0 + pr) * ne + (j0 + j)) * ne + kk, (unsigned long long)v);
    }
    __syncthreads();
  }
}

// L == 1: no layer pairs, count A directly (moe.cpp:176-178).
template <typename IdT>
__global__ void count_activation_kernel(int L, int ne, int K, const IdT* __restrict__ ids,
                                        int64_t T, unsigned long long* __restrict__ A,
                                        uint32_t* __restrict__ flags) {
  extern __shared__ uint32_t hist[];
  const int cells = L * ne;
  for (int i = threadIdx.x; i < cells; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t n = T * L * K;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = (uint32_t)ids[i];
    const int l = (int)((i / K) % L);
    if (e >= (uint32_t)ne) {
      bad = true;
      continue;
    }
    atomicAdd(&hist[l * ne + e], 1u);
  }
  if (bad) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
  __syncthreads();
  for (int i = threadIdx.x; i < cells; i += blockDim.x)
    if (hist[i]) atomicAdd(&A[i], (unsigned long long)hist[i]);
}

// A_l(j) = sum_k E_l(j,k) / k  (l < L-1), one warp per row; A_{L-1}(k) = sum_j E_{L-2}(j,k) / k.
__global__ void derive_activation_kernel(int L, int ne, int K, const unsigned long long* __restrict__ E,
                                         unsigned long long* __restrict__ A) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int rows = (L - 1) * ne;
  if (warp < rows) {
    const unsigned long long* r = E + (int64_t)warp * ne;
    unsigned long long s = 0;
    for (int k = lane; k < ne; k += 32) s += r[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) A[warp] = s / (unsigned long long)K;
  } else if (warp < rows + (ne + 31) / 32) {
    const int k = (warp - rows) * 32 + lane;
    if (k < ne) {
      const unsigned long long* blk = E + (int64_t)(L - 2) * ne * ne;
      unsigned long long s = 0;
      for (int j = 0; j < ne; ++j) s += blk[(int64_t)j * ne + k];
      A[(int64_t)(L - 1) * ne + k] = s / (unsigned long long)K;
    }
  }
}

__global__ void derive_w_kernel(int L, int ne, const unsigned long long* __restrict__ E,
                                unsigned long long* __restrict__ W) {
  const int64_t cells = (int64_t)ne * ne;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long s = 0;
    for (int l = 0; l + 1 < L; ++l) s += E[(int64_t)l * cells + i];
    W[i] = s;
  }
}

// flat_activation (moe.cpp:207-215) and flat_pair_weights (moe.cpp:217-231) as doubles; the
// outputs are pre-zeroed by the caller.
__global__ void flat_forms_kernel(int L, int ne, const unsigned long long* __restrict__ A,
                                  const unsigned long long* __restrict__ E, double* flatA,
                                  double* flatW) {
  const int64_t m = (int64_t)L * ne;
  const int64_t nE = (int64_t)(L - 1) * ne * ne;
  const int64_t n = (flatA ? m : 0) + (flatW ? nE : 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flatA && i < m) {
      const int64_t l = i / ne;
      flatA[l * m + i] = (double)A[i];
    } else {
      const int64_t c = flatA ? i - m : i;
      const int64_t l = c / ((int64_t)ne * ne);
      const int64_t r = c - l * ne * ne;
      const int64_t j = r / ne, kk = r - j * ne;
      const unsigned long long v = E[c];
      if (v) flatW[(l * ne + j) * m + (l + 1) * ne + kk] = (double)v;
    }
  }
}

template <typename IdT, int K>
cudaError_t launch_k(const StatsPlan& plan, const CountParams& prm, const IdT* ids,
                     unsigned long long* E, uint32_t* flags, cudaStream_t s, int grid) {
  auto kern = count_pairs_kernel<IdT, K>;
  const size_t smem = (size_t)plan.smem_words * 4;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, plan.threads, smem, s>>>(prm, ids, E, flags);
  return cudaGetLastError();
}

template <typename IdT>
cudaError_t dispatch_k(const StatsPlan& plan, const CountParams& prm, const void* ids,
                       unsigned long long* E, uint32_t* flags, cudaStream_t s, int grid) {
  const IdT* p = static_cast<const IdT*>(ids);
  const uintptr_t addr = reinterpret_cast<uintptr_t>(ids);
  const int bytes = plan.k * (int)sizeof(IdT);
  const int vec = (bytes % 8 == 0) ? 8 : (bytes % 4 == 0) ? 4 : (bytes % 2 == 0) ? 2 : 1;
  const bool aligned = (addr % (uintptr_t)vec) == 0;
  if (aligned) {
    switch (plan.k) {
      case 1: return launch_k<IdT, 1>(plan, prm, p, E, flags, s, grid);
      case 2: return launch_k<IdT, 2>(plan, prm, p, E, flags, s, grid);
      case 4: return launch_k<IdT, 4>(plan, prm, p, E, flags, s, grid);
      case 6: return launch_k<IdT, 6>(plan, prm, p, E, flags, s, grid);
      case 8: return launch_k<IdT, 8>(plan, prm, p, E, flags, s, grid);
      default: break;
    }
  }
  auto kern = count_pairs_generic_kernel<IdT>;
  const size_t smem = (size_t)plan.smem_words * 4;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, plan.threads, smem, s>>>(prm, p, E, flags);
  return cudaGetLastError();
}

}  // namespace

StatsPlan make_stats_plan(int L, int ne, int k, int sms, int max_smem_optin) {
  StatsPlan p;
  p.L = L;
  p.ne = ne;
  p.k = k;
  p.sms = sms;
  const int pairs = std::max(L - 1, 0);
  // Shared-memory budget per CTA: one 1024-thread CTA per SM, leaving room for the runtime.
  const int budget_words = std::max(1024, (std::min(max_smem_optin, 200 * 1024)) / 4);
  const int pair_words = ne * ne;
  if (pairs == 0) {
    p.n_groups = 0;
    p.n_parts = 0;
    p.rows_per_part = ne;
    p.smem_words = 0;
    return p;
  }
  if (pair_words <= budget_words) {
    p.rows_per_part = ne;
    p.n_parts = 1;
    p.pairs_per_group = std::max(1, std::min(pairs, budget_words / pair_words));
    // balance the groups so the last one is not nearly empty
    const int ng = (pairs + p.pairs_per_group - 1) / p.pairs_per_group;
    p.pairs_per_group = (pairs + ng - 1) / ng;
  } else {
    p.pairs_per_group = 1;
    const int max_rows = std::max(1, budget_words / ne);
    const int parts = (ne + max_rows - 1) / max_rows;
    p.rows_per_part = (ne + parts - 1) / parts;
    p.n_parts = parts;
  }
  p.n_groups = (pairs + p.pairs_per_group - 1) / p.pairs_per_group;
  p.smem_words = p.pairs_per_group * p.rows_per_part * ne;
  p.threads = 1024;
  p.ctas_per_sm = 1;
  return p;
}

cudaError_t launch_count_pairs(const StatsPlan& plan, const void* ids, int id_bytes, int64_t T,
                               unsigned long long* E, uint32_t* flags, cudaStream_t s) {
  if (T <= 0 || plan.n_groups == 0) return cudaSuccess;
  CountParams prm;
  prm.L = plan.L;
  prm.ne = plan.ne;
  prm.k = plan.k;
  prm.P = plan.pairs_per_group;
  prm.R = plan.rows_per_part;
  // Zipf-hot columns would otherwise put many lanes of one warp into one bank with different
  // rows; XOR-ing the low 5 column bits with the row spreads them (needs n_e % 32 == 0).
  prm.swz = (plan.ne % 32 == 0) ? 31u : 0u;
  prm.n_groups = plan.n_groups;
  prm.n_parts = plan.n_parts;
  prm.T = T;
  const int64_t base_units = (int64_t)plan.n_groups * plan.n_parts;
  const int64_t resident = (int64_t)plan.sms * plan.ctas_per_sm;
  // Enough units for ~4 waves of resident CTAs, but at least 8K tokens per unit so the one-time
  // flush of the privatised counters stays a small fraction of the counting work.
  int64_t n_chunks = std::max<int64_t>(1, (4 * resident + base_units - 1) / base_units);
  n_chunks = std::min<int64_t>(n_chunks, std::max<int64_t>(1, T / 8192));
  prm.chunk_tokens = (T + n_chunks - 1) / n_chunks;
  n_chunks = (T + prm.chunk_tokens - 1) / prm.chunk_tokens;
  prm.n_units = n_chunks * base_units;
  const int grid = (int)std::min<int64_t>(prm.n_units, resident);
  if (id_bytes == 1) return dispatch_k<uint8_t>(plan, prm, ids, E, flags, s, grid);
  return dispatch_k<int32_t>(plan, prm, ids, E, flags, s, grid);
}

cudaError_t launch_count_activation(int L, int ne, int k, const void* ids, int id_bytes, int64_t T,
                                    unsigned long long* A, uint32_t* flags, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const size_t smem = (size_t)L * ne * 4;
  const int64_t n = T * L * k;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 148, (n + 255) / 256));
  if (id_bytes == 1) {
    auto kern = count_activation_kernel<uint8_t>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 256, smem, s>>>(L, ne, k, static_cast<const uint8_t*>(ids), T, A, flags);
  } else {
    auto kern = count_activation_kernel<int32_t>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 256, smem, s>>>(L, ne, k, static_cast<const int32_t*>(ids), T, A, flags);
  }
  return cudaGetLastError();
}

cudaError_t launch_derive_activation(int L, int ne, int k, const unsigned long long* E,
                                     unsigned long long* A, cudaStream_t s) {
  if (L < 2) return cudaSuccess;
  const int warps = (L - 1) * ne + (ne + 31) / 32;
  const int threads = 256;
  const int grid = (warps * 32 + threads - 1) / threads;
  derive_activation_kernel<<<grid, threads, 0, s>>>(L, ne, k, E, A);
  return cudaGetLastError();
}

cudaError_t launch_derive_w(int L, int ne, const unsigned long long* E, unsigned long long* W,
                            cudaStream_t s) {
  const int64_t cells = (int64_t)ne * ne;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(1184, (cells + 255) / 256));
  derive_w_kernel<<<grid, 256, 0, s>>>(L, ne, E, W);
  return cudaGetLastError();
}

__global__ void add_u64_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src,
                               int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

cudaError_t launch_add_u64(unsigned long long* dst, const unsigned long long* src, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 1184, (n + 255) / 256));
  add_u64_kernel<<<grid, 256, 0, s>>>(dst, src, n);
  return cudaGetLastError();
}

cudaError_t launch_flat_forms(int L, int ne, const unsigned long long* A,
                              const unsigned long long* E, double* flatA, double* flatW,
                              cudaStream_t s) {
  const int64_t n = (int64_t)L * ne + (int64_t)(L - 1) * ne * ne;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 1184, (n + 255) / 256));
  flat_forms_kernel<<<grid, 256, 0, s>>>(L, ne, A, E, flatA, flatW);
  return cudaGetLastError();
}

}  // namespace gimbal_gpu
