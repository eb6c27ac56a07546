// Placement scoring, strong-pair (hotspot) selection and greedy re-placement on sm_100a.
//
// Reference semantics (/root/reference/proj/src/placement.cpp):
//   eval_cost          :58-85   loads(l,p) = sum_e A(l,e)[P(e)=p]; ideal_l = rowsum_l / g;
//                               D = max |loads - ideal|; cut = sum over pairs on different GPUs;
//                               objective = alpha*D + beta*cut
//   check_feasible     :30-50   ids in [0,g), every GPU exactly m/g experts (global cap)
//   build_affinity_set :186-238 pairs (w >= threshold && w > 0) sorted (w desc, a asc, b asc),
//                               top_e, endpoint union trimmed to capacity
//   greedy_place       :240-299 anchor M; order by (-total, id); home = first argmax row;
//                               least-loaded GPU with headroom, strict <
//
// cut is evaluated on E directly (W = flat_pair_weights() is never materialised): for candidate
// P, same = sum_l sum_{j,k} E_l(j,k) [P(l,j) == P(l+1,k)] and cut = total - same with
// total = tokens * (L-1) * top_k^2 (every token adds exactly top_k^2 pairings per layer pair).
// All sums are integers; converting the u64 result to double reproduces the reference's fp64
// accumulation exactly while the value stays below 2^53 (checked, GIMBAL_OVERFLOW otherwise).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "greedy_block.cuh"
#include "internal.cuh"
#include "ptx.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kEvalThreads = 256;
constexpr int kEvalCellsPerThread = 32;             // E cells held in registers per thread
constexpr int kEvalCands = 32;                      // candidates per CTA
constexpr int kEvalCellsPerCta = kEvalThreads * kEvalCellsPerThread;
constexpr int kSortLocal = 2048;  // keys per CTA in the shared-memory sort / top-K stages

// ---- cut: same[c] += sum over this CTA's E cells of E(j,k) [P(j) == P(k')] ----
// The CTA owns kEvalCellsPerCta consecutive cells of the flattened E (row r = flat expert
// f(l,j) of layer l < L-1, column k = expert of layer l+1), keeps them in registers and streams
// kEvalCands candidates at a time through shared memory.
__global__ void __launch_bounds__(kEvalThreads)
    eval_same_kernel(int L, int ne, const unsigned long long* __restrict__ E,
                     const uint8_t* __restrict__ cands, int64_t C, int64_t m,
                     unsigned long long* __restrict__ same, WidthGuard guard) {
  extern __shared__ uint8_t sm[];
  if (width_skip(guard)) return;
  const int64_t nE = (int64_t)(L - 1) * ne * ne;
  const int64_t cell0 = (int64_t)blockIdx.x * kEvalCellsPerCta;
  const int64_t row_lo = cell0 / ne;
  const int64_t cell_hi = min(nE, cell0 + kEvalCellsPerCta);
  const int64_t row_hi = (cell_hi - 1) / ne;                 // inclusive
  const int64_t span_lo = row_lo;                            // first flat id needed
  const int64_t span_hi = min(m, (row_hi / ne + 2) * ne);    // end of layer (l_hi + 1)
  const int span = (int)(span_hi - span_lo);
  unsigned long long e[kEvalCellsPerThread];
  int rowo[kEvalCellsPerThread];  // offset of P(row) in the staged span
  int colo[kEvalCellsPerThread];  // offset of P(col) in the staged span
#pragma unroll
  for (int i = 0; i < kEvalCellsPerThread; ++i) {
    const int64_t cell = cell0 + threadIdx.x + (int64_t)i * kEvalThreads;
    if (cell < cell_hi) {
      e[i] = E[cell];
      const int64_t r = cell / ne;
      const int64_t k = cell - r * ne;
      const int64_t l = r / ne;
      rowo[i] = (int)(r - span_lo);
      colo[i] = (int)((l + 1) * ne + k - span_lo);
    } else {
      e[i] = 0;
      rowo[i] = 0;
      colo[i] = 0;
    }
  }
  __shared__ unsigned long long red[kEvalThreads / 32][kEvalCands];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid.y splits the candidates so small E tensors still fill the machine
  const int64_t per_y = ((C + gridDim.y - 1) / gridDim.y + kEvalCands - 1) / kEvalCands * kEvalCands;
  const int64_t c_end = min(C, (int64_t)(blockIdx.y + 1) * per_y);
  for (int64_t c0 = (int64_t)blockIdx.y * per_y; c0 < c_end; c0 += kEvalCands) {
    const int nc = (int)min((int64_t)kEvalCands, c_end - c0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nc * span; idx += blockDim.x) {
      const int c = idx / span, o = idx - c * span;
      sm[c * span + o] = cands[(c0 + c) * m + span_lo + o];
    }
    __syncthreads();
    for (int c = 0; c < nc; ++c) {
      const uint8_t* P = sm + c * span;
      unsigned long long s = 0;
#pragma unroll
      for (int i = 0; i < kEvalCellsPerThread; ++i) s += (P[rowo[i]] == P[colo[i]]) ? e[i] : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp][c] = s;
    }
    __syncthreads();
    if (threadIdx.x < nc) {
      unsigned long long s = 0;
#pragma unroll
      for (int w = 0; w < kEvalThreads / 32; ++w) s += red[w][threadIdx.x];
      if (s) atomicAdd(&same[c0 + threadIdx.x], s);
    }
  }
}

// Fast form for n_e in {32, 64, 128, 256} and E cells < 2^27 (u32 partial sums): thread owns
// column k of 32 consecutive rows of one layer pair, so per candidate it reads its column's GPU
// once and the 32 rows' GPUs as two broadcast 16-byte shared loads.
__global__ void __launch_bounds__(kEvalThreads)
    eval_same_fast_kernel(int L, int ne, const unsigned long long* __restrict__ E,
                          const uint8_t* __restrict__ cands, int64_t C, int64_t m,
                          unsigned long long* __restrict__ same, WidthGuard guard) {
  extern __shared__ __align__(16) uint8_t sm[];
  if (width_skip(guard)) return;
  const int rows_per_cta = kEvalCellsPerCta / ne;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;          // first flat row of this CTA
  const int64_t n_rows = (int64_t)(L - 1) * ne;
  const int grp = threadIdx.x / ne;                                 // 32-row group of this thread
  const int k = threadIdx.x - grp * ne;
  const int64_t rg = r0 + (int64_t)grp * 32;                         // its first row
  const int64_t layer = rg / ne;                                     // rows rg..rg+31 share it
  const int64_t span_hi = min(m, (min(n_rows, r0 + rows_per_cta) - 1) / ne * ne + 2 * ne);
  const int span = (int)((span_hi - r0 + 15) & ~15ll);               // 16-byte aligned stride
  uint32_t e[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) e[i] = rg + i < n_rows ? (uint32_t)E[(rg + i) * ne + k] : 0u;
  const int rowo = (int)(rg - r0);
  const int colo = (int)((layer + 1) * ne + k - r0);
  const bool active = rg < n_rows;
  __shared__ unsigned long long red[kEvalThreads / 32][kEvalCands];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid.y splits the candidates so small E tensors still fill the machine
  const int64_t per_y = ((C + gridDim.y - 1) / gridDim.y + kEvalCands - 1) / kEvalCands * kEvalCands;
  const int64_t c_end = min(C, (int64_t)(blockIdx.y + 1) * per_y);
  for (int64_t c0 = (int64_t)blockIdx.y * per_y; c0 < c_end; c0 += kEvalCands) {
    const int nc = (int)min((int64_t)kEvalCands, c_end - c0);
    const int live = (int)(span_hi - r0);
    __syncthreads();
    if (((reinterpret_cast<uintptr_t>(cands) | (uintptr_t)m | (uintptr_t)r0 | (uintptr_t)live) & 3) == 0) {
      const int live4 = live >> 2;  // stage 4 GPU ids per load
      for (int idx = threadIdx.x; idx < nc * live4; idx += blockDim.x) {
        const int c = idx / live4, o = idx - c * live4;
        reinterpret_cast<uint32_t*>(sm + c * span)[o] =
            __ldg(reinterpret_cast<const uint32_t*>(cands + (c0 + c) * m + r0) + o);
      }
    } else
    for (int idx = threadIdx.x; idx < nc * live; idx += blockDim.x) {
      const int c = idx / live, o = idx - c * live;
      sm[c * span + o] = cands[(c0 + c) * m + r0 + o];
    }
    __syncthreads();
    for (int c = 0; c < nc; ++c) {
      const uint8_t* P = sm + c * span;
      uint32_t s = 0;
      if (active) {
        const uint32_t q = P[colo];
        const uint4 w0 = *reinterpret_cast<const uint4*>(P + rowo);
        const uint4 w1 = *reinterpret_cast<const uint4*>(P + rowo + 16);
        const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int i = 0; i < 32; ++i) s += (((w[i >> 2] >> (8 * (i & 3))) & 0xffu) == q) ? e[i] : 0u;
      }
      unsigned long long s64 = s;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s64 += __shfl_xor_sync(0xffffffffu, s64, o);
      if (lane == 0) red[warp][c] = s64;
    }
    __syncthreads();
    if (threadIdx.x < nc) {
      unsigned long long s = 0;
#pragma unroll
      for (int w = 0; w < kEvalThreads / 32; ++w) s += red[w][threadIdx.x];
      if (s) atomicAdd(&same[c0 + threadIdx.x], s);
    }
  }
}

__global__ void max_cell_kernel(const unsigned long long* __restrict__ E, int64_t n,
                                unsigned long long* __restrict__ out) {
  unsigned long long mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, E[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// ---- small shapes (Mixtral class): one warp per candidate, one lane per layer ----
// The whole E ((L-1) x NE x NE u32, cells < 2^27) and A sit in shared memory; lane l reads its
// candidate's GPU ids of layers l and l+1 (NE bytes each), adds E_l(j, k) for every same-GPU (j, k)
// pair, and forms layer l's per-GPU loads, |load - ideal_l| and per-GPU expert counts; the warp
// reduces them.  Replaces eval_same_kernel + eval_dev_kernel (4096 CTAs each) for small n_e.
// Shared-memory tables of the small-shape evaluators: E as u32 cells ((L-1) x NE x NE), ideal
// loads (L doubles), A (L x NE u64).  Returns the bytes used.
template <int NE>
__host__ __device__ constexpr size_t small_tables_bytes(int L) {
  return (((size_t)(L - 1) * NE * NE * 4 + 15) & ~(size_t)15) + (size_t)L * 8 + (size_t)L * NE * 8;
}

// ideal_l = A.row(l).sum() / g (placement.cpp:68); integer rowsum < 2^53 is exact in fp64
template <int NE, int G>
__device__ __forceinline__ void small_ideal(int L, const unsigned long long* sA, double* sIdeal) {
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    unsigned long long r = 0;
#pragma unroll
    for (int j = 0; j < NE; ++j) r += sA[l * NE + j];
    sIdeal[l] = __ddiv_rn((double)r, (double)G);
  }
}

struct SmallScore {
  unsigned long long same;  // sum of E over same-GPU (j, k) pairs
  double dev;               // max_l,p |loads - ideal_l|
};

// One candidate by one warp (lane per layer): same-GPU pair weight and deviation (every lane gets
// them), feasibility flagged here (check_feasible, placement.cpp:30-50).
template <int NE, int G>
__device__ __forceinline__ SmallScore small_candidate(int L, const uint32_t* sE, const unsigned long long* sA,
                                                      const double* sIdeal, const uint8_t* __restrict__ P, int64_t c,
                                                      int64_t base, uint32_t* __restrict__ flags,
                                                      long long* __restrict__ bad_index) {
  const int lane = threadIdx.x & 31;
  const int m = L * NE;
  unsigned long long sm = 0;
  double dev = 0.0;
  uint32_t cnt[G];
#pragma unroll
  for (int q = 0; q < G; ++q) cnt[q] = 0u;
  bool bad = false;
  for (int l = lane; l < L; l += 32) {
    uint32_t pl[NE], pn[NE];
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      pl[j] = P[l * NE + j];
      bad |= pl[j] >= (uint32_t)G;
    }
    unsigned long long load[G];
#pragma unroll
    for (int q = 0; q < G; ++q) load[q] = 0ull;
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const unsigned long long a = sA[l * NE + j];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        load[q] += pl[j] == (uint32_t)q ? a : 0ull;
        cnt[q] += pl[j] == (uint32_t)q ? 1u : 0u;
      }
    }
    const double ideal = sIdeal[l];
#pragma unroll
    for (int q = 0; q < G; ++q) dev = fmax(dev, fabs(__dsub_rn((double)load[q], ideal)));
    if (l + 1 < L) {
#pragma unroll
      for (int k = 0; k < NE; ++k) pn[k] = P[(l + 1) * NE + k];
      const uint32_t* El = sE + l * NE * NE;
#pragma unroll
      for (int j = 0; j < NE; ++j)
#pragma unroll
        for (int k = 0; k < NE; ++k) sm += pl[j] == pn[k] ? (unsigned long long)El[j * NE + k] : 0ull;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
#pragma unroll
    for (int q = 0; q < G; ++q) cnt[q] += __shfl_xor_sync(0xffffffffu, cnt[q], o);
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    bool infeasible = bad;
#pragma unroll
    for (int q = 0; q < G; ++q) infeasible |= cnt[q] != (uint32_t)(m / G);
    if (infeasible) {
      atomicOr(flags, (uint32_t)kFlagInfeasible);
      atomicMin(bad_index, (long long)(base + c));
    }
  }
  return SmallScore{sm, dev};
}

template <int NE, int G>
__global__ void __launch_bounds__(256)
    eval_small_kernel(int L, const unsigned long long* __restrict__ A, const unsigned long long* __restrict__ E,
                      const uint8_t* __restrict__ cands, int64_t C, int64_t base, unsigned long long* __restrict__ same,
                      double* __restrict__ D, uint32_t* __restrict__ flags, long long* __restrict__ bad_index) {
  extern __shared__ __align__(16) unsigned char sm_small[];
  uint32_t* sE = reinterpret_cast<uint32_t*>(sm_small);                       // (L-1) * NE * NE
  double* sIdeal = reinterpret_cast<double*>(sm_small + (((L - 1) * NE * NE * 4 + 15) & ~15));  // L
  unsigned long long* sA = reinterpret_cast<unsigned long long*>(sIdeal + L);  // L * NE
  for (int i = threadIdx.x; i < (L - 1) * NE * NE; i += blockDim.x) sE[i] = (uint32_t)E[i];
  for (int i = threadIdx.x; i < L * NE; i += blockDim.x) sA[i] = A[i];
  __syncthreads();
  small_ideal<NE, G>(L, sA, sIdeal);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= C) return;
  const SmallScore r = small_candidate<NE, G>(L, sE, sA, sIdeal, cands + c * (int64_t)L * NE, c, base, flags, bad_index);
  if ((threadIdx.x & 31) == 0) {
    same[c] = r.same;
    D[c] = r.dev;
  }
}

// ---- deviation + feasibility: one CTA per candidate, one warp per layer at a time ----
// Lane-private bins (g <= G <= 8): every lane adds its experts' activations into its own G bins in
// shared memory, laid out [GPU][lane] so a warp's accesses fall on its lanes' banks whatever GPU ids
// the lanes hold (no atomics, no bank conflicts); per-GPU counts ride in registers as 4-bit fields.
// The warp then sums each GPU's 32 bins with a reduce-scatter of shuffles.  Integer sums: the same
// loads as any order.
template <int G>
__global__ void __launch_bounds__(256)
    eval_dev_bins_kernel(int L, int ne, int g, const unsigned long long* __restrict__ A,
                         const uint8_t* __restrict__ cands, int64_t m, double* __restrict__ D,
                         uint32_t* __restrict__ flags, long long* __restrict__ bad_index, int64_t base) {
  constexpr int kWarps = 8;
  __shared__ unsigned long long bins[kWarps][G][32];
  __shared__ uint32_t ctot[G];
  __shared__ double dmax[kWarps];
  __shared__ int bad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x;
  const uint8_t* P = cands + c * m;
  if (threadIdx.x < G) ctot[threadIdx.x] = 0u;
  if (threadIdx.x == 0) bad = 0;
#pragma unroll
  for (int p = 0; p < G; ++p) bins[warp][p][lane] = 0ull;
  __syncthreads();
  double dev = 0.0;
  uint32_t cnt_lo = 0u, cnt_hi = 0u;  // per-GPU expert counts, 8-bit fields (GPUs 0-3, 4-7)
  bool my_bad = false;
  for (int l = warp; l < L; l += kWarps) {
    // n_e <= 256 (uint8 ids): at most 8 experts per lane, all loaded before the bin updates
    unsigned long long av[8];
    uint32_t pv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane + 32 * i;
      av[i] = e < ne ? A[(int64_t)l * ne + e] : 0ull;
      pv[i] = e < ne ? (uint32_t)P[(int64_t)l * ne + e] : 0xffffffffu;
    }
    unsigned long long rowsum = 0;
    uint32_t nib = 0u;  // this layer's counts, 4-bit fields (<= 8 experts per lane)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (lane + 32 * i >= ne) break;
      rowsum += av[i];
      if (pv[i] >= (uint32_t)g) {
        my_bad = true;
        continue;
      }
      bins[warp][pv[i]][lane] += av[i];
      nib += 1u << (4 * pv[i]);
    }
    cnt_lo += nib & 0x0f0f0f0fu;
    cnt_hi += (nib >> 4) & 0x0f0f0f0fu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rowsum += __shfl_xor_sync(0xffffffffu, rowsum, o);
    // read back (and clear) this lane's bins, then sum each GPU over the 32 lanes
    unsigned long long v[G];
#pragma unroll
    for (int p = 0; p < G; ++p) {
      v[p] = bins[warp][p][lane];
      bins[warp][p][lane] = 0ull;
    }
    // reduce-scatter: after the halving steps lane keeps GPU (lane % G)'s partial sum
#pragma unroll
    for (int h = G / 2; h >= 1; h >>= 1) {
      const bool upper = (lane & h) != 0;
#pragma unroll
      for (int p = 0; p < h; ++p) {
        const unsigned long long send = upper ? v[p] : v[p + h];
        const unsigned long long keep = upper ? v[p + h] : v[p];
        v[p] = keep + __shfl_xor_sync(0xffffffffu, send, h);
      }
    }
    unsigned long long load = v[0];
#pragma unroll
    for (int o = G; o < 32; o <<= 1) load += __shfl_xor_sync(0xffffffffu, load, o);
    // ideal_l = A.row(l).sum() / g (placement.cpp:68); integer rowsum < 2^53 is exact in fp64
    if (lane < g && lane < G) {
      const double ideal = __ddiv_rn((double)rowsum, (double)g);
      dev = fmax(dev, fabs(__dsub_rn((double)load, ideal)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
  if (lane == 0) dmax[warp] = dev;
  // counts: widen the 8-bit fields (<= 31 layers x 8 per lane: L <= 248) to 16 bits, sum the warp
  uint32_t c16[4] = {cnt_lo & 0x00ff00ffu, (cnt_lo >> 8) & 0x00ff00ffu, cnt_hi & 0x00ff00ffu, (cnt_hi >> 8) & 0x00ff00ffu};
#pragma unroll
  for (int w = 0; w < 4; ++w)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c16[w] += __shfl_xor_sync(0xffffffffu, c16[w], o);
  if (lane == 0) {
    // 16-bit fields (low, high): c16[0] GPUs 0, 4; c16[1] 2, 6; c16[2] 1, 5; c16[3] 3, 7
#pragma unroll
    for (int p = 0; p < G; ++p) {
      const uint32_t word = c16[(p & 1) * 2 + ((p >> 1) & 1)];
      atomicAdd(&ctot[p], (word >> (16 * ((p >> 2) & 1))) & 0xffffu);
    }
  }
  if (__any_sync(0xffffffffu, my_bad) && lane == 0) bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int w = 0; w < kWarps; ++w) d = fmax(d, dmax[w]);
    D[c] = d;
    const uint32_t cap = (uint32_t)(m / g);
    int infeasible = bad;
    for (int p = 0; p < g; ++p)
      if (ctot[p] != cap) infeasible = 1;
    if (infeasible) {
      atomicOr(flags, (uint32_t)kFlagInfeasible);
      atomicMin(bad_index, (long long)(base + c));
    }
  }
}

__global__ void __launch_bounds__(256)
    eval_dev_kernel(int L, int ne, int g, const unsigned long long* __restrict__ A,
                    const uint8_t* __restrict__ cands, int64_t m, double* __restrict__ D,
                    uint32_t* __restrict__ flags, long long* __restrict__ bad_index, int64_t base) {
  extern __shared__ unsigned long long sh[];  // [warps][g] loads, then [g] counts (u32)
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* loads = sh + warp * g;
  uint32_t* counts = reinterpret_cast<uint32_t*>(sh + warps * g);
  const int64_t c = blockIdx.x;
  const uint8_t* P = cands + c * m;
  for (int p = threadIdx.x; p < g; p += blockDim.x) counts[p] = 0;
  __shared__ double dmax[8];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  double dev = 0.0;
  for (int l = warp; l < L; l += warps) {
    for (int p = lane; p < g; p += 32) loads[p] = 0ull;
    __syncwarp();
    unsigned long long rowsum = 0;
    for (int e = lane; e < ne; e += 32) {
      const unsigned long long a = A[(int64_t)l * ne + e];
      const int p = P[(int64_t)l * ne + e];
      rowsum += a;
      if (p >= g) {
        bad = 1;
        continue;
      }
      atomicAdd(&loads[p], a);
      atomicAdd(&counts[p], 1u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rowsum += __shfl_xor_sync(0xffffffffu, rowsum, o);
    __syncwarp();
    // ideal_l = A.row(l).sum() / g (placement.cpp:68); integer rowsum < 2^53 is exact in fp64
    const double ideal = __ddiv_rn((double)rowsum, (double)g);
    for (int p = lane; p < g; p += 32) {
      const double d = fabs(__dsub_rn((double)loads[p], ideal));
      dev = fmax(dev, d);
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
  if (lane == 0) dmax[warp] = dev;
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int w = 0; w < warps; ++w) d = fmax(d, dmax[w]);
    D[c] = d;
    const uint32_t cap = (uint32_t)(m / g);
    int infeasible = bad;
    for (int p = 0; p < g; ++p)
      if (counts[p] != cap) infeasible = 1;
    if (infeasible) {
      atomicOr(flags, (uint32_t)kFlagInfeasible);
      atomicMin(bad_index, (long long)(base + c));
    }
  }
}

// cut/objective per candidate, then the argmin (lowest index among minima) in one CTA.
__global__ void eval_finish_kernel(int64_t C, int L, int ne, int k, const unsigned long long* __restrict__ A,
                                   double alpha, double beta, const unsigned long long* __restrict__ same,
                                   const double* __restrict__ D, double* __restrict__ cut,
                                   double* __restrict__ obj, long long* __restrict__ argmin,
                                   uint32_t* __restrict__ flags) {
  __shared__ double bv[1024];
  __shared__ long long bi[1024];
  __shared__ unsigned long long tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  if (L > 1) {  // total pair weight: (L-1) * k * (tokens * k) with tokens * k = sum_j A(0, j)
    unsigned long long a = 0;
    for (int j = threadIdx.x; j < ne; j += blockDim.x) a += A[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0 && a) atomicAdd(&tot, a);
  }
  __syncthreads();
  const unsigned long long total = tot * (unsigned long long)(L - 1) * (unsigned long long)k;
  double best = 0.0;
  long long besti = -1;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
    const unsigned long long cu = total - same[c];
    if (cu > (1ull << 53)) atomicOr(flags, (uint32_t)kFlagOverflow);
    const double cd = (double)cu;
    // objective = alpha * D + beta * cut (placement.cpp:83): two roundings, no FMA contraction
    const double o = __dadd_rn(__dmul_rn(alpha, D[c]), __dmul_rn(beta, cd));
    cut[c] = cd;
    obj[c] = o;
    if (besti < 0 || o < best) {
      best = o;
      besti = c;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = besti;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = bv[threadIdx.x + s];
      const long long i2 = bi[threadIdx.x + s];
      const long long i1 = bi[threadIdx.x];
      if (i2 >= 0 && (i1 < 0 || v2 < bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < i1))) {
        bv[threadIdx.x] = v2;
        bi[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && argmin) *argmin = bi[0];
}

// ---- per-candidate bottleneck excess (sim.cpp:132-144's hotspot measure over the counted trace):
// excess_c = sum over layers, in order, of max(0, peak_l * g / (T * k) - 1), peak_l = max over
// GPUs p of sum_{e: P_c(l, e) = p} A(l, e), T * k = sum_e A(0, e).  One CTA per candidate, one
// warp per layer at a time; the layer terms are added in layer order by one thread (the
// reference's double arithmetic, IEEE, no contraction).
__global__ void __launch_bounds__(256)
    eval_excess_kernel(int L, int ne, int g, const unsigned long long* __restrict__ A,
                       const uint8_t* __restrict__ cands, int64_t m, double* __restrict__ excess,
                       uint32_t* __restrict__ flags) {
  extern __shared__ unsigned long long ex_sh[];  // [warps][g] loads, then [L] terms (double)
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* loads = ex_sh + warp * g;
  double* term = reinterpret_cast<double*>(ex_sh + warps * g);
  __shared__ unsigned long long tk;
  if (threadIdx.x == 0) tk = 0;
  __syncthreads();
  {
    unsigned long long a = 0;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) a += A[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0 && a) atomicAdd(&tk, a);
  }
  __syncthreads();
  const double per_layer = (double)tk;
  const uint8_t* P = cands + blockIdx.x * m;
  bool bad = false;
  for (int l = warp; l < L; l += warps) {
    for (int p = lane; p < g; p += 32) loads[p] = 0;
    __syncwarp();
    for (int e = lane; e < ne; e += 32) {
      const uint32_t p = P[(int64_t)l * ne + e];
      if (p >= (uint32_t)g) {
        bad = true;
        continue;
      }
      atomicAdd(&loads[p], A[(int64_t)l * ne + e]);
    }
    __syncwarp();
    unsigned long long peak = 0;
    for (int p = lane; p < g; p += 32) peak = max(peak, loads[p]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) peak = max(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    if (lane == 0) {
      const double x = __dsub_rn(__ddiv_rn(__dmul_rn((double)peak, (double)g), per_layer), 1.0);
      term[l] = 0.0 < x ? x : 0.0;  // std::max(0.0, x)
    }
    __syncwarp();
  }
  if (bad) atomicOr(flags, (uint32_t)kFlagInfeasible);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int l = 0; l < L; ++l) s = __dadd_rn(s, term[l]);
    excess[blockIdx.x] = s;
  }
}

// ---- build_affinity_set: composite sort keys over E ----
// key = (w << 24) | (2^24 - 1 - idx) for qualifying cells, else 0; sorting keys in descending
// order yields (w desc, idx asc), and idx = (l*ne + j)*ne + k orders exactly like the
// reference's (a asc, b asc) tie-break (a = l*ne + j, b = (l+1)*ne + k).
__global__ void affinity_keys_kernel(int L, int ne, const unsigned long long* __restrict__ E,
                                     double threshold, unsigned long long* __restrict__ keys,
                                     int64_t n, int64_t n_pad, uint32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0ull;
    if (i < n) {
      const unsigned long long w = E[i];
      const double wd = (double)w;
      if (wd >= threshold && wd > 0.0) {
        if (w >= (1ull << 40)) atomicOr(flags, (uint32_t)kFlagOverflow);
        key = (w << 24) | (unsigned long long)(0xffffffll - i);
      }
    }
    keys[i] = key;
  }
}

// Top-K selection for small top_e (placement.cpp:217-219 keeps only the top_e heaviest pairs):
// each CTA sorts a 2048-key segment in shared memory (descending) and keeps its first K keys;
// repeated until one segment remains.  FROM_E builds the composite keys from E on the fly.
template <bool FROM_E>
__global__ void __launch_bounds__(1024)
    topk_segment_kernel(const unsigned long long* __restrict__ in, int64_t n, double threshold, int K,
                        unsigned long long* __restrict__ out, uint32_t* __restrict__ flags) {
  __shared__ unsigned long long s[kSortLocal];
  const int64_t base = (int64_t)blockIdx.x * kSortLocal;
  for (int i = threadIdx.x; i < kSortLocal; i += blockDim.x) {
    const int64_t idx = base + i;
    unsigned long long key = 0ull;
    if (idx < n) {
      if constexpr (FROM_E) {
        const unsigned long long w = in[idx];
        const double wd = (double)w;
        if (wd >= threshold && wd > 0.0) {
          if (w >= (1ull << 40)) atomicOr(flags, (uint32_t)kFlagOverflow);
          key = (w << 24) | (unsigned long long)(0xffffffll - idx);
        }
      } else {
        key = in[idx];
      }
    }
    s[i] = key;
  }
  __syncthreads();
  for (int k = 2; k <= kSortLocal; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < kSortLocal / 2; t += blockDim.x) {
        const int i = 2 * j * (t / j) + (t % j);
        const bool desc = ((i & k) == 0);
        const unsigned long long a = s[i], b = s[i + j];
        if (desc ? (a < b) : (a > b)) {
          s[i] = b;
          s[i + j] = a;
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < K; i += blockDim.x) out[(int64_t)blockIdx.x * K + i] = s[i];
}

// Register top-K for small K (top_e <= kRegTopK, the simulator's default is 4): every thread keeps
// its K largest composite keys sorted in registers (branch-free insertion, skipped once a key
// cannot enter), warps merge their lanes' lists by shuffles, warp 0 merges the CTA's warps, and the
// CTA writes its K keys sorted descending.  One pass over E with ~2 CTAs per SM, then one CTA over
// the survivors; replaces the 2048-key bitonic segment sorts (0.34 ms -> tens of us at DS-V3).
constexpr int kRegTopK = 8;
constexpr int kRegThreads = 256;

template <int K>
__device__ __forceinline__ void topk_insert(unsigned long long (&r)[K], unsigned long long key) {
  if (key <= r[K - 1]) return;
#pragma unroll
  for (int i = K - 1; i >= 0; --i) {
    const unsigned long long prev = i ? r[i - 1] : ~0ull;
    r[i] = key > prev ? prev : (key > r[i] ? key : r[i]);
  }
}

template <int K>
__device__ __forceinline__ void topk_warp_merge(unsigned long long (&r)[K], int first = 16) {
#pragma unroll
  for (int o = first; o > 0; o >>= 1) {
    unsigned long long other[K];
#pragma unroll
    for (int i = 0; i < K; ++i) other[i] = __shfl_xor_sync(0xffffffffu, r[i], o);
#pragma unroll
    for (int i = 0; i < K; ++i) topk_insert<K>(r, other[i]);
  }
}

template <bool FROM_E, int K>  // K = kept keys per list (4 when top_e <= 4, else 8)
__global__ void __launch_bounds__(kRegThreads)
    topk_reg_kernel(const unsigned long long* __restrict__ in, int64_t n, double threshold,
                    unsigned long long* __restrict__ out, uint32_t* __restrict__ flags) {
  __shared__ unsigned long long lists[kRegThreads / 32][K];
  unsigned long long r[K];
#pragma unroll
  for (int i = 0; i < K; ++i) r[i] = 0ull;
  bool over = false;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key;
    if constexpr (FROM_E) {
      const unsigned long long w = in[idx];
      const double wd = (double)w;
      key = 0ull;
      if (wd >= threshold && wd > 0.0) {
        over |= w >= (1ull << 40);
        key = (w << 24) | (unsigned long long)(0xffffffll - idx);
      }
    } else {
      key = in[idx];
    }
    topk_insert<K>(r, key);
  }
  if (FROM_E && __syncthreads_or(over) && threadIdx.x == 0) atomicOr(flags, (uint32_t)kFlagOverflow);
  topk_warp_merge<K>(r);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) lists[warp][i] = r[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) r[i] = lane < kRegThreads / 32 ? lists[lane][i] : 0ull;
    topk_warp_merge<K>(r);
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < K; ++i) out[(int64_t)blockIdx.x * K + i] = r[i];
    }
  }
}

// Sequential endpoint union over the sorted pairs (placement.cpp:221-237): the result is the
// union of the longest prefix (<= kept pairs) whose union fits `capacity`.
__global__ void affinity_select_kernel(int L, int ne, const unsigned long long* __restrict__ keys,
                                       int64_t n_keys, int32_t top_e, int32_t capacity,
                                       uint32_t* __restrict__ bits, int32_t* __restrict__ out,
                                       int32_t* __restrict__ n_out) {
  const int64_t m = (int64_t)L * ne;
  const int64_t words = (m + 31) / 32;
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t members = 0;
    const int64_t nn = (int64_t)ne * ne;
    for (int64_t i = 0; i < n_keys; ++i) {
      if (top_e >= 0 && i >= top_e) break;
      const unsigned long long key = keys[i];
      if (key == 0ull) break;
      const int64_t idx = 0xffffffll - (int64_t)(key & 0xffffffull);
      const int64_t a = idx / ne;
      const int64_t b = (idx / nn + 1) * ne + (idx % ne);
      const bool na = !((bits[a >> 5] >> (a & 31)) & 1u);
      const bool nb = !((bits[b >> 5] >> (b & 31)) & 1u);
      const int64_t grown = members + (na ? 1 : 0) + (nb ? 1 : 0);
      if (grown > capacity) break;
      if (na) bits[a >> 5] |= 1u << (a & 31);
      if (nb) bits[b >> 5] |= 1u << (b & 31);
      members = grown;
    }
    int32_t n = 0;
    for (int64_t w = 0; w < words; ++w) {
      uint32_t v = bits[w];
      while (v) {
        const int bit = __ffs(v) - 1;
        out[n++] = (int32_t)(w * 32 + bit);
        v &= v - 1;
      }
    }
    *n_out = n;
  }
}

// ---- greedy_place on the compact flat activation ----
// order keys = (A(e) << 24) | (2^24 - 1 - e) for unanchored experts (descending = (-total, id)),
// 0 for anchored ones and padding.
__global__ void greedy_keys_kernel(int64_t m, const unsigned long long* __restrict__ A,
                                   const uint32_t* __restrict__ anchored,
                                   unsigned long long* __restrict__ keys, int64_t n_pad,
                                   uint32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0ull;
    if (i < m && !((anchored[i >> 5] >> (i & 31)) & 1u)) {
      const unsigned long long a = A[i];
      if (a >= (1ull << 40)) atomicOr(flags, (uint32_t)kFlagOverflow);
      key = (a << 24) | (unsigned long long)(0xffffffll - i);
    }
    keys[i] = key;
  }
}

// ---- bitonic sort (descending) of u64 keys, n a power of two ----

__global__ void bitonic_local_kernel(unsigned long long* keys, int64_t n, int64_t k_start,
                                     int64_t k_end, bool full) {
  // full: run the network for k in [2, min(kSortLocal, n)] entirely in shared memory.
  // otherwise: for the current k (k_start), run the j < kSortLocal steps.
  __shared__ unsigned long long s[kSortLocal];
  const int64_t base = (int64_t)blockIdx.x * kSortLocal;
  for (int i = threadIdx.x; i < kSortLocal; i += blockDim.x) s[i] = keys[base + i];
  __syncthreads();
  const int64_t kmax = full ? min((int64_t)kSortLocal, n) : k_start;
  const int64_t kmin = full ? 2 : k_start;
  for (int64_t k = kmin; k <= kmax; k <<= 1) {
    for (int64_t j = (full ? k : kSortLocal) >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < kSortLocal / 2; t += blockDim.x) {
        const int64_t lo_local = 2 * j * (t / j) + (t % j);
        const int64_t i = base + lo_local;
        const int64_t pi = i + j;
        const bool desc = ((i & k) == 0);
        const unsigned long long a = s[lo_local], b = s[lo_local + j];
        if (desc ? (a < b) : (a > b)) {
          s[lo_local] = b;
          s[lo_local + j] = a;
        }
        (void)pi;
      }
      __syncthreads();
    }
  }
  (void)k_end;
  for (int i = threadIdx.x; i < kSortLocal; i += blockDim.x) keys[base + i] = s[i];
}

__global__ void bitonic_global_kernel(unsigned long long* keys, int64_t n, int64_t k, int64_t j) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n / 2;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = 2 * j * (t / j) + (t % j);
    const bool desc = ((i & k) == 0);
    const unsigned long long a = keys[i], b = keys[i + j];
    if (desc ? (a < b) : (a > b)) {
      keys[i] = b;
      keys[i + j] = a;
    }
  }
}

// n < kSortLocal: one CTA sorts everything in shared memory.
__global__ void bitonic_small_kernel(unsigned long long* keys, int n) {
  __shared__ unsigned long long s[kSortLocal];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = keys[i];
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
        const int i = 2 * j * (t / j) + (t % j);
        const bool desc = ((i & k) == 0);
        const unsigned long long a = s[i], b = s[i + j];
        if (desc ? (a < b) : (a > b)) {
          s[i] = b;
          s[i + j] = a;
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < n; i += blockDim.x) keys[i] = s[i];
}

// ---- the whole placement pass for small shapes in one launch (Mixtral class) ----
// gimbal_pass_async queues ~10 dependent launches (derive A, top-K, select, greedy keys, sort,
// walk, evaluator, finish); at m = 256 each runs a few microseconds and the step is launch-bound.
// Here CTA 0 derives A, builds the strong-pair set (register top-K + the reference's endpoint
// union), sorts the greedy keys in shared memory, runs the greedy walk (greedy_block.cuh) into
// candidate row 0 and scores that row, while CTAs 1.. score candidates 1..C-1 (one warp each, as
// eval_small_kernel); the last CTA to finish (completion ticket) forms cut / objective and the
// argmin.  Every step follows the standalone kernels' arithmetic, so the results are identical.
struct TinyPass {
  int L, k;
  double threshold;
  int top_e, capacity, anchor;
  int n2;                // greedy keys sorted in shared memory (next power of two >= m)
  int greedy_parallel;   // greedy_smem_bytes: layer-parallel walk fits
  const unsigned long long* E;
  unsigned long long* A_out;
  uint8_t* cands;
  int64_t C;
  double alpha, beta;
  double* scores;        // [3][C]: deviation, cut, objective
  long long* argmin;
  int32_t* placement;
  int32_t* members;
  int32_t* n_members;
  uint32_t* flags;       // handle flag words: [0] pass errors, [1] deferred evaluator errors
  unsigned long long* same;
  long long* bad_index;  // 0x7f7f.. before the launch (set once, restored by the last CTA)
  uint32_t* ticket;      // 0x7f7f7f7f before the launch (set once, restored by the last CTA)
  long long* best;       // per CTA: best objective (bits), its candidate index
  uint32_t* flags_out;   // copy of flag words 0-1 at the end, or null
  int32_t* ring;         // mapped host ring of packed results (slots x (6 + 2m) words), or null
  uint32_t* ring_seq;    // device pass counter: this pass writes slot ring_seq % ring_slots
  int ring_slots;
};

// bytes of CTA 0's scratch after the shared tables (keep in step with tiny_pass_kernel)
inline size_t tiny_prep_bytes(int n2, int KT, int m) {
  return (size_t)n2 * 16 + (size_t)64 * KT + (((size_t)(m + 31) / 32 * 4 + 15) & ~(size_t)15) +
         (((size_t)m + 15) & ~(size_t)15);
}

constexpr int kTinyThreads = 256;
constexpr uint32_t kTicketBase = 0x7f7f7f7fu;

#ifdef GIMBAL_AB_KNOBS
// phase timestamps of the fused pass's CTA 0 and last CTA (test/tool build only)
__device__ unsigned long long g_tiny_prof[16];
#define TINY_MARK(i)                                                              \
  do {                                                                           \
    if (threadIdx.x == 0) g_tiny_prof[i] = globaltimer_ns();                     \
  } while (0)
#else
#define TINY_MARK(i) \
  do {               \
  } while (0)
#endif

template <int NE>
__host__ __device__ constexpr size_t tiny_extra_offset(int L) {
  return (small_tables_bytes<NE>(L) + 15) & ~(size_t)15;
}

template <int NE, int G, int KT>
__global__ void __launch_bounds__(kTinyThreads) tiny_pass_kernel(const TinyPass p) {
  extern __shared__ __align__(16) unsigned char sm_tiny[];
  const int L = p.L;
  const int m = L * NE;
  const int nE = (L - 1) * NE * NE;
  uint32_t* sE = reinterpret_cast<uint32_t*>(sm_tiny);
  double* sIdeal = reinterpret_cast<double*>(sm_tiny + ((nE * 4 + 15) & ~15));
  unsigned long long* sA = reinterpret_cast<unsigned long long*>(sIdeal + L);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (blockIdx.x == 0) TINY_MARK(0);
  for (int i = tid; i < nE; i += kTinyThreads) sE[i] = (uint32_t)p.E[i];
  __syncthreads();
  // derive_activation_kernel: A_l(j) = sum_k E_l(j, k) / k, A_{L-1}(k) = sum_j E_{L-2}(j, k) / k
  for (int r = tid; r < m; r += kTinyThreads) {
    const int l = r / NE, x = r - l * NE;
    unsigned long long s = 0;
    if (l < L - 1) {
#pragma unroll
      for (int c = 0; c < NE; ++c) s += sE[(l * NE + x) * NE + c];
    } else {
#pragma unroll
      for (int j = 0; j < NE; ++j) s += sE[((L - 2) * NE + j) * NE + x];
    }
    sA[r] = s / (unsigned long long)p.k;
  }
  __syncthreads();
  small_ideal<NE, G>(L, sA, sIdeal);
  __syncthreads();
  double* D = p.scores;
  // CTA 0's scratch (tiny_prep_bytes): greedy keys, rank-sorted keys, top-K lists, member bits,
  // the greedy row, then greedy_walk_block's shared memory
  unsigned char* extra = sm_tiny + tiny_extra_offset<NE>(L);
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(extra);   // n2
  unsigned long long* keys2 = keys + p.n2;                                   // n2
  unsigned long long* lists = keys2 + p.n2;                                  // 8 x KT
  uint32_t* bits = reinterpret_cast<uint32_t*>(lists + 8 * KT);              // (m + 31) / 32
  uint8_t* row0 = reinterpret_cast<uint8_t*>(bits) + (((m + 31) / 32 * 4 + 15) & ~15);
  unsigned long long* gsm = reinterpret_cast<unsigned long long*>(row0 + ((m + 15) & ~15));
  __shared__ unsigned long long s_same0, s_dev0;  // row 0's score (CTA 0)
  __shared__ int s_bad0;
  if (blockIdx.x == 0) {
    __shared__ int s_nM;
    TINY_MARK(1);
    for (int r = tid; r < m; r += kTinyThreads) p.A_out[r] = sA[r];
    // build_affinity_set (placement.cpp:186-238): top_e heaviest (w desc, a asc, b asc) pairs
    // with w >= threshold and w > 0 -- composite keys as topk_reg_kernel, one CTA
    unsigned long long r[KT];
#pragma unroll
    for (int i = 0; i < KT; ++i) r[i] = 0ull;
    for (int idx = tid; idx < nE; idx += kTinyThreads) {
      const unsigned long long w = sE[idx];
      const double wd = (double)w;
      topk_insert<KT>(r, (wd >= p.threshold && wd > 0.0) ? (w << 24) | (unsigned long long)(0xffffff - idx) : 0ull);
    }
    topk_warp_merge<KT>(r);
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < KT; ++i) lists[warp * KT + i] = r[i];
    }
    for (int w = tid; w < (m + 31) / 32; w += kTinyThreads) bits[w] = 0u;
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < KT; ++i) r[i] = lane < kTinyThreads / 32 ? lists[lane * KT + i] : 0ull;
      topk_warp_merge<KT>(r, kTinyThreads / 64);  // lists in lanes 0-7 only
      if (lane == 0) {  // affinity_select_kernel: endpoint union of the longest prefix within capacity
        int members = 0;
        for (int i = 0; i < p.top_e; ++i) {
          const unsigned long long key = r[0];
#pragma unroll
          for (int q = 0; q + 1 < KT; ++q) r[q] = r[q + 1];  // pop the front (registers, static indices)
          r[KT - 1] = 0ull;
          if (key == 0ull) break;
          const int idx = 0xffffff - (int)(key & 0xffffffull);
          const int a = idx / NE;
          const int b = (idx / (NE * NE) + 1) * NE + (idx % NE);
          const bool na = !((bits[a >> 5] >> (a & 31)) & 1u);
          const bool nb = !((bits[b >> 5] >> (b & 31)) & 1u);
          const int grown = members + (na ? 1 : 0) + (nb ? 1 : 0);
          if (grown > p.capacity) break;
          if (na) bits[a >> 5] |= 1u << (a & 31);
          if (nb) bits[b >> 5] |= 1u << (b & 31);
          members = grown;
        }
        int n = 0;
        for (int w = 0; w < (m + 31) / 32; ++w) {
          uint32_t v = bits[w];
          while (v) {
            p.members[n++] = w * 32 + (__ffs(v) - 1);
            v &= v - 1;
          }
        }
        *p.n_members = n;
        s_nM = n;
      }
    }
    __syncthreads();
    TINY_MARK(2);
    // greedy_keys_kernel: (A << 24) | (2^24 - 1 - e) for unanchored experts, 0 otherwise
    for (int i = tid; i < p.n2; i += kTinyThreads)
      keys[i] = (i < m && !((bits[i >> 5] >> (i & 31)) & 1u)) ? (sA[i] << 24) | (unsigned long long)(0xffffff - i)
                                                            : 0ull;
    __syncthreads();
    unsigned long long* sorted = keys;
    if (p.n2 <= 512) {
      // rank sort (descending; equal keys -- only zeros -- by position): one pass, no barriers
      for (int i = tid; i < p.n2; i += kTinyThreads) {
        const unsigned long long ki = keys[i];
        int rank = 0;
#pragma unroll 8
        for (int j = 0; j < p.n2; ++j) {
          const unsigned long long kj = keys[j];
          rank += (kj > ki) | ((kj == ki) & (j < i));
        }
        keys2[rank] = ki;
      }
      sorted = keys2;
    } else {  // bitonic_small_kernel
      for (int kk = 2; kk <= p.n2; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
          for (int t = tid; t < p.n2 / 2; t += kTinyThreads) {
            const int i = 2 * j * (t / j) + (t % j);
            const bool desc = ((i & kk) == 0);
            const unsigned long long a = keys[i], b = keys[i + j];
            if (desc ? (a < b) : (a > b)) {
              keys[i] = b;
              keys[i + j] = a;
            }
          }
          __syncthreads();
        }
    }
    __syncthreads();
    TINY_MARK(3);
    // greedy_place (placement.cpp:240-299) into the placement and the shared copy of row 0
    if (p.greedy_parallel)
      greedy_detail::greedy_walk_block<G>(L, NE, G, sA, p.members, s_nM, nullptr, p.anchor, sorted, m, p.placement,
                                          row0, nullptr, gsm);
    else
      greedy_detail::greedy_walk_block<0>(L, NE, G, sA, p.members, s_nM, nullptr, p.anchor, sorted, m, p.placement,
                                          row0, nullptr, gsm);
    __syncthreads();
    TINY_MARK(4);
    for (int i = tid; i < m; i += kTinyThreads) p.cands[i] = row0[i];
    // row 0 scored by the whole CTA, with small_candidate's arithmetic: same-GPU pair weight,
    // per-layer GPU loads (shared u64 atomics, exact), max |load - ideal|, feasibility
    unsigned long long* ld = keys;                         // [L][G] (the sort's keys are spent)
    uint32_t* cnt0 = reinterpret_cast<uint32_t*>(lists);   // [G]
    for (int i = tid; i < L * G; i += kTinyThreads) ld[i] = 0ull;
    if (tid < G) cnt0[tid] = 0u;
    if (tid == 0) {
      s_same0 = 0ull;
      s_dev0 = 0ull;
      s_bad0 = 0;
    }
    __syncthreads();
    unsigned long long sm0 = 0;
    bool bad0 = false;
    for (int r = tid; r < m; r += kTinyThreads) {
      const int l = r / NE, j = r - l * NE;
      const uint32_t pj = row0[r];
      if (pj < (uint32_t)G) {
        atomicAdd(&ld[l * G + pj], sA[r]);
        atomicAdd(&cnt0[pj], 1u);
      } else {
        bad0 = true;
      }
      if (l + 1 < L) {
        const uint32_t* Er = sE + (l * NE + j) * NE;
#pragma unroll
        for (int kk = 0; kk < NE; ++kk) sm0 += row0[(l + 1) * NE + kk] == pj ? (unsigned long long)Er[kk] : 0ull;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sm0 += __shfl_xor_sync(0xffffffffu, sm0, o);
    if (lane == 0 && sm0) atomicAdd(&s_same0, sm0);
    if (bad0) s_bad0 = 1;
    __syncthreads();
    double dv = 0.0;
    for (int r = tid; r < L * G; r += kTinyThreads) dv = fmax(dv, fabs(__dsub_rn((double)ld[r], sIdeal[r / G])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dv = fmax(dv, __shfl_xor_sync(0xffffffffu, dv, o));
    if (lane == 0) atomicMax(&s_dev0, (unsigned long long)__double_as_longlong(dv));  // dv >= 0: bits order
    __syncthreads();
    if (tid == 0) {
      bool infeasible = s_bad0 != 0;
      for (int q = 0; q < G; ++q) infeasible |= cnt0[q] != (uint32_t)(m / G);
      if (infeasible) {
        atomicOr(p.flags + 1, (uint32_t)kFlagInfeasible);
        atomicMin(p.bad_index, 0ll);
      }
    }
  }
  // score this CTA's candidates (CTA 0: the greedy row), cut and objective included
  // (eval_finish_kernel: cut = tokens * k * (L-1) * k - same; objective = alpha * D + beta * cut,
  // placement.cpp:83, two roundings, no FMA contraction), then the CTA's best (objective, index)
  __shared__ double w_best[kTinyThreads / 32];
  __shared__ long long w_idx[kTinyThreads / 32];
  unsigned long long tot = 0;  // tokens * k = sum_j A(0, j)
#pragma unroll
  for (int j = 0; j < NE; ++j) tot += sA[j];
  const unsigned long long total = tot * (unsigned long long)(L - 1) * (unsigned long long)p.k;
  const int64_t c = blockIdx.x == 0 ? (warp == 0 ? 0 : -1) : 1 + (int64_t)(blockIdx.x - 1) * (kTinyThreads / 32) + warp;
  long long my_idx = -1;
  double my_obj = 0.0;
  if (c >= 0 && c < p.C) {
    const SmallScore r = blockIdx.x == 0 ? SmallScore{s_same0, __longlong_as_double((long long)s_dev0)}
                                         : small_candidate<NE, G>(L, sE, sA, sIdeal, p.cands + c * m, c, 0,
                                                                  p.flags + 1, p.bad_index);
    const unsigned long long cu = total - r.same;
    const double cd = (double)cu;
    my_obj = __dadd_rn(__dmul_rn(p.alpha, r.dev), __dmul_rn(p.beta, cd));
    my_idx = c;
    if (lane == 0) {
      if (cu > (1ull << 53)) atomicOr(p.flags + 1, (uint32_t)kFlagOverflow);
      D[c] = r.dev;
      p.scores[p.C + c] = cd;
      p.scores[2 * p.C + c] = my_obj;
    }
  }
  if (blockIdx.x == 0) TINY_MARK(5);
  if (lane == 0) {
    w_best[warp] = my_obj;
    w_idx[warp] = my_idx;
  }
  __syncthreads();
  __shared__ int s_last;
  if (tid == 0) {
    double b = 0.0;
    long long bi = -1;
    for (int w = 0; w < kTinyThreads / 32; ++w)  // ascending candidate order: strict < keeps the lowest index
      if (w_idx[w] >= 0 && (bi < 0 || w_best[w] < b)) {
        b = w_best[w];
        bi = w_idx[w];
      }
    p.best[2 * blockIdx.x] = __double_as_longlong(b);
    p.best[2 * blockIdx.x + 1] = bi;
    __threadfence();
    s_last = (atomicAdd(p.ticket, 1u) - kTicketBase) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  TINY_MARK(6);
  __threadfence();
  // the last CTA: argmin over the CTAs' bests (lowest index among minima), flags read back
  __shared__ double bv[kTinyThreads];
  __shared__ long long bix[kTinyThreads];
  double best = 0.0;
  long long besti = -1;
  for (int b = tid; b < (int)gridDim.x; b += kTinyThreads) {
    const long long i2 = __ldcg(p.best + 2 * b + 1);
    const double v2 = __longlong_as_double(__ldcg(p.best + 2 * b));
    if (i2 >= 0 && (besti < 0 || v2 < best || (v2 == best && i2 < besti))) {
      best = v2;
      besti = i2;
    }
  }
  bv[tid] = best;
  bix[tid] = besti;
  __syncthreads();
  for (int s = kTinyThreads / 2; s > 0; s >>= 1) {
    if (tid < s) {
      const double v2 = bv[tid + s];
      const long long i2 = bix[tid + s];
      const long long i1 = bix[tid];
      if (i2 >= 0 && (i1 < 0 || v2 < bv[tid] || (v2 == bv[tid] && i2 < i1))) {
        bv[tid] = v2;
        bix[tid] = i2;
      }
    }
    __syncthreads();
  }
  TINY_MARK(7);
  if (p.ring) {
    // the packed results straight into mapped host memory ([argmin | |M| | pad | error words |
    // M | greedy], gimbal_pass_enqueue): no device-to-host copy on the stream behind the pass
    __shared__ int32_t* slot;
    __shared__ uint32_t f0, f1;
    if (tid == 0) {
      const uint32_t seq = *p.ring_seq;
      *p.ring_seq = seq + 1;
      slot = p.ring + (size_t)(seq % (uint32_t)p.ring_slots) * (size_t)(6 + 2 * m);
      f0 = atomicOr(p.flags, 0u);
      f1 = atomicOr(p.flags + 1, 0u);
    }
    __syncthreads();
    const int nM = __ldcg(p.n_members);
    if (tid == 0) {
      const long long am = bix[0];
      slot[0] = (int32_t)(am & 0xffffffffll);
      slot[1] = (int32_t)(am >> 32);
      slot[2] = nM;
      slot[3] = 0;
      slot[4] = (int32_t)f0;
      slot[5] = (int32_t)f1;
    }
    for (int i = tid; i < nM; i += kTinyThreads) slot[6 + i] = __ldcg(p.members + i);
    for (int i = tid; i < m; i += kTinyThreads) slot[6 + m + i] = __ldcg(p.placement + i);
    __threadfence_system();
  }
  if (tid == 0) {
    *p.argmin = bix[0];
    // ready for the next launch: no memset node per pass
    *p.bad_index = 0x7f7f7f7f7f7f7f7fll;
    *p.ticket = kTicketBase;
    if (p.flags_out) {
      __threadfence();
      p.flags_out[0] = atomicOr(p.flags, 0u);
      p.flags_out[1] = atomicOr(p.flags + 1, 0u);
    }
  }
}

}  // namespace

cudaError_t sort_u64_desc(unsigned long long* keys, int64_t n, cudaStream_t s) {
  if (n <= 1) return cudaSuccess;
  if (n <= kSortLocal) {
    bitonic_small_kernel<<<1, 1024, 0, s>>>(keys, (int)n);
    return cudaGetLastError();
  }
  const int64_t blocks = n / kSortLocal;
  bitonic_local_kernel<<<(unsigned)blocks, 1024, 0, s>>>(keys, n, 0, 0, true);
  for (int64_t k = 2 * kSortLocal; k <= n; k <<= 1) {
    for (int64_t j = k >> 1; j >= kSortLocal; j >>= 1) {
      const int grid = (int)std::min<int64_t>(4 * 1184, (n / 2 + 255) / 256);
      bitonic_global_kernel<<<grid, 256, 0, s>>>(keys, n, k, j);
    }
    bitonic_local_kernel<<<(unsigned)blocks, 1024, 0, s>>>(keys, n, k, k, false);
  }
  return cudaGetLastError();
}

size_t eval_scratch_bytes(int64_t C) {
  return (size_t)C * sizeof(unsigned long long) + sizeof(long long) * 2;
}

// Candidate slices per cell block: at least ~4 CTAs per SM in total, at most one per 32 candidates.
static unsigned candidate_splits(int64_t cell_ctas, int64_t C) {
  const int64_t want = (4 * 148 + cell_ctas - 1) / cell_ctas;
  const int64_t most = (C + kEvalCands - 1) / kEvalCands;
  return (unsigned)std::max<int64_t>(1, std::min(want, most));
}

// same[0..C) = 0 and the lowest infeasible index = "none" (a huge value) before any range runs
cudaError_t launch_eval_prepare(int64_t C, unsigned long long* scratch_same, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(scratch_same, 0, (size_t)C * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  return cudaMemsetAsync(scratch_same + C, 0x7f, sizeof(long long), s);  // 0x7f7f...7f
}

// Same-GPU weights and deviations of candidates [base, base + C) (pointers already offset to the
// range); bad_index / flags are shared by all ranges of one batch.
cudaError_t launch_eval_range(int L, int ne, int g, const unsigned long long* A, const unsigned long long* E,
                              const uint8_t* cands, int64_t C, int64_t base, unsigned long long* same, double* D,
                              uint32_t* flags, long long* bad_index, bool small_cells,
                              const unsigned long long* device_max_cell, cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  const int64_t m = (int64_t)L * ne;
  cudaError_t e = cudaSuccess;
  // width decided on the device: the small-cell form and the generic form both launch, guarded
  const bool guarded = device_max_cell != nullptr;
  if (guarded) small_cells = true;
  const WidthGuard g_small{device_max_cell, 1}, g_any{device_max_cell, 0};
  bool small_ran = false;
  if (!guarded && small_cells && L > 1 && L <= 256 && (L - 1) * ne * ne * 4 <= 32 * 1024 && !GIMBAL_KNOB("GIMBAL_EVAL_NO_SMALL")) {
    auto kern = ne == 8 && g == 8   ? eval_small_kernel<8, 8>
              : ne == 8 && g == 4   ? eval_small_kernel<8, 4>
              : ne == 8 && g == 2   ? eval_small_kernel<8, 2>
              : ne == 16 && g == 8  ? eval_small_kernel<16, 8>
              : ne == 16 && g == 4  ? eval_small_kernel<16, 4>
              : ne == 16 && g == 16 ? eval_small_kernel<16, 16>
                                    : nullptr;
    if (kern) {
      const size_t smem = (((size_t)(L - 1) * ne * ne * 4 + 15) & ~(size_t)15) + (size_t)L * 8 + (size_t)L * ne * 8;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<(unsigned)((C + 7) / 8), 256, smem, s>>>(L, A, E, cands, C, base, same, D, flags, bad_index);
      return cudaGetLastError();
    }
  }
  const bool fast = small_cells && ne % 32 == 0 && 256 % ne == 0;
  // tensor cores: E byte planes x one-hot assignment (eval_mma.cu); a handful of candidates (the
  // greedy row scored after the overlapped walk) is cheaper on the integer path, which reads E once
  // instead of building every unit's byte planes (DS-V3: 8.5 us vs 0.12 ms for the one row)
  if (small_cells && eval_mma_supported(L, ne, g, cands, C) && !(C <= 8 && ne % 32 == 0 && 256 % ne == 0)) {
    e = launch_eval_mma(L, ne, g, E, cands, C, same, g_small, s);
    if (e != cudaSuccess) return e;
    small_ran = true;
  } else if (L > 1 && fast) {
    const int64_t rows = (int64_t)(L - 1) * ne;
    const int rows_per_cta = kEvalCellsPerCta / ne;
    const int64_t ctas = (rows + rows_per_cta - 1) / rows_per_cta;
    const int64_t span = (std::min<int64_t>(m, rows_per_cta + 2 * ne) + 15) & ~15ll;
    const size_t smem = (size_t)kEvalCands * (size_t)span;
    e = cudaFuncSetAttribute(eval_same_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    eval_same_fast_kernel<<<dim3((unsigned)ctas, candidate_splits(ctas, C)), kEvalThreads, smem, s>>>(
        L, ne, E, cands, C, m, same, g_small);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    small_ran = true;
  }
  if (L > 1 && (!small_ran || guarded)) {  // any cell width (guarded: only when a cell >= 2^27)
    const int64_t nE = (int64_t)(L - 1) * ne * ne;
    const int64_t ctas = (nE + kEvalCellsPerCta - 1) / kEvalCellsPerCta;
    // staged span per candidate: rows of this CTA plus the next layer
    const int64_t max_span = std::min<int64_t>(m, (int64_t)kEvalCellsPerCta / ne + 3 * ne);
    const size_t smem = (size_t)kEvalCands * (size_t)max_span;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(eval_same_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    eval_same_kernel<<<dim3((unsigned)ctas, candidate_splits(ctas, C)), kEvalThreads, smem, s>>>(
        L, ne, E, cands, C, m, same, small_ran ? g_any : WidthGuard{});
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (g <= 8 && L <= 248 && !GIMBAL_KNOB("GIMBAL_EVAL_DEV_ATOMIC")) {
    auto kern = g <= 1 ? eval_dev_bins_kernel<1> : g <= 2 ? eval_dev_bins_kernel<2> : g <= 4 ? eval_dev_bins_kernel<4>
                : eval_dev_bins_kernel<8>;
    // eight 16 KB CTAs per SM need a large shared-memory carveout
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)C, 256, 0, s>>>(L, ne, g, A, cands, m, D, flags, bad_index, base);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  } else {
    const int threads = 256;
    const size_t smem = (size_t)(threads / 32) * g * 8 + (size_t)g * 4 + 8;
    e = cudaFuncSetAttribute(eval_dev_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    eval_dev_kernel<<<(unsigned)C, threads, smem, s>>>(L, ne, g, A, cands, m, D, flags, bad_index, base);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_eval_costs(int L, int ne, int g, const unsigned long long* A,
                              const unsigned long long* E, const uint8_t* cands, int64_t C,
                              double alpha, double beta, unsigned long long* scratch_same,
                              double* D, double* cut, double* obj, long long* argmin,
                              uint32_t* flags, bool small_cells, const unsigned long long* device_max_cell,
                              cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  cudaError_t e = launch_eval_prepare(C, scratch_same, s);
  if (e != cudaSuccess) return e;
  return launch_eval_range(L, ne, g, A, E, cands, C, 0, scratch_same, D, flags,
                           reinterpret_cast<long long*>(scratch_same + C), small_cells, device_max_cell, s);
}

cudaError_t launch_max_cell(const unsigned long long* E, int64_t n, unsigned long long* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256));
  max_cell_kernel<<<grid, 256, 0, s>>>(E, n, out);
  return cudaGetLastError();
}

cudaError_t launch_eval_excess(int L, int ne, int g, const unsigned long long* A, const uint8_t* cands, int64_t C,
                               double* excess, uint32_t* flags, cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  const size_t smem = (size_t)8 * g * 8 + (size_t)L * 8;
  cudaError_t e = cudaFuncSetAttribute(eval_excess_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  eval_excess_kernel<<<(unsigned)C, 256, smem, s>>>(L, ne, g, A, cands, (int64_t)L * ne, excess, flags);
  return cudaGetLastError();
}

cudaError_t launch_eval_finish(int64_t C, int L, int ne, int k, const unsigned long long* A, double alpha,
                               double beta, const unsigned long long* same, const double* D, double* cut,
                               double* obj, long long* argmin, uint32_t* flags, cudaStream_t s) {
  eval_finish_kernel<<<1, 1024, 0, s>>>(C, L, ne, k, A, alpha, beta, same, D, cut, obj, argmin, flags);
  return cudaGetLastError();
}

cudaError_t launch_affinity_keys(int L, int ne, const unsigned long long* E,
                                       double threshold, unsigned long long* keys, int64_t n_pad,
                                       uint32_t* flags, cudaStream_t s) {
  const int64_t n = (int64_t)(L - 1) * ne * ne;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 1184, (n_pad + 255) / 256));
  affinity_keys_kernel<<<grid, 256, 0, s>>>(L, ne, E, threshold, keys, n, n_pad, flags);
  return cudaGetLastError();
}

// Reduces (L-1)*ne^2 cells to the sorted top-K keys in `a`/`b` ping-pong buffers (each >=
// ceil(n/2048)*K keys); returns the buffer holding the final sorted K keys.
cudaError_t launch_affinity_topk(int L, int ne, const unsigned long long* E, double threshold, int K,
                                 unsigned long long* a, unsigned long long* b, uint32_t* flags,
                                 unsigned long long** result, cudaStream_t s) {
  const int64_t n = (int64_t)(L - 1) * ne * ne;
  if (K <= kRegTopK && !GIMBAL_KNOB("GIMBAL_TOPK_SORT")) {
    // a/b hold >= n_pad / 2 keys each (n_pad = next pow2 of n >= 2 * 296 * 8 here, else 1 block)
    int grid = (int)std::min<int64_t>(296, (n + kRegThreads * 16 - 1) / (kRegThreads * 16));
    grid = std::max(grid, 1);
    const int kk = K <= 4 ? 4 : kRegTopK;  // keys kept per list (>= K, the caller reads K of them)
    (kk == 4 ? topk_reg_kernel<true, 4> : topk_reg_kernel<true, kRegTopK>)<<<grid, kRegThreads, 0, s>>>(
        E, n, threshold, a, flags);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (grid == 1) {
      *result = a;
      return cudaSuccess;
    }
    (kk == 4 ? topk_reg_kernel<false, 4> : topk_reg_kernel<false, kRegTopK>)<<<1, kRegThreads, 0, s>>>(
        a, (int64_t)grid * kk, 0.0, b, flags);
    *result = b;
    return cudaGetLastError();
  }
  int64_t blocks = (n + kSortLocal - 1) / kSortLocal;
  topk_segment_kernel<true><<<(unsigned)blocks, 1024, 0, s>>>(E, n, threshold, K, a, flags);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t cur = blocks * K;
  unsigned long long* src = a;
  unsigned long long* dst = b;
  do {  // at least one pass so the survivors come out globally sorted
    blocks = (cur + kSortLocal - 1) / kSortLocal;
    topk_segment_kernel<false><<<(unsigned)blocks, 1024, 0, s>>>(src, cur, 0.0, K, dst, flags);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cur = blocks * K;
    std::swap(src, dst);
  } while (blocks > 1);
  *result = src;
  return cudaSuccess;
}

cudaError_t launch_affinity_select(int L, int ne, const unsigned long long* sorted_keys,
                                   int64_t n_keys, int32_t top_e, int32_t capacity,
                                   uint32_t* member_bits, int32_t* out, int32_t* n_out,
                                   cudaStream_t s) {
  affinity_select_kernel<<<1, 256, 0, s>>>(L, ne, sorted_keys, n_keys, top_e, capacity,
                                           member_bits, out, n_out);
  return cudaGetLastError();
}

cudaError_t launch_greedy_keys(int64_t m, const unsigned long long* A, const uint32_t* anchored,
                               unsigned long long* keys, int64_t n_pad, uint32_t* flags,
                               cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 1184, (n_pad + 255) / 256));
  greedy_keys_kernel<<<grid, 256, 0, s>>>(m, A, anchored, keys, n_pad, flags);
  return cudaGetLastError();
}

size_t tiny_scratch_bytes(int64_t C) {
  return eval_scratch_bytes(C) + (size_t)16 * (size_t)(2 + (C - 1 + kTinyThreads / 32 - 1) / (kTinyThreads / 32));
}

// The fused small-shape pass (tiny_pass_kernel), or cudaErrorNotSupported when the shape does not
// fit it (n_e in {8, 16} with a matching n_gpus, (L-1) n_e^2 u32 cells <= 32 KB, m <= 2048,
// 0 <= top_e <= 8).  `same` holds tiny_scratch_bytes(C); the caller guarantees every E cell < 2^32.
cudaError_t launch_tiny_pass(int L, int ne, int g, int k, double threshold, int top_e, int capacity, int anchor,
                             const unsigned long long* E, unsigned long long* A_out, uint8_t* cands, int64_t C,
                             double alpha, double beta, double* scores, long long* argmin, int32_t* placement,
                             int32_t* members, int32_t* n_members, uint32_t* flags, unsigned long long* same,
                             bool init_scratch, uint32_t* flags_out, int32_t* ring, uint32_t* ring_seq,
                             int ring_slots, cudaStream_t s) {
  const int64_t m = (int64_t)L * ne;
  if (L < 2 || L > 256 || m > 2048 || (int64_t)(L - 1) * ne * ne * 4 > 32 * 1024 || top_e < 0 ||
      top_e > kRegTopK || C < 1 || GIMBAL_KNOB("GIMBAL_NO_TINY_PASS"))
    return cudaErrorNotSupported;
  TinyPass p;
  p.L = L;
  p.k = k;
  p.threshold = threshold;
  p.top_e = top_e;
  p.capacity = capacity;
  p.anchor = anchor;
  int n2 = 1;
  while (n2 < m) n2 <<= 1;
  p.n2 = n2;
  bool parallel = false;
  const size_t gbytes = greedy_detail::greedy_smem_bytes(L, g, m, &parallel);
  p.greedy_parallel = parallel ? 1 : 0;
  p.E = E;
  p.A_out = A_out;
  p.cands = cands;
  p.C = C;
  p.alpha = alpha;
  p.beta = beta;
  p.scores = scores;
  p.argmin = argmin;
  p.placement = placement;
  p.members = members;
  p.n_members = n_members;
  p.flags = flags;
  p.same = same;
  p.bad_index = reinterpret_cast<long long*>(same + C);
  p.ticket = reinterpret_cast<uint32_t*>(same + C + 1);
  p.best = reinterpret_cast<long long*>(same + C + 2);  // 2 words per CTA (tiny_scratch_words)
  p.flags_out = flags_out;
  p.ring = ring;
  p.ring_seq = ring_seq;
  p.ring_slots = ring_slots;
  cudaError_t e = cudaSuccess;
  if (init_scratch) {  // bad index and ticket; every launch leaves them so for the next one
    e = cudaMemsetAsync(same + C, 0x7f, 2 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
  }
  const int KT = top_e <= 4 ? 4 : kRegTopK;
  auto pick = [&](auto k4, auto k8) { return KT == 4 ? k4 : k8; };
  void (*kern)(const TinyPass) = nullptr;
  size_t tables = 0;
  if (ne == 8) {
    tables = tiny_extra_offset<8>(L);
    kern = g == 8   ? pick(tiny_pass_kernel<8, 8, 4>, tiny_pass_kernel<8, 8, kRegTopK>)
         : g == 4   ? pick(tiny_pass_kernel<8, 4, 4>, tiny_pass_kernel<8, 4, kRegTopK>)
         : g == 2   ? pick(tiny_pass_kernel<8, 2, 4>, tiny_pass_kernel<8, 2, kRegTopK>)
                    : nullptr;
  } else if (ne == 16) {
    tables = tiny_extra_offset<16>(L);
    kern = g == 8   ? pick(tiny_pass_kernel<16, 8, 4>, tiny_pass_kernel<16, 8, kRegTopK>)
         : g == 4   ? pick(tiny_pass_kernel<16, 4, 4>, tiny_pass_kernel<16, 4, kRegTopK>)
         : g == 16  ? pick(tiny_pass_kernel<16, 16, 4>, tiny_pass_kernel<16, 16, kRegTopK>)
                    : nullptr;
  }
  if (!kern) return cudaErrorNotSupported;
  const size_t smem = tables + tiny_prep_bytes(n2, KT, (int)m) + gbytes;
  if (smem > 160 * 1024) return cudaErrorNotSupported;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)(1 + (C - 1 + kTinyThreads / 32 - 1) / (kTinyThreads / 32));
  kern<<<grid, kTinyThreads, smem, s>>>(p);
  return cudaGetLastError();
}


#ifdef GIMBAL_AB_KNOBS
extern "C" int gimbal_debug_tiny_profile(unsigned long long* out16) {
  return cudaMemcpyFromSymbol(out16, gimbal_gpu::g_tiny_prof, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : 1;
}
#endif

}  // namespace gimbal_gpu
