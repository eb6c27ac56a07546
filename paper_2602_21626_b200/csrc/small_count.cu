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

// The k x k increments of one token's layer pairs, ids checked per token-layer (a pair with an
// out-of-range id on either side is left out and flagged).
template <int K>
__device__ __forceinline__ bool small_count_row(const uint8_t* row, int L, int ne, uint32_t* tab) {
  bool bad = false;
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
  return bad;
}

// Top-2 rows with a compile-time expert count NE (8 or 16; L even): the row is read as 32-bit
// words (two layers each), all ids checked at once, and each pair's four cell addresses are one
// add of precomputed row / column offsets (half the instructions of the byte-wise loop, which is
// issue-bound at Mixtral).  Rows with an out-of-range id take small_count_row.
template <int NE>
__device__ __forceinline__ bool small_count_row2(const uint32_t* row, int L, uint32_t* tab) {
  constexpr uint32_t kBad = 0x01010101u * (uint32_t)(0x100 - NE);  // any id byte >= NE
  constexpr int kShift = NE == 8 ? 3 : 4;
  uint32_t acc = 0;
  for (int w = 0; w < L / 2; ++w) acc |= row[w];
  if (acc & kBad) return small_count_row<2>(reinterpret_cast<const uint8_t*>(row), L, NE, tab);
  const uint32_t tab_s = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  uint32_t w = row[0];
  // byte offsets: column k -> 4k, row j -> 4 NE j
  uint32_t j0 = (w & 0xffu) << (2 + kShift), j1 = ((w >> 8) & 0xffu) << (2 + kShift);
  uint32_t base = tab_s;
  for (int lw = 0; lw < L / 2; ++lw) {
    // pair (2 lw, 2 lw + 1): columns from the high half of word lw
    const uint32_t k0 = ((w >> 16) & 0xffu) << 2, k1 = (w >> 24) << 2;
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + j0 + k0) : "memory");
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + j0 + k1) : "memory");
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + j1 + k0) : "memory");
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + j1 + k1) : "memory");
    base += NE * NE * 4;
    if (lw + 1 == L / 2) break;
    // pair (2 lw + 1, 2 lw + 2): rows = those columns, columns from the low half of word lw + 1
    w = row[lw + 1];
    const uint32_t n0 = (w & 0xffu) << 2, n1 = ((w >> 8) & 0xffu) << 2;
    const uint32_t r0 = k0 << kShift, r1 = k1 << kShift;
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + r0 + n0) : "memory");
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + r0 + n1) : "memory");
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + r1 + n0) : "memory");
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + r1 + n1) : "memory");
    base += NE * NE * 4;
    j0 = n0 << kShift;
    j1 = n1 << kShift;
  }
  return false;
}

// NE = 0: runtime expert count, byte-wise rows; NE > 0 (K = 2 only): small_count_row2.
template <int K, int NE, int THREADS>
__global__ void __launch_bounds__(THREADS)
    count_small_tm_kernel(int L, int ne, const uint8_t* __restrict__ trace, int64_t T, int row_bytes,
                          int stride, unsigned long long* __restrict__ E, uint32_t* __restrict__ flags) {
  constexpr int kSmallThreads = THREADS;
  extern __shared__ __align__(16) uint8_t sm[];
  const int cells = (L - 1) * ne * ne;
  uint32_t* tab = reinterpret_cast<uint32_t*>(sm);
  uint8_t* rows = sm + ((cells * 4 + 15) & ~15);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) tab[i] = 0u;
  bool bad = false;
  const bool vec = (row_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(trace) & 15) == 0;
  if constexpr (NE > 0) {
    // 16-byte rows (checked by the launcher): the next block's chunks are prefetched into
    // registers while this block is counted, so one CTA per SM keeps its loads in flight
    constexpr int kPf = 8;
    const int q = row_bytes >> 4;
    const int64_t step = (int64_t)gridDim.x * kSmallThreads;
    uint4 pre[kPf];
    auto load = [&](int64_t t0) {
      const int n = (int)min((int64_t)kSmallThreads, T - t0);
      const uint4* src = reinterpret_cast<const uint4*>(trace + t0 * row_bytes);
#pragma unroll
      for (int r = 0; r < kPf; ++r) {
        const int i = threadIdx.x + r * kSmallThreads;
        if (i < n * q) pre[r] = __ldcs(src + i);
      }
    };
    int64_t t0 = (int64_t)blockIdx.x * kSmallThreads;
    if (t0 < T) load(t0);
    for (; t0 < T; t0 += step) {
      const int n = (int)min((int64_t)kSmallThreads, T - t0);
      __syncthreads();  // the previous block's rows are consumed (and the table is zeroed)
#pragma unroll
      for (int r = 0; r < kPf; ++r) {
        const int i = threadIdx.x + r * kSmallThreads;
        if (i < n * q) {
          const int rr = i / q, w = i - rr * q;
          uint32_t* d = reinterpret_cast<uint32_t*>(rows + rr * stride + w * 16);
          d[0] = pre[r].x;
          d[1] = pre[r].y;
          d[2] = pre[r].z;
          d[3] = pre[r].w;
        }
      }
      __syncthreads();
      if (t0 + step < T) load(t0 + step);
      if (threadIdx.x < n)
        bad |= small_count_row2<NE>(reinterpret_cast<const uint32_t*>(rows + threadIdx.x * stride), L, tab);
    }
  } else {
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
        if constexpr (NE > 0)
          bad |= small_count_row2<NE>(reinterpret_cast<const uint32_t*>(row), L, tab);
        else
          bad |= small_count_row<K>(row, L, ne, tab);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cells; i += blockDim.x)
    if (tab[i]) atomicAdd(E + i, (unsigned long long)tab[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
}

// ---- Top-2 over 8 experts (Mixtral): one shared atomic per token-pair instead of four ----
// A token-layer's two ids form an unordered multiset t = {lo, hi} of 8 experts: tri(t) =
// hi (hi + 1) / 2 + lo, 36 values.  A token-pair (layers l, l+1) is one event (tri_l, tri_l+1) out of
// 36 x 36 = 1296, counted in a u16 histogram per pair (red.shared.add on packed halves).  At the end
//   E_l(j, k) = sum over the 8 multisets t containing j, the 8 t' containing k of
//               H_l(t, t') * m(j, t) * m(k, t'),   m(x, t) = multiplicity of x in t (1 or 2),
// exactly the reference's k x k pairing count with multiplicity (moe.cpp:179-188).  Rows with an
// out-of-range id take small_count_row into a per-CTA E table instead (flagged there).
constexpr int kEvThreads = 1024;
constexpr int kEvTri = 36;
constexpr int kEvBinWords = kEvTri * kEvTri / 2;  // 648 u32 words = 1296 u16 bins per layer pair
constexpr int kEvMaxBlocks = 63;                   // <= 64512 tokens per CTA: u16 bins cannot overflow

__device__ __forceinline__ uint32_t ev_tri(uint32_t a, uint32_t b) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  return ((hi * (hi + 1u)) >> 1) + lo;
}

// Both layers of a row word at once (bytes a0 b0 a1 b1, ids < 8): the two ids of each layer go to
// 16-bit lanes, min / max per lane (min.u16x2 / max.u16x2), one byte permute of the triangular-number
// table for both his: tri of layer 0 in the low half, of layer 1 in the high half.
__device__ __forceinline__ uint32_t ev_tri2(uint32_t w) {
  const uint32_t a = __byte_perm(w, 0u, 0x4240), b = __byte_perm(w, 0u, 0x4341);
  uint32_t lo, hi;
  asm("min.u16x2 %0, %1, %2;" : "=r"(lo) : "r"(a), "r"(b));
  asm("max.u16x2 %0, %1, %2;" : "=r"(hi) : "r"(a), "r"(b));
  return __byte_perm(0x06030100u, 0x1c150f0au, hi | (hi >> 8)) + lo;
}

__device__ __forceinline__ void ev_add(uint32_t hist_s, uint32_t bin) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(hist_s + (bin >> 1) * 4), "r"(1u << ((bin & 1u) << 4))
               : "memory");
}

// Q = 16-byte chunks per row (L = 8 Q layers of two ids).  Rows are staged with 16-byte stores at a
// stride of an odd number of chunks and read back with 16-byte loads (conflict-free per quarter
// warp); each thread then holds its token's whole row in registers.
template <int Q>
__global__ void __launch_bounds__(kEvThreads, 1)
    count_events8_kernel(const uint8_t* __restrict__ trace, int64_t T, unsigned long long* __restrict__ E,
                         uint32_t* __restrict__ flags) {
  constexpr int L = 8 * Q, pairs = L - 1, kRowBytes = 16 * Q;
  constexpr int kStride16 = (Q & 1) ? Q + 2 : Q + 1;  // odd
  static_assert(pairs * kEvTri * 8 * 4 <= kEvThreads * kStride16 * 16, "the expansion's G fits the row staging");
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm);  // [pairs][648]
  uint32_t* tab = hist + pairs * kEvBinWords;        // [pairs][64] cells of rows with bad ids
  uint4* rows = reinterpret_cast<uint4*>(tab + pairs * 64);
  for (int i = threadIdx.x; i < pairs * (kEvBinWords + 64); i += kEvThreads) hist[i] = 0u;
  bool bad = false;
  const uint32_t hist_s = static_cast<uint32_t>(__cvta_generic_to_shared(hist));
  const int64_t step = (int64_t)gridDim.x * kEvThreads;
  uint4 pre[Q];
  auto load = [&](int64_t t0) {
    const int n = (int)min((int64_t)kEvThreads, T - t0);
    const uint4* src = reinterpret_cast<const uint4*>(trace + t0 * kRowBytes);
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      const int i = threadIdx.x + r * kEvThreads;
      if (i < n * Q) pre[r] = __ldcs(src + i);
    }
  };
  int64_t t0 = (int64_t)blockIdx.x * kEvThreads;
  if (t0 < T) load(t0);
  for (; t0 < T; t0 += step) {
    const int n = (int)min((int64_t)kEvThreads, T - t0);
    __syncthreads();  // the previous block's rows are consumed (and the tables are zeroed)
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      const int i = threadIdx.x + r * kEvThreads;
      if (i < n * Q) {
        const int rr = i / Q, c = i - rr * Q;
        rows[rr * kStride16 + c] = pre[r];
      }
    }
    __syncthreads();
    if (t0 + step < T) load(t0 + step);
    if (threadIdx.x < n) {
      uint32_t w[4 * Q];
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        const uint4 v = rows[threadIdx.x * kStride16 + c];
        w[4 * c] = v.x;
        w[4 * c + 1] = v.y;
        w[4 * c + 2] = v.z;
        w[4 * c + 3] = v.w;
      }
      uint32_t acc = 0;
#pragma unroll
      for (int i = 0; i < 4 * Q; ++i) acc |= w[i];
      if (acc & 0xf8f8f8f8u) {
        bad |= small_count_row<2>(reinterpret_cast<const uint8_t*>(rows + threadIdx.x * kStride16), L, 8, tab);
      } else {
        uint32_t base = hist_s;
        uint32_t t2 = ev_tri2(w[0]);
#pragma unroll
        for (int lw = 0; lw < 4 * Q; ++lw) {
          const uint32_t tp = t2 & 0xffffu, tn = t2 >> 16;  // layers 2 lw, 2 lw + 1
          ev_add(base, tp * kEvTri + tn);
          base += kEvBinWords * 4;
          if (lw + 1 < 4 * Q) {
            t2 = ev_tri2(w[lw + 1]);
            ev_add(base, tn * kEvTri + (t2 & 0xffffu));  // layers 2 lw + 1, 2 lw + 2
            base += kEvBinWords * 4;
          }
        }
      }
    }
  }
  __syncthreads();
  // expand the events into the pair's 8 x 8 cells in two steps (no atomics; the row staging area
  // holds the intermediate):
  //   G_l(t, k) = sum over the 8 multisets t' containing k of H_l(t, t') m(k, t')   (36 x 8 per pair)
  //   E_l(j, k) = sum over the 8 multisets t containing j of m(j, t) G_l(t, k)
  // 72 bin reads per cell instead of 64 per cell of the one-step sum, 31 % fewer in all
  uint32_t* Gt = reinterpret_cast<uint32_t*>(rows);  // [pairs][36][8]
  for (int idx = threadIdx.x; idx < pairs * kEvTri * 8; idx += kEvThreads) {
    const int p = idx / (kEvTri * 8), r = idx - p * (kEvTri * 8), t = r >> 3, kk = r & 7;
    const uint32_t* H = hist + p * kEvBinWords;
    uint32_t g = 0;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const uint32_t bin = (uint32_t)t * kEvTri + ev_tri((uint32_t)kk, (uint32_t)y);
      const uint32_t c = (H[bin >> 1] >> ((bin & 1u) << 4)) & 0xffffu;
      g += y == kk ? 2u * c : c;
    }
    Gt[idx] = g;
  }
  __syncthreads();
  for (int cell = threadIdx.x; cell < pairs * 64; cell += kEvThreads) {
    const int p = cell >> 6, j = (cell >> 3) & 7, kk = cell & 7;
    const uint32_t* Gp = Gt + p * (kEvTri * 8);
    unsigned long long sum = tab[cell];
#pragma unroll
    for (int x = 0; x < 8; ++x)
      sum += (unsigned long long)(x == j ? 2u : 1u) * Gp[ev_tri((uint32_t)j, (uint32_t)x) * 8 + kk];
    if (sum) atomicAdd(E + cell, sum);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
}

size_t events8_smem(int L) {
  const int q = L / 8;
  const int stride16 = (q & 1) ? q + 2 : q + 1;
  return (size_t)(L - 1) * (kEvBinWords + 64) * 4 + (size_t)kEvThreads * stride16 * 16;
}

size_t small_smem(int L, int ne, int k, int threads = kSmallThreads) {
  const size_t table = ((size_t)(L - 1) * ne * ne * 4 + 15) & ~(size_t)15;
  return table + (size_t)threads * ((size_t)L * k + 4);
}

// Top-2 rows of 8 or 16 experts, L even, row stride an odd number of words: the word-wise kernel,
// 1024 threads and one CTA per SM (its flush adds every cell of the CTA's table to E with a global
// atomic, so fewer, larger CTAs mean fewer same-address atomics: 148 x 1984 at Mixtral instead of
// 1184 x 1984 with 256-thread CTAs).
constexpr int kSmall2Threads = 1024;
bool small2_applies(int L, int ne, int k, const uint8_t* trace) {
  return k == 2 && (ne == 8 || ne == 16) && (L * 2) % 16 == 0 && L * 2 <= 8 * 16 && ((L * 2 + 4) / 4) % 2 == 1 &&
         (reinterpret_cast<uintptr_t>(trace) & 15) == 0 && small_smem(L, ne, k, kSmall2Threads) <= 200 * 1024;
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
  if (ne == 8 && small2_applies(L, ne, k, trace) && L % 8 == 0 && L * k <= 64 && events8_smem(L) <= 200 * 1024 &&
      !GIMBAL_KNOB("GIMBAL_SMALL_BYTEWISE") && !GIMBAL_KNOB("GIMBAL_SMALL_NO_EVENTS")) {
    const int64_t blocks = (T + kEvThreads - 1) / kEvThreads;
    int64_t grid = std::min<int64_t>(sms, blocks);
    grid = std::max<int64_t>(grid, (blocks + kEvMaxBlocks - 1) / kEvMaxBlocks);  // u16 bins
    const size_t smem = events8_smem(L);
    auto go = [&](auto kern) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<(unsigned)grid, kEvThreads, smem, s>>>(trace, T, E, flags);
      return cudaGetLastError();
    };
    switch (L / 8) {
      case 1: return go(count_events8_kernel<1>);
      case 2: return go(count_events8_kernel<2>);
      case 3: return go(count_events8_kernel<3>);
      default: return go(count_events8_kernel<4>);
    }
  }
  if (small2_applies(L, ne, k, trace) && !GIMBAL_KNOB("GIMBAL_SMALL_BYTEWISE")) {
    const size_t smem = small_smem(L, ne, k, kSmall2Threads);
    int64_t grid = std::min<int64_t>(sms, (T + kSmall2Threads - 1) / kSmall2Threads);
    const int64_t min_grid = T * k * k / ((int64_t)1 << 31) + 1;  // u32 cells per CTA
    grid = std::max<int64_t>(grid, std::min<int64_t>(min_grid, (T + kSmall2Threads - 1) / kSmall2Threads));
    auto kern = ne == 8 ? count_small_tm_kernel<2, 8, kSmall2Threads> : count_small_tm_kernel<2, 16, kSmall2Threads>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, kSmall2Threads, smem, s>>>(L, ne, trace, T, L * k, L * k + 4, E, flags);
    return cudaGetLastError();
  }
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
    case 1: return go(count_small_tm_kernel<1, 0, kSmallThreads>);
    case 2: return go(count_small_tm_kernel<2, 0, kSmallThreads>);
    case 3: return go(count_small_tm_kernel<3, 0, kSmallThreads>);
    case 4: return go(count_small_tm_kernel<4, 0, kSmallThreads>);
    case 5: return go(count_small_tm_kernel<5, 0, kSmallThreads>);
    case 6: return go(count_small_tm_kernel<6, 0, kSmallThreads>);
    case 7: return go(count_small_tm_kernel<7, 0, kSmallThreads>);
    case 8: return go(count_small_tm_kernel<8, 0, kSmallThreads>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gimbal_gpu
