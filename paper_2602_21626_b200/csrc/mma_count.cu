// Transition counting on the 5th-generation tensor cores (tcgen05, kind::i8) for n_e <= 128.
//
// E_l = X_l^T X_{l+1}, where X_l is the T x n_e multi-hot matrix of layer l's routing choices
// (X_l(t, e) = number of slots of token t at layer l that chose e).  Every product of the
// reference's k x k pairing loop (moe.cpp:179-188) is one term of this contraction, multiplicity
// included, so the integer result is exactly the reference's E.
//
// Per CTA work unit = (group of P <= 4 consecutive layer pairs, token range).  For each tile of
// 128 tokens the CTA builds the P+1 layer tiles as u8 operands in shared memory, laid out
// MN-major (a token's 128 expert indicators contiguous, the canonical no-swizzle UMMA layout:
// core matrix = 16 experts x 8 tokens = 128 B), one elected thread issues
// tcgen05.mma.cta_group::1.kind::i8 (M = 128 experts j, N = 128 experts k, K = 32 tokens) into a
// per-pair s32 accumulator in tensor memory (4 x 128 of the 512 TMEM columns), and
// tcgen05.commit releases the stage through an mbarrier while the other stage is being built.
// At the end of the unit the accumulators are read back with tcgen05.ld and added to the u64 E.
//
// Dense work is n_e^2 MACs per token-pair against k^2 useful ones: 64x at Qwen3's 128 experts /
// top-8 and 114x at DS-V2-Lite's 64 / top-6, which the int8 tensor rate (~7.7 K MAC/clk/SM)
// absorbs with the shared-memory tile construction as the co-bottleneck.  At 256 experts the
// ratio is 1024x and the shared-memory counting kernels (ingest.cu) win instead.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace gimbal_gpu {

namespace {

#ifndef GIMBAL_MMA_TOK
#define GIMBAL_MMA_TOK 128
#endif
constexpr int kTok = GIMBAL_MMA_TOK;       // tokens per tile (MMA K, kTok / 32 instructions of 32)
constexpr int kRows = 128;                 // experts per tile row block (MMA M, N <= 128)
constexpr int kTileBytes = kTok * kRows;   // 16 KB u8 operand tile
#ifndef GIMBAL_MMA_PAIRS
// 4 pairs x 128 TMEM columns, 1 CTA per SM: at Qwen3 count 31.70 vs 32.13 ms and 27.1 vs 59.4 GB of DRAM
// reads for 2 pairs x 2 CTAs per SM (half the groups re-read each trace row; profiles/r2e_qwen3_geometry.txt)
#define GIMBAL_MMA_PAIRS 4
#endif
constexpr int kMaxPairs = GIMBAL_MMA_PAIRS;  // accumulators: kMaxPairs x 128 TMEM columns
constexpr int kTmemCols = kMaxPairs <= 2 ? 256 : 512;
#ifndef GIMBAL_MMA_CTAS
#define GIMBAL_MMA_CTAS (GIMBAL_MMA_PAIRS <= 2 ? 2 : 1)
#endif
#ifndef GIMBAL_MMA_STAGES
#define GIMBAL_MMA_STAGES 2
#endif
constexpr int kCtasPerSm = GIMBAL_MMA_CTAS;  // two CTAs (TMEM halves) overlap barrier stalls
constexpr int kStages = GIMBAL_MMA_STAGES;
constexpr int kThreads = (kMaxPairs + 1) * 128;            // one token-layer row per thread per 128 tokens
constexpr int kIdSlots = 3;                                 // TMA ring of id word tiles
constexpr int kIdCols = kMaxPairs + 2;                      // token-major box: 6 layers (16-B aligned start)
constexpr int kIdSlotWords = kIdCols * kTok;                // >= 5 layers x 128 tokens (layer-major)
constexpr int kSmemBytes = kStages * (kMaxPairs + 1) * kTileBytes + kIdSlots * kIdSlotWords * 8;
constexpr int kStageBytes = (kMaxPairs + 1) * kTileBytes;

struct MmaParams {
  int L, ne, N;      // N = MMA n (n_e rounded up to 16)
  int P;             // pairs per group
  int n_groups;
  int64_t n_units;
  int64_t range_tokens;  // tokens per unit
  int64_t T, ld;
  uint32_t idesc;
  uint32_t* flags;  // LM8: kFlagDuplicates from the transposition; token-major: id errors raised here
  uint32_t* pace;   // per-range pacing counters (token-major path), or null
  int pace_tiles;   // tiles per pacing epoch
};

// Shared-memory matrix descriptor: no swizzle, MN-major.  Core matrix = 8 K-rows of 16 bytes;
// K-groups (8 tokens) are LBO = 1024 B apart, MN-groups (16 experts) SBO = 128 B apart.
__device__ __forceinline__ uint64_t operand_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fffu);
  d |= (uint64_t)((1024u >> 4) & 0x3fffu) << 16;  // leading byte offset (K direction)
  d |= (uint64_t)((128u >> 4) & 0x3fffu) << 32;   // stride byte offset (MN direction)
  d |= (uint64_t)1 << 46;                          // descriptor version 1 (sm_100)
  return d;                                        // base offset 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// TM = ids come from the token-major trace through a 2-D tensor map (box: kIdCols layers from
// l0 & ~1 x 128 tokens; row tt of the box is token t0 + tt), with range and repeat checks done
// per row here; otherwise from the layer-major LM8 buffer X by 1-D bulk copies.
template <int K, bool TM>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    count_mma_kernel(const __grid_constant__ CUtensorMap tmap, MmaParams prm,
                     const unsigned long long* __restrict__ X, unsigned long long* __restrict__ E) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kStages + 1];
  __shared__ uint64_t id_bars[kIdSlots];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* ids = reinterpret_cast<unsigned long long*>(smem + kStages * kStageBytes);
  uint32_t fill_count = 0;  // id-ring fills issued (identical in every thread)

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s <= kStages; ++s) mbar_init(&bars[s], 1);
    for (int s = 0; s < kIdSlots; ++s) mbar_init(&id_bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  const int ne = prm.ne;
  const bool dup = !TM && (*prm.flags & kFlagDuplicates) != 0;  // repeated ids: count, else set
  bool bad = false;
  uint32_t it_global = 0;        // tiles issued by this CTA (stage = it % 2, commit index = it / 2)
  uint32_t final_waits = 0;      // commits of the end-of-unit barrier
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int group = (int)(unit % prm.n_groups);
    const int64_t range = unit / prm.n_groups;
    const int l0 = group * prm.P;
    const int np = min(prm.P, prm.L - 1 - l0);
    const int64_t t_begin = range * prm.range_tokens;
    const int64_t t_end = min(prm.T, t_begin + prm.range_tokens);
    const int n_tiles = (int)((t_end - t_begin + kTok - 1) / kTok);
    const int n_rows = (np + 1) * kTok;  // token-layer rows per tile
    // The LM8 words of a tile (np+1 layers x 128 tokens, 1 KB contiguous per layer) arrive by TMA
    // bulk copies into a 3-slot ring, two tiles ahead of construction.
    auto fetch = [&](int it) {
      const uint32_t slot = fill_count % kIdSlots;
      if (TM && threadIdx.x == 0) {
        // the groups of one token range read the same trace rows: keep them within an epoch of
        // each other so every row is fetched from HBM once and served to the others from L2
        if (prm.pace != nullptr && it > 0 && it % prm.pace_tiles == 0)
          pace_arrive_wait(prm.pace + range, (uint32_t)(prm.n_groups * (it / prm.pace_tiles)), kPaceTimeoutNs);
        const int64_t t0 = t_begin + (int64_t)it * kTok;
        mbar_arrive_expect_tx(&id_bars[slot], kTok * kIdCols * 8);
        tma_load_2d(ids + slot * kIdSlotWords, &tmap, &id_bars[slot], l0 & ~1, (int)t0);
      } else if (threadIdx.x == 0) {
        const int64_t t0 = t_begin + (int64_t)it * kTok;
        const uint32_t bytes = (uint32_t)(((min((int64_t)kTok, t_end - t0) * 8) + 15) & ~15ll);
        const uint32_t bar = smem_u32(&id_bars[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * (np + 1))
                     : "memory");
        for (int q = 0; q <= np; ++q) {
          const unsigned long long* src = X + (int64_t)(l0 + q) * prm.ld + t0;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(ids + slot * kIdSlotWords + q * kTok)),
                       "l"(src), "r"(bytes), "r"(bar)
                       : "memory");
        }
      }
      ++fill_count;
    };
    fetch(0);
    if (n_tiles > 1) fetch(1);
    for (int it = 0; it < n_tiles; ++it, ++it_global) {
      if (it + 2 < n_tiles) fetch(it + 2);
      const uint32_t use = fill_count - (uint32_t)min(2, n_tiles - 1 - it) - 1;  // fill index of tile it
      mbar_wait(&id_bars[use % kIdSlots], (use / kIdSlots) & 1);
      const unsigned long long* w_tile = ids + (use % kIdSlots) * kIdSlotWords;
      const int s = (int)(it_global % kStages);
      if (it_global >= kStages) mbar_wait(&bars[s], ((it_global / kStages) - 1) & 1);
      uint8_t* stage = smem + s * kStageBytes;
      const int64_t t0 = t_begin + (int64_t)it * kTok;
      // one thread per token-layer row: zero its 128 expert bytes (8 chunks, SBO apart), then
      // count its ids (read-modify-write keeps repeated ids' multiplicity)
      for (int r = threadIdx.x; r < n_rows; r += kThreads) {
        const int q = r / kTok, tt = r - q * kTok;
        uint8_t* row = stage + q * kTileBytes + (tt >> 3) * 1024 + (tt & 7) * 16;
        const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(row + c * 128) = z;
        if (t0 + tt < t_end) {
          const unsigned long long w =
              TM ? w_tile[tt * kIdCols + (l0 & 1) + q] : w_tile[q * kTok + tt];
          bool count = dup;
          if constexpr (TM) {
            if (has_ge8(w, (uint32_t)ne)) {  // out-of-range ids: flag, leave the row empty
              bad = true;
              continue;
            }
            count = has_dup8(w);
          }
#pragma unroll
          for (int a = 0; a < K; ++a) {
            const uint32_t e = (uint32_t)(w >> (8 * a)) & 0xffu;
            uint8_t* p = row + (e >> 4) * 128 + (e & 15);
            *p = count ? (uint8_t)(*p + 1) : (uint8_t)1;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = smem_u32(stage);
        for (int p = 0; p < np; ++p) {
#pragma unroll
          for (int kk = 0; kk < kTok / 32; ++kk) {
            const uint64_t a = operand_desc(base + p * kTileBytes + kk * 4 * 1024);
            const uint64_t bdesc = operand_desc(base + (p + 1) * kTileBytes + kk * 4 * 1024);
            mma_i8(tmem + p * kRows, a, bdesc, prm.idesc, (it > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit(&bars[s]);
      }
    }
    // all MMAs of this unit complete -> read the accumulators
    if (threadIdx.x == 0) mma_commit(&bars[kStages]);
    mbar_wait(&bars[kStages], final_waits & 1);
    ++final_waits;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
      const int j = warp * 32 + lane;  // accumulator row = TMEM lane = expert j of layer l
      for (int p = 0; p < np; ++p) {
        for (int c0 = 0; c0 < prm.N; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(p * kRows + c0), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (j < ne) {
            unsigned long long* row = E + ((int64_t)(l0 + p) * ne + j) * ne;
#pragma unroll
            for (int c = 0; c < 16; ++c)
              if (v[c] != 0u && c0 + c < ne) atomicAdd(row + c0 + c, (unsigned long long)v[c]);
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  }
  if (TM && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(prm.flags, (uint32_t)kFlagIdOutOfRange);
  // drain: every commit on the stage barriers has been waited for except the last one per stage
  for (uint32_t d = 1; d <= (uint32_t)kStages && d <= it_global; ++d) {
    const uint32_t g = it_global - d;
    mbar_wait(&bars[g % kStages], (g / kStages) & 1);
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

template <int K, bool TM>
cudaError_t launch_k(const CUtensorMap& tmap, const MmaParams& prm, const unsigned long long* X,
                     unsigned long long* E, cudaStream_t s, int grid) {
  auto kern = count_mma_kernel<K, TM>;
  const int smem = kSmemBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, s>>>(tmap, prm, X, E);
  return cudaGetLastError();
}

// Units = (group of kMaxPairs pairs, token range): ranges so that groups x ranges fills the SMs;
// s32 accumulators hold per-unit counts up to tokens * k^2 < 2^31.
MmaParams make_params(int L, int ne, int k, int sms, int64_t T, int64_t ld, uint32_t* flags, int* grid) {
  MmaParams prm;
  prm.L = L;
  prm.ne = ne;
  prm.N = (ne + 15) / 16 * 16;
  prm.P = kMaxPairs;
  prm.n_groups = (L - 1 + prm.P - 1) / prm.P;
  prm.T = T;
  prm.ld = ld;
  prm.flags = flags;
  prm.pace = nullptr;
  prm.pace_tiles = 0;
  // c = s32, a = b = u8, a and b MN-major, N >> 3 at bit 17, M >> 4 at bit 24
  prm.idesc = (2u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(prm.N >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
  int64_t ranges = std::max<int64_t>(1, kCtasPerSm * sms / prm.n_groups);
  const int64_t cap = ((int64_t)1 << 31) / ((int64_t)k * k) - kTok;
  int64_t per = (T + ranges - 1) / ranges;
  if (per > cap) per = cap;
  per = (per + kTok - 1) / kTok * kTok;
  ranges = (T + per - 1) / per;
  prm.range_tokens = per;
  prm.n_units = ranges * prm.n_groups;
  *grid = (int)std::min<int64_t>(prm.n_units, (int64_t)kCtasPerSm * sms);
  return prm;
}

}  // namespace

// Measured on B200 (profiles/r1_summary.md): the contraction beats shared-memory counting at
// n_e = 128 (Qwen3: 1.07 vs 1.28 ns/token) but not at n_e = 64 (DS-V2-Lite: 0.54 vs 0.45 ns),
// where the 128-row operand tiles are half padding.
bool mma_count_supported(int L, int ne, int k) { return L > 1 && k >= 1 && k <= 8 && ne > 64 && ne <= 128; }

cudaError_t launch_count_mma(int L, int ne, int k, int sms, const unsigned long long* X, int64_t T, int64_t ld,
                             unsigned long long* E, const uint32_t* flags, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  int grid = 0;
  const MmaParams prm = make_params(L, ne, k, sms, T, ld, const_cast<uint32_t*>(flags), &grid);
  CUtensorMap none{};
  switch (k) {
    case 1: return launch_k<1, false>(none, prm, X, E, s, grid);
    case 2: return launch_k<2, false>(none, prm, X, E, s, grid);
    case 3: return launch_k<3, false>(none, prm, X, E, s, grid);
    case 4: return launch_k<4, false>(none, prm, X, E, s, grid);
    case 5: return launch_k<5, false>(none, prm, X, E, s, grid);
    case 6: return launch_k<6, false>(none, prm, X, E, s, grid);
    case 7: return launch_k<7, false>(none, prm, X, E, s, grid);
    case 8: return launch_k<8, false>(none, prm, X, E, s, grid);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_count_mma_direct(int L, int ne, int sms, const uint8_t* trace, int64_t T,
                                    unsigned long long* E, uint32_t* flags, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  CUtensorMap tmap;
  if (!mma_count_supported(L, ne, 8) || !encode_trace_map(&tmap, trace, T, L, kIdCols, kTok))
    return cudaErrorNotSupported;
  int grid = 0;
  MmaParams prm = make_params(L, ne, 8, sms, T, 0, flags, &grid);
  // pacing needs every group of a range resident together: whole ranges per wave of units
  const int64_t ranges = prm.n_units / prm.n_groups;
  const int pt = pace_tiles(0);  // off: profiles/r2_pacing_ab.md
  if (pt > 0 && grid % prm.n_groups == 0 && ranges <= kPaceWords && prm.range_tokens >= 2 * pt * kTok) {
    prm.pace = flags + kPaceOffset;
    prm.pace_tiles = pt;
    cudaError_t e = cudaMemsetAsync(prm.pace, 0, (size_t)ranges * 4, s);
    if (e != cudaSuccess) return e;
  }
  return launch_k<8, true>(tmap, prm, nullptr, E, s, grid);
}

}  // namespace gimbal_gpu
