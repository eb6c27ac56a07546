// Transition counting on the tcgen05 tensor cores for 64-expert layers (DeepSeek-V2-Lite class),
// with two layers stacked into one 128-row operand.
//
// E_l = X_l^T X_{l+1} with X_l the T x 64 multi-hot matrix of layer l (moe.cpp:179-188 counts
// every slot pairing with multiplicity, which is exactly this contraction).  A 64-expert layer
// fills only half of a 128-row MMA operand, so instead of padding, one
//   tcgen05.mma.cta_group::1.kind::i8  M = 128, N = 64, K = 32 tokens
// takes A = [X_l ; X_{l+2}] (experts of layer l in rows 0-63, of layer l+2 in rows 64-127) and
// B = X_{l+1}:  accumulator rows 0-63 are E_l(j, k), rows 64-127 are X_{l+2}^T X_{l+1} =
// E_{l+1}^T.  Two layer pairs per instruction and no wasted MACs: a group of up to 16 pairs
// needs 8 MMAs into 8 x 64 of the 512 TMEM columns.
//
// Operands (u8, MN-major, no swizzle; core matrix = 8 tokens x 16 experts = 128 B): within a
// stage the even layers of the group (offsets 0, 2, 4, ...) sit side by side along MN, 512 B
// (4 core matrices) per layer, so the A operand of MMA i is the 1 KB window starting at even
// slot i; the odd layers form the B tile the same way.  One K-group (8 tokens) of a tile is
// slots x 512 B (the descriptor's K stride).
//
// Ids come straight from the token-major [T][L][k] uint8 trace: each 64-token tile's rows are one
// contiguous 1-D bulk copy (cp.async.bulk, mbarrier completion) into a 3-slot ring, two tiles
// ahead; one thread per token-layer row zeroes its 64 operand bytes and sets (or, with repeated
// ids, increments) one byte per slot.  Ids are range-checked here (kFlagIdOutOfRange, the row is
// left empty), so no transposition or validation pass precedes the kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kNe = 64;              // experts per layer (one half of the M = 128 operand)
#ifndef GIMBAL_STACK_TOK
#define GIMBAL_STACK_TOK 64
#endif
constexpr int kTok = GIMBAL_STACK_TOK;  // tokens per tile (K = 32 MMA steps), a power of two
constexpr int kSlotBytes = 512;      // one layer's 64 experts x 8 tokens (4 core matrices)
#ifndef GIMBAL_STACK_CTAS
#define GIMBAL_STACK_CTAS 1  // 2 (half the pairs per group, 2 stages): 4.95 vs 4.75 ms at DS-V2-Lite
#endif
constexpr int kCtasPerSm = GIMBAL_STACK_CTAS;             // CTAs per SM (TMEM and smem split)
#ifndef GIMBAL_STACK_MAXPAIRS
#define GIMBAL_STACK_MAXPAIRS (16 / GIMBAL_STACK_CTAS)
#endif
#ifndef GIMBAL_STACK_STAGES
#define GIMBAL_STACK_STAGES (GIMBAL_STACK_CTAS > 1 ? 2 : 3)
#endif
#ifndef GIMBAL_STACK_THREADS
#define GIMBAL_STACK_THREADS 512
#endif
constexpr int kMaxPairs = GIMBAL_STACK_MAXPAIRS;          // kMaxPairs / 2 accumulators of 64 TMEM columns
constexpr int kTmemCols = 512 / kCtasPerSm;
constexpr int kStages = GIMBAL_STACK_STAGES;
constexpr int kIdSlots = 3;
constexpr int kThreads = GIMBAL_STACK_THREADS;
constexpr int kTokShift = kTok == 128 ? 7 : 6;
static_assert(kTok == 64 || kTok == 128, "tile of 64 or 128 tokens");

struct StackParams {
  int L, k, row_bytes;    // trace row = L * k bytes per token
  int ppg, n_groups;      // pairs per group, groups
  int even_slots, odd_slots;
  int stage_bytes, id_slot_bytes;
  int64_t n_units, range_tokens, T;
  uint32_t idesc;
  uint32_t* flags;
  uint32_t* pace;  // per-range pacing counters (the groups of a range read the same rows), or null
  int pace_tiles;
};

__device__ __forceinline__ uint64_t operand_desc(uint32_t saddr, uint32_t k_stride) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fffu);
  d |= (uint64_t)((k_stride >> 4) & 0x3fffu) << 16;  // K-group (8 tokens) stride
  d |= (uint64_t)((128u >> 4) & 0x3fffu) << 32;       // MN stride between 16-expert core matrices
  d |= (uint64_t)1 << 46;                              // descriptor version (sm_100)
  return d;
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

template <int K>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    count_mma_stack_kernel(StackParams prm, const uint8_t* __restrict__ trace, unsigned long long* __restrict__ E) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kStages + 1];
  __shared__ uint64_t id_bars[kIdSlots];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ids = smem + kStages * prm.stage_bytes;

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

  const int row_bytes = prm.row_bytes;
  const uint32_t even_k = (uint32_t)prm.even_slots * kSlotBytes;  // K-group strides
  const uint32_t odd_k = (uint32_t)prm.odd_slots * kSlotBytes;
  const uint32_t even_tile = (kTok / 8) * even_k;
  bool bad = false;
  uint32_t fills = 0;        // id-ring fills issued (same in every thread)
  uint32_t it_global = 0;    // tiles issued (stage = it % kStages)
  uint32_t final_waits = 0;
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int group = (int)(unit % prm.n_groups);
    const int64_t range = unit / prm.n_groups;
    const int p0 = group * prm.ppg;
    const int np = min(prm.ppg, prm.L - 1 - p0);  // pairs p0 .. p0 + np - 1, layers p0 .. p0 + np
    const int n_mma = (np + 1) >> 1;
    const int64_t t_begin = range * prm.range_tokens;
    const int64_t t_end = min(prm.T, t_begin + prm.range_tokens);
    const int n_tiles = (int)((t_end - t_begin + kTok - 1) / kTok);
    const int n_rows = (np + 1) * kTok;

    auto fetch = [&](int it) {  // called by every thread (fills stays uniform)
      if (threadIdx.x == 0) {
        if (prm.pace != nullptr && it > 0 && it % prm.pace_tiles == 0)
          pace_arrive_wait(prm.pace + range, (uint32_t)(prm.n_groups * (it / prm.pace_tiles)), kPaceTimeoutNs);
        const uint32_t slot = fills % kIdSlots;
        uint8_t* dst = ids + slot * prm.id_slot_bytes;
        const int64_t t0 = t_begin + (int64_t)it * kTok;
        const int n = (int)min((int64_t)kTok, t_end - t0);
        const uint32_t bytes = (uint32_t)n * row_bytes;
        const uint32_t bulk = bytes & ~15u;
        const uint8_t* src = trace + t0 * row_bytes;
        for (uint32_t b = bulk; b < bytes; ++b) dst[b] = src[b];  // < 16 tail bytes of the last tile
        mbar_arrive_expect_tx(&id_bars[slot], bulk);
        if (bulk)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(dst)),
                       "l"(src), "r"(bulk), "r"(smem_u32(&id_bars[slot]))
                       : "memory");
      }
      ++fills;
    };
    fetch(0);
    if (n_tiles > 1) fetch(1);
    for (int it = 0; it < n_tiles; ++it, ++it_global) {
      if (it + 2 < n_tiles) fetch(it + 2);
      const uint32_t use = fills - (uint32_t)min(2, n_tiles - 1 - it) - 1;  // fill index of tile it
      mbar_wait(&id_bars[use % kIdSlots], (use / kIdSlots) & 1);
      const uint8_t* id_tile = ids + (use % kIdSlots) * prm.id_slot_bytes;
      const int s = it_global % kStages;
      if (it_global >= kStages) mbar_wait(&bars[s], ((it_global / kStages) - 1) & 1);
      uint8_t* stage = smem + s * prm.stage_bytes;
      uint8_t* odd = stage + even_tile;
      const int64_t t0 = t_begin + (int64_t)it * kTok;
      for (int r = threadIdx.x; r < n_rows; r += kThreads) {
        const int q = r >> kTokShift, tt = r & (kTok - 1);  // layer offset, token in tile
        uint8_t* row = ((q & 1) ? odd + (tt >> 3) * odd_k : stage + (tt >> 3) * even_k) + (q >> 1) * kSlotBytes +
                       (tt & 7) * 16;
        const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < kNe / 16; ++c) *reinterpret_cast<uint4*>(row + c * 128) = z;
        if (t0 + tt < t_end) {
          const uint8_t* p = id_tile + tt * row_bytes + (p0 + q) * K;
          uint32_t e[K];
#pragma unroll
          for (int a = 0; a < K; ++a) e[a] = p[a];
          bool oor = false, dup = false;
#pragma unroll
          for (int a = 0; a < K; ++a) {
            oor |= e[a] >= (uint32_t)kNe;
#pragma unroll
            for (int b = a + 1; b < K; ++b) dup |= e[a] == e[b];
          }
          if (oor) {  // out-of-range ids: flag, leave the row empty
            bad = true;
            continue;
          }
          if (dup) {
#pragma unroll
            for (int a = 0; a < K; ++a) row[(e[a] >> 4) * 128 + (e[a] & 15)] += 1;
          } else {
#pragma unroll
            for (int a = 0; a < K; ++a) row[(e[a] >> 4) * 128 + (e[a] & 15)] = 1;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ebase = smem_u32(stage), obase = smem_u32(odd);
#pragma unroll
        for (int kk = 0; kk < kTok / 32; ++kk) {
          for (int i = 0; i < n_mma; ++i) {
            const uint64_t a = operand_desc(ebase + kk * 4 * even_k + i * kSlotBytes, even_k);
            const uint64_t b = operand_desc(obase + kk * 4 * odd_k + i * kSlotBytes, odd_k);
            mma_i8(tmem + i * kNe, a, b, prm.idesc, (it > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit(&bars[s]);
      }
    }
    // all MMAs of the unit done -> accumulators to E
    if (threadIdx.x == 0) mma_commit(&bars[kStages]);
    mbar_wait(&bars[kStages], final_waits & 1);
    ++final_waits;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
      const int r = warp * 32 + lane;  // accumulator row (TMEM lane)
      for (int i = 0; i < n_mma; ++i) {
        const int pair = 2 * i + (r >> 6);  // rows 0-63: pair 2i (E), rows 64-127: pair 2i+1 (E^T)
        for (int c0 = 0; c0 < kNe; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(i * kNe + c0), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (pair < np) {
            unsigned long long* El = E + (int64_t)(p0 + pair) * kNe * kNe;
            const int x = r & (kNe - 1);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              if (v[c] == 0u) continue;
              unsigned long long* cell = (r < kNe) ? El + x * kNe + c0 + c : El + (c0 + c) * kNe + x;
              atomicAdd(cell, (unsigned long long)v[c]);
            }
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(prm.flags, (uint32_t)kFlagIdOutOfRange);
  // every stage barrier's last commit not yet waited for
  for (uint32_t d = 1; d <= (uint32_t)kStages && d <= it_global; ++d) {
    const uint32_t g = it_global - d;
    mbar_wait(&bars[g % kStages], (g / kStages) & 1);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

bool make_params(int L, int k, int sms, int max_smem, int64_t T, uint32_t* flags, StackParams* prm, int* grid,
                 size_t* smem) {
  const int pairs = L - 1;
  if (pairs < 1) return false;
  prm->L = L;
  prm->k = k;
  prm->row_bytes = L * k;
  prm->id_slot_bytes = (kTok * prm->row_bytes + 127) & ~127;
  // fewest groups (each re-reads the trace rows) whose stages fit shared memory
  for (prm->n_groups = (pairs + kMaxPairs - 1) / kMaxPairs;; ++prm->n_groups) {
    if (prm->n_groups > pairs) return false;
    prm->ppg = (pairs + prm->n_groups - 1) / prm->n_groups;
    // even layer offsets 0, 2, .., ppg plus the lower half of the last MMA's A window when ppg
    // is odd (its rows are read, never written back); odd offsets 1, 3, .., < ppg + 1
    prm->even_slots = prm->ppg / 2 + 1 + (prm->ppg & 1);
    prm->odd_slots = (prm->ppg + 1) / 2;
    prm->stage_bytes = (prm->even_slots + prm->odd_slots) * (kTok / 8) * kSlotBytes;
    *smem = (size_t)kStages * prm->stage_bytes + (size_t)kIdSlots * prm->id_slot_bytes;
    if (*smem <= (size_t)(max_smem / kCtasPerSm) - 2048) break;
  }
  prm->T = T;
  prm->flags = flags;
  prm->pace = nullptr;
  prm->pace_tiles = 0;
  // c = s32, a = b = u8, both MN-major; N >> 3 at bit 17, M >> 4 at bit 24
  prm->idesc = (2u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(kNe >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // ranges x groups ~ 2 waves of units; s32 accumulators hold tokens * k^2 < 2^31 per unit
  int64_t ranges = std::max<int64_t>(1, (2 * sms + prm->n_groups - 1) / prm->n_groups);
  const int64_t cap = ((int64_t)1 << 31) / ((int64_t)k * k) - kTok;
  int64_t per = (T + ranges - 1) / ranges;
  per = std::max<int64_t>(per, 16 * kTok);
  if (per > cap) per = cap;
  per = (per + kTok - 1) / kTok * kTok;
  ranges = (T + per - 1) / per;
  prm->range_tokens = per;
  prm->n_units = ranges * prm->n_groups;
  *grid = (int)std::min<int64_t>(prm->n_units, (int64_t)kCtasPerSm * sms);
  return true;
}

template <int K>
cudaError_t launch_k(const StackParams& prm, const uint8_t* trace, unsigned long long* E, cudaStream_t s, int grid,
                     size_t smem) {
  auto kern = count_mma_stack_kernel<K>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, s>>>(prm, trace, E);
  return cudaGetLastError();
}

}  // namespace

bool mma_stack_supported(int L, int ne, int k, int id_bytes, const void* ids) {
  return ne == kNe && L > 1 && k >= 1 && k <= 8 && id_bytes == 1 && (reinterpret_cast<uintptr_t>(ids) & 15) == 0;
}

cudaError_t launch_count_mma_stack(int L, int ne, int k, int sms, int max_smem, const uint8_t* trace, int64_t T,
                                   unsigned long long* E, uint32_t* flags, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (!mma_stack_supported(L, ne, k, 1, trace)) return cudaErrorNotSupported;
  StackParams prm;
  int grid = 0;
  size_t smem = 0;
  if (!make_params(L, k, sms, max_smem, T, flags, &prm, &grid, &smem)) return cudaErrorNotSupported;
  // pacing needs every group of a range resident together: whole ranges per wave of units
  const int64_t ranges = prm.n_units / prm.n_groups;
  const int pt = pace_tiles(0);  // off: profiles/r2_pacing_ab.md
  if (pt > 0 && prm.n_groups > 1 && grid % prm.n_groups == 0 && ranges <= kPaceWords &&
      prm.range_tokens >= 2 * pt * kTok) {
    prm.pace = flags + kPaceOffset;
    prm.pace_tiles = pt;
    cudaError_t e = cudaMemsetAsync(prm.pace, 0, (size_t)ranges * 4, s);
    if (e != cudaSuccess) return e;
  }
  switch (k) {
    case 1: return launch_k<1>(prm, trace, E, s, grid, smem);
    case 2: return launch_k<2>(prm, trace, E, s, grid, smem);
    case 3: return launch_k<3>(prm, trace, E, s, grid, smem);
    case 4: return launch_k<4>(prm, trace, E, s, grid, smem);
    case 5: return launch_k<5>(prm, trace, E, s, grid, smem);
    case 6: return launch_k<6>(prm, trace, E, s, grid, smem);
    case 7: return launch_k<7>(prm, trace, E, s, grid, smem);
    case 8: return launch_k<8>(prm, trace, E, s, grid, smem);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gimbal_gpu
