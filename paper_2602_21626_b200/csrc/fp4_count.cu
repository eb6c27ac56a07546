// Transition counting for 256-expert top-8 traces (DeepSeek-V3 class) on the block-scaled FP4
// tensor cores: tcgen05.mma.kind::mxf4, the densest MMA the sm_100a tensor core offers.
//
// E_l = X_l^T X_{l+1} (moe.cpp:179-188: every slot pairing counted).  The multi-hot operands are
// stored as e2m1 nibbles (0x2 = 1.0; every other nibble 0) with all block scale factors 2^0, so
// each product is 1 x 1 and the fp32 accumulator holds the exact pair count (integers < 2^24:
// units are capped well below that).  One CTA work unit = (layer pair l, half h of layer l's
// experts, token range):  D[m][n] = sum_t A[m][t] B[n][t], A = experts 128h..128h+127 of layer l,
// B = all 256 experts of layer l+1, M = 128, N = 256, K = 64 tokens per instruction; the
// accumulator is 256 of the 512 TMEM columns and the scale factors sit in columns 256-287.
//
// Operand layout: block-scaled FP4 operands must be K-major (tokens contiguous per expert row).
// Core matrix = 8 expert rows x 32 tokens (16 bytes per row); the four 32-token chunks of a
// 256-token tile are 128 B apart (LBO) and 8-row expert groups 1 KB apart (SBO).  A token sets
// its experts' nibbles with shared-memory atomicOr (a 32-bit word holds 8 tokens of one expert
// row); each stage is zeroed one tile ahead with 16-byte stores.  Token-layer id words arrive by
// TMA (2-D box of layers (l & ~1) .. +3 over the token-major trace viewed as [T][L] u64; a box
// must start 16-byte aligned in the row), so no transposition pass runs.
//
// Measured on B200 at DS-V3 shape (profiles/r1c_fp4_vs_u15.md): bit-exact, but 223 ms per 64 Mi
// tokens against 106 ms for the shared-memory u15 counter, so it is opt-in
// (GIMBAL_COUNT_PATH=fp4).  The tensor core is not the limit (25% active): building K-major
// nibble operands costs about as many shared-memory wavefronts per token-pair as counting them
// directly (zeroing 1.5, half-filtered atomicOr 1.6, id loads 0.9 per token), with a block-wide
// barrier per tile on top.  Zero-filling stages with out-of-bounds TMA boxes and two-lanes-per-
// token layouts were both slower (372 ms).
//
// A token that repeats an expert within layer l or l+1 (multiplicity > 1, never produced by the
// generator but legal input) is left out of the operands and its pairings are added straight to
// the u64 tensor by the CTA owning half h of its layer-l ids.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kNe = 256;
constexpr int kTok = 256;                          // tokens per tile (four K = 64 instructions)
constexpr int kStages = 3;
constexpr int kIdSlots = 3;
constexpr int kThreads = 2 * kTok;                 // two threads per token of a tile
constexpr int kIdCols = 4;                         // TMA box: layers (l & ~1) .. +3 (box starts 16-B aligned)
constexpr int kATile = 128 * kTok / 2;             // 16 KB: 128 experts x 256 tokens x 4 bit
constexpr int kBTile = 256 * kTok / 2;             // 32 KB
constexpr int kStageBytes = kATile + kBTile;
constexpr int kIdSlotBytes = kTok * kIdCols * 8;   // 8 KB
constexpr int kSmemBytes = kStages * kStageBytes + kIdSlots * kIdSlotBytes;
constexpr int kLbo = 128;                          // 32-token chunk stride
constexpr int kSbo = 128 * (kTok / 32);            // 8-expert group stride
constexpr uint32_t kSfCol = 256;                   // scale factors in TMEM columns 256 .. 287
constexpr int64_t kMaxRangeTokens = (1 << 24) - kTok;  // fp32 accumulators stay exact
struct Fp4Params {
  int L;
  int combos;              // 2 * (L - 1): (pair, half)
  int64_t n_units, range_tokens, T;
  uint32_t idesc;
};

__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fffu);
  d |= (uint64_t)((kLbo >> 4) & 0x3fffu) << 16;  // K direction: next 32-token chunk
  d |= (uint64_t)((kSbo >> 4) & 0x3fffu) << 32;  // M/N direction: next 8-expert group
  d |= (uint64_t)1 << 46;                         // descriptor version (sm_100); SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ void mma_mxf4(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate, uint32_t tsfa, uint32_t tsfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(tsfa), "r"(tsfb));
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

__device__ __forceinline__ void tmem_st16(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}

// 32-bit word of expert row r, token t in a K-major FP4 tile, and the bits of t's 1.0 nibble
__device__ __forceinline__ uint32_t nib_word(uint32_t r, uint32_t t) {
  return (r >> 3) * (kSbo / 4) + (t >> 5) * (kLbo / 4) + (r & 7) * 4 + ((t & 31) >> 3);
}
__device__ __forceinline__ uint32_t nib_one(uint32_t t) { return 2u << (4 * (t & 7)); }

__global__ void __launch_bounds__(kThreads, 1)
    count_fp4_kernel(const __grid_constant__ CUtensorMap tmap, Fp4Params prm, unsigned long long* __restrict__ E) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kStages + 1];
  __shared__ uint64_t id_bars[kIdSlots];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned long long* ids = reinterpret_cast<const unsigned long long*>(smem + kStages * kStageBytes);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s <= kStages; ++s) mbar_init(&bars[s], 1);
    for (int s = 0; s < kIdSlots; ++s) mbar_init(&id_bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // stage 0 zeroed before the first tile; the others one tile ahead of their use
  static_assert(kStageBytes % (16 * kThreads) == 0, "zeroing splits evenly");
  for (int i = tid; i < kStageBytes / 16; i += kThreads) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (warp < 4) {  // every block scale factor = 2^0 (ue8m0 127) in columns kSfCol .. kSfCol + 31
    const uint32_t lanes = (uint32_t)(warp * 32) << 16;
    tmem_st16(tmem + lanes + kSfCol, 0x7f7f7f7fu);
    tmem_st16(tmem + lanes + kSfCol + 16, 0x7f7f7f7fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tsfa = tmem + kSfCol, tsfb = tmem + kSfCol + 16;

  uint32_t it_global = 0, fills = 0, final_waits = 0;
  const int tok = tid & (kTok - 1);
  const bool role_a = tid < kTok;  // A ids (this half of layer l) + B slots 0-1; else B slots 2-7
  // slot order rotated by token (one funnel shift per word): a hot expert, usually drawn into the
  // same slot by every token, reaches the shared words at different steps
  const uint32_t rot = 8u * ((uint32_t)tok & 7u);
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int combo = (int)(unit % prm.combos);
    const int64_t range = unit / prm.combos;
    const int l = combo >> 1;
    const uint32_t h = (uint32_t)(combo & 1);
    const int64_t t_begin = range * prm.range_tokens;
    const int64_t t_end = min(prm.T, t_begin + prm.range_tokens);
    const int n_tiles = (int)((t_end - t_begin + kTok - 1) / kTok);
    unsigned long long* El = E + (int64_t)l * kNe * kNe;
    // id tiles by TMA into a kIdSlots ring, kIdSlots - 1 tiles ahead (fill index = fill0 + tile);
    // a slot is refilled only after the per-tile barrier that follows its last reader
    const uint32_t fill0 = fills;
    auto fetch = [&](int it) {  // thread 0
      const uint32_t slot = (fill0 + (uint32_t)it) % kIdSlots;
      mbar_arrive_expect_tx(&id_bars[slot], kIdSlotBytes);
      tma_load_2d(smem + kStages * kStageBytes + slot * kIdSlotBytes, &tmap, &id_bars[slot], l & ~1,
                  (int)(t_begin + (int64_t)it * kTok));
    };
    if (tid == 0)
      for (int i = 0; i < min(n_tiles, kIdSlots - 1); ++i) fetch(i);
    fills += (uint32_t)n_tiles;
    for (int it = 0; it < n_tiles; ++it, ++it_global) {
      const uint32_t use = fill0 + (uint32_t)it;
      mbar_wait(&id_bars[use % kIdSlots], (use / kIdSlots) & 1);
      const int s = it_global % kStages;
      uint32_t* a_w = reinterpret_cast<uint32_t*>(smem + s * kStageBytes);
      uint32_t* b_w = a_w + kATile / 4;
      if (t_begin + (int64_t)it * kTok + tok < t_end) {
        const unsigned long long* row = ids + ((use % kIdSlots) * kTok + tok) * kIdCols;
        unsigned long long cur, nxt;
        if (l & 1) {  // words 1, 2 of the row
          cur = row[1];
          nxt = row[2];
        } else {      // words 0, 1: one 16-byte load
          const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(row);
          cur = w.x;
          nxt = w.y;
        }
        const uint32_t one = nib_one((uint32_t)tok);
        const unsigned long long nxt_r = (nxt >> rot) | (nxt << ((64u - rot) & 63u));
        if (role_a) {
          if (has_dup8(cur) | has_dup8(nxt)) {  // multiplicity: straight to the u64 tensor
#pragma unroll 1
            for (int a = 0; a < 8; ++a) {
              const uint32_t j = id_byte(cur, a);
              if ((j >> 7) != h) continue;
#pragma unroll 1
              for (int b = 0; b < 8; ++b) atomicAdd(El + j * kNe + id_byte(nxt, b), 1ull);
            }
          } else {
            const unsigned long long cur_r = (cur >> rot) | (cur << ((64u - rot) & 63u));
#pragma unroll
            for (int a = 0; a < 8; ++a) {
              const uint32_t j = id_byte(cur_r, a);
              if ((j >> 7) == h) atomicOr(a_w + nib_word(j & 127u, (uint32_t)tok), one);
            }
          }
#pragma unroll
          for (int b = 0; b < 2; ++b) atomicOr(b_w + nib_word(id_byte(nxt_r, b), (uint32_t)tok), one);
        } else {
#pragma unroll
          for (int b = 2; b < 8; ++b) atomicOr(b_w + nib_word(id_byte(nxt_r, b), (uint32_t)tok), one);
        }
      }
      // zero the next tile's stage once the MMAs that read it (tile it_global + 1 - kStages) are done
      {
        const uint32_t gn = it_global + 1;
        const int sn = gn % kStages;
        if (gn >= kStages) mbar_wait(&bars[sn], ((gn / kStages) - 1) & 1);
        uint4* z = reinterpret_cast<uint4*>(smem + sn * kStageBytes);
#pragma unroll
        for (int i = 0; i < kStageBytes / 16 / kThreads; ++i) z[tid + i * kThreads] = make_uint4(0, 0, 0, 0);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(a_w), b0 = smem_u32(b_w);
#pragma unroll
        for (int kk = 0; kk < kTok / 64; ++kk)
          mma_mxf4(tmem, kmajor_desc(a0 + kk * 2 * kLbo), kmajor_desc(b0 + kk * 2 * kLbo), prm.idesc,
                   (it > 0 || kk > 0) ? 1u : 0u, tsfa, tsfb);
        mma_commit(&bars[s]);
        if (it + kIdSlots - 1 < n_tiles) fetch(it + kIdSlots - 1);
      }
    }
    // all MMAs of the unit done -> counts to E (fp32 accumulators hold exact integers)
    if (tid == 0) mma_commit(&bars[kStages]);
    mbar_wait(&bars[kStages], final_waits & 1);
    ++final_waits;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
      const uint32_t j = h * 128u + (uint32_t)(warp * 32 + lane);  // TMEM lane = expert of layer l
      unsigned long long* rowE = El + (int64_t)j * kNe;
      for (int c0 = 0; c0 < kNe; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float f = __uint_as_float(v[c]);
          if (f != 0.0f) atomicAdd(rowE + c0 + c, (unsigned long long)f);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  }
  // drain: the last commit of each stage barrier that no zeroing pass waited for
  for (uint32_t d = 1; d <= (uint32_t)kStages - 1 && d <= it_global; ++d) {
    const uint32_t g = it_global - d;
    mbar_wait(&bars[g % kStages], (g / kStages) & 1);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace

bool fp4_count_supported(int L, int ne, int k, int id_bytes, const void* ids, int64_t T) {
  return ne == kNe && k == 8 && L > 1 && (L & 1) == 0 && id_bytes == 1 &&
         (reinterpret_cast<uintptr_t>(ids) & 15) == 0 && T < (int64_t)INT32_MAX;
}

cudaError_t launch_count_fp4(int L, int sms, const uint8_t* trace, int64_t T, unsigned long long* E,
                             cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  CUtensorMap tmap;
  if (!encode_trace_map(&tmap, trace, T, L, kIdCols, kTok)) return cudaErrorNotSupported;
  Fp4Params prm;
  prm.L = L;
  prm.combos = 2 * (L - 1);
  prm.T = T;
  // idesc (kind::mxf4): a/b = E2M1 (1) K-major, scale = UE8M0, N = 256 (>>3 at bit 17),
  // M = 128 (>>4 at bit 24), K = 64, scale-factor ids 0
  prm.idesc = (1u << 7) | (1u << 10) | ((uint32_t)(kNe >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
  // ranges so that combos x ranges is just under a whole number of waves of persistent CTAs
  int64_t best_r = 1;
  double best_eff = 0.0;
  for (int64_t r = 1; r <= 64; ++r) {
    const int64_t per = (T + r - 1) / r;
    if (per > kMaxRangeTokens) continue;
    const int64_t units = r * prm.combos;
    const int64_t waves = (units + sms - 1) / sms;
    const double eff = (double)units / (double)(waves * sms) - 0.002 * (double)r;  // epilogue cost per range
    if (eff > best_eff) {
      best_eff = eff;
      best_r = r;
    }
  }
  int64_t per = (T + best_r - 1) / best_r;
  per = (per + kTok - 1) / kTok * kTok;
  prm.range_tokens = per;
  prm.n_units = ((T + per - 1) / per) * prm.combos;
  const int grid = (int)std::min<int64_t>(prm.n_units, sms);
  cudaError_t e = cudaFuncSetAttribute(count_fp4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e != cudaSuccess) return e;
  count_fp4_kernel<<<grid, kThreads, kSmemBytes, s>>>(tmap, prm, E);
  return cudaGetLastError();
}

}  // namespace gimbal_gpu
