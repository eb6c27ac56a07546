// Transition counting for 256-expert top-8 traces (DeepSeek-V3 class) on CTA pairs with the
// block-scaled FP4 tensor cores: tcgen05.mma.cta_group::2.kind::mxf4, M = 256 x N = 256 x K = 64.
//
// E_l = X_l^T X_{l+1} (moe.cpp:179-188: every slot pairing counted) where X_l is the T x 256
// multi-hot of layer l.  A CTA pair owns one unit = (layer pair l, token range): CTA r holds the
// experts [128 r, 128 r + 128) of layer l as its half of A (M) and of layer l + 1 as its half of B
// (N), so each SM builds 128 + 128 operand rows per token instead of the 128 + 256 a one-SM
// M = 128 x N = 256 contraction needs (fp4_count.cu).  The leader CTA issues the MMAs; the
// accumulator (fp32, exact below 2^24: ranges are capped) is TMEM columns [0, 256) of both CTAs
// (rows = that CTA's 128 experts of layer l), the unit block scale factors (ue8m0 127 = 2^0)
// columns [256, 320).
//
// Operands: K-major e2m1 nibble tiles (1.0 = 0x2) of 256 tokens.  Token tt of a tile sits at word
// tt % 32 of its expert row, nibble tt / 32, so the 32 lanes of a builder warp (32 consecutive
// tokens) write 32 different words of a row; the 32-token K chunks are 144 B apart (a 16 B gap
// per chunk), which puts those 32 words on 32 different banks (a hot expert shared by the warp's
// tokens costs one wavefront, not eight).  A and B use the same token -> K mapping, so the
// contraction is unchanged.  Each builder thread owns one token: two id words from the TMA-staged
// trace rows (two-layer [256][2] boxes: one 16-byte load for even l, two 8-byte loads for odd l);
// builder warps 2-9 OR a nibble into the A half for each of the token's layer-l ids that falls in
// this CTA's half (about 4 of 8), warps 10-17 the same for layer l + 1 into the B half, and all 16
// take a 16-byte-store share of zeroing the stage two tiles ahead.
//
// Warp roles (576 threads per CTA): warp 0 lane 0 = TMA producer of the id tiles (each CTA loads
// its own), warp 1 = TMEM allocation + (leader CTA) the MMA issuer, warps 2-17 = builders (warps
// 2 + q and 10 + q build nibble q of every word), of which warps 2-5 (one per TMEM lane quarter) also drain
// the accumulator into the u64 tensor at the end of each unit.  Barriers: id_full / id_empty
// (TMA ring, per CTA), stage_full (both CTAs' builders -> the leader's issuer, remote arrives),
// stage_empty (tcgen05.commit multicast to both CTAs), acc_full (commit multicast, last tile of a
// unit) / acc_empty (both CTAs' drains -> the leader, before the next unit's first MMA).
//
// A token repeating an expert within layer l or l + 1 (multiplicity, legal input the generator
// never produces) is left out of the operands; the CTA owning half h of its layer-l ids adds its
// pairings straight to the u64 tensor.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kNe = 256;
constexpr int kTok = 256;                        // tokens per tile (four K = 64 MMAs)
constexpr int kStages = 4;                       // operand stages
constexpr int kIdSlots = 4;                      // id tile ring
constexpr int kBuilders = 16;                    // builder warps: 8 for A (layer l), 8 for B (layer l + 1)
constexpr int kThreads = (2 + kBuilders) * 32;
constexpr int kSbo = 128;                        // 8-expert row groups adjacent: row r at r * 16
constexpr int kLbo = 16 * 128 + 16;              // 32-token K chunk stride (2048 B + a 16 B gap)
constexpr int kHalfBytes = 8 * kLbo;             // 128 rows x 256 tokens, 16512 B
constexpr int kStageBytes = 2 * kHalfBytes;      // A half + B half
constexpr int kIdCols = 2;                       // TMA box: two layers (16 B per token; 16-B aligned start)
constexpr int kIdSlotBytes = 2 * kTok * kIdCols * 8;  // 8 KB: one box (even l) or two (odd l)
constexpr int kSmemBytes = kStages * kStageBytes + kIdSlots * kIdSlotBytes;
constexpr uint32_t kSfCol = 256;                 // scale factors: columns 256 .. 319
constexpr int64_t kMaxRangeTokens = (1 << 24) - kTok;
static_assert(kStageBytes % 16 == 0 && kHalfBytes % 16 == 0, "16-byte zeroing");

struct Fp4x2Params {
  int pairs;            // L - 1
  int64_t n_units;      // ranges x pairs, range-major
  int64_t range_tokens; // multiple of kTok
  int64_t T;
  uint32_t idesc;
};

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_index() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the leader CTA's (rank 0) copy of a barrier at the same shared offset
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
// Arrive on a (possibly remote) barrier of the pair without a release fence: a cluster-scope
// release compiles to MEMBAR.ALL.GPU (measured: a fifth of all stall samples).  What the waiter needs
// ordered is this CTA's own completed work -- operand stores made visible to the tensor core by
// each writer's fence.proxy.async, or TMEM reads retired by tcgen05.wait::ld -- before the arrive
// is issued, which those fences already guarantee.
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Zero the operand bytes of a stage (the 2048-byte chunk bodies of both halves; the 16-byte gaps
// only ever receive the out-of-half ORs and are never read): 4 x 16 B per builder thread.
__device__ __forceinline__ void zero_stage(uint8_t* stage, int btid) {
  static_assert(2 * 8 * 2048 / 16 == 4 * kBuilders * 32, "exact split");
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int v = btid + r * kBuilders * 32;       // 16-byte vector 0 .. 2047
    const int h = v >> 10, c = (v >> 7) & 7, o = v & 127;
    *reinterpret_cast<uint4*>(stage + h * kHalfBytes + c * kLbo + o * 16) = make_uint4(0, 0, 0, 0);
  }
}

__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fffu);
  d |= (uint64_t)((kLbo >> 4) & 0x3fffu) << 16;  // K direction: next 32-token chunk
  d |= (uint64_t)((kSbo >> 4) & 0x3fffu) << 32;  // M / N direction: next 8-expert group
  d |= (uint64_t)1 << 46;                         // descriptor version (sm_100); SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ void mma_mxf4_x2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate, uint32_t tsfa, uint32_t tsfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(tsfa), "r"(tsfb));
}

// completion of all prior MMAs of this thread -> arrive on `bar` in both CTAs of the pair
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
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

// byte offset of word w (tokens w + 32 q) of expert row r < 128 in a half tile: r * 16 plus a
// per-lane constant; the 16-byte gap per chunk puts word w of a row on bank (c + w) mod 32
__device__ __forceinline__ uint32_t lane_off(uint32_t w) { return (w >> 2) * kLbo + (w & 3) * 4; }

// For each of the 8 id bytes of w: x = id ^ (rank << 7) is < 128 exactly when the id falls in
// this CTA's half; min(x, 128) turns the other ids into "row 128", whose word at `base` + 2048 is the
// 16-byte gap after the chunk -- never read by the MMA -- so every lane issues its 8 ORs without a
// branch or predicate (ptxas turns predicated shared atomics into branch regions).
__device__ __forceinline__ void or_ids(unsigned long long w, uint32_t rank_bits, uint32_t base, uint32_t nib) {
  asm volatile(
      "{\n\t.reg .b32 lo, hi, x, a;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
#define GIMBAL_OR_ONE(SRC, SEL) \
  "prmt.b32 x, " SRC ", 0, " SEL "; xor.b32 x, x, %1; min.u32 x, x, 128; mad.lo.u32 a, x, 16, %2; red.shared.or.b32 [a], %3;\n\t"
      GIMBAL_OR_ONE("lo", "0x4440") GIMBAL_OR_ONE("lo", "0x4441") GIMBAL_OR_ONE("lo", "0x4442") GIMBAL_OR_ONE("lo", "0x4443")
      GIMBAL_OR_ONE("hi", "0x4440") GIMBAL_OR_ONE("hi", "0x4441") GIMBAL_OR_ONE("hi", "0x4442") GIMBAL_OR_ONE("hi", "0x4443")
#undef GIMBAL_OR_ONE
      "}" ::"l"(w), "r"(rank_bits), "r"(base), "r"(nib)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    count_fp4x2_kernel(const __grid_constant__ CUtensorMap tmap, Fp4x2Params prm, unsigned long long* __restrict__ E) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t id_full[kIdSlots], id_empty[kIdSlots];
  __shared__ uint64_t stage_full[kStages], stage_empty[kStages], zeroed[kStages];
  __shared__ uint64_t acc_full, acc_empty;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  uint8_t* ids_base = smem + kStages * kStageBytes;

  if (tid == 0) {
    for (int s = 0; s < kIdSlots; ++s) {
      mbar_init(&id_full[s], 1);
      mbar_init(&id_empty[s], kBuilders);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&stage_full[s], 2 * kBuilders);  // both CTAs' builder warps (leader's copy is used)
      mbar_init(&stage_empty[s], 1);
      mbar_init(&zeroed[s], kBuilders);  // every builder warp's share of zeroing the stage is done
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, 2 * 4);  // the four drain warps of both CTAs
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (warp >= 2 && warp < 6) {  // unit block scale factors in columns kSfCol .. kSfCol + 63
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
#pragma unroll
    for (int c = 0; c < 64; c += 16) tmem_st16(tmem + lanes + kSfCol + c, 0x7f7f7f7fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tsfa = tmem + kSfCol, tsfb = tmem + kSfCol + 32;

  const uint32_t ncl = cluster_count(), cl = cluster_index();
  if (warp == 0) {
    // ---------------- id tiles by TMA (this CTA's copy) ----------------
    if (lane == 0) {
      uint32_t f = 0;
      for (int64_t u = cl; u < prm.n_units; u += ncl) {
        const int l = (int)(u % prm.pairs);
        const int64_t t_begin = (u / prm.pairs) * prm.range_tokens;
        const int64_t t_end = min(prm.T, t_begin + prm.range_tokens);
        for (int64_t t0 = t_begin; t0 < t_end; t0 += kTok, ++f) {
          const uint32_t s = f % kIdSlots;
          if (f >= kIdSlots) mbar_wait(&id_empty[s], ((f / kIdSlots) - 1) & 1);
          // even l: layers (l, l + 1) as one [256][2] box; odd l: (l - 1, l) and (l + 1, l + 2)
          mbar_arrive_expect_tx(&id_full[s], kTok * 16 * ((l & 1) + 1));
          tma_load_2d(ids_base + s * kIdSlotBytes, &tmap, &id_full[s], l & ~1, (int)t0);
          if (l & 1) tma_load_2d(ids_base + s * kIdSlotBytes + kTok * 16, &tmap, &id_full[s], l + 1, (int)t0);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0 && lane == 0) {
      uint32_t it = 0, units = 0;
      for (int64_t u = cl; u < prm.n_units; u += ncl, ++units) {
        const int64_t t_begin = (u / prm.pairs) * prm.range_tokens;
        const int64_t t_end = min(prm.T, t_begin + prm.range_tokens);
        const uint32_t n_tiles = (uint32_t)((t_end - t_begin + kTok - 1) / kTok);
        // the previous unit's accumulator has been drained by both CTAs
        if (units > 0) wait_cluster(&acc_empty, (units - 1) & 1);
        for (uint32_t i = 0; i < n_tiles; ++i, ++it) {
          const uint32_t s = it % kStages;
          wait_cluster(&stage_full[s], (it / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(smem + s * kStageBytes), b0 = a0 + kHalfBytes;
#pragma unroll
          for (int kk = 0; kk < kTok / 64; ++kk)
            mma_mxf4_x2(tmem, kdesc(a0 + kk * 2 * kLbo), kdesc(b0 + kk * 2 * kLbo), prm.idesc,
                        (i > 0 || kk > 0) ? 1u : 0u, tsfa, tsfb);
          commit_both(&stage_empty[s]);
          if (i + 1 == n_tiles) commit_both(&acc_full);
        }
      }
    }
  } else {
    // ---------------- builders (+ accumulator drain on warps 2-5) ----------------
    // warps 2-9 set layer l's ids in the A half, warps 10-17 layer l + 1's in the B half
    const bool role_b = warp >= 2 + kBuilders / 2;
    const int q = (warp - 2) & (kBuilders / 2 - 1);
    const uint32_t nib = 2u << (4 * q);  // e2m1 1.0 at nibble q of the word
    const int bt = q * 32 + lane;        // this thread's token within a tile
    const int btid = tid - 64;           // 0 .. 511 among the builders
    const uint32_t rank_bits = rank << 7;
    const uint32_t leader_full0 = leader_addr(&stage_full[0]);
    for (int s0 = 0; s0 < 2; ++s0) {  // the first two stages; later ones two tiles ahead of use
      zero_stage(smem + s0 * kStageBytes, btid);
      __syncwarp();
      if (lane == 0) mbar_arrive(&zeroed[s0]);
    }
    const uint32_t leader_acc_empty = leader_addr(&acc_empty);
    uint32_t it = 0, units = 0;
    for (int64_t u = cl; u < prm.n_units; u += ncl, ++units) {
      const int l = (int)(u % prm.pairs);
      const int64_t t_begin = (u / prm.pairs) * prm.range_tokens;
      const int64_t t_end = min(prm.T, t_begin + prm.range_tokens);
      const uint32_t n_tiles = (uint32_t)((t_end - t_begin + kTok - 1) / kTok);
      unsigned long long* El = E + (int64_t)l * kNe * kNe;
      for (uint32_t i = 0; i < n_tiles; ++i, ++it) {
        const uint32_t slot = it % kIdSlots, s = it % kStages;
        mbar_wait(&id_full[slot], (it / kIdSlots) & 1);
        const unsigned long long* box = reinterpret_cast<const unsigned long long*>(ids_base + slot * kIdSlotBytes);
        unsigned long long cur = 0, nxt;
        if (role_b) {  // layer l + 1 only
          nxt = (l & 1) ? box[kTok * 2 + bt * 2] : box[bt * 2 + 1];
        } else if (l & 1) {  // 16-byte row stride: two 8-byte loads
          cur = box[bt * 2 + 1];
          nxt = box[kTok * 2 + bt * 2];
        } else {             // one 16-byte load
          const ulonglong2 v = reinterpret_cast<const ulonglong2*>(box)[bt];
          cur = v.x;
          nxt = v.y;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&id_empty[slot]);
        // this tile's stage was zeroed during tile it - 2 (the first two at the start)
        mbar_wait(&zeroed[s], (it / kStages) & 1);
        const uint32_t half = smem_u32(smem + s * kStageBytes) + (role_b ? kHalfBytes : 0u);
        if (t_begin + (int64_t)i * kTok + bt < t_end) {
          if (role_b) {
            // a token the A role sends to the u64 path contributes A row 0 to the MMA, so its
            // B nibbles are harmless: no duplicate check here
            or_ids(nxt, rank_bits, half + lane_off((uint32_t)lane), nib);
          } else if (has_dup8(cur) | has_dup8(nxt)) {  // multiplicity: straight to the u64 tensor
#pragma unroll 1
            for (int a = 0; a < 8; ++a) {
              const uint32_t j = id_byte(cur, a);
              if ((j >> 7) != rank) continue;
#pragma unroll 1
              for (int b = 0; b < 8; ++b) atomicAdd(El + j * kNe + id_byte(nxt, b), 1ull);
            }
          } else {
            or_ids(cur, rank_bits, half + lane_off((uint32_t)lane), nib);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive_remote(leader_full0 + s * 8);
        // zero the stage of tile it + 2 once its previous MMAs (tile it + 2 - kStages) are done
        {
          const uint32_t g2 = it + 2, s2 = g2 % kStages;
          if (g2 >= kStages) mbar_wait(&stage_empty[s2], ((g2 / kStages) - 1) & 1);
          zero_stage(smem + s2 * kStageBytes, btid);
          __syncwarp();
          if (lane == 0) mbar_arrive(&zeroed[s2]);
        }
      }
      if (warp < 6) {
        // drain: this CTA's 128 rows (experts 128 rank + TMEM lane) x 256 columns -> u64 E
        mbar_wait(&acc_full, units & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t quarter = (uint32_t)(warp & 3);
        const uint32_t j = rank * 128u + quarter * 32u + (uint32_t)lane;
        unsigned long long* rowE = El + (int64_t)j * kNe;
        for (int c0 = 0; c0 < kNe; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + ((quarter * 32u) << 16) + (uint32_t)c0, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float f = __uint_as_float(v[c]);
            if (f != 0.0f) atomicAdd(rowE + c0 + c, (unsigned long long)f);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive_remote(leader_acc_empty);
      }
    }
  }
  // teardown: the last unit was drained (its MMAs completed) before the drain warps got here
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace

bool fp4x2_count_supported(int L, int ne, int k, int id_bytes, const void* ids, int64_t T) {
  return ne == kNe && k == 8 && L > 1 && (L & 1) == 0 && id_bytes == 1 &&
         (reinterpret_cast<uintptr_t>(ids) & 15) == 0 && T < (int64_t)INT32_MAX;
}

cudaError_t launch_count_fp4x2(int L, int sms, const uint8_t* trace, int64_t T, unsigned long long* E,
                               cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  CUtensorMap tmap;
  if (!encode_trace_map(&tmap, trace, T, L, kIdCols, kTok)) return cudaErrorNotSupported;
  const int clusters = std::max(1, sms / 2);
  Fp4x2Params prm;
  prm.pairs = L - 1;
  prm.T = T;
  // idesc (kind::mxf4): a/b = E2M1 (1) K-major, scale factors UE8M0, N = 256 (>>3 at bit 17),
  // M = 256 (>>4 at bit 24: a CTA pair), scale-factor ids 0
  prm.idesc = (1u << 7) | (1u << 10) | ((uint32_t)(kNe >> 3) << 17) | (1u << 23) | ((uint32_t)(256 >> 4) << 24);
  // token ranges so that pairs x ranges is just under a whole number of waves of clusters; each
  // unit drains a 256 x 256 accumulator (64 Ki global atomics), so ranges stay long
  int64_t best_r = 1;
  double best_eff = -1.0;
  for (int64_t r = 1; r <= 512; ++r) {
    const int64_t per = (T + r - 1) / r;
    if (per > kMaxRangeTokens) continue;
    if (r > 1 && per < 64 * kTok) break;
    const int64_t units = r * prm.pairs;
    const int64_t waves = (units + clusters - 1) / clusters;
    const double eff = (double)units / (double)(waves * clusters) - 0.0005 * (double)r;
    if (eff > best_eff) {
      best_eff = eff;
      best_r = r;
    }
  }
  int64_t per = (T + best_r - 1) / best_r;
  per = (per + kTok - 1) / kTok * kTok;
  prm.range_tokens = per;
  prm.n_units = ((T + per - 1) / per) * prm.pairs;
  const int grid = 2 * (int)std::min<int64_t>(prm.n_units, clusters);
  cudaError_t e = cudaFuncSetAttribute(count_fp4x2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e != cudaSuccess) return e;
  count_fp4x2_kernel<<<grid, kThreads, kSmemBytes, s>>>(tmap, prm, E);
  return cudaGetLastError();
}

}  // namespace gimbal_gpu
