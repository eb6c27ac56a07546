// Placement scoring on the tensor cores (tcgen05.mma kind::i8): the "same-GPU" weight of every
// candidate placement, i.e. the complement of eval_cost's cut (placement.cpp:58-85).
//
// For layer pair l and candidate c with GPU assignment P_c:
//     same_c(l) = sum_j sum_k E_l(j, k) [P_c(l, j) == P_c(l+1, k)]
//               = sum_j X_c[j][P_c(l, j)],   X_c = E_l * H_c,   H_c[k][p] = [P_c(l+1, k) == p],
// a GEMM against the one-hot matrix of the next layer's assignment followed by a per-row gather.
// E cells are < 2^27 on this path (the host's small-cell test), so E_l is split into four u8 byte
// planes and each plane is an exact u8 x u8 -> s32 product (<= 255 * n_e per accumulator).
//
// CTA work unit = (pair l, block of 128 rows j, candidate range).  Warp roles (288 threads):
//  * warps 4-7 (producers) build the unit's four A planes once (128 rows x n_e, K-major: core
//    matrix = 8 rows x 16 bytes) from the u64 E, then per group of 64/g candidates the one-hot
//    B tile H = [(candidate, gpu) x k] (K-major, __vcmpeq4 on four GPU ids at a time);
//  * warp 8 (issuer) bulk-copies each group's candidate id rows (cp.async.bulk, one copy per lane)
//    two groups ahead into a 4-slot ring, and one lane issues 4 planes x n_e/32 instructions
//    (M = 128 rows, N = 64 (c, p) columns, K = 32) into one of two TMEM buffers (4 planes x 64
//    columns each) and commits them;
//  * warps 0-3 (epilogue) read the finished buffer back with tcgen05.ld (lane = row j), pick the
//    candidate's column P_c(l, j), recombine the planes (sum v_b << 8b), release the buffer and
//    reduce-scatter the rows over the warp into same[c] (u64 atomics),
// so a group's epilogue overlaps the next groups' one-hot builds and MMAs.  mbarriers: ids full
// (TMA tx), B full (4 producer warps), MMA done (tcgen05.commit), TMEM free (4 epilogue warps).
//
// Work per candidate is 4 x (L-1) x n_e^2 x g MACs on the tensor pipe instead of (L-1) x n_e^2
// compare-and-adds on the integer pipe (eval_same_fast_kernel, placement.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "internal.cuh"
#include "ptx.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kRowsBlk = 128;  // MMA M: rows j of one layer-l block
constexpr int kN = 64;         // MMA N: (candidate, gpu) columns per group
constexpr int kPlanes = 4;     // byte planes of a cell < 2^27
constexpr int kThreads = 288;  // warps 0-3 epilogue, warps 4-7 producers, warp 8 issuer
constexpr int kBStages = 2;    // one-hot tiles = TMEM buffers
constexpr int kIdSlotsMax = 16;  // candidate-id ring: 4, 8 or 16 slots (what shared memory holds), filled
                                 // slots - 2 groups ahead so the bulk copies' latency is hidden
constexpr int kIssuerWarp = 8;

struct EvalMmaParams {
  int L, ne, g;
  int n_jb, n_cr;  // row blocks per pair, candidate ranges
  int64_t C, m, range_cands, n_units;
  uint32_t idesc;
  int id_shift;  // log2 of the id-ring slots
};

// K-major, no swizzle: core matrix = 8 rows x 16 bytes; K-adjacent core matrices LBO = 128 B apart,
// 8-row groups SBO apart.
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fffu);
  d |= (uint64_t)((128u >> 4) & 0x3fffu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;
}

// r = c ? a : b as a real select (a plain ?: chain over v[p] is turned into an indexed local-memory
// load of the accumulator row by the compiler)
__device__ __forceinline__ uint32_t selp(uint32_t c, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tselp.b32 %0, %2, %3, q;\n\t}" : "=r"(r) : "r"(c), "r"(a), "r"(b));
  return r;
}

// v[o + p] for p < G by a binary select tree on the bits of p
template <int G>
__device__ __forceinline__ uint32_t pick(const uint32_t* v, uint32_t p) {
  uint32_t t[G];
#pragma unroll
  for (int i = 0; i < G; ++i) t[i] = v[i];
#pragma unroll
  for (int w = G / 2, bit = 1; w >= 1; w >>= 1, bit <<= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) t[i] = selp(p & (uint32_t)bit, t[2 * i + 1], t[2 * i]);
  return t[0];
}

__device__ __forceinline__ uint32_t kmajor_off(int row, int k, uint32_t sbo) {
  return (uint32_t)(row >> 3) * sbo + (uint32_t)(k >> 4) * 128u + (uint32_t)(row & 7) * 16u + (uint32_t)(k & 15);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
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

// One-hot B tile of one group from its staged GPU ids (ids[ci][0..n_e) = P_c(l+1, .)): row
// n = ci * G + p, column k, byte = [P_c(l+1, k) == p].  Stacked mode (n_e = 64, ST): rows
// [0, 32) hold pair l's one-hot of layer l+1, rows [32, 64) pair l+1's of layer l+2.  Each lane writes one 4-byte word of a core
// matrix (lane = row-in-core * 4 + word), so a warp's stores cover 128 contiguous bytes.
template <int G, bool ST>
__device__ __forceinline__ void build_onehot(uint8_t* B, const uint8_t* ids, int ids_stride, int ne, int n_live,
                                             uint32_t sbo, int pwarp, int lane, int halves_live) {
  // warp w covers 8-row groups ng = w, w + 4, ...; a lane's row n and candidate/GPU (ci, p) are
  // fixed per row group, so the k loop is shifts and adds only
#pragma unroll
  for (int ng = pwarp; ng < kN / 8; ng += 4) {
    const int n = ng * 8 + (lane >> 2);
    // stacked (n_e = 64): columns [0, 32) one-hot layer l+1 (pair l), [32, 64) layer l+2 (pair l+1)
    const int h = ST ? n >> 5 : 0, nn = ST ? n & 31 : n;
    const int ci = nn / G, p = nn % G;
    const uint32_t pat = (uint32_t)p * 0x01010101u;
    const bool on = ci < n_live && h < halves_live;
    const uint32_t* src =
        reinterpret_cast<const uint32_t*>(ids + ci * ids_stride + (ST ? (1 + h) * ne : 0)) + (lane & 3);
    uint8_t* dst = B + (uint32_t)ng * sbo + (uint32_t)(lane >> 2) * 16u + (uint32_t)(lane & 3) * 4u;
    for (int kc = 0; kc < (ne >> 4); ++kc) {
      const uint32_t w = on ? (__vcmpeq4(src[kc * 4], pat) & 0x01010101u) : 0u;
      *reinterpret_cast<uint32_t*>(dst + kc * 128) = w;
    }
  }
}

template <int G, bool ST>
__global__ void __launch_bounds__(kThreads, 1)
    eval_mma_kernel(EvalMmaParams prm, const unsigned long long* __restrict__ E, const uint8_t* __restrict__ cands,
                    unsigned long long* __restrict__ same, WidthGuard guard) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (width_skip(guard)) return;  // a cell >= 2^27: the generic evaluator runs instead
  __shared__ uint64_t mma_done[kBStages], tmem_free[kBStages], b_full[kBStages], id_full[kIdSlotsMax];
  __shared__ uint32_t tmem_slot;
  // stacked (n_e = 64, ST): A rows [0, 64) = E_l, [64, 128) = E_l+1, each half of the N = 64
  // columns serves one pair, so a group holds 32 / G candidates
  constexpr int kCols = ST ? kN / 2 : kN;  // accumulator columns one row reads
  constexpr int kCpg = kCols / G;          // candidates per group
  const int ne = prm.ne;
  const int64_t m = prm.m;
  const uint32_t sbo = (uint32_t)(ne >> 4) * 128u;
  const int plane_bytes = kRowsBlk * ne;
  const int b_bytes = kN * ne;
  // per candidate: P_c(l+1, 0..n_e) then P_c(l, j0..j0+128); stacked: P_c(l), P_c(l+1), P_c(l+2)
  const int ids_stride = ST ? 3 * ne : ne + kRowsBlk;
  const int ids_bytes = kCpg * ids_stride;
  const int R = 1 << prm.id_shift;  // id-ring slots
  uint8_t* A = smem;
  uint8_t* Bst = smem + kPlanes * plane_bytes;
  uint8_t* idst = Bst + kBStages * b_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&mma_done[s], 1);
      mbar_init(&tmem_free[s], 4);  // one arrival per epilogue warp
      mbar_init(&b_full[s], 4);     // one arrival per producer warp
    }
    for (int s = 0; s < kIdSlotsMax; ++s) mbar_init(&id_full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  // issuer warp: bulk-copy the GPU ids one group needs into id slot `slot` (16-byte aligned
  // rows), one copy per lane (candidate ci = lane / 2, lane & 1 = layer l+1 row / layer l slice)
  auto fetch_ids = [&](uint32_t slot, int l, int j0, int64_t c0, int n_live) {
    uint8_t* dst = idst + slot * ids_bytes;
    const uint32_t bar = smem_u32(&id_full[slot]);
    // the slot's previous readers (producers, epilogue) released it through b_full / tmem_free,
    // which this warp acquired; order those generic-proxy reads before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (ST) {  // one copy per candidate: layers l .. min(l + 2, L - 1)
      const int bytes = min(3, prm.L - l) * ne;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)(n_live * bytes))
                     : "memory");
      __syncwarp();
      for (int ci = lane; ci < n_live; ci += 32)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(dst + ci * ids_stride)),
                     "l"(cands + (c0 + ci) * m + (int64_t)l * ne), "r"(bytes), "r"(bar)
                     : "memory");
      return;
    }
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"((uint32_t)(n_live * (ne + kRowsBlk)))
                   : "memory");
    __syncwarp();
    for (int i = lane; i < 2 * n_live; i += 32) {
      const int ci = i >> 1;
      const uint8_t* row = cands + (c0 + ci) * m;
      const bool lo = (i & 1) == 0;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst + ci * ids_stride + (lo ? 0 : ne))),
                   "l"(lo ? row + (int64_t)(l + 1) * ne : row + (int64_t)l * ne + j0), "r"(lo ? ne : kRowsBlk),
                   "r"(bar)
                   : "memory");
    }
  };

  // Both roles walk the same (unit, group) sequence; G_ counts this CTA's groups: B stage / TMEM
  // buffer = G & 1 (barrier parity (G >> 1) & 1), id slot = G mod R (parity (G / R) & 1), R = id-ring slots.
  uint32_t G_ = 0;
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int cr = (int)(unit % prm.n_cr);
    const int64_t rest = unit / prm.n_cr;
    const int jb = (int)(rest % prm.n_jb);
    const int l = ST ? 2 * (int)rest : (int)(rest / prm.n_jb);  // stacked: pairs l and l + 1
    const int j0 = jb * kRowsBlk;
    const int halves_live = ST ? min(2, prm.L - 1 - l) : 1;
    const int64_t c_begin = (int64_t)cr * prm.range_cands;
    const int64_t c_end = min(prm.C, c_begin + prm.range_cands);
    if (c_begin >= c_end) continue;
    const int n_groups = (int)((c_end - c_begin + kCpg - 1) / kCpg);
    auto live = [&](int gi) { return (int)min((int64_t)kCpg, c_end - c_begin - (int64_t)gi * kCpg); };

    if (warp == kIssuerWarp) {
      // ---------------- issuer: id fetches + MMAs ----------------
      // groups up to G_ - 3 have finished their epilogues (tmem_free waits): their slots are free
      for (int gi = 0; gi < min(R - 2, n_groups); ++gi)
        fetch_ids((G_ + gi) & (R - 1), l, j0, c_begin + (int64_t)gi * kCpg, live(gi));
      for (int gi = 0; gi < n_groups; ++gi) {
        const uint32_t Gg = G_ + gi, s = Gg & 1;
        mbar_wait(&b_full[s], (Gg >> 1) & 1);                          // A (first group) and B(Gg) built
        if (Gg >= 2) mbar_wait(&tmem_free[s], ((Gg - 2) >> 1) & 1);   // epilogue of Gg - 2 read buffer s
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t a0 = smem_u32(A), b0 = smem_u32(Bst + s * b_bytes);
          const uint32_t d0 = tmem + s * (kPlanes * kN);
          for (int b = 0; b < kPlanes; ++b)
            for (int kk = 0; kk < ne / 32; ++kk)
              mma_i8(d0 + (uint32_t)(b * kN), kmajor_desc(a0 + b * plane_bytes + kk * 256, sbo),
                     kmajor_desc(b0 + kk * 256, sbo), prm.idesc, kk > 0 ? 1u : 0u);
          mma_commit(&mma_done[s]);
        }
        __syncwarp();
        // the slot of group Gg + R - 2 last served group Gg - 2, whose epilogue has finished
        if (gi + R - 2 < n_groups)
          fetch_ids((Gg + R - 2) & (R - 1), l, j0, c_begin + (int64_t)(gi + R - 2) * kCpg, live(gi + R - 2));
      }
    } else if (warp >= 4) {
      // ---------------- producers: A planes once per unit, a one-hot tile per group ----------------
      const int pwarp = warp - 4;
      // the previous unit's MMAs read the A planes: wait for the last of them
      if (G_ >= 1) mbar_wait(&mma_done[(G_ - 1) & 1], ((G_ - 1) >> 1) & 1);
      {
        const int kcs = ne >> 4, kcs_shift = ne == 256 ? 4 : ne == 128 ? 3 : 2;
        const int n_cm = (kRowsBlk / 8) * kcs;
        for (int cm0 = pwarp; cm0 < n_cm; cm0 += 4 * 4) {
          ulonglong2 v[4][2];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cm = cm0 + u * 4;
            if (cm < n_cm) {
              const int rg = cm >> kcs_shift, kc = cm & (kcs - 1);
              const int row = rg * 8 + (lane >> 2), k = kc * 16 + (lane & 3) * 4;
              // E is [(L-1)][n_e][n_e]: rows l * n_e + 64 .. of the stacked block are E_l+1's; rows
              // past the last pair load a valid row and are zeroed at use (loads stay batched)
              const int64_t grow = min((int64_t)l * ne + j0 + row, (int64_t)(prm.L - 1) * ne - 1);
              const ulonglong2* src = reinterpret_cast<const ulonglong2*>(E + grow * ne + k);
              v[u][0] = __ldg(src);
              v[u][1] = __ldg(src + 1);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cm = cm0 + u * 4;
            if (cm < n_cm) {
              const int rg = cm >> kcs_shift, kc = cm & (kcs - 1);
              const int row = rg * 8 + (lane >> 2), k = kc * 16 + (lane & 3) * 4;
              const uint32_t live_row = (int64_t)l * ne + j0 + row < (int64_t)(prm.L - 1) * ne ? ~0u : 0u;
              const uint32_t c0 = (uint32_t)v[u][0].x & live_row, c1 = (uint32_t)v[u][0].y & live_row;
              const uint32_t c2 = (uint32_t)v[u][1].x & live_row, c3 = (uint32_t)v[u][1].y & live_row;
              const uint32_t off = kmajor_off(row, k, sbo);
#pragma unroll
              for (int b = 0; b < kPlanes; ++b) {
                const uint32_t sel = (uint32_t)b | ((uint32_t)(4 + b) << 4);
                const uint32_t lo = __byte_perm(c0, c1, sel), hi = __byte_perm(c2, c3, sel);
                *reinterpret_cast<uint32_t*>(A + b * plane_bytes + off) = __byte_perm(lo, hi, 0x5410);
              }
            }
          }
        }
      }
      for (int gi = 0; gi < n_groups; ++gi) {
        const uint32_t Gg = G_ + gi, s = Gg & 1;
        // one-hot tile: ids landed, and the stage's previous MMAs (group Gg - 2) are done
        mbar_wait(&id_full[Gg & (R - 1)], (Gg >> prm.id_shift) & 1);
        if (Gg >= 2) mbar_wait(&mma_done[s], ((Gg - 2) >> 1) & 1);
        build_onehot<G, ST>(Bst + s * b_bytes, idst + (Gg & (R - 1)) * ids_bytes, ids_stride, ne, live(gi), sbo, pwarp,
                            lane, halves_live);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_full[s]);
      }
    } else {
      // ---------------- epilogue ----------------
      const int jr = warp * 32 + lane;  // row of the block = TMEM lane
      for (int gi = 0; gi < n_groups; ++gi) {
        const uint32_t Gg = G_ + gi, s = Gg & 1;
        const int64_t c0 = c_begin + (int64_t)gi * kCpg;
        const int n_live = live(gi);
        mbar_wait(&mma_done[s], (Gg >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // row jr's assignment P_c(l, j0 + jr); stacked: P_c(l + jr / 64, jr % 64)
        const uint8_t* ids = idst + (Gg & (R - 1)) * ids_bytes + (ST ? (jr >> 6) * ne + (jr & 63) : ne + jr);
        unsigned long long acc[kCpg];
        uint32_t pj[kCpg];
#pragma unroll
        for (int ci = 0; ci < kCpg; ++ci) {
          acc[ci] = 0ull;
          pj[ci] = ci < n_live ? (uint32_t)ids[ci * ids_stride] : 0u;
        }
        // stacked: rows [64, 128) (warps 2-3) read the upper half of the columns
        const uint32_t d0 = tmem + ((uint32_t)(warp * 32) << 16) + s * (kPlanes * kN) + (ST && warp >= 2 ? kCols : 0);
#pragma unroll
        for (int b = 0; b < kPlanes; ++b) {
#pragma unroll
          for (int ch = 0; ch < kCols / 16; ch += 2) {
            uint32_t v[2][16];
            tmem_ld16(d0 + (uint32_t)(b * kN + ch * 16), v[0]);
            tmem_ld16(d0 + (uint32_t)(b * kN + ch * 16 + 16), v[1]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int q = 0; q < 16 / G; ++q) {
                const int ci = (ch + h) * (16 / G) + q;
                const uint32_t x = pick<G>(&v[h][q * G], pj[ci]);
                acc[ci] += (unsigned long long)x << (8 * b);
              }
          }
        }
        // the buffer is read: let the issuer reuse it for group Gg + 2
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_free[s]);
        // reduce-scatter over the warp: after log2(kCpg) halvings lane groups hold one candidate
        // each, then a plain butterfly finishes the 32 / kCpg lanes that share it
#pragma unroll
        for (int half = kCpg / 2; half >= 1; half >>= 1) {
          const bool upper = (lane & (half * (32 / kCpg))) != 0;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const unsigned long long send = upper ? acc[i] : acc[i + half];
            const unsigned long long keep = upper ? acc[i + half] : acc[i];
            acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, half * (32 / kCpg));
          }
        }
        unsigned long long s64 = acc[0];
#pragma unroll
        for (int o = 32 / kCpg / 2; o > 0; o >>= 1) s64 += __shfl_xor_sync(0xffffffffu, s64, o);
        int ci = 0;  // lane bits above log2(32 / kCpg) name the candidate this lane group holds
#pragma unroll
        for (int half = kCpg / 2; half >= 1; half >>= 1)
          if (lane & (half * (32 / kCpg))) ci |= half;
        if ((lane & (32 / kCpg - 1)) == 0 && s64 != 0ull && ci < n_live) atomicAdd(&same[c0 + ci], s64);
      }
    }
    G_ += (uint32_t)n_groups;
  }
  // every commit was waited by the epilogue; every TMEM read finished before its arrive
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace

size_t eval_mma_smem(int ne, int g, int slots = 4);

bool eval_mma_supported(int L, int ne, int g, const uint8_t* cands, int64_t C) {
  if (GIMBAL_KNOB("GIMBAL_EVAL_ALU")) return false;
  if (!(L > 1 && C > 0 && (ne == 64 || ne == 128 || ne == 256) && (g == 4 || g == 8 || g == 16) &&
        (reinterpret_cast<uintptr_t>(cands) & 15) == 0))  // 16-B aligned bulk copies
    return false;
  return eval_mma_smem(ne, g, 4) <= 227 * 1024;
}

size_t eval_mma_smem(int ne, int g, int slots) {
  if (ne == 64)  // stacked pairs: 32 / g candidates per group, three id rows each
    return (size_t)kPlanes * kRowsBlk * ne + (size_t)kBStages * kN * ne + (size_t)slots * (kN / 2 / g) * (3 * ne);
  return (size_t)kPlanes * kRowsBlk * ne + (size_t)kBStages * kN * ne + (size_t)slots * (kN / g) * (ne + kRowsBlk);
}

// same[c] += sum over pairs of the same-GPU weight (same[] zeroed by the caller); E cells < 2^27.
cudaError_t launch_eval_mma(int L, int ne, int g, const unsigned long long* E, const uint8_t* cands, int64_t C,
                            unsigned long long* same, WidthGuard guard, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  EvalMmaParams prm;
  prm.L = L;
  prm.ne = ne;
  prm.g = g;
  const bool st = ne == 64;
  prm.n_jb = st ? 1 : ne / kRowsBlk;
  prm.C = C;
  prm.m = (int64_t)L * ne;
  const int cpg = (st ? kN / 2 : kN) / g;
  const int64_t base = st ? (int64_t)(L - 1 + 1) / 2 : (int64_t)(L - 1) * prm.n_jb;
  const int64_t groups = (C + cpg - 1) / cpg;
  // enough units for ~2 per SM, each rebuilding its A planes (n_e x 128 x 8 B of E) once
  prm.n_cr = (int)std::max<int64_t>(1, std::min<int64_t>(groups, (2 * sms + base - 1) / base));
  prm.range_cands = (groups + prm.n_cr - 1) / prm.n_cr * cpg;
  prm.n_cr = (int)((C + prm.range_cands - 1) / prm.range_cands);
  prm.n_units = base * prm.n_cr;
  // c = s32, a = b = u8, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
  prm.idesc = (2u << 4) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kRowsBlk >> 4) << 24);
  int slots = kIdSlotsMax;
  if (const char* e = GIMBAL_KNOB("GIMBAL_EVAL_ID_SLOTS")) slots = std::atoi(e);
  while (slots > 4 && eval_mma_smem(ne, g, slots) > 227 * 1024) slots >>= 1;
  prm.id_shift = slots == 16 ? 4 : slots == 8 ? 3 : 2;
  const size_t smem = eval_mma_smem(ne, g, 1 << prm.id_shift);
  // one SM stays free: the greedy walk (one CTA, up to 200 KB of shared memory) of the same pass
  // runs beside the scoring of the other candidates (capi.cu gimbal_pass_async)
  const int grid = (int)std::min<int64_t>(prm.n_units, std::max(1, sms - 1));
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(prm, E, cands, same, guard);
    return cudaGetLastError();
  };
  switch (g * 2 + (st ? 1 : 0)) {
    case 8: return go(eval_mma_kernel<4, false>);
    case 9: return go(eval_mma_kernel<4, true>);
    case 16: return go(eval_mma_kernel<8, false>);
    case 17: return go(eval_mma_kernel<8, true>);
    case 32: return go(eval_mma_kernel<16, false>);
    case 33: return go(eval_mma_kernel<16, true>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gimbal_gpu
