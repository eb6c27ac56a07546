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
// CTA work unit = (pair l, block of 128 rows j, candidate range).  The unit's four A planes
// (128 rows x n_e, K-major: core matrix = 8 rows x 16 bytes) are built once from the u64 E; then
// per group of 128/g candidates the B tile H = [(candidate, gpu) x k] one-hot (K-major, built with
// __vcmpeq4 from four GPU ids at a time) is staged in a 2-deep ring while the previous group's MMAs
// run, and one thread issues 4 planes x n_e/32 instructions (M = 128 rows, N = 128 (c, p) columns,
// K = 32) into four 128-column s32 accumulators (all 512 TMEM columns).  Four warps read their
// rows back with tcgen05.ld, pick column P_c(l, j) per candidate, recombine the planes
// (sum v_b << 8b) and reduce the rows of the block into same[c] (u64 atomics).
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
constexpr int kN = 128;        // MMA N: (candidate, gpu) columns per group
constexpr int kPlanes = 4;     // byte planes of a cell < 2^27
constexpr int kThreads = 256;
constexpr int kBStages = 2;
constexpr int kIdSlots = 3;  // candidate-id ring, filled two groups ahead

struct EvalMmaParams {
  int L, ne, g, cpg;  // cpg = candidates per group (kN / g)
  int n_jb, n_cr;     // row blocks per pair, candidate ranges
  int64_t C, m, range_cands, n_units;
  uint32_t idesc;
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
// n = ci * G + p, column k, byte = [P_c(l+1, k) == p].  Each lane writes one 4-byte word of a core
// matrix (lane = row-in-core * 4 + word), so a warp's stores cover 128 contiguous bytes.
template <int G>
__device__ __forceinline__ void build_onehot(uint8_t* B, const uint8_t* ids, int ids_stride, int ne, int n_live,
                                             uint32_t sbo) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kcs = ne >> 4;
  for (int cm = warp; cm < (kN / 8) * kcs; cm += kThreads / 32) {
    const int ng = cm / kcs, kc = cm - ng * kcs;
    const int n = ng * 8 + (lane >> 2), k = kc * 16 + (lane & 3) * 4;
    const int ci = n / G, p = n - ci * G;
    uint32_t w = 0u;
    if (ci < n_live) {
      const uint32_t v = *reinterpret_cast<const uint32_t*>(ids + ci * ids_stride + k);
      w = __vcmpeq4(v, (uint32_t)p * 0x01010101u) & 0x01010101u;
    }
    *reinterpret_cast<uint32_t*>(B + kmajor_off(n, k, sbo)) = w;
  }
}

template <int G>
__global__ void __launch_bounds__(kThreads, 1)
    eval_mma_kernel(EvalMmaParams prm, const unsigned long long* __restrict__ E, const uint8_t* __restrict__ cands,
                    unsigned long long* __restrict__ same) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kBStages], id_bars[kIdSlots];
  __shared__ uint32_t tmem_slot;
  constexpr int kCpg = kN / G;
  const int ne = prm.ne;
  const int64_t m = prm.m;
  const uint32_t sbo = (uint32_t)(ne >> 4) * 128u;
  const int plane_bytes = kRowsBlk * ne;
  const int b_bytes = kN * ne;
  const int ids_stride = ne + kRowsBlk;  // per candidate: P_c(l+1, 0..n_e) then P_c(l, j0..j0+128)
  uint8_t* A = smem;
  uint8_t* Bst = smem + kPlanes * plane_bytes;
  uint8_t* idst = Bst + kBStages * b_bytes;  // kIdSlots slots of kCpg * ids_stride bytes
  const int ids_bytes = kCpg * ids_stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBStages; ++s) mbar_init(&bars[s], 1);
    for (int s = 0; s < kIdSlots; ++s) mbar_init(&id_bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  // thread 0: bulk-copy the GPU ids one group needs into id slot `slot` (16-byte aligned rows)
  auto fetch_ids = [&](uint32_t slot, int l, int j0, int64_t c0, int n_live) {
    uint8_t* dst = idst + slot * ids_bytes;
    const uint32_t bar = smem_u32(&id_bars[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)(n_live * (ne + kRowsBlk)))
                 : "memory");
    for (int ci = 0; ci < n_live; ++ci) {
      const uint8_t* row = cands + (c0 + ci) * m;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst + ci * ids_stride)),
                   "l"(row + (int64_t)(l + 1) * ne), "r"(ne), "r"(bar)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst + ci * ids_stride + ne)),
                   "l"(row + (int64_t)l * ne + j0), "r"(kRowsBlk), "r"(bar)
                   : "memory");
    }
  };

  // groups of this CTA so far: B stage = & 1 (MMA barrier phase (>> 1) & 1); id slot = % 3 (phase (/ 3) & 1)
  uint32_t grp_global = 0;
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int cr = (int)(unit % prm.n_cr);
    const int64_t rest = unit / prm.n_cr;
    const int jb = (int)(rest % prm.n_jb);
    const int l = (int)(rest / prm.n_jb);
    const int j0 = jb * kRowsBlk;
    const int64_t c_begin = (int64_t)cr * prm.range_cands;
    const int64_t c_end = min(prm.C, c_begin + prm.range_cands);
    if (c_begin >= c_end) continue;
    const int n_groups = (int)((c_end - c_begin + kCpg - 1) / kCpg);
    auto live = [&](int gi) { return (int)min((int64_t)kCpg, c_end - c_begin - (int64_t)gi * kCpg); };
    if (threadIdx.x == 0) {
      fetch_ids(grp_global % kIdSlots, l, j0, c_begin, live(0));
      if (n_groups > 1) fetch_ids((grp_global + 1) % kIdSlots, l, j0, c_begin + kCpg, live(1));
    }
    // A planes: byte b of the 128 x n_e block of E_l; eight 32-byte loads in flight per lane
    {
      const int kcs = ne >> 4;
      const int n_cm = (kRowsBlk / 8) * kcs;
      for (int cm0 = warp; cm0 < n_cm; cm0 += 8 * (kThreads / 32)) {
        ulonglong2 v[8][2];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int cm = cm0 + u * (kThreads / 32);
          if (cm < n_cm) {
            const int rg = cm / kcs, kc = cm - rg * kcs;
            const int row = rg * 8 + (lane >> 2), k = kc * 16 + (lane & 3) * 4;
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(E + ((int64_t)l * ne + j0 + row) * ne + k);
            v[u][0] = __ldg(src);
            v[u][1] = __ldg(src + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int cm = cm0 + u * (kThreads / 32);
          if (cm < n_cm) {
            const int rg = cm / kcs, kc = cm - rg * kcs;
            const int row = rg * 8 + (lane >> 2), k = kc * 16 + (lane & 3) * 4;
            const uint32_t c0 = (uint32_t)v[u][0].x, c1 = (uint32_t)v[u][0].y;
            const uint32_t c2 = (uint32_t)v[u][1].x, c3 = (uint32_t)v[u][1].y;
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
    mbar_wait(&id_bars[grp_global % kIdSlots], (grp_global / kIdSlots) & 1);
    build_onehot<G>(Bst + (grp_global & 1) * b_bytes, idst + (grp_global % kIdSlots) * ids_bytes, ids_stride, ne,
                    live(0), sbo);
    for (int gi = 0; gi < n_groups; ++gi, ++grp_global) {
      const uint32_t s = grp_global & 1;
      const int64_t c0 = c_begin + (int64_t)gi * kCpg;
      const int n_live = live(gi);
      // A planes and B(gi) written; the previous group's accumulators and ids have been read
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(A), b0 = smem_u32(Bst + s * b_bytes);
        for (int b = 0; b < kPlanes; ++b)
          for (int kk = 0; kk < ne / 32; ++kk)
            mma_i8(tmem + (uint32_t)(b * kN), kmajor_desc(a0 + b * plane_bytes + kk * 256, sbo),
                   kmajor_desc(b0 + kk * 256, sbo), prm.idesc, kk > 0 ? 1u : 0u);
        mma_commit(&bars[s]);
        // slot of group gi+2 was last read by group gi-1 (finished before the barrier above)
        if (gi + 2 < n_groups) fetch_ids((grp_global + 2) % kIdSlots, l, j0, c0 + 2 * kCpg, live(gi + 2));
      }
      // the next group's one-hot tile goes to the other stage (its MMAs completed last round)
      if (gi + 1 < n_groups) {
        const uint32_t nx = grp_global + 1;
        mbar_wait(&id_bars[nx % kIdSlots], (nx / kIdSlots) & 1);
        build_onehot<G>(Bst + (s ^ 1) * b_bytes, idst + (nx % kIdSlots) * ids_bytes, ids_stride, ne, live(gi + 1),
                        sbo);
      }
      mbar_wait(&bars[s], (grp_global >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (warp < 4) {
        const int jr = warp * 32 + lane;  // row of the block = TMEM lane
        const uint8_t* ids = idst + (grp_global % kIdSlots) * ids_bytes + ne + jr;
        unsigned long long acc[kCpg];
        uint32_t pj[kCpg];
#pragma unroll
        for (int ci = 0; ci < kCpg; ++ci) {
          acc[ci] = 0ull;
          pj[ci] = ci < n_live ? (uint32_t)ids[ci * ids_stride] : 0u;
        }
#pragma unroll
        for (int b = 0; b < kPlanes; ++b) {
#pragma unroll
          for (int ch = 0; ch < kN / 16; ch += 2) {
            uint32_t v[2][16];
            const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * kN + ch * 16);
            tmem_ld16(base, v[0]);
            tmem_ld16(base + 16, v[1]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int q = 0; q < 16 / G; ++q) {
                const int ci = (ch + h) * (16 / G) + q;
                uint32_t x = v[h][q * G];
#pragma unroll
                for (int p = 1; p < G; ++p) x = pj[ci] == (uint32_t)p ? v[h][q * G + p] : x;
                acc[ci] += (unsigned long long)x << (8 * b);
              }
          }
        }
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
        {
          unsigned long long s64 = acc[0];
#pragma unroll
          for (int o = 32 / kCpg / 2; o > 0; o >>= 1) s64 += __shfl_xor_sync(0xffffffffu, s64, o);
          // lane bits above log2(32/kCpg) name the candidate this lane group now holds
          int ci = 0;
#pragma unroll
          for (int half = kCpg / 2; half >= 1; half >>= 1)
            if (lane & (half * (32 / kCpg))) ci |= half;
          if ((lane & (32 / kCpg - 1)) == 0 && s64 != 0ull && ci < n_live) atomicAdd(&same[c0 + ci], s64);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // A planes are rebuilt for the next unit
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace

size_t eval_mma_smem(int ne, int g);

bool eval_mma_supported(int L, int ne, int g, const uint8_t* cands, int64_t C) {
  if (std::getenv("GIMBAL_EVAL_ALU")) return false;
  if (!(L > 1 && C > 0 && (ne == 128 || ne == 256) && (g == 4 || g == 8 || g == 16) &&
        (reinterpret_cast<uintptr_t>(cands) & 15) == 0))  // 16-B aligned bulk copies
    return false;
  return eval_mma_smem(ne, g) <= 227 * 1024;  // n_e = 256 with g = 4 does not fit
}

size_t eval_mma_smem(int ne, int g) {
  return (size_t)kPlanes * kRowsBlk * ne + (size_t)kBStages * kN * ne + (size_t)kIdSlots * (kN / g) * (ne + kRowsBlk);
}

// same[c] += sum over pairs of the same-GPU weight (same[] zeroed by the caller); E cells < 2^27.
cudaError_t launch_eval_mma(int L, int ne, int g, const unsigned long long* E, const uint8_t* cands, int64_t C,
                            unsigned long long* same, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  EvalMmaParams prm;
  prm.L = L;
  prm.ne = ne;
  prm.g = g;
  prm.cpg = kN / g;
  prm.n_jb = ne / kRowsBlk;
  prm.C = C;
  prm.m = (int64_t)L * ne;
  const int64_t base = (int64_t)(L - 1) * prm.n_jb;
  const int64_t groups = (C + prm.cpg - 1) / prm.cpg;
  // enough units for ~2 per SM, each rebuilding its A planes (n_e x 128 x 8 B of E) once
  prm.n_cr = (int)std::max<int64_t>(1, std::min<int64_t>(groups, (2 * sms + base - 1) / base));
  prm.range_cands = (groups + prm.n_cr - 1) / prm.n_cr * prm.cpg;
  prm.n_cr = (int)((C + prm.range_cands - 1) / prm.range_cands);
  prm.n_units = base * prm.n_cr;
  // c = s32, a = b = u8, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
  prm.idesc = (2u << 4) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kRowsBlk >> 4) << 24);
  const size_t smem = eval_mma_smem(ne, g);
  const int grid = (int)std::min<int64_t>(prm.n_units, sms);
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(prm, E, cands, same);
    return cudaGetLastError();
  };
  switch (g) {
    case 4: return go(eval_mma_kernel<4>);
    case 8: return go(eval_mma_kernel<8>);
    case 16: return go(eval_mma_kernel<16>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gimbal_gpu
