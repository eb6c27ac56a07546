// Routing-trace ingestion and transition counting on sm_100a (the DS-V3-class fast path).
//
// 1. transpose_lm8_kernel: token-major uint8 trace [T][L][k] (the reference's RoutedStream order,
//    moe.hpp:75-83) -> layer-major packed form "LM8" [L][T] uint64, each word holding one token's
//    k <= 8 ids of one layer.  Whole token rows are read coalesced (one HBM pass over the trace),
//    ids are range-checked here (moe.cpp:176-187 leaves out-of-range ids undefined; we flag them).
// 2. count_lm8_kernel: one CTA work unit = (token chunk, group of consecutive layer pairs, slice
//    of rows j).  It streams the two layers of each pair it owns as contiguous 8-byte words and
//    increments u32 counters privatised in shared memory (ATOMS.POPC.INC), then flushes them to
//    the u64 tensor once.  When a pair's 256x256 table does not fit shared memory the rows are
//    split; the row filter would leave lanes idle in every atomic, so each warp first compacts
//    its passing (row, token) items into a shared queue and then drains the queue with all 32
//    lanes issuing atomics.
//
// Counting: E_l(j,k) += 1 for every (j in slots_l, k in slots_{l+1}) pairing of every token,
// with multiplicity (moe.cpp:179-188).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include <cudaTypedefs.h>

#include "internal.cuh"
#include "ptx.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kTransposeTile = 64;   // tokens per transposition CTA
constexpr int kBatch = 128;          // tokens per warp batch in the split kernel
constexpr int kSplitWarps = 24;      // warps per CTA in the split kernel

template <int K>
__global__ void __launch_bounds__(256)
    transpose_lm8_kernel(const uint8_t* __restrict__ trace, int64_t T, int L, int ne,
                         unsigned long long* __restrict__ X, int64_t ld, uint32_t* __restrict__ flags) {
  extern __shared__ uint8_t tile[];  // kTransposeTile * L * K bytes
  const int64_t t0 = (int64_t)blockIdx.x * kTransposeTile;
  const int n = (int)min((int64_t)kTransposeTile, T - t0);
  const int row = L * K;
  const int bytes = n * row;
  const uint8_t* src = trace + t0 * row;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(src);
  if ((row & 15) == 0 && (addr & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(tile);
    for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) d4[i] = __ldcs(s4 + i);
  } else if ((row & 3) == 0 && (addr & 3) == 0) {
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d4 = reinterpret_cast<uint32_t*>(tile);
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) d4[i] = __ldcs(s4 + i);
  } else {
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) tile[i] = src[i];
  }
  __syncthreads();
  bool bad = false;
  int dup = 0;
  for (int idx = threadIdx.x; idx < L * kTransposeTile; idx += blockDim.x) {
    const int l = idx / kTransposeTile, i = idx - l * kTransposeTile;
    if (i >= n) continue;
    const uint8_t* p = tile + i * row + l * K;
    unsigned long long w = 0;
    uint32_t e_[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const uint32_t e = p[a];
      e_[a] = e;
      bad |= e >= (uint32_t)ne;
      w |= (unsigned long long)e << (8 * a);
    }
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) dup |= e_[a] == e_[b];
    X[(int64_t)l * ld + t0 + i] = w;
  }
  if (bad) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
  // repeated ids within a token-layer (legal, counted with multiplicity) disable the
  // one-count-per-cell fast paths of the counting kernels
  if (__syncthreads_or(dup) && threadIdx.x == 0) atomicOr(flags, (uint32_t)kFlagDuplicates);
}

struct Lm8Params {
  int L, ne;
  int P, R;        // pairs per group, rows per part
  uint32_t swz;    // column XOR swizzle (row r stores column k at k ^ (r & swz))
  int n_groups, n_parts;
  int64_t n_units;
  int64_t chunk_tokens;
  int64_t T;       // tokens in X
  int64_t ld;      // row stride of X (tokens)
  int rolling = 0;     // TMA u16 counter: rolling drain without barriers (AB)
  int drain_blocks = 32; // TMA u16 counter, block-wide drain: blocks between drains (<= 32)
  int scalar_scan = 0;  // TMA u16 counter, block-wide drain: scan one word per load (AB)
  int roll_sync = 0;   // TMA u16 counter, rolling drain: a block barrier every roll_sync blocks (AB)
};

__device__ __forceinline__ uint32_t id_of(unsigned long long w, int a) {
  return (uint32_t)(w >> (8 * a)) & 0xffu;
}

// Whole layer pairs per unit: every slot passes, no filtering.
template <int K>
__global__ void __launch_bounds__(1024, 1)
    count_lm8_pairs_kernel(Lm8Params prm, const unsigned long long* __restrict__ X,
                           unsigned long long* __restrict__ E) {
  extern __shared__ uint32_t cnt[];
  const int ne = prm.ne;
  const int upc = prm.n_groups;
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int64_t chunk = unit / upc;
    const int group = (int)(unit % upc);
    const int l0 = group * prm.P;
    const int l1 = min(l0 + prm.P, prm.L - 1);
    const int words = (l1 - l0) * ne * ne;
    for (int w = threadIdx.x; w < words; w += blockDim.x) cnt[w] = 0u;
    __syncthreads();
    const int64_t t_begin = chunk * prm.chunk_tokens;
    const int64_t t_end = min(prm.T, t_begin + prm.chunk_tokens);
    for (int64_t t = t_begin + threadIdx.x; t < t_end; t += blockDim.x) {
      unsigned long long cur = __ldcs(X + (int64_t)l0 * prm.ld + t);
      for (int l = l0; l < l1; ++l) {
        const unsigned long long nxt = __ldcs(X + (int64_t)(l + 1) * prm.ld + t);
        uint32_t* blk = cnt + (l - l0) * ne * ne;
#pragma unroll
        for (int a = 0; a < K; ++a) {
          const uint32_t j = id_of(cur, a);
          uint32_t* rowp = blk + j * ne;
          const uint32_t sw = j & prm.swz;
#pragma unroll
          for (int b = 0; b < K; ++b) atomicAdd(rowp + (id_of(nxt, b) ^ sw), 1u);
        }
        cur = nxt;
      }
    }
    __syncthreads();
    const int nn = ne * ne;
    for (int w = threadIdx.x; w < words; w += blockDim.x) {
      const uint32_t v = cnt[w];
      if (v == 0u) continue;
      const int pr = w / nn;
      const int r = w - pr * nn;
      const int j = r / ne;
      const int kk = (r - j * ne) ^ (j & prm.swz);
      atomicAdd(E + ((int64_t)(l0 + pr) * ne + j) * ne + kk, (unsigned long long)v);
    }
    __syncthreads();
  }
}

// Work split of the u15 kernels over the (chunk, pair) units, chunk-major (u = chunk * pairs +
// pair): whole units round-robin (unit b + r * grid in round r, so the CTAs counting different
// pairs of the same chunk start together and share its trace rows through L2), then the units
// left over after the last full round are split evenly over all CTAs ("stream-K" tail: CTA b owns
// positions [b * per, (b + 1) * per) of their token space), so no SM idles through a partial wave.
struct WorkCursor {
  int64_t round, rounds;  // whole-unit rounds done / total
  int64_t p, p_end;       // tail positions (unit * chunk_tokens + token offset)
};

__device__ __forceinline__ WorkCursor work_begin(const Lm8Params& prm) {
  WorkCursor c;
  c.round = 0;
  c.rounds = prm.n_units / gridDim.x;
  const int64_t tail0 = c.rounds * gridDim.x * prm.chunk_tokens;
  const int64_t span = prm.n_units * prm.chunk_tokens - tail0;
  const int64_t per = (span + gridDim.x - 1) / gridDim.x;
  c.p = tail0 + min(span, (int64_t)blockIdx.x * per);
  c.p_end = tail0 + min(span, (int64_t)(blockIdx.x + 1) * per);
  return c;
}

// Next non-empty segment [t0, t1) of pair l; false when the CTA's work is done.
__device__ __forceinline__ bool next_segment(const Lm8Params& prm, WorkCursor& c, int& l, int64_t& t0,
                                             int64_t& t1) {
  const int pairs = prm.L - 1;
  const int64_t CH = prm.chunk_tokens;
  while (c.round < c.rounds) {
    const int64_t u = c.round * gridDim.x + blockIdx.x;
    ++c.round;
    const int64_t chunk = u / pairs;
    l = (int)(u - chunk * pairs);
    t0 = chunk * CH;
    t1 = min(prm.T, t0 + CH);
    if (t0 < t1) return true;
  }
  while (c.p < c.p_end) {
    const int64_t u = c.p / CH;
    const int64_t base = u * CH;
    const int64_t off0 = c.p - base, off1 = min(CH, c.p_end - base);
    c.p = base + off1;
    const int64_t chunk = u / pairs;
    l = (int)(u - chunk * pairs);
    t0 = chunk * CH + off0;
    t1 = min(prm.T, chunk * CH + off1);
    if (t0 < t1) return true;
  }
  return false;
}

// The k x k increments of one token into a 15-bit-counter pair table (see below).
template <int K>
__device__ __forceinline__ void u15_count_token(uint32_t* cnt, int wpr, unsigned long long* El, int ne,
                                                unsigned long long cur, unsigned long long nxt) {
#pragma unroll
  for (int a = 0; a < K; ++a) {
    const uint32_t j = id_of(cur, a);
    uint32_t* rowp = cnt + j * wpr;
    const uint32_t sw = j & 31u;
    uint32_t old[K];
    bool full = false;
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const uint32_t k = id_of(nxt, b);
      const uint32_t shift = (k & 1u) << 4;
      old[b] = atomicAdd(rowp + ((k >> 1) ^ sw), 1u << shift);
      full |= ((old[b] >> shift) & 0x7fffu) == 0x7fffu;  // this increment filled the half
    }
    if (full) {  // rare: one branch per row instead of one per increment
#pragma unroll
      for (int b = 0; b < K; ++b) {
        const uint32_t k = id_of(nxt, b);
        const uint32_t shift = (k & 1u) << 4;
        if (((old[b] >> shift) & 0x7fffu) == 0x7fffu) {
          atomicSub(rowp + ((k >> 1) ^ sw), 0x8000u << shift);
          atomicAdd(El + (int64_t)j * ne + k, 32768ull);
        }
      }
    }
  }
}

// Add a 15-bit-counter pair table to the u64 tensor (caller synchronises around it).
__device__ __forceinline__ void u15_flush(const uint32_t* cnt, int wpr, unsigned long long* El, int ne) {
  for (int w = threadIdx.x; w < ne * wpr; w += blockDim.x) {
    const uint32_t v = cnt[w];
    if (v == 0u) continue;
    const int j = w / wpr;
    const int k0 = 2 * ((w - j * wpr) ^ (j & 31));
    unsigned long long* rowE = El + (int64_t)j * ne;
    if (v & 0xffffu) atomicAdd(rowE + k0, (unsigned long long)(v & 0xffffu));
    if (v >> 16) atomicAdd(rowE + k0 + 1, (unsigned long long)(v >> 16));
  }
}

// One whole layer pair per unit with 15-bit counters, two per 32-bit word (k even: bits 0-14,
// k odd: bits 16-30; bits 15 and 31 are guards), so a 256 x 256 pair fits in 128 KB and no row
// filter is needed.  An increment that carries a half into its guard bit (the half held 0x7FFF)
// is detected from the atomic's return value: that thread moves 32768 to the u64 tensor and
// clears the guard, so counts never wrap and never carry into the neighbour.
// TM = read the token-major trace directly (top_k = 8: one u64 per token-layer, row = L words)
// instead of the layer-major buffer; used when every uint8 id is valid by construction
// (n_e = 256), so no transposition pass is needed.
template <int K, bool TM>
__global__ void __launch_bounds__(1024, 1)
    count_lm8_u15_kernel(Lm8Params prm, const unsigned long long* __restrict__ X,
                         unsigned long long* __restrict__ E) {
  extern __shared__ uint32_t cnt[];
  const int ne = prm.ne;
  const int wpr = ne >> 1;  // words per row
  WorkCursor wc = work_begin(prm);
  int l;
  int64_t t_begin, t_end;
  while (next_segment(prm, wc, l, t_begin, t_end)) {
    for (int w = threadIdx.x; w < ne * wpr; w += blockDim.x) cnt[w] = 0u;
    __syncthreads();
    const unsigned long long* Xl = X + (int64_t)l * prm.ld;
    const unsigned long long* Xn = Xl + prm.ld;
    unsigned long long* El = E + (int64_t)l * ne * ne;
    auto fetch = [&](int64_t t, unsigned long long& c, unsigned long long& n) {
      if constexpr (TM) {  // the other pairs' CTAs read the same rows: keep them cacheable
        const unsigned long long* row = X + t * prm.L + l;
        c = __ldg(row);
        n = __ldg(row + 1);
      } else {
        c = __ldcs(Xl + t);
        n = __ldcs(Xn + t);
      }
    };
    unsigned long long cur = 0, nxt = 0, cur_n = 0, nxt_n = 0;
    if (t_begin + threadIdx.x < t_end) fetch(t_begin + threadIdx.x, cur, nxt);
    for (int64_t t = t_begin + threadIdx.x; t < t_end; t += blockDim.x) {
      // the next token's ids are in flight while this token's 64 increments issue
      if (t + blockDim.x < t_end) fetch(t + blockDim.x, cur_n, nxt_n);
      u15_count_token<K>(cnt, wpr, El, ne, cur, nxt);
      cur = cur_n;
      nxt = nxt_n;
    }
    __syncthreads();
    u15_flush(cnt, wpr, El, ne);
    __syncthreads();
  }
}

// Direct token-major counting with the ids staged by the tensor memory accelerator: every
// 1024-token block of the pair's two columns is one set of 2-D TMA boxes, so the SM's load/store
// pipe serves only the shared-memory atomics and two short shared reads per token instead of two
// 32-line gathers per warp.  A box must start 16-byte aligned in the row, so boxes hold two
// layers: (l, l+1) for even l, read as one 16-byte load per token; (l-1, l) and (l+1, l+2) for
// odd l, read as two 8-byte loads at a 16-byte stride (conflict-free); columns past the last
// layer are zero-filled and never read.  A 3-stage full/empty mbarrier ring keeps the next
// blocks in flight while the current one is counted.
constexpr int kTmaStages = 3;
constexpr int kTmaBlock = 1024;  // tokens per stage = threads per CTA
constexpr int kTmaBox = 256;     // rows per TMA box (hardware limit)
constexpr int kTmaCols = 4;      // u64 words per token in a stage (two 2-layer boxes of 16 B)
constexpr int kU15Bytes = 256 * 128 * 4;

constexpr int kDrainBlocks = 32;  // u16 mode: drain every 32 x 1024 = 32768 tokens
#ifdef GIMBAL_AB_KNOBS
#define U15_ROLL_SYNC prm.roll_sync
#define U15_DRAIN_BLOCKS prm.drain_blocks
#define U15_SCALAR_SCAN prm.scalar_scan
#define U15_ROLLING prm.rolling
#else
#define U15_ROLLING 0
#define U15_SCALAR_SCAN 0
#define U15_ROLL_SYNC 0
#define U15_DRAIN_BLOCKS kDrainBlocks
#endif

// U16 = full 16-bit halves and increments without return values (a warp issues its 64 increments
// back to back), drained block-wide every 32 blocks: between two drains a token whose ids are
// distinct within each layer adds at most 1 to any cell, so a half below 32768 stays below 65536.
// The drain scans the table with 16-byte loads behind two block barriers and moves bit 15 of each
// half to the u64 tensor.  Tokens with a repeated id (multiplicity up to 64 per cell) add straight
// to the u64 tensor instead.
// AB knob GIMBAL_U15_ROLLING: a rolling drain with no barrier (each thread checks one table word
// after every block, every word once per 32 blocks, and moves a half's top two bits (>= 16384) out
// by an atomic subtract; 35 blocks of growth from below 16384 cannot pass 65535).  It is 0.5 %
// faster (103.1-103.3 vs 103.7-103.9 ms per 64 Mi DS-V3 tokens) but reads 3x the DRAM bytes
// (190-215 vs 68-73 GB; 31 GB algorithmic): the 57 CTAs counting the pairs of one chunk read the
// same rows, L2 serves the later ones only while they stay close, and the drain pauses keep them
// close (a barrier alone every 32 blocks does not; every 8 blocks does, at 4 % time).  The pass
// runs beside the serving engine that produces the trace, so HBM bandwidth left to it matters more
// than 0.5 %: the block-wide drain ships.  profiles/r2c_dsv3_drain_traffic.md has the A/B.
// !U16 = guarded 15-bit halves with per-increment overflow detection (u15_count_token).
// AGG (issue-order experiments, U16 only; the AB build selects them with GIMBAL_TMA_AGG):
//   0 = slot order as drawn (default);
//   1 = both id words rotated by a lane-dependent number of slots, so the lanes of one atomic
//       instruction read different draw positions (a hot expert, usually drawn into the same
//       slot by every token, no longer lands on one address in one instruction);
//   2 = warp aggregation: lanes with equal (j, k) cells in one instruction are merged with
//       __match_any_sync and the leader adds the group size (the north_star's prescription).
template <bool U16, int AGG = 0>
__global__ void __launch_bounds__(kTmaBlock, 1)
    count_tm_u15_tma_kernel(const __grid_constant__ CUtensorMap tmap, Lm8Params prm,
                            unsigned long long* __restrict__ E) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw);
  unsigned long long* stage = reinterpret_cast<unsigned long long*>(smem_raw + kU15Bytes);
  __shared__ uint64_t full_bar[kTmaStages], empty_bar[kTmaStages];
  constexpr int ne = 256, wpr = 128;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kTmaBlock / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t it = 0;  // stage uses so far (CTA-uniform)
  WorkCursor wc = work_begin(prm);
  int l;
  int64_t t_begin, t_end;
  while (next_segment(prm, wc, l, t_begin, t_end)) {
    for (int w = tid; w < ne * wpr; w += kTmaBlock) cnt[w] = 0u;
    const uint32_t nb = (uint32_t)((t_end - t_begin + kTmaBlock - 1) / kTmaBlock);
    unsigned long long* El = E + (int64_t)l * ne * ne;
    auto issue = [&](uint32_t blk, uint32_t g) {  // thread 0
      const uint32_t s = g % kTmaStages;
      if (g >= kTmaStages) mbar_wait(&empty_bar[s], (g / kTmaStages - 1) & 1u);
      // boxes of two layers (16 B per token, 16-byte aligned in the row): layers l, l+1 when l
      // is even; layers l-1, l and l+1, l+2 (two half-stages) when l is odd
      mbar_arrive_expect_tx(&full_bar[s], kTmaBlock * 16 * ((l & 1) + 1));
      const int64_t t0 = t_begin + (int64_t)blk * kTmaBlock;
#pragma unroll
      for (int q = 0; q < kTmaBlock / kTmaBox; ++q) {
        unsigned long long* dst = stage + (s * kTmaBlock + q * kTmaBox) * kTmaCols;
        tma_load_2d(dst, &tmap, &full_bar[s], l & ~1, (int)(t0 + q * kTmaBox));
        if (l & 1) tma_load_2d(dst + kTmaBox * 2, &tmap, &full_bar[s], l + 1, (int)(t0 + q * kTmaBox));
      }
    };
    if (tid == 0)
      for (uint32_t i = 0; i < min(nb, (uint32_t)kTmaStages); ++i) issue(i, it + i);
    __syncthreads();  // counters zeroed
    for (uint32_t i = 0; i < nb; ++i) {
      const uint32_t g = it + i, s = g % kTmaStages;
      mbar_wait(&full_bar[s], (g / kTmaStages) & 1u);
      // per 256-token box: [256][2] words of layers (l & ~1, +1), then (odd l) [256][2] of l+1, l+2
      const unsigned long long* box = stage + (s * kTmaBlock + (tid & ~(kTmaBox - 1))) * kTmaCols;
      const int r = tid & (kTmaBox - 1);
      unsigned long long cur, nxt;
      if (l & 1) {  // 16-byte row stride: conflict-free 8-byte loads
        cur = box[r * 2 + 1];
        nxt = box[kTmaBox * 2 + r * 2];
      } else {      // one 16-byte load
        const ulonglong2 v = reinterpret_cast<const ulonglong2*>(box)[r];
        cur = v.x;
        nxt = v.y;
      }
      if (t_begin + (int64_t)i * kTmaBlock + tid < t_end) {
        if constexpr (U16) {
          if (!(has_dup8(cur) | has_dup8(nxt))) {
            if constexpr (AGG == 1) {
              const uint32_t rc = 8u * (uint32_t)(lane & 7), rn = 8u * (uint32_t)((lane >> 3) & 7);
              cur = (cur >> rc) | (cur << ((64u - rc) & 63u));
              nxt = (nxt >> rn) | (nxt << ((64u - rn) & 63u));
            }
            uint32_t col[8], inc[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              const uint32_t k = id_of(nxt, b);
              col[b] = k >> 1;
              inc[b] = 1u << ((k & 1u) << 4);
            }
#pragma unroll
            for (int a = 0; a < 8; ++a) {
              const uint32_t j = id_of(cur, a);
              uint32_t* rowp = cnt + j * wpr;
              const uint32_t sw = j & 31u;
              if constexpr (AGG == 2) {
                const uint32_t act = __activemask();
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                  const uint32_t grp = __match_any_sync(act, (j << 8) | id_of(nxt, b));
                  if ((grp & ((1u << lane) - 1u)) == 0u)  // lowest lane of its group adds for all
                    atomicAdd(rowp + (col[b] ^ sw), inc[b] * (uint32_t)__popc(grp));
                }
              } else {
#pragma unroll
                for (int b = 0; b < 8; ++b) atomicAdd(rowp + (col[b] ^ sw), inc[b]);
              }
            }
          } else {
#pragma unroll 1
            for (int a = 0; a < 8; ++a)
#pragma unroll 1
              for (int b = 0; b < 8; ++b) atomicAdd(El + id_of(cur, a) * ne + id_of(nxt, b), 1ull);
          }
        } else {
          u15_count_token<8>(cnt, wpr, El, ne, cur, nxt);
        }
      }
      // release the stage only once its words have been consumed: a shared load can still sit
      // in the queue behind this warp's atomics when an early arrive would let TMA overwrite it
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
      if (tid == 0 && i + kTmaStages < nb) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(i + kTmaStages, g + kTmaStages);
      }
      if (U16 && U15_ROLLING) {
        // (AB) rolling drain, no barrier: after each 1024-token block a thread checks one word of
        // one 32nd of the table (every word once per 32 blocks) and moves a half's top two bits
        // (>= 16384) to the u64 tensor by an atomic subtract, safe beside the other warps'
        // increments.  Between two checks a half gains at most (32 + 3 stages of drift) x 1024
        // = 35840 from at most 16383, so it never passes 65535
        const int w = (int)(i & 31u) * kTmaBlock + tid;
        const uint32_t v = cnt[w];
        if (v & 0xc000c000u) {
          const int j = w / wpr;
          const int k0 = 2 * ((w - j * wpr) ^ (j & 31));
          const uint32_t lo = v & 0xc000u, hi = v & 0xc0000000u;
          if (lo) {
            atomicSub(cnt + w, lo);
            atomicAdd(El + (int64_t)j * ne + k0, (unsigned long long)lo);
          }
          if (hi) {
            atomicSub(cnt + w, hi);
            atomicAdd(El + (int64_t)j * ne + k0 + 1, (unsigned long long)(hi >> 16));
          }
        }
        if (U15_ROLL_SYNC && (i + 1) % (uint32_t)U15_ROLL_SYNC == 0) __syncthreads();
      } else if (U16 && (i + 1) % (uint32_t)U15_DRAIN_BLOCKS == 0 && i + 1 < nb) {
        __syncthreads();
        for (int w4 = tid; w4 < (U15_SCALAR_SCAN ? 0 : ne * wpr / 4); w4 += kTmaBlock) {  // 16-byte loads
          const uint4 q = reinterpret_cast<const uint4*>(cnt)[w4];
          if ((q.x | q.y | q.z | q.w) & 0x80008000u) {
            const uint32_t vs[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t v = vs[c];
              if (v & 0x80008000u) {
                const int w = 4 * w4 + c;
                const int j = w / wpr;
                const int k0 = 2 * ((w - j * wpr) ^ (j & 31));
                if (v & 0x8000u) atomicAdd(El + (int64_t)j * ne + k0, 32768ull);
                if (v & 0x80000000u) atomicAdd(El + (int64_t)j * ne + k0 + 1, 32768ull);
                cnt[w] = v & 0x7fff7fffu;
              }
            }
          }
        }
        for (int w = tid; w < (U15_SCALAR_SCAN ? ne * wpr : 0); w += kTmaBlock) {  // AB: one word per load
          const uint32_t v = cnt[w];
          if (v & 0x80008000u) {
            const int j = w / wpr;
            const int k0 = 2 * ((w - j * wpr) ^ (j & 31));
            if (v & 0x8000u) atomicAdd(El + (int64_t)j * ne + k0, 32768ull);
            if (v & 0x80000000u) atomicAdd(El + (int64_t)j * ne + k0 + 1, 32768ull);
            cnt[w] = v & 0x7fff7fffu;
          }
        }
        __syncthreads();
      }
    }
    it += nb;
    __syncthreads();
    u15_flush(cnt, wpr, El, ne);
    __syncthreads();
  }
}

// One layer pair, rows [j0, j0 + R) per unit, with warp-level compaction of the row filter.
template <int K>
__global__ void __launch_bounds__(kSplitWarps * 32, 1)
    count_lm8_split_kernel(Lm8Params prm, const unsigned long long* __restrict__ X,
                           unsigned long long* __restrict__ E) {
  extern __shared__ uint32_t cnt[];
  const int ne = prm.ne;
  const int R = prm.R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* stage =
      reinterpret_cast<unsigned long long*>(cnt + R * ne) + warp * kBatch;  // next-layer ids
  uint16_t* queue = reinterpret_cast<uint16_t*>(
                        reinterpret_cast<unsigned long long*>(cnt + R * ne) + kSplitWarps * kBatch) +
                    warp * (kBatch * K);
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int upc = prm.n_groups * prm.n_parts;
  for (int64_t unit = blockIdx.x; unit < prm.n_units; unit += gridDim.x) {
    const int64_t chunk = unit / upc;
    const int rem = (int)(unit % upc);
    const int l = rem / prm.n_parts;
    const int part = rem - l * prm.n_parts;
    const int j0 = part * R;
    const int jR = min(R, ne - j0);
    const int words = R * ne;
    for (int w = threadIdx.x; w < words; w += blockDim.x) cnt[w] = 0u;
    __syncthreads();
    const int64_t t_begin = chunk * prm.chunk_tokens;
    const int64_t t_end = min(prm.T, t_begin + prm.chunk_tokens);
    const unsigned long long* Xl = X + (int64_t)l * prm.ld;
    const unsigned long long* Xn = X + (int64_t)(l + 1) * prm.ld;
    for (int64_t base = t_begin + (int64_t)warp * kBatch; base < t_end;
         base += (int64_t)kSplitWarps * kBatch) {
      unsigned long long cur[kBatch / 32];
      bool valid[kBatch / 32];
#pragma unroll
      for (int q = 0; q < kBatch / 32; ++q) {
        const int64_t t = base + q * 32 + lane;
        valid[q] = t < t_end;
        cur[q] = valid[q] ? __ldcs(Xl + t) : 0ull;
        stage[q * 32 + lane] = valid[q] ? __ldcs(Xn + t) : 0ull;
      }
      int n_items = 0;
#pragma unroll
      for (int q = 0; q < kBatch / 32; ++q) {
#pragma unroll
        for (int a = 0; a < K; ++a) {
          const uint32_t j = id_of(cur[q], a) - (uint32_t)j0;
          const bool pass = valid[q] && j < (uint32_t)jR;
          const uint32_t m = __ballot_sync(0xffffffffu, pass);
          if (pass) queue[n_items + __popc(m & lt_mask)] = (uint16_t)(j | ((q * 32 + lane) << 8));
          n_items += __popc(m);
        }
      }
      __syncwarp();
      for (int i = lane; i < n_items; i += 32) {
        const uint32_t it = queue[i];
        const uint32_t r = it & 0xffu;
        const unsigned long long nx = stage[it >> 8];
        uint32_t* rowp = cnt + r * ne;
        const uint32_t sw = r & prm.swz;
#pragma unroll
        for (int b = 0; b < K; ++b) atomicAdd(rowp + (id_of(nx, b) ^ sw), 1u);
      }
      __syncwarp();
    }
    __syncthreads();
    for (int w = threadIdx.x; w < jR * ne; w += blockDim.x) {
      const uint32_t v = cnt[w];
      if (v == 0u) continue;
      const int j = w / ne;
      const int kk = (w - j * ne) ^ (j & prm.swz);
      atomicAdd(E + ((int64_t)l * ne + (j0 + j)) * ne + kk, (unsigned long long)v);
    }
    __syncthreads();
  }
}

template <int K>
cudaError_t launch_transpose_k(const uint8_t* trace, int64_t T, int L, int ne, unsigned long long* X,
                               int64_t ld, uint32_t* flags, cudaStream_t s) {
  const size_t smem = (size_t)kTransposeTile * L * K;
  auto kern = transpose_lm8_kernel<K>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = (T + kTransposeTile - 1) / kTransposeTile;
  kern<<<(unsigned)grid, 256, smem, s>>>(trace, T, L, ne, X, ld, flags);
  return cudaGetLastError();
}

template <int K>
cudaError_t launch_count_k(const Lm8Plan& plan, const Lm8Params& prm, const unsigned long long* X,
                           unsigned long long* E, cudaStream_t s, int grid) {
  if (plan.u15) {
    auto kern = count_lm8_u15_kernel<K, false>;
    const size_t smem = (size_t)plan.ne * plan.ne * 2;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 1024, smem, s>>>(prm, X, E);
  } else if (plan.split) {
    auto kern = count_lm8_split_kernel<K>;
    const size_t smem = (size_t)plan.R * plan.ne * 4 + (size_t)kSplitWarps * kBatch * 8 +
                        (size_t)kSplitWarps * kBatch * K * 2;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kSplitWarps * 32, smem, s>>>(prm, X, E);
  } else {
    auto kern = count_lm8_pairs_kernel<K>;
    const size_t smem = (size_t)plan.P * plan.ne * plan.ne * 4;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 1024, smem, s>>>(prm, X, E);
  }
  return cudaGetLastError();
}

}  // namespace

bool lm8_supported(int L, int ne, int k, int id_bytes) {
  return id_bytes == 1 && L > 1 && k >= 1 && k <= 8 && ne <= 256 && (int64_t)kTransposeTile * L * k <= 200 * 1024;
}

Lm8Plan make_lm8_plan(int L, int ne, int k, int sms, int max_smem_optin) {
  Lm8Plan p;
  p.L = L;
  p.ne = ne;
  p.k = k;
  p.sms = sms;
  const int pairs = L - 1;
  if (pairs < 1) return p;  // no layer pairs: A is counted directly (stats.cu)
  const int budget = std::min(max_smem_optin, 200 * 1024);
  const int pair_bytes = ne * ne * 4;
  if (pair_bytes <= budget) {
    p.split = false;
    p.R = ne;
    p.n_parts = 1;
    p.P = std::max(1, std::min(pairs, budget / pair_bytes));
    const int ng = (pairs + p.P - 1) / p.P;
    p.P = (pairs + ng - 1) / ng;
    p.n_groups = (pairs + p.P - 1) / p.P;
  } else if (ne % 64 == 0 && ne * ne * 2 <= budget && !knob_is(GIMBAL_KNOB("GIMBAL_COUNT_PATH"), "split")) {
    p.u15 = true;
    p.P = 1;
    p.R = ne;
    p.n_parts = 1;
    p.n_groups = pairs;
  } else {
    p.split = true;
    p.P = 1;
    const int queue_bytes = kSplitWarps * kBatch * (8 + 2 * k);
    const int split_budget = max_smem_optin - 4096;
    const int max_rows = std::max(1, std::min(256, (split_budget - queue_bytes) / (ne * 4)));
    p.n_parts = (ne + max_rows - 1) / max_rows;
    p.R = (ne + p.n_parts - 1) / p.n_parts;
    p.n_groups = pairs;
  }
  return p;
}

cudaError_t launch_transpose_lm8(const uint8_t* trace, int64_t T, int L, int ne, int k,
                                 unsigned long long* X, int64_t ld, uint32_t* flags, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  switch (k) {
    case 1: return launch_transpose_k<1>(trace, T, L, ne, X, ld, flags, s);
    case 2: return launch_transpose_k<2>(trace, T, L, ne, X, ld, flags, s);
    case 3: return launch_transpose_k<3>(trace, T, L, ne, X, ld, flags, s);
    case 4: return launch_transpose_k<4>(trace, T, L, ne, X, ld, flags, s);
    case 5: return launch_transpose_k<5>(trace, T, L, ne, X, ld, flags, s);
    case 6: return launch_transpose_k<6>(trace, T, L, ne, X, ld, flags, s);
    case 7: return launch_transpose_k<7>(trace, T, L, ne, X, ld, flags, s);
    case 8: return launch_transpose_k<8>(trace, T, L, ne, X, ld, flags, s);
    default: return cudaErrorInvalidValue;
  }
}

// Tensor map over the token-major top-8 trace viewed as a [T][L] u64 matrix, box = cols layers x
// rows tokens.  Needs a 16-byte row pitch (L even) and base; false = caller uses plain loads.
bool encode_trace_map(CUtensorMap* map, const uint8_t* trace, int64_t T, int L, int cols, int rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode || (L & 1) || (reinterpret_cast<uintptr_t>(trace) & 15) || T >= (int64_t)INT32_MAX ||
      GIMBAL_KNOB("GIMBAL_NO_TMA"))
    return false;
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
  if (const char* e = GIMBAL_KNOB("GIMBAL_TMA_PROMO")) {
    const int v = std::atoi(e);
    promo = v >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
            : v >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
            : v >= 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                       : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)L, (cuuint64_t)T};
  const cuuint64_t strides[1] = {(cuuint64_t)L * 8};
  const cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint8_t*>(trace), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int pace_tiles(int dflt) {
  if (const char* e = GIMBAL_KNOB("GIMBAL_PACE")) return std::max(0, std::atoi(e));
  return dflt;
}

bool direct_u15_supported(const Lm8Plan& plan, int id_bytes, const void* ids) {
  return plan.u15 && plan.k == 8 && plan.ne == 256 && id_bytes == 1 &&
         (reinterpret_cast<uintptr_t>(ids) & 7) == 0;
}

cudaError_t launch_count_direct_u15(const Lm8Plan& plan, const uint8_t* trace, int64_t T,
                                    unsigned long long* E, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  Lm8Params prm;
  prm.L = plan.L;
  prm.ne = plan.ne;
  prm.P = 1;
  prm.R = plan.ne;
  prm.swz = 31u;
  prm.n_groups = plan.n_groups;
  prm.n_parts = 1;
  prm.T = T;
  prm.ld = 0;
  const int64_t resident = plan.sms;
  // chunks bound how far apart (in tokens) the CTAs counting different pairs of the same trace
  // rows drift, i.e. the L2 footprint of the shared rows: at 64 Mi DS-V3 tokens 21 chunks read
  // 101 GB from DRAM per launch, 96 chunks 53 GB (31 GB algorithmic), same time; the stream-K
  // tail keeps the split balanced for any count.  Every unit zeroes and flushes a 128 KB table
  // (up to 64 Ki u64 global atomics), so chunks stay >= 512 Ki tokens: a 1 Mi-token streaming
  // window counts in 2 chunks (measured 2.08 ms/window vs 2.53 ms with 16 Ki-token chunks)
  int64_t n_chunks = std::min<int64_t>(96, std::max<int64_t>(1, T >> 19));
  if (const char* e = GIMBAL_KNOB("GIMBAL_DIRECT_CHUNKS")) n_chunks = std::max(1, std::atoi(e));
  n_chunks = std::min<int64_t>(n_chunks, std::max<int64_t>(1, T / 16384));
  prm.chunk_tokens = (T + n_chunks - 1) / n_chunks;
  n_chunks = (T + prm.chunk_tokens - 1) / prm.chunk_tokens;
  prm.n_units = n_chunks * plan.n_groups;
  const int grid = (int)resident;
  CUtensorMap tmap;
  if (encode_trace_map(&tmap, trace, T, plan.L, 2, kTmaBox)) {
    const size_t smem = (size_t)kU15Bytes + (size_t)kTmaStages * kTmaBlock * kTmaCols * 8;
    static const bool u16 = !knob_is(GIMBAL_KNOB("GIMBAL_TMA_MODE"), "u15");
    prm.rolling = GIMBAL_KNOB("GIMBAL_U15_ROLLING") ? 1 : 0;
    if (const char* e = GIMBAL_KNOB("GIMBAL_U15_DRAIN_BLOCKS")) prm.drain_blocks = std::min(32, std::max(1, std::atoi(e)));
    prm.scalar_scan = GIMBAL_KNOB("GIMBAL_U15_SCALAR_SCAN") ? 1 : 0;
    if (const char* e = GIMBAL_KNOB("GIMBAL_U15_ROLL_SYNC")) prm.roll_sync = std::max(0, std::atoi(e));
    static const int agg = [] {
      const char* e = GIMBAL_KNOB("GIMBAL_TMA_AGG");
      return e ? std::atoi(e) : 0;
    }();
    auto kern = !u16      ? count_tm_u15_tma_kernel<false>
                : agg == 1 ? count_tm_u15_tma_kernel<true, 1>
                : agg == 2 ? count_tm_u15_tma_kernel<true, 2>
                           : count_tm_u15_tma_kernel<true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kTmaBlock, smem, s>>>(tmap, prm, E);
    return cudaGetLastError();
  }
  auto kern = count_lm8_u15_kernel<8, true>;
  const size_t smem = (size_t)plan.ne * plan.ne * 2;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 1024, smem, s>>>(prm, reinterpret_cast<const unsigned long long*>(trace), E);
  return cudaGetLastError();
}

cudaError_t launch_count_lm8(const Lm8Plan& plan, const unsigned long long* X, int64_t T, int64_t ld,
                             unsigned long long* E, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  Lm8Params prm;
  prm.L = plan.L;
  prm.ne = plan.ne;
  prm.P = plan.P;
  prm.R = plan.R;
  prm.swz = (plan.ne % 32 == 0) ? 31u : 0u;
  prm.n_groups = plan.n_groups;
  prm.n_parts = plan.n_parts;
  prm.T = T;
  prm.ld = ld;
  const int64_t base_units = (int64_t)plan.n_groups * plan.n_parts;
  const int64_t resident = plan.sms;
  // ~4 waves of units for load balance (hot rows make units uneven), at least 16K tokens each
  // u15 units are whole pairs with no flush pressure: more, smaller units balance hot pairs
  const int64_t waves = plan.u15 ? 8 : 4;
  int64_t n_chunks = std::max<int64_t>(1, (waves * resident + base_units - 1) / base_units);
  n_chunks = std::min<int64_t>(n_chunks, std::max<int64_t>(1, T / 16384));
  prm.chunk_tokens = (T + n_chunks - 1) / n_chunks;
  n_chunks = (T + prm.chunk_tokens - 1) / prm.chunk_tokens;
  prm.n_units = n_chunks * base_units;
  // the u15 kernel splits its work evenly over however many CTAs run it
  const int grid = plan.u15 ? (int)resident : (int)std::min<int64_t>(prm.n_units, resident);
  switch (plan.k) {
    case 1: return launch_count_k<1>(plan, prm, X, E, s, grid);
    case 2: return launch_count_k<2>(plan, prm, X, E, s, grid);
    case 3: return launch_count_k<3>(plan, prm, X, E, s, grid);
    case 4: return launch_count_k<4>(plan, prm, X, E, s, grid);
    case 5: return launch_count_k<5>(plan, prm, X, E, s, grid);
    case 6: return launch_count_k<6>(plan, prm, X, E, s, grid);
    case 7: return launch_count_k<7>(plan, prm, X, E, s, grid);
    case 8: return launch_count_k<8>(plan, prm, X, E, s, grid);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gimbal_gpu
