// greedy_place (placement.cpp:240-299, paper Alg. 3) as a device routine of one CTA, shared by the
// standalone walk kernel (greedy.cu) and the fused small-shape pass (placement.cu tiny_pass_kernel).
// See greedy.cu for the algorithm.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace gimbal_gpu {
namespace greedy_detail {

constexpr int kGreedyThreads = 256;
constexpr int kGreedyMaxLayers = kGreedyThreads;  // layer-parallel phase needs one thread per layer

__device__ __forceinline__ int key_expert(unsigned long long key) { return 0xffffff - (int)(key & 0xffffffull); }
__device__ __forceinline__ unsigned long long key_total(unsigned long long key) { return key >> 24; }

template <int G>
__device__ __forceinline__ int argmin_first(const unsigned long long (&v)[G], const int (&cnt)[G], int cap) {
  int best = -1;
  unsigned long long bv = 0ull;
#pragma unroll
  for (int p = 0; p < G; ++p)
    if (cnt[p] < cap && (best < 0 || v[p] < bv)) {
      best = p;
      bv = v[p];
    }
  return best;
}

// Sequential tail: positions [start, n_valid) with shared loads/counts (placement.cpp:286-297).
__device__ inline void sequential_walk(int g, int cap, const unsigned long long* __restrict__ keys, int64_t start,
                                int64_t n_valid, unsigned long long inv_ne, unsigned long long* load, int* counts,
                                int32_t* __restrict__ out, uint8_t* __restrict__ out_u8) {
  for (int64_t i = start; i < n_valid; ++i) {
    const unsigned long long key = keys[i];
    const int e = key_expert(key);
    const unsigned long long a = key_total(key);
    const int layer = (int)(((unsigned long long)e * inv_ne) >> 40);
    const unsigned long long* lr = load + (a > 0 ? layer : 0) * g;
    int best = -1;
    unsigned long long bv = 0ull;
    for (int p = 0; p < g; ++p) {
      if (counts[p] >= cap) continue;
      if (best < 0 || lr[p] < bv) {
        best = p;
        bv = lr[p];
      }
    }
    out[e] = best;
    if (out_u8) out_u8[e] = (uint8_t)best;
    load[layer * g + best] += a;
    counts[best] += 1;
  }
}

// The whole walk by one CTA of kGreedyThreads threads; `load` = the CTA's greedy shared memory
// (greedy_smem_bytes): [L][g] loads, [g] counts, then the staged keys / lists of the parallel path.
template <int G>  // G = n_gpus (<= 32) for the layer-parallel path; 0 = fully sequential
__device__ void greedy_walk_block(int L, int ne, int g, const unsigned long long* __restrict__ A,
                                  const int32_t* __restrict__ M, int32_t nM, const int32_t* __restrict__ nM_dev,
                                  int32_t anchor, const unsigned long long* __restrict__ keys, int64_t n_keys,
                                  int32_t* __restrict__ out, uint8_t* __restrict__ out_u8, uint8_t* __restrict__ tent,
                                  unsigned long long* __restrict__ load) {
  int* counts = reinterpret_cast<int*>(load + (int64_t)L * g);
  __shared__ long long s_nvalid, s_npos;
  const int64_t m = (int64_t)L * ne;
  const int cap = (int)(m / g);
  const unsigned long long inv_ne = ((1ull << 40) + (unsigned long long)ne - 1) / (unsigned long long)ne;
  for (int64_t i = threadIdx.x; i < (int64_t)L * g; i += blockDim.x) load[i] = 0ull;
  for (int p = threadIdx.x; p < g; p += blockDim.x) counts[p] = 0;
  if (threadIdx.x == 0) {
    s_nvalid = n_keys;
    s_npos = n_keys;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int32_t n_set = nM >= 0 ? nM : *nM_dev;  // device count: set built by affinity_select
    for (int i = 0; i < n_set; ++i) {  // placement.cpp:272-279: the strong-pair set on the anchor
      const int e = M[i];
      out[e] = anchor;
      if (out_u8) out_u8[e] = (uint8_t)anchor;
      load[(int64_t)(e / ne) * g + anchor] += A[e];
      counts[anchor] += 1;
    }
  }
  // boundaries of the sorted keys: [0, n_pos) positive totals, [n_pos, n_valid) zero totals
  for (int64_t i = threadIdx.x; i < n_keys; i += blockDim.x) {
    const unsigned long long k0 = keys[i];
    const unsigned long long k1 = i + 1 < n_keys ? keys[i + 1] : 0ull;
    if (k0 != 0ull && k1 == 0ull) s_nvalid = i + 1;
    if (key_total(k0) > 0 && key_total(k1) == 0) s_npos = i + 1;
    if (i == 0 && key_total(k0) == 0) s_npos = 0;
    if (i == 0 && k0 == 0ull) s_nvalid = 0;
  }
  __syncthreads();
  const int64_t n_valid = s_nvalid;
  const int64_t n_pos = min((int64_t)s_npos, n_valid);

  if constexpr (G > 0) {
    // sorted keys, each position's layer, its tentative GPU, and per-layer position lists staged
    // in shared memory (the launcher only picks this path when they fit)
    unsigned long long* skeys = reinterpret_cast<unsigned long long*>(counts + 4 * ((g + 3) / 4));
    const int64_t n_pad = (n_pos + 15) & ~15ll;
    uint16_t* list = reinterpret_cast<uint16_t*>(skeys + n_pad);  // positions grouped by layer, ascending
    uint8_t* lay = reinterpret_cast<uint8_t*>(list + n_pad);
    tent = lay + n_pad;
    __shared__ int l_start[kGreedyMaxLayers + 1];
    __shared__ long long w_star[kGreedyThreads / 32];
    __shared__ int w_cnt[kGreedyThreads / 32][32];
    __shared__ uint32_t s_full;
    for (int l = threadIdx.x; l <= L; l += blockDim.x) l_start[l] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n_pad; i += blockDim.x) {
      const unsigned long long key = i < n_pos ? keys[i] : 0ull;
      skeys[i] = key;
      const int l = i < n_pos ? (int)(((unsigned long long)key_expert(key) * inv_ne) >> 40) : 0xff;
      lay[i] = (uint8_t)l;
      if (i < n_pos) atomicAdd(&l_start[l + 1], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int l = 0; l < L; ++l) l_start[l + 1] += l_start[l];
      uint32_t f = 0;
      for (int p = 0; p < G; ++p) f |= (counts[p] >= cap ? 1u : 0u) << p;
      s_full = f;
    }
    __syncthreads();
    // one pass per layer thread over the layer map (16 layer bytes per shared load, exact
    // zero-byte test on word ^ layer) writes its positions in ascending order
    if (threadIdx.x < L) {
      const int l = threadIdx.x;
      const uint32_t lw = 0x01010101u * (uint32_t)l;
      int w = l_start[l];
      for (int64_t c = 0; c < n_pos; c += 16) {
        const uint4 w4 = *reinterpret_cast<const uint4*>(lay + c);
        const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t x = ws[q] ^ lw;
          uint32_t z = ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);  // 0x80 where byte == 0
          while (z) {
            list[w++] = (uint16_t)(c + q * 4 + ((__ffs(z) - 1) >> 3));
            z &= z - 1;
          }
        }
      }
    }
    __syncthreads();
    // Rounds: with the set F of full GPUs fixed, every other GPU has room, so the walk is again a
    // set of independent per-layer walks.  A round runs them from the first unplaced position,
    // finds the first position whose GPU would overflow and commits everything before it; that
    // GPU is then full, so there are at most g rounds and every committed position is exact.
    const int l_me = threadIdx.x;
    int cursor = l_me < L ? l_start[l_me] : 0;  // first uncommitted entry of this layer's list
    const int l_end = l_me < L ? l_start[l_me + 1] : 0;
    int64_t pos = 0;
    while (pos < n_pos) {
      const uint32_t full = s_full;
      // ---- A: per-layer walks over the GPUs outside F (cap ignored), tentative GPUs ----
      if (l_me < L) {
        unsigned long long v[G];
#pragma unroll
        for (int p = 0; p < G; ++p) v[p] = load[l_me * G + p];
        for (int idx = cursor; idx < l_end; ++idx) {
          const int i = list[idx];
          const unsigned long long a = key_total(skeys[i]);
          int best = -1;
          unsigned long long bv = 0ull;
#pragma unroll
          for (int p = 0; p < G; ++p)
            if (!((full >> p) & 1u) && (best < 0 || v[p] < bv)) {
              best = p;
              bv = v[p];
            }
#pragma unroll
          for (int p = 0; p < G; ++p) v[p] += (p == best) ? a : 0ull;
          tent[i] = (uint8_t)best;
        }
      }
      __syncthreads();
      // ---- B: first position >= pos whose tentative GPU is already at its cap.  Each warp
      // counts its segment's positions per GPU, then scans the segment with the headroom left
      // by the segments before it; the earliest overflow over all warps is the round's end ----
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      const int n_warps = blockDim.x >> 5;
      const int64_t seg = ((n_pos - pos + n_warps - 1) / n_warps + 31) & ~31ll;
      const int64_t s_lo = min(n_pos, pos + warp * seg), s_hi = min(n_pos, s_lo + seg);
      {
        int taken = 0;  // lane q: positions of this segment on GPU q
        for (int64_t base = s_lo; base < s_hi; base += 32) {
          const int64_t i = base + lane;
          const int p = i < s_hi ? tent[i] : -1;
#pragma unroll
          for (int q = 0; q < G; ++q) {
            const unsigned b = __ballot_sync(0xffffffffu, p == q);
            if (lane == q) taken += __popc(b);
          }
        }
        w_cnt[warp][lane] = taken;
      }
      __syncthreads();
      {
        int room = 0;  // lane p: GPU p's headroom at the start of this segment
        if (lane < G) {
          room = cap - counts[lane];
          for (int w2 = 0; w2 < warp; ++w2) room -= w_cnt[w2][lane];
        }
        long long star = n_pos;
        for (int64_t base = s_lo; base < s_hi; base += 32) {
          const int64_t i = base + lane;
          const int p = i < s_hi ? tent[i] : -1;
          int used_before = 0;  // earlier positions of this chunk on the same GPU
          int taken = 0;        // lane q: positions of this chunk on GPU q
#pragma unroll
          for (int q = 0; q < G; ++q) {
            const unsigned b = __ballot_sync(0xffffffffu, p == q);
            if (p == q) used_before = __popc(b & ((1u << lane) - 1u));
            if (lane == q) taken = __popc(b);
          }
          const int room_p = __shfl_sync(0xffffffffu, room, p < 0 ? 0 : p);
          const unsigned vb = __ballot_sync(0xffffffffu, p >= 0 && used_before >= room_p);
          if (vb) {  // the earliest position of this segment whose GPU would hold cap experts
            star = base + __ffs(vb) - 1;
            break;
          }
          room -= taken;
        }
        if (lane == 0) w_star[warp] = star;
      }
      __syncthreads();
      long long star = n_pos;
      for (int w2 = 0; w2 < n_warps; ++w2) star = min(star, w_star[w2]);
#ifdef GIMBAL_DEBUG_GREEDY
      if (threadIdx.x == 0) printf("greedy round: pos %lld star %lld n_pos %lld full %x\n", (long long)pos,
                                   (long long)star, (long long)n_pos, full);
#endif
      // ---- C: commit [pos, star): loads per layer, counts per GPU, output ----
      if (l_me < L) {
        unsigned long long v[G];
#pragma unroll
        for (int p = 0; p < G; ++p) v[p] = load[l_me * G + p];
        int c[G];
#pragma unroll
        for (int p = 0; p < G; ++p) c[p] = 0;
        for (; cursor < l_end; ++cursor) {
          const int i = list[cursor];
          if (i >= star) break;
          const unsigned long long key = skeys[i];
          const int e = key_expert(key);
          const int p = tent[i];
#pragma unroll
          for (int q = 0; q < G; ++q) {
            v[q] += (q == p) ? key_total(key) : 0ull;
            c[q] += (q == p);
          }
          out[e] = p;
          if (out_u8) out_u8[e] = (uint8_t)p;
        }
#pragma unroll
        for (int p = 0; p < G; ++p) {
          load[l_me * G + p] = v[p];
          if (c[p]) atomicAdd(&counts[p], c[p]);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t f = 0;
        for (int p = 0; p < G; ++p) f |= (counts[p] >= cap ? 1u : 0u) << p;
        s_full = f;
      }
      __syncthreads();
      pos = star;
    }
    // experts with zero activation (home row 0, no load change) after every positive one
    if (threadIdx.x == 0) sequential_walk(g, cap, keys, n_pos, n_valid, inv_ne, load, counts, out, out_u8);
  } else {
    (void)tent;
    __syncthreads();
    if (threadIdx.x == 0) sequential_walk(g, cap, keys, 0, n_valid, inv_ne, load, counts, out, out_u8);
  }
}


// Shared memory of greedy_walk_block, and whether the layer-parallel path applies.
inline size_t greedy_smem_bytes(int L, int g, int64_t n_keys, bool* parallel) {
  const size_t base = (size_t)L * g * 8 + (size_t)4 * ((g + 3) / 4) * 4;
  const size_t n_pad = (size_t)((n_keys + 15) & ~15ll);
  const size_t staged = base + n_pad * 12;  // key (8 B) + list entry (2) + layer + tentative GPU per position
  *parallel = L <= kGreedyMaxLayers && L < 255 && n_pad < 65536 && staged <= 200 * 1024 &&
              (g == 2 || g == 4 || g == 8 || g == 16 || g == 32);
  return *parallel ? staged : base;
}

}  // namespace greedy_detail
}  // namespace gimbal_gpu
