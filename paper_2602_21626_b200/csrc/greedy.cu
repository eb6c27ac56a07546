// greedy_place (placement.cpp:240-299, paper Alg. 3) on the compact flat activation, sm_100a.
//
// The reference walks the unanchored experts in (-total, id) order and puts each on the GPU with
// headroom whose load in the expert's home row is lowest (strict <, lowest GPU first), then adds
// the expert's activation column to that GPU.  On the flat activation an expert of layer l with
// A > 0 has home row l and only changes row l; an expert with A = 0 (home row 0) changes nothing
// and sorts after every positive expert.  So until some GPU reaches its cardinality cap m/g, the
// walk decomposes into independent per-layer walks, and after that it does again for as long as
// the set of full GPUs stays the same.  The kernel groups the positions by layer once, then runs
// rounds, each from the first unplaced position with the current full set F:
//   A. every layer's walk in parallel (one thread per layer, its load row in registers) over the
//      GPUs outside F, cap ignored, recording each position's tentative GPU;
//   B. s*, the first position whose tentative GPU would already be full (each warp counts a
//      segment per GPU with ballots, then scans it with the headroom the earlier segments leave);
//   C. commits positions before s*; the GPU at s* is now full.
// At most g rounds; positions before each s* are provably identical to the sequential walk.  The
// A = 0 experts (no load change, sorted last) finish with the exact sequential walk.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "greedy_block.cuh"
#include "internal.cuh"

namespace gimbal_gpu {

namespace {

using namespace greedy_detail;

template <int G>
__global__ void __launch_bounds__(kGreedyThreads)
    greedy_walk_kernel(int L, int ne, int g, const unsigned long long* __restrict__ A,
                       const int32_t* __restrict__ M, int32_t nM, const int32_t* __restrict__ nM_dev,
                       int32_t anchor, const unsigned long long* __restrict__ keys, int64_t n_keys,
                       int32_t* __restrict__ out, uint8_t* __restrict__ out_u8, uint8_t* __restrict__ tent) {
  extern __shared__ unsigned long long greedy_smem[];
  greedy_walk_block<G>(L, ne, g, A, M, nM, nM_dev, anchor, keys, n_keys, out, out_u8, tent, greedy_smem);
}

}  // namespace

cudaError_t launch_greedy_walk(int L, int ne, int g, const unsigned long long* A, const int32_t* M, int32_t nM,
                               int32_t anchor, const unsigned long long* keys, int64_t n_keys, int32_t* out,
                               uint8_t* out_u8, uint8_t* tent_scratch, cudaStream_t s, const int32_t* nM_dev) {
  bool parallel = false;
  const size_t smem = greedy_smem_bytes(L, g, n_keys, &parallel);
  parallel = parallel && tent_scratch != nullptr;
  auto kern = !parallel ? greedy_walk_kernel<0>
            : g == 8    ? greedy_walk_kernel<8>
            : g == 4    ? greedy_walk_kernel<4>
            : g == 2    ? greedy_walk_kernel<2>
            : g == 16   ? greedy_walk_kernel<16>
            : g == 32   ? greedy_walk_kernel<32>
                        : greedy_walk_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<1, kGreedyThreads, smem, s>>>(L, ne, g, A, M, nM, nM_dev, anchor, keys, n_keys, out, out_u8, tent_scratch);
  return cudaGetLastError();
}

}  // namespace gimbal_gpu
