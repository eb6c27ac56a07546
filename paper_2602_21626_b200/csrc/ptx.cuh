// Thin inline-PTX wrappers for mbarriers and the tensor memory accelerator (sm_100a).
#pragma once

#include <cuda.h>  // CUtensorMap (type only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>

#include <cstdint>

namespace gimbal_gpu {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// Spin until the phase with the given parity has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// 2-D tiled TMA load of one box at (c0 = innermost, c1) into shared memory, completing on bar.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Pacing barrier among the CTAs that read the same trace rows (the units of one token range):
// arrive on the counter, then wait until `target` arrivals, so no CTA runs more than one epoch
// ahead of the others and the rows they share are still in L2 when the last one reads them.  No
// data passes through it (relaxed ordering suffices), so it is only a speed hint: the wait gives
// up after `timeout_ns` (co-residency is not guaranteed when other kernels share the GPU).
__device__ __forceinline__ void pace_arrive_wait(uint32_t* ctr, uint32_t target, uint64_t timeout_ns) {
  atomicAdd(ctr, 1u);
  if (*reinterpret_cast<volatile uint32_t*>(ctr) >= target) return;
  const uint64_t t0 = globaltimer_ns();
  while (*reinterpret_cast<volatile uint32_t*>(ctr) < target) {
    if (globaltimer_ns() - t0 > timeout_ns) break;
    __nanosleep(256);
  }
}

// ---- packed top-8 uint8 id words (one u64 per token-layer) ----

__device__ __forceinline__ uint32_t id_byte(unsigned long long w, int a) {
  return (uint32_t)(w >> (8 * a)) & 0xffu;
}

// true when two of the eight id bytes are equal (every pair compared once: within each half at
// byte distance 1 and 2, across the halves at all four rotations; "has a zero byte" test)
__device__ __forceinline__ bool has_dup8(unsigned long long x) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  auto z = [](uint32_t v) { return (v - 0x01010101u) & ~v & 0x80808080u; };
  uint32_t acc = z(lo ^ __byte_perm(lo, 0, 0x0321)) | z(lo ^ __byte_perm(lo, 0, 0x1032));
  acc |= z(hi ^ __byte_perm(hi, 0, 0x0321)) | z(hi ^ __byte_perm(hi, 0, 0x1032));
  acc |= z(lo ^ hi) | z(lo ^ __byte_perm(hi, 0, 0x0321));
  acc |= z(lo ^ __byte_perm(hi, 0, 0x1032)) | z(lo ^ __byte_perm(hi, 0, 0x2103));
  return acc != 0u;
}

// true when some id byte is >= n (1 <= n <= 128): bytes below 128 gain bit 7 from + (128 - n)
// exactly when they reach n, bytes from 128 up carry it already
__device__ __forceinline__ bool has_ge8(unsigned long long w, uint32_t n) {
  const unsigned long long add = (unsigned long long)(128u - n) * 0x0101010101010101ull;
  return (((w & 0x7f7f7f7f7f7f7f7full) + add) | w) & 0x8080808080808080ull;
}

}  // namespace gimbal_gpu
