// Internal helpers shared by the sm_100a translation units of libgimbal_gpu.so.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "gimbal_gpu.h"

namespace gimbal_gpu {

// Thread-local last error (gimbal_last_error()).
void set_error(const std::string& msg);
const std::string& last_error();

struct Status {
  int code = GIMBAL_OK;
  std::string msg;
};

// Error flags raised inside kernels (sticky per handle).
enum KernelFlag : uint32_t {
  kFlagIdOutOfRange = 1u,
  kFlagInfeasible = 2u,
  kFlagOverflow = 4u,
  kFlagDuplicates = 8u,  // not an error: some token-layer repeats an id (multiplicity > 1)
};

// A handle's flag words (64 B) are followed by the pacing counters of its counting kernels
// (ptx.cuh pace_arrive_wait): flags + kPaceOffset, kPaceWords of them, zeroed by the launcher
// before each kernel that paces its CTAs.
constexpr int kPaceOffset = 16;
constexpr int kPaceWords = 1024;
constexpr size_t kFlagAllocBytes = (size_t)(kPaceOffset + kPaceWords) * 4;
constexpr uint64_t kPaceTimeoutNs = 300000;
// Tiles (or blocks) per pacing epoch for a counting kernel: `dflt`, or the AB knob GIMBAL_PACE
// (0 = no pacing) in the test/tool build.
int pace_tiles(int dflt);

#define GIMBAL_CUDA_TRY(expr)                                                          \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      ::gimbal_gpu::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));     \
      return GIMBAL_CUDA_ERROR;                                                        \
    }                                                                                  \
  } while (0)

#define GIMBAL_TRY(expr)            \
  do {                              \
    int s_ = (expr);                \
    if (s_ != GIMBAL_OK) return s_; \
  } while (0)

// A stats handle's device tensors and stream (capi.cu), for kernels that count into it directly
// (online.cu).  Callers hold *mu while queueing and call stats_note_added afterwards.
struct StatsInternals {
  unsigned long long* dE = nullptr;
  unsigned long long* dA = nullptr;
  uint32_t* dflags = nullptr;
  cudaStream_t stream = nullptr;
  int device = 0;
  gimbal_topology topo{};
  std::mutex* mu = nullptr;
};
StatsInternals stats_internals(gimbal_stats_t h);
void stats_note_added(gimbal_stats_t h, int64_t n);
int stats_resolve_tokens(gimbal_stats_t h);

// NCCL (dist.cu, resolved at run time): in-place u64 SUM all-reduce; objectives scatter + MIN
// all-reduce + argmin (lowest index).  `comm` is an ncclComm_t.
int nccl_allreduce_u64_sum(unsigned long long* buf, size_t n, void* comm, cudaStream_t s);
int nccl_merge_argmin(const double* local, int64_t n_local, int64_t offset, double* global, int64_t n_total,
                      long long* argmin, void* comm, cudaStream_t s);

// Experiment knobs (alternate kernels for A/B timing and engine-specific tests).  Compiled in only
// for the test/tool build lib/libgimbal_gpu_ab.so (-DGIMBAL_AB_KNOBS); in the shipped
// libgimbal_gpu.so every knob reads as unset, so the kernel choice depends on the inputs alone.
#ifdef GIMBAL_AB_KNOBS
#define GIMBAL_KNOB(name) std::getenv(name)
#else
#define GIMBAL_KNOB(name) (static_cast<const char*>(nullptr))
#endif
// true when knob `name` is set to exactly `value` (never in the shipped build)
inline bool knob_is(const char* knob_value, const char* value) {
  if (!knob_value) return false;
  while (*knob_value && *knob_value == *value) {
    ++knob_value;
    ++value;
  }
  return *knob_value == *value;
}

inline int invalid(const std::string& msg) {
  set_error(msg);
  return GIMBAL_INVALID_ARGUMENT;
}

// MoeTopology::validate (moe.cpp:12-24) with the reference's messages.
int validate_topology(const gimbal_topology& t);

// Scoped device guard.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---- kernel launchers (stream-ordered, return cudaError_t of the launch) ----

// Statistics plan: which layer pairs / row slices one CTA privatises in shared memory.
struct StatsPlan {
  int L = 0, ne = 0, k = 0;
  int pairs_per_group = 1;   // consecutive layer pairs per CTA work unit
  int rows_per_part = 0;     // rows j of E per CTA work unit
  int n_groups = 0, n_parts = 0;
  int smem_words = 0;        // u32 counters per CTA
  int threads = 1024;
  int ctas_per_sm = 1;
  int sms = 148;
};
StatsPlan make_stats_plan(int L, int ne, int k, int sms, int max_smem_optin);

// Layer-major packed ingest path (ingest.cu): uint8 ids, top_k <= 8.
struct Lm8Plan {
  int L = 0, ne = 0, k = 0, sms = 148;
  bool split = false;  // rows of one pair split over units (with warp compaction)
  bool u15 = false;    // whole pair with guarded 15-bit counters (n_e^2 * 2 B fits, n_e % 64 == 0)
  int P = 1, R = 0, n_groups = 0, n_parts = 1;
};
bool lm8_supported(int L, int ne, int k, int id_bytes);
// whole-E-in-shared-memory counting straight from the token-major uint8 trace (small_count.cu)
bool small_count_supported(int L, int ne, int k, int id_bytes, int64_t T);
cudaError_t launch_count_small(int L, int ne, int k, int sms, const uint8_t* trace, int64_t T,
                               unsigned long long* E, uint32_t* flags, cudaStream_t s);
Lm8Plan make_lm8_plan(int L, int ne, int k, int sms, int max_smem_optin);
cudaError_t launch_transpose_lm8(const uint8_t* trace, int64_t T, int L, int ne, int k,
                                 unsigned long long* X, int64_t ld, uint32_t* flags, cudaStream_t s);
cudaError_t launch_count_lm8(const Lm8Plan& plan, const unsigned long long* X, int64_t T, int64_t ld,
                             unsigned long long* E, cudaStream_t s);
// n_e = 256, top_k = 8, uint8 ids (always in range): count straight from the token-major trace
bool direct_u15_supported(const Lm8Plan& plan, int id_bytes, const void* ids);
cudaError_t launch_count_direct_u15(const Lm8Plan& plan, const uint8_t* trace, int64_t T,
                                    unsigned long long* E, cudaStream_t s);

// Tensor map over a token-major top-8 uint8 trace as a [T][L] u64 matrix (ingest.cu).
bool encode_trace_map(CUtensorMap* map, const uint8_t* trace, int64_t T, int L, int cols, int rows);

// tcgen05 int8 multi-hot contraction (mma_count.cu), n_e in (64, 128], top_k <= 8, on LM8 input.
bool mma_count_supported(int L, int ne, int k);
cudaError_t launch_count_mma(int L, int ne, int k, int sms, const unsigned long long* X, int64_t T, int64_t ld,
                             unsigned long long* E, const uint32_t* flags, cudaStream_t s);
// Same contraction reading the token-major trace through TMA (top-8 uint8, L even, 16-byte
// aligned base; ids range-checked and repeated ids detected in the kernel).  Returns
// cudaErrorNotSupported when the trace cannot be mapped.
cudaError_t launch_count_mma_direct(int L, int ne, int sms, const uint8_t* trace, int64_t T,
                                    unsigned long long* E, uint32_t* flags, cudaStream_t s);

// Same contraction for 64-expert layers with two layers stacked per 128-row operand, reading the
// token-major uint8 trace (16-byte aligned) by bulk copies (mma_stack.cu).  cudaErrorNotSupported
// when the shape does not fit.
bool mma_stack_supported(int L, int ne, int k, int id_bytes, const void* ids);
cudaError_t launch_count_mma_stack(int L, int ne, int k, int sms, int max_smem, const uint8_t* trace, int64_t T,
                                   unsigned long long* E, uint32_t* flags, cudaStream_t s);

// Block-scaled FP4 on CTA pairs (fp4x2_count.cu): M = 256 x N = 256 per pair of SMs.
bool fp4x2_count_supported(int L, int ne, int k, int id_bytes, const void* ids, int64_t T);
cudaError_t launch_count_fp4x2(int L, int sms, const uint8_t* trace, int64_t T, unsigned long long* E,
                               cudaStream_t s);
// Block-scaled FP4 tensor-core contraction for 256-expert top-8 uint8 traces (fp4_count.cu):
// L even, 16-byte aligned base, T < 2^31.  cudaErrorNotSupported when the trace cannot be mapped.
bool fp4_count_supported(int L, int ne, int k, int id_bytes, const void* ids, int64_t T);
cudaError_t launch_count_fp4(int L, int sms, const uint8_t* trace, int64_t T, unsigned long long* E,
                             cudaStream_t s);

cudaError_t launch_count_pairs(const StatsPlan& plan, const void* ids, int id_bytes, int64_t T,
                               unsigned long long* E, uint32_t* flags, cudaStream_t s);
cudaError_t launch_count_activation(int L, int ne, int k, const void* ids, int id_bytes, int64_t T,
                                    unsigned long long* A, uint32_t* flags, cudaStream_t s);
cudaError_t launch_derive_activation(int L, int ne, int k, const unsigned long long* E,
                                     unsigned long long* A, cudaStream_t s);
cudaError_t launch_derive_w(int L, int ne, const unsigned long long* E, unsigned long long* W,
                            cudaStream_t s);
cudaError_t launch_add_u64(unsigned long long* dst, const unsigned long long* src, int64_t n, cudaStream_t s);
cudaError_t launch_flat_forms(int L, int ne, const unsigned long long* A,
                              const unsigned long long* E, double* flatA, double* flatW,
                              cudaStream_t s);

// placement
cudaError_t launch_eval_costs(int L, int ne, int g, const unsigned long long* A,
                              const unsigned long long* E, const uint8_t* cands, int64_t C,
                              double alpha, double beta, unsigned long long* scratch_same,
                              double* D, double* cut, double* obj, long long* argmin,
                              uint32_t* flags, bool small_cells, const unsigned long long* device_max_cell,
                              cudaStream_t s);
size_t eval_scratch_bytes(int64_t C);
// max over E cells (for choosing 32-bit partial sums in the evaluator)
cudaError_t launch_max_cell(const unsigned long long* E, int64_t n, unsigned long long* out, cudaStream_t s);

// Which evaluator kernels may run: the u32-partial-sum / byte-plane forms need every E cell
// < 2^27.  When the host can bound the cells (tokens * k^2 < 2^27, or a known max) it launches one
// form; otherwise (`max_cell` != nullptr: written on the device by launch_max_cell just before) both
// forms are launched and each returns at once unless the device max matches its `want_small`, so
// the choice needs no host synchronisation.
struct WidthGuard {
  const unsigned long long* max_cell = nullptr;
  int want_small = 0;
};
__device__ __forceinline__ bool width_skip(const WidthGuard& g) {
  return g.max_cell != nullptr && ((*g.max_cell < (1ull << 27)) != (g.want_small != 0));
}

// tensor-core same-GPU weights (eval_mma.cu): n_e in {128, 256}, g in {4, 8, 16}, cells < 2^27
bool eval_mma_supported(int L, int ne, int g, const uint8_t* cands, int64_t C);
cudaError_t launch_eval_mma(int L, int ne, int g, const unsigned long long* E, const uint8_t* cands, int64_t C,
                            unsigned long long* same, WidthGuard guard, cudaStream_t s);
cudaError_t launch_eval_prepare(int64_t C, unsigned long long* scratch_same, cudaStream_t s);
cudaError_t launch_eval_range(int L, int ne, int g, const unsigned long long* A, const unsigned long long* E,
                              const uint8_t* cands, int64_t C, int64_t base, unsigned long long* same, double* D,
                              uint32_t* flags, long long* bad_index, bool small_cells,
                              const unsigned long long* device_max_cell, cudaStream_t s);
// cut = total - same with total = sum_l sum E_l = (L-1) * k * sum_j A(0, j) (every token adds k^2
// pairings per layer pair and k activations per layer), read from the device A, so scoring needs
// no host-side token count (after an all-reduce it is only known on the device).
cudaError_t launch_eval_finish(int64_t C, int L, int ne, int k, const unsigned long long* A, double alpha,
                               double beta, const unsigned long long* same, const double* D, double* cut,
                               double* obj, long long* argmin, uint32_t* flags, cudaStream_t s);

// per-candidate bottleneck excess sum_l max(0, peak_l * g / (T k) - 1) over the handle's A
cudaError_t launch_eval_excess(int L, int ne, int g, const unsigned long long* A, const uint8_t* cands, int64_t C,
                               double* excess, uint32_t* flags, cudaStream_t s);

cudaError_t launch_affinity_keys(int L, int ne, const unsigned long long* E, double threshold,
                                 unsigned long long* keys, int64_t n_pad, uint32_t* flags,
                                 cudaStream_t s);
cudaError_t launch_affinity_topk(int L, int ne, const unsigned long long* E, double threshold, int K,
                                 unsigned long long* a, unsigned long long* b, uint32_t* flags,
                                 unsigned long long** result, cudaStream_t s);
constexpr int kTopkMax = 1024;  // top_e up to this uses segment top-K instead of a full sort
cudaError_t launch_affinity_select(int L, int ne, const unsigned long long* sorted_keys,
                                   int64_t n_keys, int32_t top_e, int32_t capacity,
                                   uint32_t* member_bits, int32_t* out, int32_t* n_out,
                                   cudaStream_t s);

cudaError_t launch_greedy_keys(int64_t m, const unsigned long long* A, const uint32_t* anchored,
                               unsigned long long* keys, int64_t n_pad, uint32_t* flags,
                               cudaStream_t s);
cudaError_t launch_greedy_walk(int L, int ne, int g, const unsigned long long* A, const int32_t* M,
                               int32_t nM, int32_t anchor, const unsigned long long* keys,
                               int64_t n_keys, int32_t* out, uint8_t* out_u8, uint8_t* tent_scratch,
                               cudaStream_t s, const int32_t* nM_dev = nullptr);  // nM < 0: read *nM_dev

// Sort uint64 keys descending in place (bitonic; n must be a power of two).
cudaError_t sort_u64_desc(unsigned long long* keys, int64_t n, cudaStream_t s);
// The whole placement pass for small shapes in one launch (placement.cu tiny_pass_kernel):
// cudaErrorNotSupported when the shape does not fit it.  Every E cell must be < 2^32; `same` holds
// tiny_scratch_bytes(C).
size_t tiny_scratch_bytes(int64_t C);
cudaError_t launch_tiny_pass(int L, int ne, int g, int k, double threshold, int top_e, int capacity, int anchor,
                             const unsigned long long* E, unsigned long long* A_out, uint8_t* cands, int64_t C,
                             double alpha, double beta, double* scores, long long* argmin, int32_t* placement,
                             int32_t* members, int32_t* n_members, uint32_t* flags, unsigned long long* same,
                             bool init_scratch, uint32_t* flags_out, int32_t* ring, uint32_t* ring_seq,
                             int ring_slots, cudaStream_t s);

cudaError_t launch_comm_cost(int L, int ne, int k, const void* ids, int id_bytes, int64_t T,
                             const int32_t* assign, unsigned long long* out, uint32_t* flags,
                             cudaStream_t s);

cudaError_t launch_generate_trace(int L, int ne, int k, const uint32_t* cdf, uint64_t thr_base,
                                  uint64_t thr_unif, uint64_t seed, int64_t t0, int64_t T,
                                  uint8_t* out, cudaStream_t s);

inline int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace gimbal_gpu
