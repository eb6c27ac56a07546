// C ABI (include/gimbal_gpu.h) over the sm_100a kernels: handles, ingest, readback, placement.
//
// Host-side logic here is limited to argument validation (with the reference's messages),
// buffer management and stream ordering; every numeric result is produced on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace gimbal_gpu {

namespace {
thread_local std::string t_err;
}
void set_error(const std::string& msg) { t_err = msg; }
const std::string& last_error() { return t_err; }

int validate_topology(const gimbal_topology& t) {
  if (t.n_layers < 1) return invalid("MoeTopology: n_layers must be >= 1");
  if (t.n_experts < 1) return invalid("MoeTopology: n_experts must be >= 1");
  if (t.top_k < 1 || t.top_k > t.n_experts) return invalid("MoeTopology: top_k must be in [1, n_experts]");
  if (t.n_gpus < 1 || t.n_gpus > t.n_experts) return invalid("MoeTopology: n_gpus must be in [1, n_experts]");
  if (t.n_experts % t.n_gpus != 0) return invalid("MoeTopology: n_experts must be divisible by n_gpus");
  return GIMBAL_OK;
}

namespace {

// Device buffer that grows on demand (per handle; freed with the handle).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t n) {
    if (n <= bytes) return GIMBAL_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    GIMBAL_CUDA_TRY(cudaMalloc(&p, n));
    bytes = n;
    return GIMBAL_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int flags_to_status(uint32_t f) {
  if (f & kFlagIdOutOfRange) {
    set_error("add_token: expert id out of range [0, n_experts)");
    return GIMBAL_OUT_OF_RANGE;
  }
  if (f & kFlagOverflow) {
    set_error("count exceeds the exactly representable range");
    return GIMBAL_OVERFLOW;
  }
  return GIMBAL_OK;
}

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace
}  // namespace gimbal_gpu

using namespace gimbal_gpu;

struct gimbal_stats_s {
  gimbal_topology topo{};
  int device = 0;
  int sms = 148;
  int smem_optin = 0;
  StatsPlan plan;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  unsigned long long* dE = nullptr;  // (L-1)*ne*ne
  unsigned long long* dA = nullptr;  // L*ne
  unsigned long long* dW = nullptr;  // ne*ne
  uint32_t* dflags = nullptr;
  int64_t tokens = 0;
  bool derived = true;
  // evaluator cell width (pick_cell_width): bounded on the host from the token count, else decided
  // on the device from a max-cell probe that is re-run only when the counts changed
  int64_t count_version = 0;     // bumped by every reset / add / merge / reduction
  int64_t probed_version = -1;   // count state the device probe (`probe`) was taken on
  bool small_cells = false;
  const unsigned long long* width_guard = nullptr;
  // after an all-reduce without a known global total the token count lives on the device only
  // (as sum_j A(0, j) / k); gimbal_stats_tokens reads it back on demand
  bool tokens_on_device = false;
  // host-ingest staging (double-buffered)
  static constexpr int kStages = 2;
  size_t stage_bytes = 0;
  void* dstage[kStages] = {nullptr, nullptr};
  void* hstage[kStages] = {nullptr, nullptr};
  cudaEvent_t ev_copied[kStages] = {nullptr, nullptr};
  cudaEvent_t ev_consumed[kStages] = {nullptr, nullptr};
  // layer-major ingest buffers (ingest.cu)
  static constexpr int64_t kLm8BufferBytes = (int64_t)4 << 30;
  Lm8Plan lm8_plan;
  bool use_mma = false;  // tcgen05 contraction instead of shared-memory counting (n_e <= 128)
  bool use_stack = false;  // tcgen05 contraction with two 64-expert layers per operand
  bool use_fp4 = false;    // block-scaled FP4 tcgen05 contraction (256 experts, top-8)
  bool use_fp4x2 = false;  // the same on CTA pairs (cta_group::2)
  cudaStream_t t_stream = nullptr;
  unsigned long long* lm8[kStages] = {nullptr, nullptr};
  int64_t lm8_tokens = 0;
  int lm8_next = 0;
  cudaEvent_t ev_lm8_ready[kStages] = {nullptr, nullptr};
  cudaEvent_t ev_lm8_free[kStages] = {nullptr, nullptr};
  cudaEvent_t ev_order = nullptr;
  // optional event pairs around each counting launch (gimbal_stats_count_timing)
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
  size_t tev_used = 0;
  // gimbal_pass_graph: the step recorded as a CUDA graph (reset + count + pass), replayed while the
  // arguments stay the same; its counting kernels are timed by event-record nodes (g_tev)
  bool capturing = false;
  struct GraphKey {
    const void* ids = nullptr;
    int id_bytes = 0;
    int64_t n = 0;
    double threshold = 0, alpha = 0, beta = 0;
    int32_t top_e = 0, capacity = 0, anchor = 0;
    uint8_t* cands = nullptr;
    int64_t C = 0;
    double* scores = nullptr;
    int64_t* argmin = nullptr;
    int32_t *placement = nullptr, *members = nullptr, *n_members = nullptr;
    uint32_t* flags = nullptr;
    int sms = 0;
    bool operator==(const GraphKey& o) const {
      return ids == o.ids && id_bytes == o.id_bytes && n == o.n && threshold == o.threshold && alpha == o.alpha &&
             beta == o.beta && top_e == o.top_e && capacity == o.capacity && anchor == o.anchor && cands == o.cands &&
             C == o.C && scores == o.scores && argmin == o.argmin && placement == o.placement &&
             members == o.members && n_members == o.n_members && flags == o.flags && sms == o.sms;
    }
  };
  GraphKey gkey;
  int gseen = 0;  // eager runs with gkey (the first allocates every scratch buffer)
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;  // kept: its event-record nodes are re-pointed per timed replay
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_tev;        // recorded at capture
  std::vector<std::pair<cudaGraphNode_t, cudaGraphNode_t>> g_nodes;  // their record nodes
  // timed replays: every replay records into a fresh event pair (the exec's record nodes are
  // re-pointed before the launch), so no replay waits on the host for the previous one's timing;
  // the pairs are read when the timing is collected (or when too many are outstanding)
  using EvPair = std::pair<cudaEvent_t, cudaEvent_t>;
  std::vector<EvPair> g_pool, g_inflight;
  double g_ms = 0.0;
  int64_t g_launches = 0;
  int harvest_graph_timing(bool accumulate = true) {
    for (auto& pr : g_inflight) {
      if (accumulate) {
        GIMBAL_CUDA_TRY(cudaEventSynchronize(pr.second));
        float ms = 0.f;
        GIMBAL_CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
        g_ms += ms;
        ++g_launches;
      }
      g_pool.push_back(pr);
    }
    g_inflight.clear();
    return GIMBAL_OK;
  }
  // before a timed replay: fresh event pairs into the exec's record nodes
  int arm_graph_timing() {
    if (g_inflight.size() >= 4096) GIMBAL_TRY(harvest_graph_timing());
    for (auto& nd : g_nodes) {
      EvPair pr;
      if (!g_pool.empty()) {
        pr = g_pool.back();
        g_pool.pop_back();
      } else {
        GIMBAL_CUDA_TRY(cudaEventCreate(&pr.first));
        GIMBAL_CUDA_TRY(cudaEventCreate(&pr.second));
      }
      GIMBAL_CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(gexec, nd.first, pr.first));
      GIMBAL_CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(gexec, nd.second, pr.second));
      g_inflight.push_back(pr);
    }
    return GIMBAL_OK;
  }
  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    gexec = nullptr;
    graph = nullptr;
    for (auto* v : {&g_tev, &g_pool, &g_inflight})
      for (auto& pr : *v) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
      }
    g_tev.clear();
    g_pool.clear();
    g_inflight.clear();
    g_nodes.clear();
  }

  int timing_begin() {
    if (capturing) {  // an event-record node in the graph, timed on every replay
      cudaEvent_t a, b;
      GIMBAL_CUDA_TRY(cudaEventCreate(&a));
      GIMBAL_CUDA_TRY(cudaEventCreate(&b));
      g_tev.emplace_back(a, b);
      GIMBAL_CUDA_TRY(cudaEventRecordWithFlags(a, stream, cudaEventRecordExternal));
      return GIMBAL_OK;
    }
    if (!timing) return GIMBAL_OK;
    if (tev_used == tev.size()) {
      cudaEvent_t a, b;
      GIMBAL_CUDA_TRY(cudaEventCreate(&a));
      GIMBAL_CUDA_TRY(cudaEventCreate(&b));
      tev.emplace_back(a, b);
    }
    GIMBAL_CUDA_TRY(cudaEventRecord(tev[tev_used].first, stream));
    return GIMBAL_OK;
  }
  int timing_end() {
    if (capturing) {
      GIMBAL_CUDA_TRY(cudaEventRecordWithFlags(g_tev.back().second, stream, cudaEventRecordExternal));
      return GIMBAL_OK;
    }
    if (!timing) return GIMBAL_OK;
    GIMBAL_CUDA_TRY(cudaEventRecord(tev[tev_used].second, stream));
    ++tev_used;
    return GIMBAL_OK;
  }
  // scratch
  DevBuf cand, same, dout, keys, misc, ints, probe, dscr;
  // side stream of gimbal_pass_async: the greedy walk runs there beside the candidate scoring
  cudaStream_t g_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_caller = nullptr, ev_back = nullptr;  // gimbal_pass_enqueue's stream joins
  // the fused small-shape pass leaves its ticket / bad index ready in `same`: set once per buffer
  const unsigned long long* tiny_ready_same = nullptr;
  int64_t tiny_ready_C = -1;
  bool last_pass_tiny = false;  // the latest gimbal_pass_async took the fused small-shape path
  // the fused pass writes its packed results into a mapped host ring (slot = device counter
  // dflags[8] modulo the slots); host_seq mirrors that counter (every executed fused pass, never a
  // capture), ran_tiny / ring_slot describe the latest executed pass
  static constexpr int kRingSlots = 64;
  int32_t* ring_host = nullptr;
  int32_t* ring_dev = nullptr;
  uint64_t host_seq = 0;
  int ring_slot = 0;
  bool ran_tiny = false;
  void note_tiny_run() {
    ring_slot = (int)(host_seq % kRingSlots);
    ++host_seq;
    ran_tiny = true;
  }
  bool g_uses_tiny = false;     // ... while the replayed graph was being recorded
  // scratch buffers the recorded graph points into; a replay needs all of them unchanged
  std::vector<const void*> scratch_snapshot() const {
    return {cand.p, same.p, dout.p, keys.p, misc.p, ints.p, probe.p, dscr.p, lm8[0], lm8[1]};
  }
  std::vector<const void*> g_scratch;
  std::mutex mu;
  // strong-pair set resident in `ints` for the asynchronous window path (streaming windows keep
  // M fixed, sim.cpp:94-104, so it is uploaded once): valid while ints.p == m_cached_buf
  std::vector<int32_t> m_cached;
  int32_t m_cached_anchor = -1;
  void* m_cached_buf = nullptr;

  int64_t m() const { return (int64_t)topo.n_layers * topo.n_experts; }
  int64_t nE() const { return (int64_t)(topo.n_layers - 1) * topo.n_experts * topo.n_experts; }

  // A is derived from E for every placement; W = sum_l E_l only when it is read back (the
  // placement pass scores cuts on E directly), which saves a launch per pass and per window
  bool w_derived = true;
  void set_derived(bool d) {
    derived = d;
    w_derived = d;
  }
  int derive() {
    if (derived) return GIMBAL_OK;
    const int L = topo.n_layers, ne = topo.n_experts;
    if (L > 1) GIMBAL_CUDA_TRY(launch_derive_activation(L, ne, topo.top_k, dE, dA, stream));
    derived = true;
    return GIMBAL_OK;
  }
  int derive_w() {
    GIMBAL_TRY(derive());
    if (w_derived) return GIMBAL_OK;
    if (topo.n_layers > 1) GIMBAL_CUDA_TRY(launch_derive_w(topo.n_layers, topo.n_experts, dE, dW, stream));
    w_derived = true;
    return GIMBAL_OK;
  }

  // Host token count after an all-reduce that left it on the device: every token adds k
  // activations to layer 0, so tokens = sum_j A(0, j) / k (one small read-back, synchronising).
  int resolve_tokens() {
    if (!tokens_on_device) return GIMBAL_OK;
    GIMBAL_TRY(derive());
    std::vector<unsigned long long> a0((size_t)topo.n_experts);
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(a0.data(), dA, a0.size() * 8, cudaMemcpyDeviceToHost, stream));
    GIMBAL_CUDA_TRY(cudaStreamSynchronize(stream));
    unsigned long long s = 0;
    for (unsigned long long v : a0) s += v;
    tokens = (int64_t)(s / (unsigned long long)topo.top_k);
    tokens_on_device = false;
    return GIMBAL_OK;
  }

  int check_flags() {
    uint32_t f = 0;
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(&f, dflags, sizeof(f), cudaMemcpyDeviceToHost, stream));
    GIMBAL_CUDA_TRY(cudaStreamSynchronize(stream));
    return flags_to_status(f & (kFlagIdOutOfRange | kFlagOverflow));
  }

  // Layer-major ingest: the trace is transposed chunk by chunk on t_stream into one of two LM8
  // buffers while the previous chunk is counted on `stream`.
  int count_lm8(const uint8_t* ids, int64_t n) {
    const int L = topo.n_layers, ne = topo.n_experts, k = topo.top_k;
    const int64_t per_token = (int64_t)L * 8;
    const int64_t cap_tokens = std::max<int64_t>(1, kLm8BufferBytes / per_token);
    // row stride (tokens) a multiple of 16 so every layer row is 16-byte aligned for TMA bulk
    // copies; 64 B of slack for the rounded-up tail copy of the last row
    const int64_t ch = (std::min<int64_t>(n, cap_tokens) + 15) / 16 * 16;
    if (ch > lm8_tokens) {
      for (int b = 0; b < kStages; ++b) {
        if (lm8[b]) {
          GIMBAL_CUDA_TRY(cudaStreamSynchronize(stream));
          cudaFree(lm8[b]);
          lm8[b] = nullptr;
        }
        GIMBAL_CUDA_TRY(cudaMalloc(&lm8[b], (size_t)ch * per_token + 64));
      }
      lm8_tokens = ch;
    }
    const int64_t row = (int64_t)L * k;
    // the first transposition cannot overlap counting: keep that chunk short (1/8 of a buffer)
    const int64_t first = n > ch ? std::max<int64_t>(16, (ch / 8 + 15) / 16 * 16) : ch;
    for (int64_t t0 = 0; t0 < n;) {
      const int b = lm8_next;
      lm8_next ^= 1;
      const int64_t cnt = std::min<int64_t>(t0 == 0 ? first : ch, n - t0);
      const int64_t t_this = t0;
      t0 += cnt;
      GIMBAL_CUDA_TRY(cudaStreamWaitEvent(t_stream, ev_lm8_free[b], 0));
      GIMBAL_CUDA_TRY(launch_transpose_lm8(ids + t_this * row, cnt, L, ne, k, lm8[b], lm8_tokens, dflags, t_stream));
      GIMBAL_CUDA_TRY(cudaEventRecord(ev_lm8_ready[b], t_stream));
      GIMBAL_CUDA_TRY(cudaStreamWaitEvent(stream, ev_lm8_ready[b], 0));
      GIMBAL_TRY(timing_begin());
      if (use_mma) {
        GIMBAL_CUDA_TRY(launch_count_mma(L, ne, k, sms, lm8[b], cnt, lm8_tokens, dE, dflags, stream));
      } else {
        GIMBAL_CUDA_TRY(launch_count_lm8(lm8_plan, lm8[b], cnt, lm8_tokens, dE, stream));
      }
      GIMBAL_TRY(timing_end());
      GIMBAL_CUDA_TRY(cudaEventRecord(ev_lm8_free[b], stream));
    }
    return GIMBAL_OK;
  }

  int count_device(const void* ids, int id_bytes, int64_t n) {
    const int L = topo.n_layers;
    if (use_stack && mma_stack_supported(L, topo.n_experts, topo.top_k, id_bytes, ids) &&
        !GIMBAL_KNOB("GIMBAL_NO_DIRECT")) {
      // 64-expert layers: two layers per 128-row tensor-core operand, straight from the trace
      GIMBAL_TRY(timing_begin());
      const cudaError_t e = launch_count_mma_stack(L, topo.n_experts, topo.top_k, sms, smem_optin,
                                                   static_cast<const uint8_t*>(ids), n, dE, dflags, stream);
      if (e != cudaErrorNotSupported) {
        GIMBAL_CUDA_TRY(e);
        GIMBAL_TRY(timing_end());
        return GIMBAL_OK;
      }
      cudaGetLastError();  // shape does not fit the stacked kernel: fall through (timing slot reused)
    }
    if (use_fp4x2 && fp4x2_count_supported(L, topo.n_experts, topo.top_k, id_bytes, ids, n) &&
        !GIMBAL_KNOB("GIMBAL_NO_DIRECT")) {
      // 256 experts, top-8: block-scaled FP4 on CTA pairs straight from the trace
      GIMBAL_TRY(timing_begin());
      const cudaError_t e = launch_count_fp4x2(L, sms, static_cast<const uint8_t*>(ids), n, dE, stream);
      if (e != cudaErrorNotSupported) {
        GIMBAL_CUDA_TRY(e);
        GIMBAL_TRY(timing_end());
        return GIMBAL_OK;
      }
      cudaGetLastError();  // not mappable: fall through (timing slot reused)
    }
    if (use_fp4 && fp4_count_supported(L, topo.n_experts, topo.top_k, id_bytes, ids, n) &&
        !GIMBAL_KNOB("GIMBAL_NO_DIRECT")) {
      // 256 experts, top-8: block-scaled FP4 tensor-core contraction straight from the trace
      GIMBAL_TRY(timing_begin());
      const cudaError_t e = launch_count_fp4(L, sms, static_cast<const uint8_t*>(ids), n, dE, stream);
      if (e != cudaErrorNotSupported) {
        GIMBAL_CUDA_TRY(e);
        GIMBAL_TRY(timing_end());
        return GIMBAL_OK;
      }
      cudaGetLastError();  // not mappable: fall through (timing slot reused)
    }
    if (!use_mma && direct_u15_supported(lm8_plan, id_bytes, ids) && !GIMBAL_KNOB("GIMBAL_NO_DIRECT")) {
      // every uint8 id is a valid expert at n_e = 256: no validation / transposition pass
      GIMBAL_TRY(timing_begin());
      GIMBAL_CUDA_TRY(launch_count_direct_u15(lm8_plan, static_cast<const uint8_t*>(ids), n, dE, stream));
      GIMBAL_TRY(timing_end());
      return GIMBAL_OK;
    }
    if (use_mma && id_bytes == 1 && topo.top_k == 8 && L % 2 == 0 && (reinterpret_cast<uintptr_t>(ids) & 15) == 0 &&
        n < INT32_MAX && !GIMBAL_KNOB("GIMBAL_NO_DIRECT") && !GIMBAL_KNOB("GIMBAL_NO_TMA")) {
      // tensor-core contraction straight from the token-major trace (TMA-mapped rows)
      GIMBAL_TRY(timing_begin());
      GIMBAL_CUDA_TRY(launch_count_mma_direct(L, topo.n_experts, sms, static_cast<const uint8_t*>(ids), n, dE,
                                              dflags, stream));
      GIMBAL_TRY(timing_end());
      return GIMBAL_OK;
    }
    if (small_count_supported(L, topo.n_experts, topo.top_k, id_bytes, n) && !GIMBAL_KNOB("GIMBAL_NO_SMALL")) {
      // the whole E fits every CTA's shared memory (Mixtral class): one pass, no transposition
      GIMBAL_TRY(timing_begin());
      GIMBAL_CUDA_TRY(launch_count_small(L, topo.n_experts, topo.top_k, sms, static_cast<const uint8_t*>(ids), n,
                                         dE, dflags, stream));
      GIMBAL_TRY(timing_end());
      return GIMBAL_OK;
    }
    if (lm8_supported(L, topo.n_experts, topo.top_k, id_bytes)) {
      // the transposition must see work already queued on `stream` (e.g. host staging)
      GIMBAL_CUDA_TRY(cudaEventRecord(ev_order, stream));
      GIMBAL_CUDA_TRY(cudaStreamWaitEvent(t_stream, ev_order, 0));
      return count_lm8(static_cast<const uint8_t*>(ids), n);
    }
    if (L > 1) {
      GIMBAL_TRY(timing_begin());
      GIMBAL_CUDA_TRY(launch_count_pairs(plan, ids, id_bytes, n, dE, dflags, stream));
      GIMBAL_TRY(timing_end());
    } else {
      GIMBAL_CUDA_TRY(launch_count_activation(L, topo.n_experts, topo.top_k, ids, id_bytes, n, dA,
                                              dflags, stream));
    }
    return GIMBAL_OK;
  }

  int ensure_staging() {
    if (stage_bytes) return GIMBAL_OK;
    const size_t row = (size_t)topo.n_layers * topo.top_k * 4;
    stage_bytes = std::max<size_t>(row, (size_t)1 << 30);
    for (int b = 0; b < kStages; ++b) {
      GIMBAL_CUDA_TRY(cudaMalloc(&dstage[b], stage_bytes));
      GIMBAL_CUDA_TRY(cudaEventCreateWithFlags(&ev_copied[b], cudaEventDisableTiming));
      GIMBAL_CUDA_TRY(cudaEventCreateWithFlags(&ev_consumed[b], cudaEventDisableTiming));
    }
    return GIMBAL_OK;
  }

  // Host trace: chunks are copied on copy_stream into alternating device stages while the
  // previous chunk is counted on `stream`.  Pageable sources go through pinned bounce buffers.
  int count_host(const void* ids, int id_bytes, int64_t n) {
    GIMBAL_TRY(ensure_staging());
    const bool pinned = is_pinned_host(ids);
    if (!pinned && !hstage[0]) {
      for (int b = 0; b < kStages; ++b) GIMBAL_CUDA_TRY(cudaMallocHost(&hstage[b], stage_bytes));
    }
    const size_t row = (size_t)topo.n_layers * topo.top_k * id_bytes;
    const int64_t per = (int64_t)(stage_bytes / row);
    const char* src = static_cast<const char*>(ids);
    int b = 0;
    for (int64_t t0 = 0; t0 < n; t0 += per, b ^= 1) {
      const int64_t cnt = std::min<int64_t>(per, n - t0);
      const size_t bytes = (size_t)cnt * row;
      GIMBAL_CUDA_TRY(cudaStreamWaitEvent(copy_stream, ev_consumed[b], 0));
      const void* from = src + (size_t)t0 * row;
      if (!pinned) {
        // the bounce buffer is free once its previous H2D completed
        GIMBAL_CUDA_TRY(cudaEventSynchronize(ev_copied[b]));
        std::memcpy(hstage[b], from, bytes);
        from = hstage[b];
      }
      GIMBAL_CUDA_TRY(cudaMemcpyAsync(dstage[b], from, bytes, cudaMemcpyHostToDevice, copy_stream));
      GIMBAL_CUDA_TRY(cudaEventRecord(ev_copied[b], copy_stream));
      GIMBAL_CUDA_TRY(cudaStreamWaitEvent(stream, ev_copied[b], 0));
      GIMBAL_TRY(count_device(dstage[b], id_bytes, cnt));
      GIMBAL_CUDA_TRY(cudaEventRecord(ev_consumed[b], stream));
    }
    return GIMBAL_OK;
  }
};

namespace {

int check_handle(gimbal_stats_t h) {
  if (!h) return invalid("null gimbal_stats_t handle");
  return GIMBAL_OK;
}

int copy_out(void* dst, const void* src, size_t bytes, int mem, cudaStream_t s) {
  if (!dst || bytes == 0) return GIMBAL_OK;
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes,
                                  mem == GIMBAL_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                           : cudaMemcpyDeviceToHost,
                                  s));
  return GIMBAL_OK;
}

}  // namespace

extern "C" {

int gimbal_abi_version(void) { return GIMBAL_ABI_VERSION; }
const char* gimbal_last_error(void) { return last_error().c_str(); }

int gimbal_topology_validate(const gimbal_topology* topo) {
  if (!topo) return invalid("null topology");
  return validate_topology(*topo);
}

int gimbal_stats_create(const gimbal_topology* topo, int device, gimbal_stats_t* out) {
  if (!topo || !out) return invalid("gimbal_stats_create: null argument");
  GIMBAL_TRY(validate_topology(*topo));
  int ndev = 0;
  GIMBAL_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return invalid("gimbal_stats_create: device out of range");
  DeviceGuard g(device);
  auto* h = new gimbal_stats_s();
  h->topo = *topo;
  h->device = device;
  int optin = 0;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  h->plan = make_stats_plan(topo->n_layers, topo->n_experts, topo->top_k, h->sms, optin);
  auto fail = [&](int st) {
    gimbal_stats_destroy(h);
    return st;
  };
  h->lm8_plan = make_lm8_plan(topo->n_layers, topo->n_experts, topo->top_k, h->sms, optin);
  {
    // GIMBAL_COUNT_PATH=atomic|lm8|split|fp4 overrides the default (tensor cores where supported)
    const char* path = GIMBAL_KNOB("GIMBAL_COUNT_PATH");
    const bool want_mma = !(path && std::string(path) == "atomic");
    h->use_mma = want_mma && mma_count_supported(topo->n_layers, topo->n_experts, topo->top_k);
    h->use_stack = want_mma && !(path && std::string(path) == "lm8");
    // opt-in: measured slower than the atomic u15 kernel at DS-V3 (fp4_count.cu header)
    h->use_fp4 = path && std::string(path) == "fp4";
    h->use_fp4x2 = path && std::string(path) == "fp4x2";
  }
  h->smem_optin = optin;
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->t_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->g_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_order, cudaEventDisableTiming) != cudaSuccess) {
    set_error("gimbal_stats_create: stream creation failed");
    return fail(GIMBAL_CUDA_ERROR);
  }
  for (int b = 0; b < gimbal_stats_s::kStages; ++b) {
    if (cudaEventCreateWithFlags(&h->ev_lm8_ready[b], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_lm8_free[b], cudaEventDisableTiming) != cudaSuccess) {
      set_error("gimbal_stats_create: event creation failed");
      return fail(GIMBAL_CUDA_ERROR);
    }
  }
  const int64_t nA = (int64_t)topo->n_layers * topo->n_experts;
  const int64_t nW = (int64_t)topo->n_experts * topo->n_experts;
  const int64_t nE = std::max<int64_t>(h->nE(), 1);
  if (cudaMalloc(&h->dE, nE * 8) != cudaSuccess || cudaMalloc(&h->dA, nA * 8) != cudaSuccess ||
      cudaMalloc(&h->dW, nW * 8) != cudaSuccess || cudaMalloc(&h->dflags, kFlagAllocBytes) != cudaSuccess) {
    set_error("gimbal_stats_create: device allocation failed");
    return fail(GIMBAL_CUDA_ERROR);
  }
  *out = h;
  if (cudaMemset(h->dflags, 0, kFlagAllocBytes) != cudaSuccess) {
    *out = nullptr;
    set_error("gimbal_stats_create: flag init failed");
    return fail(GIMBAL_CUDA_ERROR);
  }
  int st = gimbal_stats_reset(h);
  if (st != GIMBAL_OK) {
    *out = nullptr;
    return fail(st);
  }
  return GIMBAL_OK;
}

int gimbal_stats_destroy(gimbal_stats_t h) {
  if (!h) return GIMBAL_OK;
  {
    DeviceGuard g(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
    cudaFree(h->dE);
    cudaFree(h->dA);
    cudaFree(h->dW);
    cudaFree(h->dflags);
    for (int b = 0; b < gimbal_stats_s::kStages; ++b) {
      if (h->dstage[b]) cudaFree(h->dstage[b]);
      if (h->hstage[b]) cudaFreeHost(h->hstage[b]);
      if (h->ev_copied[b]) cudaEventDestroy(h->ev_copied[b]);
      if (h->ev_consumed[b]) cudaEventDestroy(h->ev_consumed[b]);
    }
    if (h->g_stream) cudaStreamSynchronize(h->g_stream);
    h->drop_graph();
    for (DevBuf* b : {&h->cand, &h->same, &h->dout, &h->keys, &h->misc, &h->ints, &h->probe, &h->dscr}) b->release();
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_caller) cudaEventDestroy(h->ev_caller);
    if (h->ring_host) cudaFreeHost(h->ring_host);
    if (h->ev_back) cudaEventDestroy(h->ev_back);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->t_stream) cudaStreamSynchronize(h->t_stream);
    for (int b = 0; b < gimbal_stats_s::kStages; ++b) {
      if (h->lm8[b]) cudaFree(h->lm8[b]);
      if (h->ev_lm8_ready[b]) cudaEventDestroy(h->ev_lm8_ready[b]);
      if (h->ev_lm8_free[b]) cudaEventDestroy(h->ev_lm8_free[b]);
    }
    if (h->ev_order) cudaEventDestroy(h->ev_order);
    for (auto& pr : h->tev) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->t_stream) cudaStreamDestroy(h->t_stream);
    if (h->g_stream) cudaStreamDestroy(h->g_stream);
  }
  delete h;
  return GIMBAL_OK;
}

int gimbal_stats_reset(gimbal_stats_t h) {
  GIMBAL_TRY(check_handle(h));
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  const int64_t nA = h->m();
  const int64_t nW = (int64_t)h->topo.n_experts * h->topo.n_experts;
  GIMBAL_CUDA_TRY(cudaMemsetAsync(h->dE, 0, std::max<int64_t>(h->nE(), 1) * 8, h->stream));
  GIMBAL_CUDA_TRY(cudaMemsetAsync(h->dA, 0, nA * 8, h->stream));
  GIMBAL_CUDA_TRY(cudaMemsetAsync(h->dW, 0, nW * 8, h->stream));
  GIMBAL_CUDA_TRY(cudaMemsetAsync(h->dflags, 0, 4, h->stream));  // word 1 (deferred) survives
  h->tokens = 0;
  h->tokens_on_device = false;
  ++h->count_version;
  h->set_derived(true);
  return GIMBAL_OK;
}

int gimbal_stats_add_tokens(gimbal_stats_t h, const void* ids, int id_bytes, int64_t n_tokens, int mem) {
  GIMBAL_TRY(check_handle(h));
  if (id_bytes != 1 && id_bytes != 4) return invalid("add_token: id_bytes must be 1 or 4");
  if (id_bytes == 1 && h->topo.n_experts > 256) return invalid("add_token: uint8 ids need n_experts <= 256");
  if (n_tokens < 0) return invalid("add_token: negative token count");
  if (n_tokens == 0) return GIMBAL_OK;
  if (!ids) return invalid("add_token: null ids");
  std::lock_guard<std::mutex> lk(h->mu);
  {
    DeviceGuard g(h->device);
    GIMBAL_TRY(h->resolve_tokens());
  }
  DeviceGuard g(h->device);
  if (mem == GIMBAL_MEM_DEVICE) {
    GIMBAL_TRY(h->count_device(ids, id_bytes, n_tokens));
  } else {
    GIMBAL_TRY(h->count_host(ids, id_bytes, n_tokens));
  }
  h->tokens += n_tokens;
  ++h->count_version;
  h->set_derived(false);
  return GIMBAL_OK;
}

int gimbal_stats_tokens(gimbal_stats_t h, int64_t* tokens) {
  GIMBAL_TRY(check_handle(h));
  if (!tokens) return invalid("null tokens");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  GIMBAL_TRY(h->resolve_tokens());
  *tokens = h->tokens;
  return GIMBAL_OK;
}

int gimbal_stats_sync(gimbal_stats_t h) {
  GIMBAL_TRY(check_handle(h));
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  uint32_t f[2] = {0, 0};
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(f, h->dflags, sizeof(f), cudaMemcpyDeviceToHost, h->stream));
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (f[1]) {  // deferred evaluator flags of gimbal_window_place_async: report once, then clear
    GIMBAL_CUDA_TRY(cudaMemset(h->dflags + 1, 0, 4));
    if (f[1] & kFlagInfeasible)
      return invalid("placement: a queued candidate batch is infeasible (ids must be in [0, g) with exactly "
                     "m/g experts per GPU)");
    GIMBAL_TRY(flags_to_status(f[1]));
  }
  return flags_to_status(f[0] & (kFlagIdOutOfRange | kFlagOverflow));
}

int gimbal_stats_read(gimbal_stats_t h, uint64_t* A, uint64_t* E, uint64_t* W, int mem) {
  GIMBAL_TRY(check_handle(h));
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  GIMBAL_TRY(h->derive_w());
  const int64_t ne = h->topo.n_experts;
  GIMBAL_TRY(copy_out(A, h->dA, h->m() * 8, mem, h->stream));
  if (h->nE() > 0) GIMBAL_TRY(copy_out(E, h->dE, h->nE() * 8, mem, h->stream));
  GIMBAL_TRY(copy_out(W, h->dW, ne * ne * 8, mem, h->stream));
  return h->check_flags();
}

int gimbal_stats_flat(gimbal_stats_t h, double* flatA, double* flatW, int mem) {
  GIMBAL_TRY(check_handle(h));
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  GIMBAL_TRY(h->derive());
  const int L = h->topo.n_layers, ne = h->topo.n_experts;
  const int64_t m = h->m();
  const size_t bA = (size_t)L * m * 8, bW = (size_t)m * m * 8;
  double* dA = nullptr;
  double* dW = nullptr;
  DevBuf tmpA, tmpW;
  if (flatA) {
    if (mem == GIMBAL_MEM_DEVICE) dA = flatA;
    else {
      GIMBAL_TRY(tmpA.ensure(bA));
      dA = tmpA.as<double>();
    }
    GIMBAL_CUDA_TRY(cudaMemsetAsync(dA, 0, bA, h->stream));
  }
  if (flatW) {
    if (mem == GIMBAL_MEM_DEVICE) dW = flatW;
    else {
      GIMBAL_TRY(tmpW.ensure(bW));
      dW = tmpW.as<double>();
    }
    GIMBAL_CUDA_TRY(cudaMemsetAsync(dW, 0, bW, h->stream));
  }
  if (L > 1 || dA) GIMBAL_CUDA_TRY(launch_flat_forms(L, ne, h->dA, h->dE, dA, L > 1 ? dW : nullptr, h->stream));
  if (mem != GIMBAL_MEM_DEVICE) {
    if (flatA) GIMBAL_CUDA_TRY(cudaMemcpyAsync(flatA, dA, bA, cudaMemcpyDeviceToHost, h->stream));
    if (flatW) GIMBAL_CUDA_TRY(cudaMemcpyAsync(flatW, dW, bW, cudaMemcpyDeviceToHost, h->stream));
  }
  int st = h->check_flags();
  tmpA.release();
  tmpW.release();
  return st;
}

int gimbal_stats_device_buffers(gimbal_stats_t h, uint64_t** E, uint64_t** A, void** stream) {
  GIMBAL_TRY(check_handle(h));
  if (E) *E = h->nE() > 0 ? reinterpret_cast<uint64_t*>(h->dE) : nullptr;
  if (A) *A = reinterpret_cast<uint64_t*>(h->dA);
  if (stream) *stream = h->stream;
  return GIMBAL_OK;
}

int gimbal_stats_count_timing(gimbal_stats_t h, int enable, double* count_ms, int64_t* launches) {
  GIMBAL_TRY(check_handle(h));
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  if (count_ms || launches) {
    GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
    GIMBAL_TRY(h->harvest_graph_timing());
    double total = h->g_ms;
    for (size_t i = 0; i < h->tev_used; ++i) {
      float ms = 0.f;
      GIMBAL_CUDA_TRY(cudaEventElapsedTime(&ms, h->tev[i].first, h->tev[i].second));
      total += ms;
    }
    if (count_ms) *count_ms = total;
    if (launches) *launches = (int64_t)h->tev_used + h->g_launches;
  }
  if (enable != (h->timing ? 1 : 0) || enable) {
    if (!count_ms && !launches) {
      GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
      GIMBAL_TRY(h->harvest_graph_timing(false));  // replays before this point are not counted
    }
    h->tev_used = 0;
    h->g_ms = 0.0;
    h->g_launches = 0;
  }
  h->timing = enable != 0;
  return GIMBAL_OK;
}

int gimbal_stats_merge(gimbal_stats_t h, const uint64_t* counts, int64_t tokens, int mem) {
  GIMBAL_TRY(check_handle(h));
  if (tokens < 0) return invalid("merge: negative token count");
  if (!counts) return invalid("merge: null counts");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  GIMBAL_TRY(h->resolve_tokens());
  const bool pairs = h->topo.n_layers > 1;
  const int64_t n = pairs ? h->nE() : h->m();
  unsigned long long* dst = pairs ? h->dE : h->dA;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(counts);
  DevBuf tmp;
  if (mem != GIMBAL_MEM_DEVICE) {
    GIMBAL_TRY(tmp.ensure((size_t)n * 8));
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(tmp.p, counts, (size_t)n * 8, cudaMemcpyHostToDevice, h->stream));
    src = tmp.as<unsigned long long>();
  }
  GIMBAL_CUDA_TRY(launch_add_u64(dst, src, n, h->stream));
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
  tmp.release();
  h->tokens += tokens;
  ++h->count_version;
  h->set_derived(!pairs);
  return GIMBAL_OK;
}

int gimbal_stats_mark_reduced(gimbal_stats_t h, int64_t global_tokens) {
  GIMBAL_TRY(check_handle(h));
  if (global_tokens < 0) return invalid("mark_reduced: negative token count");
  std::lock_guard<std::mutex> lk(h->mu);
  h->tokens = global_tokens;
  h->tokens_on_device = false;
  ++h->count_version;
  h->set_derived(h->topo.n_layers < 2);
  return GIMBAL_OK;
}

namespace {

int pick_cell_width(gimbal_stats_t h);

// Queues the batch evaluator (eval_same + eval_dev + eval_finish) for C device candidates on the
// handle's stream.  The only host synchronisation is the one-off max-cell probe when the token
// count alone cannot bound every E cell below 2^27.
int enqueue_eval(gimbal_stats_t h, const uint8_t* dc, int64_t C, double alpha, double beta, double* dD,
                 double* dcut, double* dobj, long long* darg, uint32_t* flags) {
  const int L = h->topo.n_layers, ne = h->topo.n_experts, gg = h->topo.n_gpus, k = h->topo.top_k;
  GIMBAL_TRY(h->same.ensure(eval_scratch_bytes(C)));
  h->tiny_ready_same = nullptr;  // the evaluators overwrite the fused pass's ticket words
  GIMBAL_TRY(pick_cell_width(h));
  GIMBAL_CUDA_TRY(launch_eval_costs(L, ne, gg, h->dA, h->dE, dc, C, alpha, beta,
                                    h->same.as<unsigned long long>(), dD, dcut, dobj, darg,
                                    flags, h->small_cells, h->width_guard, h->stream));
  GIMBAL_CUDA_TRY(launch_eval_finish(C, L, ne, k, h->dA, alpha, beta, h->same.as<unsigned long long>(), dD, dcut,
                                     dobj, darg, flags, h->stream));
  return GIMBAL_OK;
}

// E cells < 2^27 lets the evaluators keep 32-bit partial sums / four byte planes.  Decided on the
// host when the token count bounds every cell (a token adds at most k^2 to a cell); otherwise a
// max-cell probe is queued (once per count state) and the evaluators pick their form on the
// device (WidthGuard), so a pass never waits on the host.
int pick_cell_width(gimbal_stats_t h) {
  const int k = h->topo.top_k;
  if (!h->tokens_on_device && (unsigned long long)h->tokens * (unsigned long long)(k * k) < (1ull << 27)) {
    h->small_cells = true;
    h->width_guard = nullptr;
    return GIMBAL_OK;
  }
  if (h->probed_version != h->count_version) {
    GIMBAL_TRY(h->probe.ensure(64));  // not `misc`: it may hold a queued pass's member bits
    GIMBAL_CUDA_TRY(launch_max_cell(h->dE, h->topo.n_layers > 1 ? h->nE() : 0, h->probe.as<unsigned long long>(),
                                    h->stream));
    h->probed_version = h->count_version;
  }
  h->small_cells = true;
  h->width_guard = h->probe.as<unsigned long long>();
  return GIMBAL_OK;
}

}  // namespace

int gimbal_eval_costs(gimbal_stats_t h, const uint8_t* candidates, int64_t C, int cand_mem,
                      double alpha, double beta, double* deviation, double* cut, double* objective,
                      int64_t* argmin, int out_mem) {
  GIMBAL_TRY(check_handle(h));
  if (!(alpha > 0.0) || !(beta > 0.0)) return invalid("PlacementProblem: alpha and beta must be > 0");
  if (C < 0) return invalid("eval_costs: negative candidate count");
  if (C == 0) {
    if (argmin) *argmin = -1;
    return GIMBAL_OK;
  }
  if (!candidates || !deviation || !cut || !objective) return invalid("eval_costs: null argument");
  if (h->topo.n_gpus > 255) return invalid("eval_costs: uint8 candidates need n_gpus <= 255");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  GIMBAL_TRY(h->derive());
  const int64_t m = h->m();
  const uint8_t* dc = candidates;
  if (cand_mem != GIMBAL_MEM_DEVICE) {
    GIMBAL_TRY(h->cand.ensure((size_t)C * m));
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(h->cand.p, candidates, (size_t)C * m, cudaMemcpyHostToDevice, h->stream));
    dc = h->cand.as<uint8_t>();
  }
  double *dD = deviation, *dcut = cut, *dobj = objective;
  GIMBAL_TRY(h->dout.ensure((size_t)C * 24 + 16));
  if (out_mem != GIMBAL_MEM_DEVICE) {
    dD = h->dout.as<double>();
    dcut = dD + C;
    dobj = dcut + C;
  }
  long long* darg = reinterpret_cast<long long*>(h->dout.as<double>() + 3 * C);
  GIMBAL_TRY(enqueue_eval(h, dc, C, alpha, beta, dD, dcut, dobj, darg, h->dflags));
  uint32_t f = 0;
  long long bad = 0, am = -1;
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(&f, h->dflags, 4, cudaMemcpyDeviceToHost, h->stream));
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(&bad, h->same.as<unsigned long long>() + C, 8, cudaMemcpyDeviceToHost,
                                  h->stream));
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(&am, darg, 8, cudaMemcpyDeviceToHost, h->stream));
  if (out_mem != GIMBAL_MEM_DEVICE) {
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(deviation, dD, C * 8, cudaMemcpyDeviceToHost, h->stream));
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(cut, dcut, C * 8, cudaMemcpyDeviceToHost, h->stream));
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(objective, dobj, C * 8, cudaMemcpyDeviceToHost, h->stream));
  }
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (f & kFlagInfeasible) {
    // clear the non-sticky flag, report like check_feasible (placement.cpp:30-50)
    GIMBAL_CUDA_TRY(cudaMemsetAsync(h->dflags, 0, 4, h->stream));
    uint32_t keep = f & ~(uint32_t)kFlagInfeasible;
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(h->dflags, &keep, 4, cudaMemcpyHostToDevice, h->stream));
    GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return invalid("placement: candidate " + std::to_string(bad) +
                   " is infeasible (ids must be in [0, g) with exactly m/g experts per GPU)");
  }
  GIMBAL_TRY(flags_to_status(f));
  if (argmin) *argmin = am;
  return GIMBAL_OK;
}

namespace {

// Queues build_affinity_set on the handle's E: member bitmask `bits` (m bits), sorted member ids
// `dout` and their count `dn` (device), no host synchronisation.  L >= 2, (L-1)*n_e^2 < 2^24.
int enqueue_affinity(gimbal_stats_t h, double threshold, int32_t top_e, int32_t capacity, uint32_t* bits,
                     int32_t* dout, int32_t* dn) {
  const int L = h->topo.n_layers, ne = h->topo.n_experts;
  const int64_t n = h->nE();
  const int64_t n_pad = next_pow2(n);
  GIMBAL_TRY(h->keys.ensure((size_t)n_pad * 8));
  if (top_e >= 1 && top_e <= kTopkMax) {
    // only the top_e heaviest pairs can survive truncation: segment top-K, no full sort
    // two halves: segment survivors ((n / 2048) * top_e keys) or register top-K partials (<= 4096)
    const int64_t half = std::max<int64_t>({n_pad / 2, (n + 2047) / 2048 * (int64_t)top_e, 4096});
    GIMBAL_TRY(h->keys.ensure((size_t)half * 16));
    unsigned long long* ka = h->keys.as<unsigned long long>();
    unsigned long long* kb = ka + half;
    unsigned long long* sorted = nullptr;
    GIMBAL_CUDA_TRY(launch_affinity_topk(L, ne, h->dE, threshold, top_e, ka, kb, h->dflags, &sorted, h->stream));
    GIMBAL_CUDA_TRY(launch_affinity_select(L, ne, sorted, top_e, top_e, capacity, bits, dout, dn, h->stream));
  } else {
    GIMBAL_CUDA_TRY(launch_affinity_keys(L, ne, h->dE, threshold, h->keys.as<unsigned long long>(), n_pad,
                                         h->dflags, h->stream));
    GIMBAL_CUDA_TRY(sort_u64_desc(h->keys.as<unsigned long long>(), n_pad, h->stream));
    GIMBAL_CUDA_TRY(launch_affinity_select(L, ne, h->keys.as<unsigned long long>(), n, top_e, capacity, bits,
                                           dout, dn, h->stream));
  }
  return GIMBAL_OK;
}

}  // namespace

int gimbal_affinity_set(gimbal_stats_t h, double threshold, int32_t top_e, int32_t capacity,
                        int32_t anchor_gpu, int32_t* out, int32_t* n_out) {
  GIMBAL_TRY(check_handle(h));
  if (!out || !n_out) return invalid("build_affinity_set: null output");
  if (anchor_gpu < 0 || anchor_gpu >= h->topo.n_gpus)
    return invalid("build_affinity_set: anchor_gpu out of range");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  if (h->topo.n_layers < 2) {
    *n_out = 0;
    return h->check_flags();
  }
  if (h->nE() >= (1ll << 24)) {
    set_error("build_affinity_set: (L-1)*n_experts^2 must be < 2^24");
    return GIMBAL_NOT_SUPPORTED;
  }
  const int64_t m = h->m();
  GIMBAL_TRY(h->misc.ensure((size_t)((m + 31) / 32) * 4 + (size_t)m * 4 + 16));
  uint32_t* bits = h->misc.as<uint32_t>();
  int32_t* dout = reinterpret_cast<int32_t*>(bits + (m + 31) / 32);
  int32_t* dn = dout + m;
  GIMBAL_TRY(enqueue_affinity(h, threshold, top_e, capacity, bits, dout, dn));
  int32_t cnt = 0;
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(&cnt, dn, 4, cudaMemcpyDeviceToHost, h->stream));
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (cnt > 0) {
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(out, dout, (size_t)cnt * 4, cudaMemcpyDeviceToHost, h->stream));
  }
  *n_out = cnt;
  return h->check_flags();
}

// Reference validation order and messages (placement.cpp:243-252, 272-279).
static int validate_greedy(int64_t m, int g, const int32_t* M, int32_t nM, int32_t anchor,
                           std::vector<uint32_t>& bits) {
  if (g < 1 || m < 1 || m % g != 0) return invalid("greedy_place: experts must be divisible by g");
  const int64_t cap = m / g;
  if (anchor < 0 || anchor >= g) return invalid("greedy_place: anchor_gpu out of range");
  if (nM > cap) return invalid("greedy_place: affinity set exceeds anchor capacity");
  bits.assign((size_t)((m + 31) / 32), 0u);
  for (int i = 0; i < nM; ++i) {
    const int64_t e = M[i];
    if (e < 0 || e >= m) return invalid("greedy_place: affinity id out of range");
    if ((bits[e >> 5] >> (e & 31)) & 1u) return invalid("greedy_place: duplicate affinity id");
    bits[e >> 5] |= 1u << (e & 31);
  }
  return GIMBAL_OK;
}

namespace {

// Scratch layout in h->ints for greedy: [anchored bits][M][result m int32][tent m bytes].
struct GreedyScratch {
  uint32_t* bits;
  int32_t* M;
  int32_t* res;
  uint8_t* tent;
};

int greedy_scratch(gimbal_stats_t h, size_t words, int32_t nM, GreedyScratch& g) {
  const int64_t m = h->m();
  GIMBAL_TRY(h->keys.ensure((size_t)next_pow2(m) * 8));
  GIMBAL_TRY(h->ints.ensure(words * 4 + (size_t)std::max(nM, 1) * 4 + (size_t)m * 4 + (size_t)m + 64));
  g.bits = h->ints.as<uint32_t>();
  g.M = reinterpret_cast<int32_t*>(g.bits + words);
  g.res = g.M + std::max(nM, 1);
  g.tent = reinterpret_cast<uint8_t*>(g.res + m);  // per-position scratch
  return GIMBAL_OK;
}

// greedy_keys -> sort -> walk on the handle's stream (anchored bits and M already on the device).
int enqueue_greedy(gimbal_stats_t h, const GreedyScratch& gs, int32_t nM, int32_t anchor, int32_t* dres,
                   uint8_t* out_u8) {
  const int L = h->topo.n_layers, ne = h->topo.n_experts, g = h->topo.n_gpus;
  const int64_t m = h->m();
  const int64_t n_pad = next_pow2(m);
  GIMBAL_CUDA_TRY(launch_greedy_keys(m, h->dA, gs.bits, h->keys.as<unsigned long long>(), n_pad, h->dflags,
                                     h->stream));
  GIMBAL_CUDA_TRY(sort_u64_desc(h->keys.as<unsigned long long>(), n_pad, h->stream));
  GIMBAL_CUDA_TRY(launch_greedy_walk(L, ne, g, h->dA, gs.M, nM, anchor, h->keys.as<unsigned long long>(),
                                     m, dres, out_u8, gs.tent, h->stream));
  return GIMBAL_OK;
}

}  // namespace

int gimbal_greedy_place(gimbal_stats_t h, const int32_t* M, int32_t nM, int32_t anchor, int32_t* out,
                        int out_mem, uint8_t* out_u8) {
  GIMBAL_TRY(check_handle(h));
  if (!out && !out_u8) return invalid("greedy_place: null output");
  if (nM < 0 || (nM > 0 && !M)) return invalid("greedy_place: bad affinity set");
  const int64_t m = h->m();
  std::vector<uint32_t> bits;
  GIMBAL_TRY(validate_greedy(m, h->topo.n_gpus, M, nM, anchor, bits));
  if (m >= (1ll << 24)) {
    set_error("greedy_place: m must be < 2^24");
    return GIMBAL_NOT_SUPPORTED;
  }
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard dg(h->device);
  GIMBAL_TRY(h->derive());
  GreedyScratch gs{};
  GIMBAL_TRY(greedy_scratch(h, bits.size(), nM, gs));
  h->m_cached_buf = nullptr;  // this call overwrites the resident strong-pair set
  int32_t* dres = (out && out_mem == GIMBAL_MEM_DEVICE) ? out : gs.res;
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(gs.bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, h->stream));
  if (nM > 0) GIMBAL_CUDA_TRY(cudaMemcpyAsync(gs.M, M, (size_t)nM * 4, cudaMemcpyHostToDevice, h->stream));
  GIMBAL_TRY(enqueue_greedy(h, gs, nM, anchor, dres, out_u8));
  if (out && out_mem != GIMBAL_MEM_DEVICE)
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(out, dres, (size_t)m * 4, cudaMemcpyDeviceToHost, h->stream));
  return h->check_flags();
}

int gimbal_window_place_async(gimbal_stats_t h, const int32_t* M, int32_t nM, int32_t anchor,
                              uint8_t* candidates, int64_t C, double alpha, double beta, double* scores,
                              int64_t* argmin, int32_t* placement) {
  GIMBAL_TRY(check_handle(h));
  if (!(alpha > 0.0) || !(beta > 0.0)) return invalid("PlacementProblem: alpha and beta must be > 0");
  if (C < 1 || !candidates || !scores || !argmin || !placement)
    return invalid("window_place: needs C >= 1 device candidates and device outputs");
  if (nM < 0 || (nM > 0 && !M)) return invalid("greedy_place: bad affinity set");
  if (h->topo.n_gpus > 255) return invalid("eval_costs: uint8 candidates need n_gpus <= 255");
  const int64_t m = h->m();
  if (m >= (1ll << 24)) {
    set_error("greedy_place: m must be < 2^24");
    return GIMBAL_NOT_SUPPORTED;
  }
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard dg(h->device);
  const int64_t words = (m + 31) / 32;
  GreedyScratch gs{};
  GIMBAL_TRY(greedy_scratch(h, (size_t)words, nM, gs));
  const bool same_set = h->m_cached_buf == h->ints.p && h->m_cached_anchor == anchor &&
                        h->m_cached.size() == (size_t)nM &&
                        std::equal(M, M + nM, h->m_cached.begin());
  if (!same_set) {
    std::vector<uint32_t> bits;
    GIMBAL_TRY(validate_greedy(m, h->topo.n_gpus, M, nM, anchor, bits));
    // a new set is rare (once per stream): upload synchronously so the host vectors may go
    GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
    GIMBAL_CUDA_TRY(cudaMemcpy(gs.bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice));
    if (nM > 0) GIMBAL_CUDA_TRY(cudaMemcpy(gs.M, M, (size_t)nM * 4, cudaMemcpyHostToDevice));
    h->m_cached.assign(M, M + nM);
    h->m_cached_anchor = anchor;
    h->m_cached_buf = h->ints.p;
  }
  GIMBAL_TRY(h->derive());
  GIMBAL_TRY(enqueue_greedy(h, gs, nM, anchor, placement, candidates));
  // evaluator flags go to the deferred word (dflags[1]): reset() clears only the count-state word,
  // so an infeasible candidate in any queued window is still reported by gimbal_stats_sync
  return enqueue_eval(h, candidates, C, alpha, beta, scores, scores + C, scores + 2 * C,
                      reinterpret_cast<long long*>(argmin), h->dflags + 1);
}

int gimbal_pass_async(gimbal_stats_t h, double threshold, int32_t top_e, int32_t capacity, int32_t anchor,
                      uint8_t* candidates, int64_t C, double alpha, double beta, double* scores, int64_t* argmin,
                      int32_t* placement, int32_t* members, int32_t* n_members, uint32_t* flags_out) {
  GIMBAL_TRY(check_handle(h));
  if (!(alpha > 0.0) || !(beta > 0.0)) return invalid("PlacementProblem: alpha and beta must be > 0");
  if (anchor < 0 || anchor >= h->topo.n_gpus) return invalid("build_affinity_set: anchor_gpu out of range");
  if (C < 1 || !candidates || !scores || !argmin || !placement || !members || !n_members)
    return invalid("pass: needs C >= 1 device candidates and device outputs");
  if (h->topo.n_gpus > 255) return invalid("eval_costs: uint8 candidates need n_gpus <= 255");
  const int64_t m = h->m();
  // greedy_place rejects |M| > m/g (placement.cpp:252); with capacity <= m/g that cannot happen,
  // so the whole pass can be queued without looking at |M|
  if (capacity > m / h->topo.n_gpus) return invalid("pass: capacity must be <= m/g (greedy_place anchor capacity)");
  if (m >= (1ll << 24) || h->nE() >= (1ll << 24)) {
    set_error("pass: m and (L-1)*n_experts^2 must be < 2^24");
    return GIMBAL_NOT_SUPPORTED;
  }
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard dg(h->device);
  // small shapes (Mixtral class): the whole pass in one launch when every E cell fits 32 bits
  // (the token count bounds it: a token adds at most k^2 to a cell)
  const unsigned long long kk2 = (unsigned long long)h->topo.top_k * (unsigned long long)h->topo.top_k;
  if (!h->tokens_on_device && h->tokens >= 0 && (unsigned long long)h->tokens * kk2 < (1ull << 32)) {
    GIMBAL_TRY(h->same.ensure(tiny_scratch_bytes(C)));
    unsigned long long* same = h->same.as<unsigned long long>();
    const bool init = h->tiny_ready_same != same || h->tiny_ready_C != C;
    if (!h->ring_host) {
      void* host = nullptr;
      GIMBAL_CUDA_TRY(cudaHostAlloc(&host, (size_t)gimbal_stats_s::kRingSlots * (size_t)(6 + 2 * m) * 4,
                                    cudaHostAllocMapped));
      h->ring_host = static_cast<int32_t*>(host);
      void* dev = nullptr;
      GIMBAL_CUDA_TRY(cudaHostGetDevicePointer(&dev, host, 0));
      h->ring_dev = static_cast<int32_t*>(dev);
    }
    const cudaError_t e = launch_tiny_pass(
        h->topo.n_layers, h->topo.n_experts, h->topo.n_gpus, h->topo.top_k, threshold, top_e, capacity, anchor, h->dE,
        h->dA, candidates, C, alpha, beta, scores, reinterpret_cast<long long*>(argmin), placement, members, n_members,
        h->dflags, same, init, flags_out, h->ring_dev, h->dflags + 8, gimbal_stats_s::kRingSlots, h->stream);
    if (e != cudaErrorNotSupported) {
      GIMBAL_CUDA_TRY(e);
      h->tiny_ready_same = same;
      h->tiny_ready_C = C;
      h->last_pass_tiny = true;
      if (!h->capturing) h->note_tiny_run();
      h->derived = true;  // the pass wrote A
      return GIMBAL_OK;
    }
    cudaGetLastError();
  }
  h->last_pass_tiny = false;
  h->ran_tiny = false;
  GIMBAL_TRY(h->derive());
  // scratch sized before anything is queued (a regrown buffer is freed, not stream-ordered)
  GreedyScratch gs{};
  GIMBAL_TRY(greedy_scratch(h, 0, 1, gs));  // only the walk's per-position scratch is used
  h->m_cached_buf = nullptr;
  GIMBAL_TRY(h->misc.ensure((size_t)((m + 31) / 32) * 4 + 64));
  uint32_t* bits = h->misc.as<uint32_t>();
  if (h->topo.n_layers < 2) {
    GIMBAL_CUDA_TRY(cudaMemsetAsync(bits, 0, (size_t)((m + 31) / 32) * 4, h->stream));
    GIMBAL_CUDA_TRY(cudaMemsetAsync(n_members, 0, 4, h->stream));
  } else {
    GIMBAL_TRY(enqueue_affinity(h, threshold, top_e, capacity, bits, members, n_members));
  }
  const int L = h->topo.n_layers, ne = h->topo.n_experts, g = h->topo.n_gpus;
  const int64_t n_pad = next_pow2(m);
  auto greedy_on = [&](cudaStream_t st) -> int {
    GIMBAL_CUDA_TRY(launch_greedy_keys(m, h->dA, bits, h->keys.as<unsigned long long>(), n_pad, h->dflags, st));
    GIMBAL_CUDA_TRY(sort_u64_desc(h->keys.as<unsigned long long>(), n_pad, st));
    GIMBAL_CUDA_TRY(launch_greedy_walk(L, ne, g, h->dA, members, -1, anchor, h->keys.as<unsigned long long>(), m,
                                       placement, candidates, gs.tent, st, n_members));
    return GIMBAL_OK;
  };
  // evaluator flags go to the deferred word (dflags[1]) as in gimbal_window_place_async
  // (tiny shapes: the walk is ~10 us and the extra launches cost more than it hides; measured
  // Mixtral m = 256: 0.286 vs 0.269 ms per step, DS-V2-Lite m = 1664: 5.15 vs 5.25 ms)
  if (C < 2 || m < 1024 || GIMBAL_KNOB("GIMBAL_NO_GREEDY_OVERLAP")) {
    GIMBAL_TRY(greedy_on(h->stream));
    GIMBAL_TRY(enqueue_eval(h, candidates, C, alpha, beta, scores, scores + C, scores + 2 * C,
                            reinterpret_cast<long long*>(argmin), h->dflags + 1));
    if (flags_out) GIMBAL_CUDA_TRY(cudaMemcpyAsync(flags_out, h->dflags, 8, cudaMemcpyDeviceToDevice, h->stream));
    return GIMBAL_OK;
  }
  // The greedy walk (latency-bound, one CTA) runs on the side stream while candidates 1..C-1 are
  // scored on the handle's stream; candidate 0 (the greedy row it writes) is scored after the join.
  GIMBAL_TRY(h->same.ensure(eval_scratch_bytes(C)));
  h->tiny_ready_same = nullptr;  // the evaluators overwrite the fused pass's ticket words
  GIMBAL_TRY(pick_cell_width(h));
  GIMBAL_CUDA_TRY(cudaEventRecord(h->ev_fork, h->stream));
  GIMBAL_CUDA_TRY(cudaStreamWaitEvent(h->g_stream, h->ev_fork, 0));
  GIMBAL_TRY(greedy_on(h->g_stream));
  GIMBAL_CUDA_TRY(cudaEventRecord(h->ev_join, h->g_stream));
  unsigned long long* same = h->same.as<unsigned long long>();
  long long* bad = reinterpret_cast<long long*>(same + C);
  uint32_t* flags = h->dflags + 1;
  GIMBAL_CUDA_TRY(launch_eval_prepare(C, same, h->stream));
  GIMBAL_CUDA_TRY(launch_eval_range(L, ne, g, h->dA, h->dE, candidates + m, C - 1, 1, same + 1, scores + 1, flags,
                                    bad, h->small_cells, h->width_guard, h->stream));
  GIMBAL_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  GIMBAL_CUDA_TRY(launch_eval_range(L, ne, g, h->dA, h->dE, candidates, 1, 0, same, scores, flags, bad,
                                    h->small_cells, h->width_guard, h->stream));
  GIMBAL_CUDA_TRY(launch_eval_finish(C, L, ne, h->topo.top_k, h->dA, alpha, beta, same, scores, scores + C,
                                     scores + 2 * C,
                                     reinterpret_cast<long long*>(argmin), flags, h->stream));
  if (flags_out) GIMBAL_CUDA_TRY(cudaMemcpyAsync(flags_out, h->dflags, 8, cudaMemcpyDeviceToDevice, h->stream));
  return GIMBAL_OK;
}

}  // extern "C"

namespace gimbal_gpu {

// Internals for the online hook (online.cu), which counts straight into a handle's tensors.
StatsInternals stats_internals(gimbal_stats_t h) {
  StatsInternals v;
  v.dE = h->dE;
  v.dA = h->dA;
  v.dflags = h->dflags;
  v.stream = h->stream;
  v.device = h->device;
  v.topo = h->topo;
  v.mu = &h->mu;
  return v;
}

// n tokens were counted into the handle's counted buffer behind its stream (caller holds mu)
void stats_note_added(gimbal_stats_t h, int64_t n) {
  h->tokens += n;
  ++h->count_version;
  h->set_derived(h->topo.n_layers < 2);
}

int stats_resolve_tokens(gimbal_stats_t h) { return h->resolve_tokens(); }

}  // namespace gimbal_gpu

extern "C" {

int gimbal_stats_allreduce(gimbal_stats_t h, gimbal_comm_t comm, int64_t global_tokens) {
  GIMBAL_TRY(check_handle(h));
  if (!comm) return invalid("gimbal_stats_allreduce: null communicator");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  const bool pairs = h->topo.n_layers > 1;
  // the counted buffer (A is re-derived from the reduced E on use)
  GIMBAL_TRY(nccl_allreduce_u64_sum(pairs ? h->dE : h->dA, (size_t)(pairs ? h->nE() : h->m()), comm, h->stream));
  if (global_tokens >= 0) {
    h->tokens = global_tokens;
    h->tokens_on_device = false;
  } else {
    h->tokens_on_device = true;
  }
  ++h->count_version;
  h->set_derived(!pairs);
  return GIMBAL_OK;
}

int gimbal_dist_merge_argmin(gimbal_stats_t h, gimbal_comm_t comm, const double* objectives, int64_t n_local,
                             int64_t offset, int64_t n_total, double* global, int64_t* argmin) {
  GIMBAL_TRY(check_handle(h));
  if (!comm || !global || !argmin || (n_local > 0 && !objectives)) return invalid("merge_argmin: null argument");
  if (n_local < 0 || offset < 0 || n_total < 1 || offset + n_local > n_total)
    return invalid("merge_argmin: slice outside [0, n_total)");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  return nccl_merge_argmin(objectives, n_local, offset, global, n_total, reinterpret_cast<long long*>(argmin), comm,
                           h->stream);
}

int gimbal_pass_distributed_async(gimbal_stats_t h, gimbal_comm_t comm, double threshold, int32_t top_e,
                                  int32_t capacity, int32_t anchor, uint8_t* candidates, int64_t n_local,
                                  int64_t cand_offset, int64_t n_total, double alpha, double beta, double* scores,
                                  double* global, int64_t* argmin, int32_t* placement, int32_t* members,
                                  int32_t* n_members, uint32_t* flags_out) {
  GIMBAL_TRY(check_handle(h));
  if (n_local < 0 || cand_offset < 0 || n_total < 1 || cand_offset + n_local > n_total)
    return invalid("pass_distributed: candidate slice outside [0, n_total)");
  if (!global || !argmin || !scores || !candidates) return invalid("pass_distributed: null argument");
  const int64_t lead = (cand_offset == 0 && n_local > 0) ? 0 : 1;
  const int64_t rows = n_local + lead;
  GIMBAL_TRY(gimbal_stats_allreduce(h, comm, -1));
  {
    std::lock_guard<std::mutex> lk(h->mu);
    GIMBAL_TRY(h->dscr.ensure(64));
  }
  GIMBAL_TRY(gimbal_pass_async(h, threshold, top_e, capacity, anchor, candidates, rows, alpha, beta, scores,
                               reinterpret_cast<int64_t*>(h->dscr.p), placement, members, n_members, flags_out));
  return gimbal_dist_merge_argmin(h, comm, scores + 2 * rows + lead, n_local, cand_offset, n_total, global, argmin);
}

int gimbal_eval_excess(gimbal_stats_t h, const uint8_t* candidates, int64_t C, int cand_mem, double* excess,
                       int out_mem) {
  GIMBAL_TRY(check_handle(h));
  if (C < 0) return invalid("eval_excess: negative candidate count");
  if (C == 0) return GIMBAL_OK;
  if (!candidates || !excess) return invalid("eval_excess: null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  GIMBAL_TRY(h->derive());
  const int64_t m = h->m();
  const uint8_t* dc = candidates;
  if (cand_mem != GIMBAL_MEM_DEVICE) {
    GIMBAL_TRY(h->cand.ensure((size_t)C * m));
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(h->cand.p, candidates, (size_t)C * m, cudaMemcpyHostToDevice, h->stream));
    dc = h->cand.as<uint8_t>();
  }
  double* dx = excess;
  if (out_mem != GIMBAL_MEM_DEVICE) {
    GIMBAL_TRY(h->dout.ensure((size_t)C * 8 + 16));
    dx = h->dout.as<double>();
  }
  GIMBAL_CUDA_TRY(cudaMemsetAsync(h->dflags + 2, 0, 4, h->stream));
  GIMBAL_CUDA_TRY(launch_eval_excess(h->topo.n_layers, h->topo.n_experts, h->topo.n_gpus, h->dA, dc, C, dx,
                                     h->dflags + 2, h->stream));
  uint32_t f = 0;
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(&f, h->dflags + 2, 4, cudaMemcpyDeviceToHost, h->stream));
  if (out_mem != GIMBAL_MEM_DEVICE)
    GIMBAL_CUDA_TRY(cudaMemcpyAsync(excess, dx, (size_t)C * 8, cudaMemcpyDeviceToHost, h->stream));
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (f) return invalid("eval_excess: candidate GPU id out of range [0, g)");
  return GIMBAL_OK;
}

int gimbal_pass_graph(gimbal_stats_t h, const void* ids, int id_bytes, int64_t n_tokens, double threshold,
                      int32_t top_e, int32_t capacity, int32_t anchor, uint8_t* candidates, int64_t C, double alpha,
                      double beta, double* scores, int64_t* argmin, int32_t* placement, int32_t* members,
                      int32_t* n_members, uint32_t* flags_out) {
  GIMBAL_TRY(check_handle(h));
  if (!ids || n_tokens < 1) return invalid("pass_graph: needs device ids of at least one token");
  gimbal_stats_s::GraphKey key;
  key.ids = ids;
  key.id_bytes = id_bytes;
  key.n = n_tokens;
  key.threshold = threshold;
  key.alpha = alpha;
  key.beta = beta;
  key.top_e = top_e;
  key.capacity = capacity;
  key.anchor = anchor;
  key.cands = candidates;
  key.C = C;
  key.scores = scores;
  key.argmin = argmin;
  key.placement = placement;
  key.members = members;
  key.n_members = n_members;
  key.flags = flags_out;
  key.sms = h->sms;
  if (h->gexec && key == h->gkey && h->scratch_snapshot() == h->g_scratch) {
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard g(h->device);
    if (h->g_uses_tiny && (h->tiny_ready_same != h->same.as<unsigned long long>() || h->tiny_ready_C != C)) {
      // another evaluator call reused the scratch: restore the fused pass's ticket / bad index
      GIMBAL_CUDA_TRY(cudaMemsetAsync(h->same.as<unsigned long long>() + C, 0x7f, 16, h->stream));
      h->tiny_ready_same = h->same.as<unsigned long long>();
      h->tiny_ready_C = C;
    }
    if (h->timing) GIMBAL_TRY(h->arm_graph_timing());
    GIMBAL_CUDA_TRY(cudaGraphLaunch(h->gexec, h->stream));
    if (h->g_uses_tiny)
      h->note_tiny_run();
    else
      h->ran_tiny = false;
    // host-side effects of reset + add_tokens + pass: the counts are the trace's, A derived
    h->tokens = n_tokens;
    h->tokens_on_device = false;
    ++h->count_version;
    h->derived = true;
    h->w_derived = h->topo.n_layers < 2;
    h->m_cached_buf = nullptr;
    return GIMBAL_OK;
  }
  auto eager = [&]() -> int {
    GIMBAL_TRY(gimbal_stats_reset(h));
    GIMBAL_TRY(gimbal_stats_add_tokens(h, ids, id_bytes, n_tokens, GIMBAL_MEM_DEVICE));
    return gimbal_pass_async(h, threshold, top_e, capacity, anchor, candidates, C, alpha, beta, scores, argmin,
                             placement, members, n_members, flags_out);
  };
  if (!(key == h->gkey) || h->gseen == 0 || (h->gexec && h->scratch_snapshot() != h->g_scratch)) {
    // first run with these arguments: eager (validates, sizes every scratch buffer)
    h->drop_graph();
    h->gkey = key;
    h->gseen = 0;
    GIMBAL_TRY(eager());
    h->gseen = 1;
    return GIMBAL_OK;
  }
  // second run: record the step as a graph, then launch it
  {
    DeviceGuard g(h->device);
    GIMBAL_CUDA_TRY(cudaStreamSynchronize(h->stream));
    h->drop_graph();
    GIMBAL_CUDA_TRY(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
    h->capturing = true;
    const int st = eager();
    h->capturing = false;
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
    if (st != GIMBAL_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    GIMBAL_CUDA_TRY(ce);
    h->graph = graph;
    // the record nodes of each timed counting launch (timing_begin / timing_end, in order)
    size_t n_nodes = 0;
    GIMBAL_CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &n_nodes));
    std::vector<cudaGraphNode_t> nodes(n_nodes);
    GIMBAL_CUDA_TRY(cudaGraphGetNodes(graph, nodes.data(), &n_nodes));
    h->g_nodes.assign(h->g_tev.size(), {nullptr, nullptr});
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      GIMBAL_CUDA_TRY(cudaGraphNodeGetType(nd, &ty));
      if (ty != cudaGraphNodeTypeEventRecord) continue;
      cudaEvent_t ev = nullptr;
      GIMBAL_CUDA_TRY(cudaGraphEventRecordNodeGetEvent(nd, &ev));
      for (size_t i = 0; i < h->g_tev.size(); ++i) {
        if (h->g_tev[i].first == ev) h->g_nodes[i].first = nd;
        if (h->g_tev[i].second == ev) h->g_nodes[i].second = nd;
      }
    }
    for (auto& nd : h->g_nodes)
      if (!nd.first || !nd.second) {
        set_error("pass_graph: timing record node not found in the captured graph");
        return GIMBAL_CUDA_ERROR;
      }
    // the capture-time events become the first replay's pair
    for (auto& pr : h->g_tev) h->g_pool.push_back(pr);
    h->g_tev.clear();
    h->g_uses_tiny = h->last_pass_tiny;
    h->g_scratch = h->scratch_snapshot();
    GIMBAL_CUDA_TRY(cudaGraphInstantiate(&h->gexec, graph, 0));
  }
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  if (h->timing) GIMBAL_TRY(h->arm_graph_timing());
  GIMBAL_CUDA_TRY(cudaGraphLaunch(h->gexec, h->stream));
  if (h->g_uses_tiny)
    h->note_tiny_run();
  else
    h->ran_tiny = false;
  return GIMBAL_OK;
}

int gimbal_pass_enqueue(gimbal_stats_t h, const void* ids, int id_bytes, int64_t n_tokens, double threshold,
                        int32_t top_e, int32_t capacity, int32_t anchor, uint8_t* candidates, int64_t C,
                        double alpha, double beta, double* scores, int32_t* packed, int32_t* packed_host,
                        void* caller_stream, int32_t** results_host) {
  GIMBAL_TRY(check_handle(h));
  if (!packed || !packed_host || !results_host) return invalid("pass_enqueue: null packed result buffer");
  const int64_t m = h->m();
  cudaStream_t caller = static_cast<cudaStream_t>(caller_stream);
  const bool join = caller != h->stream;
  {
    DeviceGuard g(h->device);
    if (join) {
      if (!h->ev_caller) GIMBAL_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_caller, cudaEventDisableTiming));
      GIMBAL_CUDA_TRY(cudaEventRecord(h->ev_caller, caller));
      GIMBAL_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->ev_caller, 0));
    }
  }
  // packed layout (int32 words): [0:2] argmin, [2] |M|, [3] pad, [4:6] error words, [6:6+m] M,
  // [6+m:6+2m] greedy
  GIMBAL_TRY(gimbal_pass_graph(h, ids, id_bytes, n_tokens, threshold, top_e, capacity, anchor, candidates, C, alpha,
                               beta, scores, reinterpret_cast<int64_t*>(packed), packed + 6 + m, packed + 6,
                               packed + 2, reinterpret_cast<uint32_t*>(packed + 4)));
  DeviceGuard g(h->device);
  if (h->ran_tiny) {  // the fused pass wrote its results into the mapped ring already
    *results_host = h->ring_host + (size_t)h->ring_slot * (size_t)(6 + 2 * m);
  } else {
    GIMBAL_CUDA_TRY(
        cudaMemcpyAsync(packed_host, packed, (size_t)(6 + 2 * m) * 4, cudaMemcpyDeviceToHost, h->stream));
    *results_host = packed_host;
  }
  if (join) {
    if (!h->ev_back) GIMBAL_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_back, cudaEventDisableTiming));
    GIMBAL_CUDA_TRY(cudaEventRecord(h->ev_back, h->stream));
    GIMBAL_CUDA_TRY(cudaStreamWaitEvent(caller, h->ev_back, 0));
  }
  return GIMBAL_OK;
}

int gimbal_stats_set_count_sms(gimbal_stats_t h, int n_sms) {
  GIMBAL_TRY(check_handle(h));
  std::lock_guard<std::mutex> lk(h->mu);
  int dev_sms = 0;
  GIMBAL_CUDA_TRY(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->device));
  if (n_sms < 1 || n_sms > dev_sms) return invalid("set_count_sms: n_sms must be in [1, SM count]");
  h->sms = n_sms;
  h->plan = make_stats_plan(h->topo.n_layers, h->topo.n_experts, h->topo.top_k, n_sms, h->smem_optin);
  h->lm8_plan = make_lm8_plan(h->topo.n_layers, h->topo.n_experts, h->topo.top_k, n_sms, h->smem_optin);
  return GIMBAL_OK;
}

int gimbal_static_placement(const gimbal_topology* topo, int32_t* out) {
  if (!topo || !out) return invalid("static_placement: null argument");
  GIMBAL_TRY(validate_topology(*topo));
  const int per = topo->n_experts / topo->n_gpus;
  for (int l = 0; l < topo->n_layers; ++l)
    for (int e = 0; e < topo->n_experts; ++e) out[l * topo->n_experts + e] = e / per;
  return GIMBAL_OK;
}

int gimbal_comm_cost(const gimbal_topology* topo, const void* ids, int id_bytes, int64_t T, int mem,
                     const int32_t* assign, int32_t n_assign, int device, int64_t* out) {
  if (!topo || !out) return invalid("comm_cost: null argument");
  GIMBAL_TRY(validate_topology(*topo));
  const int L = topo->n_layers, ne = topo->n_experts, k = topo->top_k;
  const int64_t m = (int64_t)L * ne;
  if (n_assign != m) return invalid("comm_cost: assignment size mismatch");
  for (int i = 0; i < n_assign; ++i)
    if (assign[i] < 0) return invalid("comm_cost: unplaced expert");
  if (id_bytes != 1 && id_bytes != 4) return invalid("comm_cost: id_bytes must be 1 or 4");
  if (k > 32) {
    set_error("comm_cost: top_k > 32");
    return GIMBAL_NOT_SUPPORTED;
  }
  // GPU ids only matter through equality: compact them to [0, 256)
  std::vector<int32_t> compact(assign, assign + n_assign);
  {
    std::vector<int32_t> vals(compact);
    std::sort(vals.begin(), vals.end());
    vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
    if (vals.size() > 256) {
      set_error("comm_cost: more than 256 distinct GPU ids");
      return GIMBAL_NOT_SUPPORTED;
    }
    for (auto& v : compact) v = (int32_t)(std::lower_bound(vals.begin(), vals.end(), v) - vals.begin());
  }
  *out = 0;
  if (T <= 0 || L < 2) return GIMBAL_OK;
  DeviceGuard dg(device);
  cudaStream_t s;
  GIMBAL_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  DevBuf dids, dassign, dres;
  int st = GIMBAL_OK;
  const void* src = ids;
  const size_t bytes = (size_t)T * L * k * id_bytes;
  if (mem != GIMBAL_MEM_DEVICE) {
    if ((st = dids.ensure(bytes)) == GIMBAL_OK) {
      if (cudaMemcpyAsync(dids.p, ids, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) st = GIMBAL_CUDA_ERROR;
      src = dids.p;
    }
  }
  if (st == GIMBAL_OK) st = dassign.ensure((size_t)m * 4);
  if (st == GIMBAL_OK) st = dres.ensure(16);
  unsigned long long crossings = 0;
  uint32_t flags = 0;
  if (st == GIMBAL_OK) {
    cudaMemcpyAsync(dassign.p, compact.data(), (size_t)m * 4, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(dres.p, 0, 16, s);
    if (launch_comm_cost(L, ne, k, src, id_bytes, T, dassign.as<int32_t>(), dres.as<unsigned long long>(),
                         reinterpret_cast<uint32_t*>(dres.as<unsigned long long>() + 1), s) != cudaSuccess) {
      set_error("comm_cost: kernel launch failed");
      st = GIMBAL_CUDA_ERROR;
    } else {
      cudaMemcpyAsync(&crossings, dres.p, 8, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(&flags, dres.as<unsigned long long>() + 1, 4, cudaMemcpyDeviceToHost, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("comm_cost: execution failed");
        st = GIMBAL_CUDA_ERROR;
      }
    }
  }
  dids.release();
  dassign.release();
  dres.release();
  cudaStreamDestroy(s);
  if (st != GIMBAL_OK) return st;
  GIMBAL_TRY(flags_to_status(flags));
  *out = (int64_t)crossings;
  return GIMBAL_OK;
}

}  // extern "C"
