// The online expert-layer hook on the GPU: MoeHook::iteration_cost (sim.cpp:113-147) and its
// token_crossings (sim.cpp:183-198), one engine iteration at a time.
//
// Per iteration the routed ids of the batch ([n][L][k], packed to uint8 on the host) go to the
// device in one copy, and three kernels do the whole per-token loop of the reference:
//   online_count_kernel  every (token, layer) unit: the layer x GPU load histogram under the
//                        current placement (layer_gpu_tokens_) and the id checks;
//   online_pairs_kernel  (beside it) the window statistics (all k x k pairings into E, as
//                        RoutingStats::add_token, moe.cpp:169-191) in shared-memory tables of a
//                        block of E rows per CTA, and the cross-GPU transitions (token_crossings);
//   online_finish_kernel per-layer peaks, the bottleneck excess sum_l max(0, peak_l g / (n k) - 1)
//                        in the reference's double arithmetic and layer order, the lifetime
//                        per-GPU activation totals (gpu_activation_total_), and the reset of the
//                        per-iteration accumulators.
// The copy (large batches only; small ones are read zero-copy from pinned memory) and the kernels are
// one CUDA graph, and the finish kernel writes {excess_sum, crossings} straight into pinned memory
// (node parameters updated per launch for the batch size); the host turns them into seconds with
// the reference's own expression.  Statistics stay device-resident: the window handle is the
// caller's gimbal_stats_t (its E/A feed maybe_relocate's greedy on the GPU).
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace gimbal_gpu {

namespace {

constexpr int kOnlineThreads = 256;

struct OnlineOut {
  double excess_sum;
  long long crossings;
};

// with_pairs = 0: the layer pairs (E, crossings) are online_pairs_kernel's; this kernel does the
// histogram, the id checks and (L = 1) the activation only.
__global__ void __launch_bounds__(kOnlineThreads)
    online_count_kernel(const uint8_t* __restrict__ ids, long long n, int L, int ne, int k, int g,
                        const uint8_t* __restrict__ place, unsigned long long* __restrict__ E,
                        unsigned long long* __restrict__ A, unsigned int* __restrict__ hist,
                        unsigned long long* __restrict__ crossings, uint32_t* __restrict__ flags, int with_pairs) {
  extern __shared__ unsigned int sh_hist[];  // [L][g]
  for (int i = threadIdx.x; i < L * g; i += blockDim.x) sh_hist[i] = 0u;
  __syncthreads();
  unsigned long long cross = 0;
  bool bad = false;
  const long long units = n * (long long)L;
  const long long nE = (long long)ne * ne;
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < units;
       u += (long long)gridDim.x * blockDim.x) {
    const long long t = u / L;
    const int l = (int)(u - t * L);
    const uint8_t* row = ids + (t * L + l) * k;
    const uint8_t* pl = place + (long long)l * ne;
    if (k <= 8) {
      // top-k <= 8: the unit's ids and the next layer's, loaded up front into two registers (the
      // small-batch graph reads them zero-copy from pinned host memory: one round trip, not one per
      // dependent id)
      const bool pairs = with_pairs && l + 1 < L;
      unsigned long long cw = 0, nw = 0;
#pragma unroll
      for (int a = 0; a < 8; ++a)
        if (a < k) {
          cw |= (unsigned long long)row[a] << (8 * a);
          if (pairs) nw |= (unsigned long long)row[k + a] << (8 * a);
        }
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        if (a >= k) break;
        const uint32_t e = (uint32_t)(cw >> (8 * a)) & 0xffu;
        if (e >= (uint32_t)ne) {
          bad = true;
          continue;
        }
        atomicAdd(&sh_hist[l * g + pl[e]], 1u);
        if (L == 1) atomicAdd(A + e, 1ull);
      }
      if (pairs) {
        const uint8_t* pn = pl + ne;
        unsigned long long* El = E + (long long)l * nE;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          if (a >= k) break;
          const uint32_t j = (uint32_t)(cw >> (8 * a)) & 0xffu;
          if (j >= (uint32_t)ne) continue;
          const uint32_t pj = pl[j];
          unsigned long long* Erow = El + (long long)j * ne;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            if (b >= k) break;
            const uint32_t kk = (uint32_t)(nw >> (8 * b)) & 0xffu;
            if (kk >= (uint32_t)ne) continue;
            atomicAdd(Erow + kk, 1ull);
            cross += (pj != pn[kk]) ? 1u : 0u;
          }
        }
      }
      continue;
    }
    for (int a = 0; a < k; ++a) {  // layer_gpu_tokens_(l, P(f(l, e))) += 1 (sim.cpp:117-126)
      const uint32_t e = row[a];
      if (e >= (uint32_t)ne) {
        bad = true;
        continue;
      }
      atomicAdd(&sh_hist[l * g + pl[e]], 1u);
      if (L == 1) atomicAdd(A + e, 1ull);  // no layer pairs: activation is the counted buffer
    }
    if (with_pairs && l + 1 < L) {
      const uint8_t* nxt = row + k;
      const uint8_t* pn = pl + ne;
      unsigned long long* El = E + (long long)l * nE;
      for (int a = 0; a < k; ++a) {
        const uint32_t j = row[a];
        if (j >= (uint32_t)ne) continue;
        const uint32_t pj = pl[j];
        unsigned long long* Erow = El + (long long)j * ne;
        for (int b = 0; b < k; ++b) {
          const uint32_t kk = nxt[b];
          if (kk >= (uint32_t)ne) continue;  // flagged by the unit owning layer l + 1
          atomicAdd(Erow + kk, 1ull);         // moe.cpp:179-188, with multiplicity
          cross += (pj != pn[kk]) ? 1u : 0u;  // token_crossings (sim.cpp:183-198)
        }
      }
    }
  }
  if (bad) atomicOr(flags, (uint32_t)kFlagIdOutOfRange);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cross += __shfl_xor_sync(0xffffffffu, cross, o);
  if ((threadIdx.x & 31) == 0 && cross) atomicAdd(crossings, cross);
  __syncthreads();
  for (int i = threadIdx.x; i < L * g; i += blockDim.x)
    if (sh_hist[i]) atomicAdd(hist + i, sh_hist[i]);
}

// The window's E for one iteration, one CTA per (layer pair l, block of `rows` rows of E_l): the
// CTA counts every token's k x k pairings whose layer-l id falls in its rows into shared u32
// cells, then adds them to E (it is the only writer of those cells in this launch: plain
// read-modify-write, no global atomics) and counts the pairings that cross GPUs under the current
// placement (token_crossings, sim.cpp:183-198: the same sum, grouped by cell).  Invalid ids are
// skipped one by one, as in online_count_kernel (which flags them).
__global__ void __launch_bounds__(kOnlineThreads)
    online_pairs_kernel(const uint8_t* __restrict__ ids, long long n, int L, int ne, int k, int rows, int parts,
                        const uint8_t* __restrict__ place, unsigned long long* __restrict__ E,
                        unsigned long long* __restrict__ crossings) {
  extern __shared__ unsigned int tab[];  // [rows][ne]
  const int l = blockIdx.x / parts;
  const int r0 = (blockIdx.x - l * parts) * rows;
  const int r1 = min(ne, r0 + rows);
  const int cells = (r1 - r0) * ne;
  for (int i = threadIdx.x; i < cells; i += blockDim.x) tab[i] = 0u;
  __syncthreads();
  if (k == 8) {  // top-8 rows: one 8-byte load per token-layer (the staging buffer is 256-B aligned)
    for (long long t = threadIdx.x; t < n; t += blockDim.x) {
      const unsigned long long* row = reinterpret_cast<const unsigned long long*>(ids) + t * L + l;
      const unsigned long long cw = __ldg(row), nw = __ldg(row + 1);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int j = (int)((cw >> (8 * a)) & 0xffu);
        if (j < r0 || j >= r1) continue;
        unsigned int* trow = tab + (j - r0) * ne;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int kk = (int)((nw >> (8 * b)) & 0xffu);
          if (kk < ne) atomicAdd(trow + kk, 1u);
        }
      }
    }
  } else {
    for (long long t = threadIdx.x; t < n; t += blockDim.x) {
      const uint8_t* cur = ids + (t * L + l) * k;
      const uint8_t* nxt = cur + k;
      for (int a = 0; a < k; ++a) {
        const int j = cur[a];
        if (j < r0 || j >= r1) continue;  // also every id >= ne
        unsigned int* trow = tab + (j - r0) * ne;
        for (int b = 0; b < k; ++b) {
          const int kk = nxt[b];
          if (kk < ne) atomicAdd(trow + kk, 1u);
        }
      }
    }
  }
  __syncthreads();
  unsigned long long cross = 0;
  const uint8_t* pl = place + (long long)l * ne;
  const uint8_t* pn = pl + ne;
  unsigned long long* El = E + ((long long)l * ne + r0) * ne;
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    const unsigned int v = tab[i];
    if (v == 0u) continue;
    const int jr = i / ne, kk = i - jr * ne;
    El[i] += v;
    cross += pl[r0 + jr] != pn[kk] ? v : 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cross += __shfl_xor_sync(0xffffffffu, cross, o);
  if ((threadIdx.x & 31) == 0 && cross) atomicAdd(crossings, cross);
}

__global__ void online_finish_kernel(long long n, int L, int k, int g, unsigned int* __restrict__ hist,
                                     unsigned long long* __restrict__ crossings,
                                     unsigned long long* __restrict__ gpu_totals, OnlineOut* __restrict__ out) {
  // gpu_activation_total_[p] += every activation placed on p this iteration
  for (int p = threadIdx.x; p < g; p += blockDim.x) {
    unsigned long long s = 0;
#pragma unroll 8
    for (int l = 0; l < L; ++l) s += hist[l * g + p];
    gpu_totals[p] += s;
  }
  if (threadIdx.x < 32) {
    // sim.cpp:132-144, operation by operation: per_layer = double(n * k); for each layer in order
    // excess_sum += max(0.0, peak * n_gpus / per_layer - 1.0)  (IEEE, no contraction).  Lane i
    // finds the peaks of layers i, i + 32, ... (independent loads); lane 0 adds the terms in layer
    // order (a single thread walking all L x g cells cost 15 us at the DS-V3 shape)
    const int lane = threadIdx.x;
    const double per_layer = (double)(n * (long long)k);
    double sum = 0.0;
    for (int l0 = 0; l0 < L; l0 += 32) {
      double x = 0.0;
      if (l0 + lane < L) {
        const unsigned int* h = hist + (l0 + lane) * g;
        unsigned int peak = 0;
        for (int p = 0; p < g; ++p) peak = max(peak, h[p]);
        x = __dsub_rn(__ddiv_rn(__dmul_rn((double)peak, (double)g), per_layer), 1.0);
      }
      const int cnt = min(32, L - l0);
      for (int i = 0; i < cnt; ++i) {
        const double xi = __shfl_sync(0xffffffffu, x, i);
        sum = __dadd_rn(sum, 0.0 < xi ? xi : 0.0);  // std::max(0.0, x)
      }
    }
    if (lane == 0) {
      out->excess_sum = sum;
      out->crossings = (long long)*crossings;
      *crossings = 0;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < L * g; i += blockDim.x) hist[i] = 0u;
}

}  // namespace

}  // namespace gimbal_gpu

using namespace gimbal_gpu;

namespace {

// A few persistent host threads that stage large batches of routed ids into the pinned buffer
// together (a 4096-token DS-V3 batch is 1.9 MB of uint8 or 7.6 MB of int32 ids; one core narrows
// int32 at ~8 GB/s).  run(f) calls f(part) for every part, part 0 on the caller, and returns when
// all have finished.  Created on the first large batch of a handle.
class HostPool {
 public:
  explicit HostPool(int parts) : parts_(parts) {
    try {
      for (int i = 1; i < parts; ++i) th_.emplace_back([this, i] { loop(i); });
    } catch (...) {  // the threads already started are stopped and joined before rethrowing
      shutdown();
      throw;
    }
  }
  ~HostPool() { shutdown(); }
  int parts() const { return parts_; }
  void run(const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      remaining_ = parts_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return remaining_ == 0; });
  }

 private:
  void shutdown() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (std::thread& t : th_) t.join();
    th_.clear();
  }
  void loop(int part) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      const std::function<void(int)>* f = job_;
      lk.unlock();
      (*f)(part);
      lk.lock();
      if (--remaining_ == 0) done_.notify_one();
    }
  }
  const int parts_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int remaining_ = 0;
  bool stop_ = false;
};

constexpr size_t kPoolMinBytes = 1u << 20;  // int32 input bytes from which narrowing is split over threads

}  // namespace

struct gimbal_online_s {
  gimbal_stats_t window = nullptr;
  StatsInternals si;
  int L = 0, ne = 0, k = 0, g = 0;
  int64_t m = 0;
  int64_t cap = 0;  // tokens the staging buffers hold
  uint8_t* d_ids = nullptr;
  uint8_t* h_ids = nullptr;  // pinned
  uint8_t* d_place = nullptr;
  unsigned int* d_hist = nullptr;
  unsigned long long* d_cross = nullptr;
  unsigned long long* d_totals = nullptr;
  OnlineOut* h_out = nullptr;      // pinned, written by online_finish_kernel through h_out_dev
  OnlineOut* h_out_dev = nullptr;  // its device address
  uint8_t* h_ids_dev = nullptr;    // device address of the pinned id staging (zero-copy reads)
  bool placed = false;
  // the iteration as a graph: [H2D ids ->] count [+ pairs] -> finish (result into pinned memory); two variants
  // (mode 0: online_count_kernel counts E with global atomics -- small batches; mode 1: the
  // shared-memory pair tables of online_pairs_kernel -- large batches)
  struct Graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t n_h2d = nullptr, n_count = nullptr, n_pairs = nullptr, n_finish = nullptr;
  } gr[2];
  int64_t iterations = 0;
  std::unique_ptr<HostPool> pool;  // host staging threads (created on the first large batch)
  bool pool_failed = false;        // thread creation failed once: stage on the calling thread

  void release() {
    for (Graph& x : gr) {
      if (x.exec) cudaGraphExecDestroy(x.exec);
      if (x.graph) cudaGraphDestroy(x.graph);
      x = Graph{};
    }
    cudaFree(d_ids);
    cudaFreeHost(h_ids);
    d_ids = nullptr;
    h_ids = nullptr;
    h_ids_dev = nullptr;
    cap = 0;
  }
};

namespace {

int grow(gimbal_online_t o, int64_t n) {
  if (n <= o->cap) return GIMBAL_OK;
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(o->si.stream));
  o->release();
  const int64_t cap = std::max<int64_t>(n, 4096);
  const size_t bytes = (size_t)cap * o->L * o->k;
  GIMBAL_CUDA_TRY(cudaMalloc(&o->d_ids, bytes));
  GIMBAL_CUDA_TRY(cudaHostAlloc(&o->h_ids, bytes, cudaHostAllocMapped));
  void* dev = nullptr;
  GIMBAL_CUDA_TRY(cudaHostGetDevicePointer(&dev, o->h_ids, 0));
  o->h_ids_dev = static_cast<uint8_t*>(dev);
  o->cap = cap;
  return GIMBAL_OK;
}

// Pair kernel geometry: rows of E_l per CTA so that a CTA's u32 cells fit 96 KB of shared memory
// (every CTA of a pair reads the pair's two id columns of the whole batch: fewer, larger CTAs).
struct PairGrid {
  int rows, parts;
  unsigned ctas;
  unsigned smem;
};
PairGrid pair_grid(const gimbal_online_s* o) {
  PairGrid pg;
  pg.rows = std::max(1, std::min(o->ne, (96 * 1024 / 4) / o->ne));
  pg.parts = (o->ne + pg.rows - 1) / pg.rows;
  pg.ctas = (unsigned)((o->L - 1) * pg.parts);
  pg.smem = (unsigned)(pg.rows * o->ne * 4);
  return pg;
}

// the iteration's kernel node parameters for batch size n (the argument arrays live in `a`)
struct NodeArgs {
  long long nn;
  int L, ne, k, g, with_pairs, rows, parts;
  const uint8_t* ids;
  const uint8_t* place;
  unsigned long long *E, *A, *cross, *totals;
  unsigned int* hist;
  uint32_t* flags;
  OnlineOut* out;
  void* cargs[13];
  void* pargs[10];
  void* fargs[8];
};

void node_params(gimbal_online_t o, int mode, int64_t n, unsigned grid, NodeArgs& a, cudaKernelNodeParams& kp,
                 cudaKernelNodeParams& pp, cudaKernelNodeParams& fp) {
  const PairGrid pg = pair_grid(o);
  a.nn = n;
  a.L = o->L;
  a.ne = o->ne;
  a.k = o->k;
  a.g = o->g;
  a.with_pairs = mode == 1 ? 0 : 1;  // mode 1: online_pairs_kernel counts E and the crossings
  a.rows = pg.rows;
  a.parts = pg.parts;
  // mode 0 (small batches) reads the ids straight from the pinned staging buffer (zero-copy: no
  // copy node); mode 1 copies them to the device first (its pair kernel reads each column once per
  // row block)
  a.ids = mode == 1 ? o->d_ids : o->h_ids_dev;
  a.place = o->d_place;
  a.E = o->si.dE;
  a.A = o->si.dA;
  a.cross = o->d_cross;
  a.totals = o->d_totals;
  a.hist = o->d_hist;
  a.flags = o->si.dflags;
  a.out = o->h_out_dev;  // the 16-byte result straight into pinned host memory (no copy node)
  void* c[] = {(void*)&a.ids, &a.nn, &a.L, &a.ne, &a.k, &a.g, (void*)&a.place, &a.E, &a.A, &a.hist, &a.cross,
               &a.flags, &a.with_pairs};
  std::copy(c, c + 13, a.cargs);
  void* q[] = {(void*)&a.ids, &a.nn, &a.L, &a.ne, &a.k, &a.rows, &a.parts, (void*)&a.place, &a.E, &a.cross};
  std::copy(q, q + 10, a.pargs);
  void* f[] = {&a.nn, &a.L, &a.k, &a.g, &a.hist, &a.cross, &a.totals, &a.out};
  std::copy(f, f + 8, a.fargs);
  kp = cudaKernelNodeParams{};
  kp.func = (void*)online_count_kernel;
  kp.gridDim = dim3(grid);
  kp.blockDim = dim3(kOnlineThreads);
  kp.sharedMemBytes = (unsigned)(o->L * o->g * 4);
  kp.kernelParams = a.cargs;
  pp = cudaKernelNodeParams{};
  pp.func = (void*)online_pairs_kernel;
  pp.gridDim = dim3(std::max(1u, pg.ctas));
  pp.blockDim = dim3(kOnlineThreads);
  pp.sharedMemBytes = pg.smem;
  pp.kernelParams = a.pargs;
  fp = cudaKernelNodeParams{};
  fp.func = (void*)online_finish_kernel;
  fp.gridDim = dim3(1);
  fp.blockDim = dim3(256);
  fp.kernelParams = a.fargs;
}

// Mode 1 (pair tables) when the batch's pairings outnumber the pair tables' cells: below that the
// tables' zeroing and read-out cost more than global atomics into the L2-resident E.
int online_mode(const gimbal_online_s* o, int64_t n) {
  return o->L > 1 && n * (int64_t)o->k * o->k >= (int64_t)o->ne * o->ne / 4 && n >= 256 ? 1 : 0;
}

// mode 1: H2D ids -> {histogram kernel, pair kernel} -> finish; mode 0: the combined kernel reading the
// pinned ids -> finish.  finish writes the result into pinned host memory.
int build_graph(gimbal_online_t o, int mode, int64_t n, unsigned grid) {
  GIMBAL_CUDA_TRY(cudaFuncSetAttribute(online_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  gimbal_online_s::Graph& x = o->gr[mode];
  GIMBAL_CUDA_TRY(cudaGraphCreate(&x.graph, 0));
  NodeArgs a;
  cudaKernelNodeParams kp, pp, fp;
  node_params(o, mode, n, grid, a, kp, pp, fp);
  const cudaGraphNode_t* first = nullptr;
  size_t n_first = 0;
  if (mode == 1) {
    GIMBAL_CUDA_TRY(cudaGraphAddMemcpyNode1D(&x.n_h2d, x.graph, nullptr, 0, o->d_ids, o->h_ids,
                                             (size_t)n * o->L * o->k, cudaMemcpyHostToDevice));
    first = &x.n_h2d;
    n_first = 1;
  }
  GIMBAL_CUDA_TRY(cudaGraphAddKernelNode(&x.n_count, x.graph, first, n_first, &kp));
  cudaGraphNode_t before_finish[2] = {x.n_count, nullptr};
  int n_before = 1;
  if (mode == 1) {
    GIMBAL_CUDA_TRY(cudaGraphAddKernelNode(&x.n_pairs, x.graph, first, n_first, &pp));
    before_finish[n_before++] = x.n_pairs;
  }
  GIMBAL_CUDA_TRY(cudaGraphAddKernelNode(&x.n_finish, x.graph, before_finish, n_before, &fp));
  GIMBAL_CUDA_TRY(cudaGraphInstantiate(&x.exec, x.graph, 0));
  return GIMBAL_OK;
}

// batch size n -> graph node parameters (copy size, kernel n and grid)
int update_graph(gimbal_online_t o, int mode, int64_t n, unsigned grid) {
  gimbal_online_s::Graph& x = o->gr[mode];
  if (mode == 1)
    GIMBAL_CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(x.exec, x.n_h2d, o->d_ids, o->h_ids,
                                                       (size_t)n * o->L * o->k, cudaMemcpyHostToDevice));
  NodeArgs a;
  cudaKernelNodeParams kp, pp, fp;
  node_params(o, mode, n, grid, a, kp, pp, fp);
  GIMBAL_CUDA_TRY(cudaGraphExecKernelNodeSetParams(x.exec, x.n_count, &kp));
  if (mode == 1) GIMBAL_CUDA_TRY(cudaGraphExecKernelNodeSetParams(x.exec, x.n_pairs, &pp));
  GIMBAL_CUDA_TRY(cudaGraphExecKernelNodeSetParams(x.exec, x.n_finish, &fp));
  return GIMBAL_OK;
}

}  // namespace

extern "C" {

int gimbal_online_create(gimbal_stats_t window, gimbal_online_t* out) {
  if (!window || !out) return invalid("gimbal_online_create: null argument");
  auto* o = new gimbal_online_s();
  o->window = window;
  o->si = stats_internals(window);
  o->L = o->si.topo.n_layers;
  o->ne = o->si.topo.n_experts;
  o->k = o->si.topo.top_k;
  o->g = o->si.topo.n_gpus;
  o->m = (int64_t)o->L * o->ne;
  if (o->ne > 256 || o->g > 255) {
    delete o;
    set_error("online hook: needs n_experts <= 256 and n_gpus <= 255 (uint8 ids / GPU ids)");
    return GIMBAL_NOT_SUPPORTED;
  }
  DeviceGuard dg(o->si.device);
  auto fail = [&](int st) {
    gimbal_online_destroy(o);
    return st;
  };
  if (cudaMalloc(&o->d_place, (size_t)o->m) != cudaSuccess ||
      cudaMalloc(&o->d_hist, (size_t)o->L * o->g * 4) != cudaSuccess ||
      cudaMalloc(&o->d_cross, 8) != cudaSuccess || cudaMalloc(&o->d_totals, (size_t)o->g * 8) != cudaSuccess ||
      cudaHostAlloc(&o->h_out, sizeof(OnlineOut), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&o->h_out_dev), o->h_out, 0) != cudaSuccess) {
    set_error("gimbal_online_create: allocation failed");
    return fail(GIMBAL_CUDA_ERROR);
  }
  if (cudaMemset(o->d_hist, 0, (size_t)o->L * o->g * 4) != cudaSuccess || cudaMemset(o->d_cross, 0, 8) != cudaSuccess ||
      cudaMemset(o->d_totals, 0, (size_t)o->g * 8) != cudaSuccess) {
    set_error("gimbal_online_create: init failed");
    return fail(GIMBAL_CUDA_ERROR);
  }
  *out = o;
  return GIMBAL_OK;
}

int gimbal_online_destroy(gimbal_online_t o) {
  if (!o) return GIMBAL_OK;
  DeviceGuard dg(o->si.device);
  // no use of the window handle here: it may already be destroyed (its destroy synchronised its
  // stream); cudaFree / cudaFreeHost wait for outstanding work on these buffers
  o->release();
  cudaFree(o->d_place);
  cudaFree(o->d_hist);
  cudaFree(o->d_cross);
  cudaFree(o->d_totals);
  cudaFreeHost(o->h_out);
  delete o;
  return GIMBAL_OK;
}

int gimbal_online_set_placement(gimbal_online_t o, const int32_t* assign, int64_t m) {
  if (!o || !assign) return invalid("online: null argument");
  if (m != o->m) return invalid("online: placement size mismatch");
  std::vector<uint8_t> p((size_t)m);
  for (int64_t i = 0; i < m; ++i) {
    if (assign[i] < 0 || assign[i] >= o->g) return invalid("online: placement GPU id out of range");
    p[(size_t)i] = (uint8_t)assign[i];
  }
  std::lock_guard<std::mutex> lk(*o->si.mu);
  DeviceGuard dg(o->si.device);
  // pageable source: the copy has consumed `p` when the call returns
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(o->d_place, p.data(), (size_t)m, cudaMemcpyHostToDevice, o->si.stream));
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(o->si.stream));
  o->placed = true;
  return GIMBAL_OK;
}

int gimbal_online_iteration(gimbal_online_t o, const void* ids, int id_bytes, int64_t n, double* excess_sum,
                            int64_t* crossings) {
  if (!o || !excess_sum || !crossings) return invalid("online: null argument");
  if (id_bytes != 1 && id_bytes != 4) return invalid("online: id_bytes must be 1 or 4");
  if (!o->placed) return invalid("online: no placement set");
  if (n <= 0) {
    *excess_sum = 0.0;
    *crossings = 0;
    return GIMBAL_OK;
  }
  if (!ids) return invalid("online: null ids");
  std::lock_guard<std::mutex> lk(*o->si.mu);
  DeviceGuard dg(o->si.device);
  GIMBAL_TRY(stats_resolve_tokens(o->window));
  GIMBAL_TRY(grow(o, n));
  const size_t cnt = (size_t)n * o->L * o->k;
  // int32 (RoutedStream::choices) -> uint8 (n_e <= 256; the reference leaves bad ids UB): a
  // branch-free (vectorisable) conversion with one range verdict per part
  const uint32_t ne = (uint32_t)o->ne;
  auto stage = [&](size_t b, size_t e) -> uint32_t {
    if (id_bytes == 1) {
      std::memcpy(o->h_ids + b, static_cast<const uint8_t*>(ids) + b, e - b);
      return 0u;
    }
    const int32_t* s = static_cast<const int32_t*>(ids);
    uint32_t bad = 0;
    for (size_t i = b; i < e; ++i) {
      const uint32_t v = (uint32_t)s[i];  // negative ids wrap above n_e
      bad |= v >= ne ? 1u : 0u;
      o->h_ids[i] = (uint8_t)v;
    }
    return bad;
  };
  uint32_t bad = 0;
  if (id_bytes == 4 && cnt * 4 >= kPoolMinBytes && !o->pool_failed) {  // (uint8: one memcpy beats woken threads)
    if (!o->pool) {
      const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
      try {
        o->pool.reset(new HostPool((int)std::min(8u, hw / 2)));
      } catch (const std::exception&) {  // no threads to be had: stage on the calling thread
        o->pool_failed = true;
      }
    }
  }
  if (o->pool && id_bytes == 4 && cnt * 4 >= kPoolMinBytes) {
    const int parts = o->pool->parts();
    std::vector<uint32_t> bads((size_t)parts, 0u);
    const size_t per = ((cnt + parts - 1) / parts + 63) & ~(size_t)63;
    o->pool->run([&](int p) {
      const size_t b = std::min(cnt, (size_t)p * per), e = std::min(cnt, b + per);
      bads[(size_t)p] = stage(b, e);
    });
    for (uint32_t x : bads) bad |= x;
  } else {
    bad = stage(0, cnt);
  }
  if (bad) {
    set_error("add_token: expert id out of range [0, n_experts)");
    return GIMBAL_OUT_OF_RANGE;
  }
  const unsigned grid =
      (unsigned)std::max<int64_t>(1, std::min<int64_t>(4 * 148, (n * o->L + kOnlineThreads - 1) / kOnlineThreads));
  const int mode = online_mode(o, n);
  if (!o->gr[mode].exec) {  // (grow() drops both graphs when the staging buffers move)
    GIMBAL_TRY(build_graph(o, mode, n, grid));
  } else {
    GIMBAL_TRY(update_graph(o, mode, n, grid));
  }
  GIMBAL_CUDA_TRY(cudaGraphLaunch(o->gr[mode].exec, o->si.stream));
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(o->si.stream));
  stats_note_added(o->window, n);
  ++o->iterations;
  *excess_sum = o->h_out->excess_sum;
  *crossings = o->h_out->crossings;
  return GIMBAL_OK;
}

int gimbal_online_gpu_totals(gimbal_online_t o, int64_t* out) {
  if (!o || !out) return invalid("online: null argument");
  std::lock_guard<std::mutex> lk(*o->si.mu);
  DeviceGuard dg(o->si.device);
  std::vector<unsigned long long> t((size_t)o->g);
  GIMBAL_CUDA_TRY(cudaMemcpyAsync(t.data(), o->d_totals, (size_t)o->g * 8, cudaMemcpyDeviceToHost, o->si.stream));
  GIMBAL_CUDA_TRY(cudaStreamSynchronize(o->si.stream));
  for (int p = 0; p < o->g; ++p) out[p] = (int64_t)t[(size_t)p];
  return GIMBAL_OK;
}

}  // extern "C"
