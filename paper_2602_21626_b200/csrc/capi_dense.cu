// C ABI, part 2: the reference's general dense forms (PlacementProblem with explicit A / W, an
// explicit AffinityTensor, greedy_place on an arbitrary activation matrix), the synthetic trace
// generator and the reference's balanced-candidate recipe.
//
// The dense forms exist so that the reference's operator API (placement.hpp:44-85) can be served
// unchanged for arbitrary inputs (tests build hand-made A / W / E).  Counts must be non-negative
// integer-valued doubles below 2^40 for the affinity/greedy forms (every reference call site
// passes counts); other values return GIMBAL_NOT_SUPPORTED.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"

using namespace gimbal_gpu;

namespace {

struct Tmp {
  std::vector<void*> ptrs;
  ~Tmp() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

// eval_cost on a dense problem (placement.cpp:58-85).  loads and the per-row sums follow the
// reference's visiting order (j ascending); the cut is summed per row j in k order and the row
// partials are combined in j order (exact for integer-valued W, within 1e-15 relative otherwise).
__global__ void dense_eval_kernel(int rows, int m, int g, const double* __restrict__ A,
                                  const double* __restrict__ W, const int32_t* __restrict__ P,
                                  double* __restrict__ row_cut, double* __restrict__ row_dev) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid < m) {
    const int j = tid;
    double c = 0.0;
    for (int k = j + 1; k < m; ++k)
      if (P[j] != P[k]) c = __dadd_rn(c, __dadd_rn(W[(int64_t)j * m + k], W[(int64_t)k * m + j]));
    row_cut[j] = c;
  }
  if (tid < rows) {
    const int i = tid;
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = __dadd_rn(s, A[(int64_t)i * m + j]);
    const double ideal = __ddiv_rn(s, (double)g);
    double dev = 0.0;
    for (int p = 0; p < g; ++p) {
      double load = 0.0;
      for (int j = 0; j < m; ++j)
        if (P[j] == p) load = __dadd_rn(load, A[(int64_t)i * m + j]);
      dev = fmax(dev, fabs(__dsub_rn(load, ideal)));
    }
    row_dev[i] = dev;
  }
}

__global__ void dense_eval_finish(int rows, int m, double alpha, double beta,
                                  const double* __restrict__ row_cut,
                                  const double* __restrict__ row_dev, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double c = 0.0, d = 0.0;
    for (int j = 0; j < m; ++j) c = __dadd_rn(c, row_cut[j]);
    for (int i = 0; i < rows; ++i) d = fmax(d, row_dev[i]);
    out[0] = d;
    out[1] = c;
    out[2] = __dadd_rn(__dmul_rn(alpha, d), __dmul_rn(beta, c));
  }
}

// Dense greedy: keys (total desc, id asc) + first-argmax home row per column.
__global__ void dense_greedy_keys(int rows, int64_t m, const unsigned long long* __restrict__ A,
                                  const uint32_t* __restrict__ anchored,
                                  unsigned long long* __restrict__ keys, int32_t* __restrict__ home,
                                  int64_t n_pad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_pad;
       e += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0ull;
    if (e < m) {
      // totals = colwise().sum(); home = first argmax row (Eigen maxCoeff keeps the first
      // strict maximum), placement.cpp:259-265
      unsigned long long tot = A[e], best = A[e];
      int h = 0;
      for (int i = 1; i < rows; ++i) {
        const unsigned long long v = A[(int64_t)i * m + e];
        tot += v;
        if (v > best) {
          best = v;
          h = i;
        }
      }
      home[e] = h;
      if (!((anchored[e >> 5] >> (e & 31)) & 1u)) key = (tot << 24) | (unsigned long long)(0xffffffll - e);
    }
    keys[e] = key;
  }
}

__global__ void dense_greedy_walk(int rows, int64_t m, int g, const unsigned long long* __restrict__ A,
                                  const int32_t* __restrict__ M, int32_t nM, int32_t anchor,
                                  const unsigned long long* __restrict__ keys,
                                  const int32_t* __restrict__ home, unsigned long long* __restrict__ load,
                                  int32_t* __restrict__ out) {
  __shared__ int counts[1024];
  __shared__ int target;
  const int cap = (int)(m / g);
  for (int p = threadIdx.x; p < g; p += blockDim.x) counts[p] = 0;
  for (int64_t i = threadIdx.x; i < (int64_t)rows * g; i += blockDim.x) load[i] = 0ull;
  __syncthreads();
  for (int a = 0; a < nM; ++a) {
    const int64_t e = M[a];
    for (int i = threadIdx.x; i < rows; i += blockDim.x) load[(int64_t)i * g + anchor] += A[(int64_t)i * m + e];
    if (threadIdx.x == 0) {
      out[e] = anchor;
      counts[anchor] += 1;
    }
    __syncthreads();
  }
  for (int64_t idx = 0; idx < m; ++idx) {
    const unsigned long long key = keys[idx];
    if (key == 0ull) break;
    const int64_t e = 0xffffffll - (int64_t)(key & 0xffffffull);
    if (threadIdx.x == 0) {
      const int row = home[e];
      int t = -1;
      for (int p = 0; p < g; ++p) {  // placement.cpp:290-295
        if (counts[p] >= cap) continue;
        if (t == -1 || load[(int64_t)row * g + p] < load[(int64_t)row * g + t]) t = p;
      }
      target = t;
      out[e] = t;
      counts[t] += 1;
    }
    __syncthreads();
    const int t = target;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) load[(int64_t)i * g + t] += A[(int64_t)i * m + e];
    __syncthreads();
  }
}

bool integer_valued(const double* v, size_t n, std::vector<unsigned long long>& out) {
  out.resize(n);
  for (size_t i = 0; i < n; ++i) {
    const double x = v[i];
    if (!(x >= 0.0) || x >= 1099511627776.0 || std::floor(x) != x) return false;
    out[i] = (unsigned long long)x;
  }
  return true;
}

}  // namespace

namespace gimbal_gpu {
cudaError_t launch_affinity_keys(int L, int ne, const unsigned long long* E, double threshold,
                                 unsigned long long* keys, int64_t n_pad, uint32_t* flags,
                                 cudaStream_t s);
}

// ---- generator helpers (host) ----
namespace {

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t mix_seed(uint64_t seed, uint64_t stream) { return splitmix64(seed ^ splitmix64(stream)); }

// The reference Rng's draws (rng.hpp:25-71) on std::mt19937_64, which the C++ standard fixes.
struct RefRng {
  std::mt19937_64 eng;
  explicit RefRng(uint64_t s) : eng(s) {}
  int64_t uniform_int(int64_t n) {
    const uint64_t bound = (uint64_t)n;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
      x = eng();
    } while (x >= limit);
    return (int64_t)(x % bound);
  }
  template <typename T>
  void shuffle(T* items, size_t n) {
    for (size_t i = n; i > 1; --i) {
      const size_t j = (size_t)uniform_int((int64_t)i);
      std::swap(items[i - 1], items[j]);
    }
  }
};

}  // namespace

extern "C" {

int gimbal_eval_cost_dense(int32_t rows, int32_t m, const double* A, const double* W, int32_t g,
                           double alpha, double beta, const int32_t* assign, double* deviation,
                           double* cut, double* objective) {
  if (!A || !W || !assign || !deviation || !cut || !objective) return invalid("eval_cost: null argument");
  // PlacementProblem::validate (placement.cpp:13-26)
  if (m < 1) return invalid("PlacementProblem: no experts");
  if (g < 1) return invalid("PlacementProblem: g must be >= 1");
  if (m % g != 0) return invalid("PlacementProblem: experts must be divisible by g");
  if (!(alpha > 0.0) || !(beta > 0.0)) return invalid("PlacementProblem: alpha and beta must be > 0");
  // check_feasible (placement.cpp:30-50)
  std::vector<int> counts((size_t)g, 0);
  for (int j = 0; j < m; ++j) {
    if (assign[j] < 0 || assign[j] >= g) return invalid("placement: expert assigned to invalid GPU");
    counts[(size_t)assign[j]] += 1;
  }
  for (int p = 0; p < g; ++p)
    if (counts[(size_t)p] != m / g)
      return invalid("placement: GPU " + std::to_string(p) + " holds " + std::to_string(counts[(size_t)p]) +
                     " experts, expected " + std::to_string(m / g));
  Tmp t;
  double* dA = t.alloc<double>((size_t)rows * m);
  double* dW = t.alloc<double>((size_t)m * m);
  int32_t* dP = t.alloc<int32_t>(m);
  double* rc = t.alloc<double>(m);
  double* rd = t.alloc<double>(std::max(rows, 1));
  double* res = t.alloc<double>(3);
  if (!dA || !dW || !dP || !rc || !rd || !res) {
    set_error("eval_cost: device allocation failed");
    return GIMBAL_CUDA_ERROR;
  }
  GIMBAL_CUDA_TRY(cudaMemcpy(dA, A, (size_t)rows * m * 8, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(cudaMemcpy(dW, W, (size_t)m * m * 8, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(cudaMemcpy(dP, assign, (size_t)m * 4, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(cudaMemset(rd, 0, std::max(rows, 1) * 8));
  const int n = std::max(rows, m);
  dense_eval_kernel<<<(n + 127) / 128, 128>>>(rows, m, g, dA, dW, dP, rc, rd);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  dense_eval_finish<<<1, 32>>>(rows, m, alpha, beta, rc, rd, res);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  double h[3];
  GIMBAL_CUDA_TRY(cudaMemcpy(h, res, sizeof(h), cudaMemcpyDeviceToHost));
  *deviation = h[0];
  *cut = h[1];
  *objective = h[2];
  return GIMBAL_OK;
}

int gimbal_affinity_set_dense(const gimbal_topology* topo, const double* E, int32_t n_blocks,
                              double threshold, int32_t top_e, int32_t capacity, int32_t anchor_gpu,
                              int32_t* out, int32_t* n_out) {
  if (!topo || !out || !n_out) return invalid("build_affinity_set: null argument");
  GIMBAL_TRY(validate_topology(*topo));
  if (anchor_gpu < 0 || anchor_gpu >= topo->n_gpus) return invalid("build_affinity_set: anchor_gpu out of range");
  if (n_blocks != std::max(0, topo->n_layers - 1)) return invalid("build_affinity_set: tensor depth mismatch");
  const int L = topo->n_layers, ne = topo->n_experts;
  *n_out = 0;
  if (L < 2) return GIMBAL_OK;
  const int64_t n = (int64_t)(L - 1) * ne * ne;
  if (n >= (1ll << 24)) {
    set_error("build_affinity_set: (L-1)*n_experts^2 must be < 2^24");
    return GIMBAL_NOT_SUPPORTED;
  }
  std::vector<unsigned long long> ev;
  if (!integer_valued(E, (size_t)n, ev)) {
    set_error("build_affinity_set: weights must be non-negative integer counts < 2^40");
    return GIMBAL_NOT_SUPPORTED;
  }
  const int64_t n_pad = next_pow2(n);
  const int64_t m = (int64_t)L * ne;
  Tmp t;
  auto* dE = t.alloc<unsigned long long>(n);
  auto* keys = t.alloc<unsigned long long>(n_pad);
  auto* bits = t.alloc<uint32_t>((m + 31) / 32);
  auto* dout = t.alloc<int32_t>(m);
  auto* dn = t.alloc<int32_t>(1);
  auto* flags = t.alloc<uint32_t>(1);
  if (!dE || !keys || !bits || !dout || !dn || !flags) {
    set_error("build_affinity_set: device allocation failed");
    return GIMBAL_CUDA_ERROR;
  }
  GIMBAL_CUDA_TRY(cudaMemcpy(dE, ev.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(cudaMemset(flags, 0, 4));
  GIMBAL_CUDA_TRY(launch_affinity_keys(L, ne, dE, threshold, keys, n_pad, flags, 0));
  GIMBAL_CUDA_TRY(sort_u64_desc(keys, n_pad, 0));
  GIMBAL_CUDA_TRY(launch_affinity_select(L, ne, keys, n, top_e, capacity, bits, dout, dn, 0));
  int32_t cnt = 0;
  GIMBAL_CUDA_TRY(cudaMemcpy(&cnt, dn, 4, cudaMemcpyDeviceToHost));
  if (cnt > 0) GIMBAL_CUDA_TRY(cudaMemcpy(out, dout, (size_t)cnt * 4, cudaMemcpyDeviceToHost));
  *n_out = cnt;
  return GIMBAL_OK;
}

int gimbal_greedy_place_dense(int32_t rows, int32_t m, const double* activation, const int32_t* M,
                              int32_t nM, int32_t anchor_gpu, int32_t g, int32_t* out) {
  if (!activation || !out || (nM > 0 && !M)) return invalid("greedy_place: null argument");
  if (g < 1 || m < 1 || m % g != 0) return invalid("greedy_place: experts must be divisible by g");
  const int cap = m / g;
  if (anchor_gpu < 0 || anchor_gpu >= g) return invalid("greedy_place: anchor_gpu out of range");
  if (nM > cap) return invalid("greedy_place: affinity set exceeds anchor capacity");
  std::vector<uint32_t> bits((size_t)((m + 31) / 32), 0u);
  for (int i = 0; i < nM; ++i) {
    const int e = M[i];
    if (e < 0 || e >= m) return invalid("greedy_place: affinity id out of range");
    if ((bits[(size_t)e >> 5] >> (e & 31)) & 1u) return invalid("greedy_place: duplicate affinity id");
    bits[(size_t)e >> 5] |= 1u << (e & 31);
  }
  if (rows < 1) return invalid("greedy_place: activation has no rows");
  if (g > 1024 || m >= (1 << 24)) {
    set_error("greedy_place: g <= 1024 and m < 2^24 required");
    return GIMBAL_NOT_SUPPORTED;
  }
  std::vector<unsigned long long> av;
  if (!integer_valued(activation, (size_t)rows * m, av)) {
    set_error("greedy_place: activation must hold non-negative integer counts < 2^40");
    return GIMBAL_NOT_SUPPORTED;
  }
  const int64_t n_pad = next_pow2(m);
  Tmp t;
  auto* dA = t.alloc<unsigned long long>((size_t)rows * m);
  auto* dbits = t.alloc<uint32_t>(bits.size());
  auto* keys = t.alloc<unsigned long long>(n_pad);
  auto* home = t.alloc<int32_t>(m);
  auto* load = t.alloc<unsigned long long>((size_t)rows * g);
  auto* dM = t.alloc<int32_t>(std::max(nM, 1));
  auto* dout = t.alloc<int32_t>(m);
  if (!dA || !dbits || !keys || !home || !load || !dM || !dout) {
    set_error("greedy_place: device allocation failed");
    return GIMBAL_CUDA_ERROR;
  }
  GIMBAL_CUDA_TRY(cudaMemcpy(dA, av.data(), av.size() * 8, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(cudaMemcpy(dbits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice));
  if (nM > 0) GIMBAL_CUDA_TRY(cudaMemcpy(dM, M, (size_t)nM * 4, cudaMemcpyHostToDevice));
  const int grid = (int)std::min<int64_t>(1184, (n_pad + 255) / 256);
  dense_greedy_keys<<<grid, 256>>>(rows, m, dA, dbits, keys, home, n_pad);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  GIMBAL_CUDA_TRY(sort_u64_desc(keys, n_pad, 0));
  dense_greedy_walk<<<1, 256>>>(rows, m, g, dA, dM, nM, anchor_gpu, keys, home, load, dout);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  GIMBAL_CUDA_TRY(cudaMemcpy(out, dout, (size_t)m * 4, cudaMemcpyDeviceToHost));
  return GIMBAL_OK;
}

int gimbal_generator_tables(const gimbal_topology* topo, double zipf_s, double lambda, double peak,
                            uint64_t model_seed, double drift, uint64_t drift_epoch, uint32_t* cdf,
                            uint64_t* thr) {
  if (!topo || !cdf || !thr) return invalid("generator: null argument");
  GIMBAL_TRY(validate_topology(*topo));
  if (lambda < 0.0 || lambda > 1.0) return invalid("RoutingParams: lambda must be in [0, 1]");
  if (peak < 0.0 || peak > 1.0) return invalid("RoutingParams: affinity_peak must be in [0, 1]");
  if (drift < 0.0 || drift > 1.0) return invalid("generator: drift must be in [0, 1]");
  const int L = topo->n_layers, ne = topo->n_experts;
  const double rest = ne > 1 ? (1.0 - peak) / (ne - 1) : 0.0;
  if (ne > 1 && peak < rest) {
    set_error("generator: affinity_peak below the uniform share is not supported");
    return GIMBAL_NOT_SUPPORTED;
  }
  // per-layer Zipf ranks over a permutation seeded like the reference (moe.cpp:61-71)
  std::vector<std::vector<int>> ranks((size_t)L, std::vector<int>((size_t)ne));
  RefRng rng(mix_seed(model_seed, 0x5a1fULL));
  for (int l = 0; l < L; ++l) {
    std::iota(ranks[(size_t)l].begin(), ranks[(size_t)l].end(), 0);
    rng.shuffle(ranks[(size_t)l].data(), (size_t)ne);
  }
  // drift (config 5): each epoch re-draws round(drift*ne) rank slots of every layer
  const int nd = (int)std::lround(drift * ne);
  for (uint64_t w = 1; w <= drift_epoch && nd > 1; ++w) {
    RefRng dr(mix_seed(mix_seed(model_seed, 0xd21fULL), w));
    std::vector<int> pos((size_t)ne);
    for (int l = 0; l < L; ++l) {
      std::iota(pos.begin(), pos.end(), 0);
      dr.shuffle(pos.data(), pos.size());  // first nd positions are the re-drawn slots
      std::vector<int> vals((size_t)nd);
      for (int i = 0; i < nd; ++i) vals[(size_t)i] = ranks[(size_t)l][(size_t)pos[(size_t)i]];
      dr.shuffle(vals.data(), vals.size());
      for (int i = 0; i < nd; ++i) ranks[(size_t)l][(size_t)pos[(size_t)i]] = vals[(size_t)i];
    }
  }
  for (int l = 0; l < L; ++l) {
    std::vector<double> w((size_t)ne);
    double sum = 0.0;
    for (int e = 0; e < ne; ++e) {
      w[(size_t)e] = 1.0 / std::pow((double)(ranks[(size_t)l][(size_t)e] + 1), zipf_s);
      sum += w[(size_t)e];
    }
    double cum = 0.0;
    for (int e = 0; e < ne; ++e) {
      cum += w[(size_t)e] / sum;
      const double q = std::floor(cum * 4294967296.0);
      cdf[(size_t)l * ne + e] = (e == ne - 1 || q >= 4294967295.0) ? 0xffffffffu : (uint32_t)q;
    }
  }
  const double two32 = 4294967296.0;
  const double pb = 1.0 - lambda;
  const double pu = lambda * rest * ne;
  thr[0] = (uint64_t)std::min(two32, std::floor(pb * two32 + 0.5));
  thr[1] = (uint64_t)std::min(two32, std::floor((pb + pu) * two32 + 0.5));
  if (lambda == 0.0) thr[0] = thr[1] = (uint64_t)two32;
  return GIMBAL_OK;
}

int gimbal_generate_trace(const gimbal_topology* topo, double zipf_s, double lambda, double peak,
                          uint64_t model_seed, uint64_t stream_seed, double drift, uint64_t drift_epoch,
                          int64_t first_token, int64_t n_tokens, uint8_t* out, int device) {
  if (!topo || (!out && n_tokens > 0)) return invalid("generator: null argument");
  GIMBAL_TRY(validate_topology(*topo));
  if (topo->n_experts > 256 || topo->top_k > 64) {
    set_error("generator: uint8 traces need n_experts <= 256, top_k <= 64");
    return GIMBAL_NOT_SUPPORTED;
  }
  const int L = topo->n_layers, ne = topo->n_experts;
  std::vector<uint32_t> cdf((size_t)L * ne);
  uint64_t thr[2];
  GIMBAL_TRY(gimbal_generator_tables(topo, zipf_s, lambda, peak, model_seed, drift, drift_epoch, cdf.data(), thr));
  if (n_tokens <= 0) return GIMBAL_OK;
  DeviceGuard g(device);
  Tmp t;
  auto* dcdf = t.alloc<uint32_t>(cdf.size());
  if (!dcdf) {
    set_error("generator: device allocation failed");
    return GIMBAL_CUDA_ERROR;
  }
  GIMBAL_CUDA_TRY(cudaMemcpy(dcdf, cdf.data(), cdf.size() * 4, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(launch_generate_trace(L, ne, topo->top_k, dcdf, thr[0], thr[1], stream_seed, first_token,
                                        n_tokens, out, 0));
  GIMBAL_CUDA_TRY(cudaDeviceSynchronize());
  return GIMBAL_OK;
}

int gimbal_shuffled_candidates(int32_t m, int32_t g, uint64_t seed, int64_t n, uint8_t* out) {
  if (!out && n > 0) return invalid("shuffled_candidates: null output");
  if (m < 1 || g < 1 || g > 255 || m % g != 0) return invalid("shuffled_candidates: need m % g == 0, g <= 255");
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < hw; ++w) {
    pool.emplace_back([=] {
      std::vector<uint8_t> a((size_t)m);
      for (int64_t c = w; c < n; c += hw) {
        for (int e = 0; e < m; ++e) a[(size_t)e] = (uint8_t)(e % g);
        RefRng r(seed + (uint64_t)c);
        r.shuffle(a.data(), a.size());
        std::memcpy(out + (size_t)c * m, a.data(), (size_t)m);
      }
    });
  }
  for (auto& th : pool) th.join();
  return GIMBAL_OK;
}

}  // extern "C"
