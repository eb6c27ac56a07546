// placement::exact_solve (placement.cpp:87-184) on the GPU: every balanced placement of up to 16
// experts on up to 4 GPUs, scored in parallel, instead of the reference's single-threaded branch
// and bound.
//
// The reference searches placements with GPU labels in first-use order (restricted growth
// strings; label symmetry broken), experts in index order and labels ascending, keeps a new
// incumbent only when strictly better and prunes on an admissible bound.  With non-negative A / W
// the bound never cuts off a strictly better leaf, so its answer is the lexicographically least
// canonical placement with the minimum objective.  Here the host lists the canonical prefixes of
// the first m - kSuffix experts in lexicographic order; GPU thread t walks every completion of
// prefix t depth-first in the same order (no pruning) and keeps its first minimum; a one-block
// reduction takes the minimum objective, ties to the lowest thread.
//
// Objective as the reference's leaf: loads(i, p) accumulated over experts in index order, ideal_i
// = rowsum_i / g, D = max |loads - ideal| (from 0.0), cut = sum over experts j of sum over k < j on
// another GPU of W(k, j) + W(j, k), objective = alpha * D + beta * cut (no fused multiply-add).
// For non-negative integer-valued A / W below 2^40 (every count-derived problem and the
// reference's tests) all sums are exact, so the answer equals the reference's bit for bit; other
// inputs return GIMBAL_NOT_SUPPORTED.  The returned cost is eval_cost of the answer, as in the
// reference (placement.cpp:182-183).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace gimbal_gpu;

namespace {

constexpr int kMaxExperts = 16;  // placement.hpp:49 kExactMaxExperts
constexpr int kMaxGpus = 4;      // placement.hpp:50 kExactMaxGpus
constexpr int kMaxRows = 64;     // rows of A (layers) held per thread
constexpr int kSuffix = 6;       // experts each thread enumerates below its prefix (10^4-10^5 threads at m = 16)

struct ExactParams {
  int rows, m, g, cap, depth;  // depth = prefix length
  int n_prefix;
  double alpha, beta;
};

__device__ __forceinline__ int label_of(uint32_t packed, int j) { return (int)((packed >> (2 * j)) & 3u); }

// One thread per canonical prefix: depth-first over the completions, labels ascending.
__global__ void __launch_bounds__(128) exact_enum_kernel(ExactParams prm, const double* __restrict__ A,
                                                          const double* __restrict__ W,
                                                          const uint32_t* __restrict__ prefixes,
                                                          double* __restrict__ best_obj,
                                                          uint32_t* __restrict__ best_assign) {
  __shared__ double sPW[kMaxExperts * kMaxExperts];  // W(k, j) + W(j, k)
  __shared__ double sIdeal[kMaxRows];
  const int m = prm.m, g = prm.g, R = prm.rows;
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
    const int k = i / m, j = i - k * m;
    sPW[i] = W[k * m + j] + W[j * m + k];
  }
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s += A[i * m + j];
    sIdeal[i] = s / (double)g;
  }
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= prm.n_prefix) return;

  double loads[kMaxRows * kMaxGpus];
  double cutd[kMaxExperts + 1];
  int lab[kMaxExperts], used[kMaxExperts + 1], cnt[kMaxGpus];
  for (int i = 0; i < R * g; ++i) loads[i] = 0.0;
  for (int p = 0; p < kMaxGpus; ++p) cnt[p] = 0;
  // apply label p to expert j (prefix or search step)
  auto place = [&](int j, int p) {
    double d = 0.0;
    for (int k = 0; k < j; ++k)
      if (lab[k] != p) d += sPW[k * m + j];
    cutd[j + 1] = cutd[j] + d;
    used[j + 1] = max(used[j], p + 1);
    lab[j] = p;
    cnt[p] += 1;
    for (int i = 0; i < R; ++i) loads[i * g + p] += A[i * m + j];
  };
  auto unplace = [&](int j) {
    const int p = lab[j];
    cnt[p] -= 1;
    for (int i = 0; i < R; ++i) loads[i * g + p] -= A[i * m + j];
    lab[j] = -1;
  };
  cutd[0] = 0.0;
  used[0] = 0;
  const uint32_t pre = prefixes[t];
  for (int j = 0; j < prm.depth; ++j) place(j, label_of(pre, j));

  double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  uint32_t best_packed = 0u;
  int j = prm.depth;
  if (j < m) lab[j] = -1;
  while (true) {
    if (j == m) {
      double dev = 0.0;
      for (int i = 0; i < R; ++i)
        for (int p = 0; p < g; ++p) dev = fmax(dev, fabs(loads[i * g + p] - sIdeal[i]));
      const double obj = __dadd_rn(__dmul_rn(prm.alpha, dev), __dmul_rn(prm.beta, cutd[m]));
      if (obj < best) {
        best = obj;
        uint32_t pk = 0u;
        for (int k = 0; k < m; ++k) pk |= (uint32_t)lab[k] << (2 * k);
        best_packed = pk;
      }
      --j;
      continue;
    }
    // next label for expert j after its current one (-1: none tried yet)
    const int cur = lab[j];
    if (cur >= 0) unplace(j);
    const int limit = min(g - 1, used[j]);
    int p = cur + 1;
    while (p <= limit && cnt[p] == prm.cap) ++p;
    if (p <= limit) {
      place(j, p);
      ++j;
      if (j < m) lab[j] = -1;
    } else {
      if (j == prm.depth) break;
      --j;
    }
  }
  best_obj[t] = best;
  best_assign[t] = best_packed;
}

// Minimum objective, ties to the lowest prefix index (the lexicographically least placement).
__global__ void __launch_bounds__(1024) exact_reduce_kernel(int n, const double* __restrict__ obj,
                                                            const uint32_t* __restrict__ assign,
                                                            uint32_t* __restrict__ out) {
  __shared__ double so[1024];
  __shared__ int si[1024];
  double b = __longlong_as_double(0x7ff0000000000000ll);
  int bi = -1;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (obj[i] < b) {  // ascending i per thread: the first minimum is kept
      b = obj[i];
      bi = i;
    }
  so[threadIdx.x] = b;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = so[threadIdx.x + s];
      const int oi = si[threadIdx.x + s];
      if (oi >= 0 && (si[threadIdx.x] < 0 || o < so[threadIdx.x] || (o == so[threadIdx.x] && oi < si[threadIdx.x]))) {
        so[threadIdx.x] = o;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = si[0] >= 0 ? assign[si[0]] : 0u;
    out[1] = si[0] >= 0 ? 1u : 0u;
  }
}

// Canonical prefixes of length `depth` (labels in first-use order, at most `cap` per label) in
// lexicographic order, packed 2 bits per expert.
void list_prefixes(int depth, int g, int cap, std::vector<uint32_t>& out) {
  std::vector<int> cnt((size_t)g, 0);
  auto rec = [&](auto&& self, int j, int used, uint32_t pk) -> void {
    if (j == depth) {
      out.push_back(pk);
      return;
    }
    for (int p = 0; p <= std::min(g - 1, used); ++p) {
      if (cnt[(size_t)p] == cap) continue;
      cnt[(size_t)p] += 1;
      self(self, j + 1, std::max(used, p + 1), pk | ((uint32_t)p << (2 * j)));
      cnt[(size_t)p] -= 1;
    }
  };
  rec(rec, 0, 0, 0u);
}

bool exact_integer(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!(v[i] >= 0.0 && v[i] < 1099511627776.0 && v[i] == std::floor(v[i]))) return false;
  return true;
}

struct DevBuf {
  std::vector<void*> ptrs;
  ~DevBuf() {
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

}  // namespace

extern "C" {

int gimbal_exact_solve_dense(int32_t rows, int32_t m, const double* A, const double* W, int32_t g, double alpha,
                             double beta, int32_t* assign_out, double* deviation, double* cut, double* objective) {
  if (!A || !W || !assign_out || !deviation || !cut || !objective) return invalid("exact_solve: null argument");
  // PlacementProblem::validate (placement.cpp:13-26), then the size limit (placement.cpp:175-179)
  if (m < 1) return invalid("PlacementProblem: no experts");
  if (g < 1) return invalid("PlacementProblem: g must be >= 1");
  if (m % g != 0) return invalid("PlacementProblem: experts must be divisible by g");
  if (!(alpha > 0.0) || !(beta > 0.0)) return invalid("PlacementProblem: alpha and beta must be > 0");
  if (m > kMaxExperts || g > kMaxGpus)
    return invalid("exact_solve: instance too large (max " + std::to_string(kMaxExperts) + " experts on " +
                   std::to_string(kMaxGpus) + " GPUs); use greedy_place");
  if (rows < 1 || rows > kMaxRows) {
    set_error("exact_solve: A must have 1.." + std::to_string(kMaxRows) + " rows");
    return GIMBAL_NOT_SUPPORTED;
  }
  if (!exact_integer(A, (size_t)rows * m) || !exact_integer(W, (size_t)m * m)) {
    set_error("exact_solve: A and W must be non-negative integer-valued doubles below 2^40");
    return GIMBAL_NOT_SUPPORTED;
  }
  ExactParams prm;
  prm.rows = rows;
  prm.m = m;
  prm.g = g;
  prm.cap = m / g;
  prm.depth = std::max(0, m - kSuffix);
  prm.alpha = alpha;
  prm.beta = beta;
  std::vector<uint32_t> pre;
  list_prefixes(prm.depth, g, prm.cap, pre);
  prm.n_prefix = (int)pre.size();

  DevBuf t;
  double* dA = t.alloc<double>((size_t)rows * m);
  double* dW = t.alloc<double>((size_t)m * m);
  uint32_t* dPre = t.alloc<uint32_t>(pre.size());
  double* dObj = t.alloc<double>(pre.size());
  uint32_t* dAs = t.alloc<uint32_t>(pre.size());
  uint32_t* dOut = t.alloc<uint32_t>(2);
  if (!dA || !dW || !dPre || !dObj || !dAs || !dOut) {
    set_error("exact_solve: device allocation failed");
    return GIMBAL_CUDA_ERROR;
  }
  GIMBAL_CUDA_TRY(cudaMemcpy(dA, A, (size_t)rows * m * 8, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(cudaMemcpy(dW, W, (size_t)m * m * 8, cudaMemcpyHostToDevice));
  GIMBAL_CUDA_TRY(cudaMemcpy(dPre, pre.data(), pre.size() * 4, cudaMemcpyHostToDevice));
  exact_enum_kernel<<<(prm.n_prefix + 127) / 128, 128>>>(prm, dA, dW, dPre, dObj, dAs);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  exact_reduce_kernel<<<1, 1024>>>(prm.n_prefix, dObj, dAs, dOut);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  uint32_t h[2];
  GIMBAL_CUDA_TRY(cudaMemcpy(h, dOut, sizeof(h), cudaMemcpyDeviceToHost));
  if (!h[1]) {
    set_error("exact_solve: no feasible placement");
    return GIMBAL_CUDA_ERROR;
  }
  for (int j = 0; j < m; ++j) assign_out[j] = (int32_t)((h[0] >> (2 * j)) & 3u);
  // the returned cost is eval_cost of the answer (placement.cpp:182-183)
  return gimbal_eval_cost_dense(rows, m, A, W, g, alpha, beta, assign_out, deviation, cut, objective);
}

}  // extern "C"
