// C entry points over the REFERENCE's own hot-path sources — ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/Makefile together with /root/reference/proj/src/moe.cpp and
// /root/reference/proj/src/placement.cpp (compiled unchanged, Eigen supplied by
// oracle/eigen_subset) into oracle/_ref/libgimbal_ref.so.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs load it.  Matrices cross this boundary
// row-major (A[l][e], E[l][j][k], W[j][k]); the reference stores them column-major in Eigen.
//
// Every function returns 0 on success, -1 on a reference exception (message via
// ref_last_error(), mirroring the std::invalid_argument text).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "gimbal/moe.hpp"
#include "gimbal/placement.hpp"
#include "gimbal/rng.hpp"

using namespace gimbal;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

moe::MoeTopology topo_of(int L, int ne, int k, int g) { return moe::MoeTopology{L, ne, k, g}; }

Eigen::MatrixXd from_rowmajor(const double* p, int rows, int cols) {
  Eigen::MatrixXd m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m(i, j) = p[static_cast<std::size_t>(i) * cols + j];
  return m;
}

void to_rowmajor(const Eigen::MatrixXd& m, double* out) {
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) out[i * m.cols() + j] = m(i, j);
}

template <typename Id>
void add_tokens(moe::RoutingStats& stats, const Id* ids, std::int64_t n, int stride) {
  std::vector<int> tok(static_cast<std::size_t>(stride));
  for (std::int64_t t = 0; t < n; ++t) {
    const Id* row = ids + t * stride;
    for (int i = 0; i < stride; ++i) tok[static_cast<std::size_t>(i)] = static_cast<int>(row[i]);
    stats.add_token(std::span<const int>(tok));
  }
}

void read_stats(const moe::RoutingStats& stats, const moe::MoeTopology& topo, double* A, double* E,
                double* W) {
  if (A) to_rowmajor(stats.activation(), A);
  if (E || W) {
    auto aff = stats.affinity();
    const std::size_t blk = static_cast<std::size_t>(topo.n_experts) * topo.n_experts;
    if (E)
      for (std::size_t l = 0; l < aff.E.size(); ++l) to_rowmajor(aff.E[l], E + l * blk);
    if (W) to_rowmajor(aff.W, W);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// record_stats (moe.cpp:233-239) over a token-major [T][L][k] trace; id_bytes 1 (uint8) or 4 (int32).
int ref_record_stats(int L, int ne, int k, int g, const void* ids, int id_bytes, std::int64_t T,
                     double* A, double* E, double* W, std::int64_t* tokens) {
  return guarded([&] {
    auto topo = topo_of(L, ne, k, g);
    moe::RoutingStats stats(topo);
    if (id_bytes == 1) add_tokens(stats, static_cast<const std::uint8_t*>(ids), T, L * k);
    else add_tokens(stats, static_cast<const std::int32_t*>(ids), T, L * k);
    read_stats(stats, topo, A, E, W);
    if (tokens) *tokens = stats.tokens();
  });
}

// flat_activation (moe.cpp:207-215) -> [L][m]; flat_pair_weights (moe.cpp:217-231) -> [m][m].
int ref_flat_forms(int L, int ne, int k, int g, const void* ids, int id_bytes, std::int64_t T,
                   double* flatA, double* flatW) {
  return guarded([&] {
    auto topo = topo_of(L, ne, k, g);
    moe::RoutingStats stats(topo);
    if (id_bytes == 1) add_tokens(stats, static_cast<const std::uint8_t*>(ids), T, L * k);
    else add_tokens(stats, static_cast<const std::int32_t*>(ids), T, L * k);
    if (flatA) to_rowmajor(stats.flat_activation(), flatA);
    if (flatW) to_rowmajor(stats.flat_pair_weights(), flatW);
  });
}

// comm_cost (moe.cpp:241-267).
int ref_comm_cost(int L, int ne, int k, int g, const void* ids, int id_bytes, std::int64_t T,
                  const std::int32_t* assign, int n_assign, std::int64_t* out) {
  return guarded([&] {
    moe::RoutedStream s;
    s.topo = topo_of(L, ne, k, g);
    s.n_tokens = T;
    s.choices.resize(static_cast<std::size_t>(T) * L * k);
    for (std::size_t i = 0; i < s.choices.size(); ++i)
      s.choices[i] = id_bytes == 1 ? static_cast<const std::uint8_t*>(ids)[i]
                                   : static_cast<const std::int32_t*>(ids)[i];
    std::vector<int> a(assign, assign + n_assign);
    *out = moe::comm_cost(s, std::span<const int>(a));
  });
}

// eval_cost (placement.cpp:58-85) on a general PlacementProblem: A [rows][m], W [m][m].
int ref_eval_cost(int rows, int m, const double* A, const double* W, int g, double alpha,
                  double beta, const std::int32_t* assign, int n_assign, double* D, double* cut,
                  double* obj) {
  return guarded([&] {
    placement::PlacementProblem p;
    p.A = from_rowmajor(A, rows, m);
    p.W = from_rowmajor(W, m, m);
    p.g = g;
    p.alpha = alpha;
    p.beta = beta;
    placement::Placement pl{std::vector<int>(assign, assign + n_assign)};
    auto c = placement::eval_cost(p, pl);
    *D = c.deviation;
    *cut = c.cut;
    *obj = c.objective;
  });
}

// exact_solve (placement.cpp:87-184): the reference's branch and bound, assignment + its cost.
int ref_exact_solve(int rows, int m, const double* A, const double* W, int g, double alpha, double beta,
                    std::int32_t* assign, double* D, double* cut, double* obj) {
  return guarded([&] {
    placement::PlacementProblem p;
    p.A = from_rowmajor(A, rows, m);
    p.W = from_rowmajor(W, m, m);
    p.g = g;
    p.alpha = alpha;
    p.beta = beta;
    auto [pl, c] = placement::exact_solve(p);
    for (int j = 0; j < m; ++j) assign[j] = pl.assign[static_cast<std::size_t>(j)];
    *D = c.deviation;
    *cut = c.cut;
    *obj = c.objective;
  });
}

// build_affinity_set (placement.cpp:186-238) from E [(L-1)][ne][ne].
int ref_build_affinity_set(int L, int ne, int k, int g, const double* E, int n_blocks,
                           double threshold, int top_e, int capacity, int anchor,
                           std::int32_t* out, int* n_out) {
  return guarded([&] {
    auto topo = topo_of(L, ne, k, g);
    moe::AffinityTensor aff;
    const std::size_t blk = static_cast<std::size_t>(ne) * ne;
    for (int l = 0; l < n_blocks; ++l) aff.E.push_back(from_rowmajor(E + l * blk, ne, ne));
    aff.W = Eigen::MatrixXd::Zero(ne, ne);
    for (const auto& e : aff.E) aff.W += e;
    auto set = placement::build_affinity_set(aff, topo, threshold, top_e, capacity, anchor);
    *n_out = static_cast<int>(set.experts.size());
    for (std::size_t i = 0; i < set.experts.size(); ++i) out[i] = set.experts[i];
  });
}

// greedy_place (placement.cpp:240-299) on a general activation [rows][m].
int ref_greedy_place(int rows, int m, const double* act, const std::int32_t* M, int nM, int anchor,
                     int g, std::int32_t* out) {
  return guarded([&] {
    placement::AffinitySet set{std::vector<int>(M, M + nM), anchor};
    auto pl = placement::greedy_place(from_rowmajor(act, rows, m), set, g);
    for (std::size_t i = 0; i < pl.assign.size(); ++i) out[i] = pl.assign[i];
  });
}

// maybe_relocate (placement.cpp:301-318). *fired = 0 off-cadence.
int ref_maybe_relocate(std::int64_t step, std::int64_t tau, const std::int32_t* M, int nM, int anchor,
                       int rows, int m, const double* act, int g, const std::int32_t* prev,
                       int n_prev, std::int32_t* out, std::int64_t* moved, int* fired) {
  return guarded([&] {
    placement::AffinitySet set{std::vector<int>(M, M + nM), anchor};
    placement::Placement previous{std::vector<int>(prev, prev + n_prev)};
    auto r = placement::maybe_relocate(step, tau, set, from_rowmajor(act, rows, m), g, previous);
    *fired = r.has_value() ? 1 : 0;
    if (r) {
      for (std::size_t i = 0; i < r->placement.assign.size(); ++i) out[i] = r->placement.assign[i];
      *moved = r->moved;
    }
  });
}

// static_placement (placement.cpp:320-331).
int ref_static_placement(int L, int ne, int k, int g, std::int32_t* out) {
  return guarded([&] {
    auto pl = placement::static_placement(topo_of(L, ne, k, g));
    for (std::size_t i = 0; i < pl.assign.size(); ++i) out[i] = pl.assign[i];
  });
}

// RoutingModel (moe.cpp:43-153) + route_token with prev = nullopt, as every reference caller
// does (test_moe.cpp:13-23, sim.cpp:96,117).  Writes T*L*k int32 ids.
int ref_route_tokens(int L, int ne, int k, int g, double zipf_s, double lambda, double peak,
                     std::uint64_t model_seed, std::uint64_t rng_seed, std::int64_t T,
                     std::int32_t* out) {
  return guarded([&] {
    moe::RoutingParams params{zipf_s, lambda, peak};
    moe::RoutingModel model(topo_of(L, ne, k, g), params, model_seed);
    Rng rng(rng_seed);
    const std::size_t stride = static_cast<std::size_t>(L) * k;
    std::vector<int> tok(stride);
    for (std::int64_t t = 0; t < T; ++t) {
      model.route_token(std::nullopt, rng, std::span<int>(tok));
      for (std::size_t i = 0; i < stride; ++i) out[static_cast<std::size_t>(t) * stride + i] = tok[i];
    }
  });
}

// RoutingModel base weights [L][ne] and kernel [ne][ne] (moe.cpp:61-80).
int ref_model_weights(int L, int ne, int k, int g, double zipf_s, double lambda, double peak,
                      std::uint64_t model_seed, double* base, double* kernel) {
  return guarded([&] {
    moe::RoutingParams params{zipf_s, lambda, peak};
    moe::RoutingModel model(topo_of(L, ne, k, g), params, model_seed);
    if (base) to_rowmajor(model.base_weights(), base);
    if (kernel) to_rowmajor(model.affinity_kernel(), kernel);
  });
}

// The reference CPU pipeline the bench times: add_token over a uint8 trace
// (sharded over n_threads RoutingStats), then affinity(), flat_activation(),
// flat_pair_weights(), build_affinity_set, greedy_place and eval_cost per candidate
// ([C][m] uint8 GPU ids).  Returns per-stage wall seconds in t[0..3]
// (add_token, flat forms + affinity set + greedy, eval, total) and the argmin candidate.
int ref_pipeline(int L, int ne, int k, int g, const std::uint8_t* ids, std::int64_t T,
                 int n_threads, const std::uint8_t* cands, int C, double threshold, int top_e,
                 int anchor, double alpha, double beta, double* objectives, std::int64_t* argmin,
                 std::int32_t* greedy_out, double* t) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double>(b - a).count();
    };
    auto topo = topo_of(L, ne, k, g);
    const int stride = L * k;
    if (n_threads < 1) n_threads = 1;
    // one RoutingStats per worker thread, constructed (and zero-filled) before the clock starts:
    // the reference builds one per pass, the other n_threads - 1 exist only because of the
    // sharding, so their fixed cost is not part of the per-token rate
    std::vector<moe::RoutingStats> shards(static_cast<std::size_t>(n_threads),
                                          moe::RoutingStats(topo));
    auto t0 = clk::now();
    {
      std::vector<std::thread> pool;
      for (int w = 0; w < n_threads; ++w) {
        pool.emplace_back([&, w] {
          const std::int64_t lo = T * w / n_threads, hi = T * (w + 1) / n_threads;
          add_tokens(shards[static_cast<std::size_t>(w)], ids + lo * stride, hi - lo, stride);
        });
      }
      for (auto& th : pool) th.join();
    }
    auto t1 = clk::now();
    // The public API has no way to merge RoutingStats, so the placement stages run once on the
    // first shard (their cost does not depend on the token count; with n_threads == 1 the
    // outputs are the reference's exact answers for the whole trace).
    auto aff = shards[0].affinity();
    Eigen::MatrixXd flatA = shards[0].flat_activation();
    Eigen::MatrixXd flatW = shards[0].flat_pair_weights();
    auto set = placement::build_affinity_set(aff, topo, threshold, top_e,
                                             topo.total_experts() / topo.n_gpus, anchor);
    auto greedy = placement::greedy_place(flatA, set, g);
    if (greedy_out)
      for (std::size_t i = 0; i < greedy.assign.size(); ++i) greedy_out[i] = greedy.assign[i];
    auto t2 = clk::now();
    placement::PlacementProblem p;
    p.A = std::move(flatA);
    p.W = std::move(flatW);
    p.g = g;
    p.alpha = alpha;
    p.beta = beta;
    const int m = topo.total_experts();
    // eval_cost per candidate (placement.cpp:58-85) is a pure function of (problem, placement):
    // candidates are scored by n_threads workers, each with its own Placement
    std::vector<double> obj(static_cast<std::size_t>(C > 0 ? C : 1));
    {
      std::vector<std::thread> pool;
      for (int w = 0; w < n_threads; ++w) {
        pool.emplace_back([&, w] {
          placement::Placement pl;
          for (int c = w; c < C; c += n_threads) {
            pl.assign.assign(cands + static_cast<std::size_t>(c) * m, cands + static_cast<std::size_t>(c + 1) * m);
            obj[static_cast<std::size_t>(c)] = placement::eval_cost(p, pl).objective;
          }
        });
      }
      for (auto& th : pool) th.join();
    }
    double best = 0.0;
    std::int64_t best_i = -1;
    for (int c = 0; c < C; ++c) {
      if (objectives) objectives[c] = obj[static_cast<std::size_t>(c)];
      if (best_i < 0 || obj[static_cast<std::size_t>(c)] < best) {
        best = obj[static_cast<std::size_t>(c)];
        best_i = c;
      }
    }
    auto t3 = clk::now();
    *argmin = best_i;
    t[0] = secs(t0, t1);
    t[1] = secs(t1, t2);
    t[2] = secs(t2, t3);
    t[3] = secs(t0, t3);
  });
}

// Rng helpers (rng.hpp:11-74) for fixture generation.
std::uint64_t ref_mix_seed(std::uint64_t seed, std::uint64_t stream) { return mix_seed(seed, stream); }

// The reference's balanced random candidate recipe (acceptance_main.cpp:344-351):
// assign[e] = e % g, then Rng(seed).shuffle.
void ref_shuffled_balanced(int m, int g, std::uint64_t seed, std::int32_t* out) {
  std::vector<int> a(static_cast<std::size_t>(m));
  for (int e = 0; e < m; ++e) a[static_cast<std::size_t>(e)] = e % g;
  Rng r(seed);
  r.shuffle(std::span<int>(a));
  for (int e = 0; e < m; ++e) out[e] = a[static_cast<std::size_t>(e)];
}

}  // extern "C"

// ---- MoeSubsystem::iteration_cost's per-token work (sim.cpp:113-147, token_crossings
// sim.cpp:183-198) restated over the reference's own RoutingStats: the oracle (and the host
// timing baseline) for the GPU hook gimbal_online_iteration.  Routing is not part of it (the
// caller passes the routed ids, as the GPU hook receives them).
namespace {
struct RefHook {
  moe::MoeTopology topo;
  moe::RoutingStats lifetime, window;
  std::vector<int> assign;
  Eigen::MatrixXd layer_gpu;
  std::vector<std::int64_t> totals;
  RefHook(const moe::MoeTopology& t)
      : topo(t), lifetime(t), window(t), layer_gpu(Eigen::MatrixXd::Zero(t.n_layers, t.n_gpus)),
        totals(static_cast<std::size_t>(t.n_gpus), 0) {}
};
}  // namespace

extern "C" {

void* ref_hook_create(int L, int ne, int k, int g, const std::int32_t* assign) {
  auto* h = new RefHook(topo_of(L, ne, k, g));
  h->assign.assign(assign, assign + static_cast<std::size_t>(L) * ne);
  return h;
}

void ref_hook_destroy(void* p) { delete static_cast<RefHook*>(p); }

void ref_hook_set_placement(void* p, const std::int32_t* assign) {
  auto* h = static_cast<RefHook*>(p);
  h->assign.assign(assign, assign + h->assign.size());
}

void ref_hook_reset_window(void* p) { static_cast<RefHook*>(p)->window.reset(); }

int ref_hook_iteration(void* p, const std::int32_t* ids, std::int64_t n, double* excess_sum, std::int64_t* crossings) {
  auto* h = static_cast<RefHook*>(p);
  return guarded([&] {
    const auto& topo = h->topo;
    const int per = topo.n_layers * topo.top_k;
    h->layer_gpu.setZero();
    std::int64_t cross = 0;
    std::vector<int> tok(static_cast<std::size_t>(per));
    for (std::int64_t t = 0; t < n; ++t) {
      for (int i = 0; i < per; ++i) tok[static_cast<std::size_t>(i)] = ids[t * per + i];
      h->lifetime.add_token(std::span<const int>(tok));
      h->window.add_token(std::span<const int>(tok));
      for (int l = 0; l < topo.n_layers; ++l)
        for (int a = 0; a < topo.top_k; ++a) {
          const int gpu = h->assign[static_cast<std::size_t>(topo.flat_id(l, tok[static_cast<std::size_t>(l * topo.top_k + a)]))];
          h->layer_gpu(l, gpu) += 1.0;
          h->totals[static_cast<std::size_t>(gpu)] += 1;
        }
      for (int l = 0; l + 1 < topo.n_layers; ++l)
        for (int a = 0; a < topo.top_k; ++a) {
          const int ga = h->assign[static_cast<std::size_t>(topo.flat_id(l, tok[static_cast<std::size_t>(l * topo.top_k + a)]))];
          for (int b = 0; b < topo.top_k; ++b)
            if (ga != h->assign[static_cast<std::size_t>(
                          topo.flat_id(l + 1, tok[static_cast<std::size_t>((l + 1) * topo.top_k + b)]))])
              ++cross;
        }
    }
    const double per_layer = static_cast<double>(n * topo.top_k);
    double s = 0.0;
    for (int l = 0; l < topo.n_layers; ++l) {
      const double peak = h->layer_gpu.row(l).maxCoeff();
      s += std::max(0.0, peak * topo.n_gpus / per_layer - 1.0);
    }
    *excess_sum = s;
    *crossings = cross;
  });
}

// window A [L][ne], window E [(L-1)][ne][ne] (row-major doubles, either may be NULL), GPU totals [g]
int ref_hook_stats(void* p, double* A, double* E, std::int64_t* totals) {
  auto* h = static_cast<RefHook*>(p);
  return guarded([&] {
    if (A) to_rowmajor(h->window.activation(), A);
    if (E) {
      const auto aff = h->window.affinity();
      const std::size_t blk = static_cast<std::size_t>(h->topo.n_experts) * h->topo.n_experts;
      for (std::size_t l = 0; l < aff.E.size(); ++l) to_rowmajor(aff.E[l], E + l * blk);
    }
    if (totals)
      for (std::size_t i = 0; i < h->totals.size(); ++i) totals[i] = h->totals[i];
  });
}

}  // extern "C"
