// gimbal::placement over the B200 C ABI (include/gimbal_gpu.h).  Replaces the reference's
// proj/src/placement.cpp: eval_cost, build_affinity_set and greedy_place execute on the GPU
// (placement.cpp:58-85, 186-299); validation keeps the reference's order and messages.
// exact_solve is the reference's m <= 16 correctness oracle and stays a host search here.
#include <algorithm>
#include <charconv>
#include <fstream>
#include <limits>
#include <stdexcept>

#include "gimbal/placement.hpp"
#include "status.hpp"

namespace gimbal::placement {

using gpu_shim::check;

namespace {

std::vector<double> rowmajor(const Eigen::MatrixXd& m) {
  std::vector<double> v(static_cast<std::size_t>(m.rows() * m.cols()));
  for (Eigen::Index r = 0; r < m.rows(); ++r)
    for (Eigen::Index c = 0; c < m.cols(); ++c) v[static_cast<std::size_t>(r * m.cols() + c)] = m(r, c);
  return v;
}

}  // namespace

void PlacementProblem::validate() const {  // placement.cpp:13-26
  const int m = experts();
  if (m < 1) throw std::invalid_argument("PlacementProblem: no experts");
  if (g < 1) throw std::invalid_argument("PlacementProblem: g must be >= 1");
  if (m % g != 0) throw std::invalid_argument("PlacementProblem: experts must be divisible by g");
  if (W.rows() != m || W.cols() != m) throw std::invalid_argument("PlacementProblem: W must be experts x experts");
  if (!(alpha > 0.0) || !(beta > 0.0)) throw std::invalid_argument("PlacementProblem: alpha and beta must be > 0");
}

PlacementCost eval_cost(const PlacementProblem& problem, const Placement& placement) {
  problem.validate();
  const int m = problem.experts();
  if (static_cast<int>(placement.assign.size()) != m) throw std::invalid_argument("placement: assignment size mismatch");
  const auto A = rowmajor(problem.A);
  const auto W = rowmajor(problem.W);
  std::vector<std::int32_t> a(placement.assign.begin(), placement.assign.end());
  PlacementCost cost;
  check(gimbal_eval_cost_dense(static_cast<std::int32_t>(problem.A.rows()), m, A.data(), W.data(), problem.g,
                               problem.alpha, problem.beta, a.data(), &cost.deviation, &cost.cut, &cost.objective),
        "eval_cost");
  return cost;
}

// Every balanced placement scored on the GPU (gimbal_exact_solve_dense, csrc/exact.cu): the
// objective-minimal one, lexicographically least among ties -- what placement.cpp:87-184's branch
// and bound returns -- and its eval_cost.
std::pair<Placement, PlacementCost> exact_solve(const PlacementProblem& problem) {
  problem.validate();
  const int m = problem.experts();
  const auto A = rowmajor(problem.A);
  const auto W = rowmajor(problem.W);
  std::vector<std::int32_t> a(static_cast<std::size_t>(std::max(m, 1)));
  PlacementCost cost;
  check(gimbal_exact_solve_dense(static_cast<std::int32_t>(problem.A.rows()), m, A.data(), W.data(), problem.g,
                                 problem.alpha, problem.beta, a.data(), &cost.deviation, &cost.cut, &cost.objective),
        "exact_solve");
  Placement pl{std::vector<int>(a.begin(), a.begin() + m)};
  return {pl, cost};
}

AffinitySet build_affinity_set(const moe::AffinityTensor& affinity, const moe::MoeTopology& topo, double threshold,
                               int top_e, int capacity, int anchor_gpu) {
  topo.validate();
  if (anchor_gpu < 0 || anchor_gpu >= topo.n_gpus)
    throw std::invalid_argument("build_affinity_set: anchor_gpu out of range");
  if (static_cast<int>(affinity.E.size()) != std::max(0, topo.n_layers - 1))
    throw std::invalid_argument("build_affinity_set: tensor depth mismatch");
  const int n = topo.n_experts;
  std::vector<double> E;
  E.reserve(affinity.E.size() * static_cast<std::size_t>(n) * n);
  for (const auto& b : affinity.E) {
    if (b.rows() != n || b.cols() != n) throw std::invalid_argument("build_affinity_set: block shape mismatch");
    const auto rm = rowmajor(b);
    E.insert(E.end(), rm.begin(), rm.end());
  }
  const gimbal_topology t{topo.n_layers, topo.n_experts, topo.top_k, topo.n_gpus};
  std::vector<std::int32_t> out(static_cast<std::size_t>(std::max(1, topo.total_experts())));
  std::int32_t n_out = 0;
  check(gimbal_affinity_set_dense(&t, E.empty() ? nullptr : E.data(), static_cast<std::int32_t>(affinity.E.size()),
                                  threshold, top_e, capacity, anchor_gpu, out.data(), &n_out),
        "build_affinity_set");
  return AffinitySet{std::vector<int>(out.begin(), out.begin() + n_out), anchor_gpu};
}

Placement greedy_place(const Eigen::MatrixXd& activation, const AffinitySet& affinity, int g) {
  const int m = static_cast<int>(activation.cols());
  const auto A = rowmajor(activation);
  std::vector<std::int32_t> M(affinity.experts.begin(), affinity.experts.end());
  std::vector<std::int32_t> out(static_cast<std::size_t>(std::max(m, 1)));
  check(gimbal_greedy_place_dense(static_cast<std::int32_t>(activation.rows()), m, A.data(),
                                  M.empty() ? nullptr : M.data(), static_cast<std::int32_t>(M.size()),
                                  affinity.anchor_gpu, g, out.data()),
        "greedy_place");
  return Placement{std::vector<int>(out.begin(), out.begin() + m)};
}

std::optional<Relocation> maybe_relocate(std::int64_t step_count, std::int64_t tau, const AffinitySet& affinity,
                                         const Eigen::MatrixXd& recent_activation, int g, const Placement& previous) {
  if (tau < 1) throw std::invalid_argument("maybe_relocate: tau must be >= 1");
  if (step_count % tau != 0) return std::nullopt;  // placement.cpp:305-306 cadence
  Relocation r;
  r.placement = greedy_place(recent_activation, affinity, g);
  const std::size_t m = r.placement.assign.size();
  if (previous.assign.size() == m) {
    for (std::size_t e = 0; e < m; ++e) r.moved += previous.assign[e] != r.placement.assign[e];
  } else {
    r.moved = static_cast<std::int64_t>(m);
  }
  return r;
}

Placement static_placement(const moe::MoeTopology& topo) {
  topo.validate();
  const gimbal_topology t{topo.n_layers, topo.n_experts, topo.top_k, topo.n_gpus};
  std::vector<std::int32_t> out(static_cast<std::size_t>(topo.total_experts()));
  check(gimbal_static_placement(&t, out.data()), "static_placement");
  return Placement{std::vector<int>(out.begin(), out.end())};
}

// Two-column text files "expert_id,gpu_id" (placement.cpp:333-372 format).
void write_placement(const std::string& path, const Placement& placement) {
  std::ofstream os(path);
  if (!os) throw std::runtime_error("cannot open placement file for writing: " + path);
  os << "expert_id,gpu_id\n";
  for (std::size_t e = 0; e < placement.assign.size(); ++e) os << e << ',' << placement.assign[e] << '\n';
  if (!os) throw std::runtime_error("failed writing placement file: " + path);
}

Placement read_placement(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw std::runtime_error("cannot open placement file: " + path);
  std::string line;
  if (!std::getline(is, line) || (line != "expert_id,gpu_id" && line != "expert_id,gpu_id\r"))
    throw std::runtime_error("placement header must be 'expert_id,gpu_id': " + path);
  Placement pl;
  std::size_t no = 1;
  while (std::getline(is, line)) {
    ++no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const auto comma = line.find(',');
    std::int64_t id = -1;
    int gpu = -1;
    const char* end = line.data() + line.size();
    const bool ok = comma != std::string::npos &&
                    std::from_chars(line.data(), line.data() + comma, id).ec == std::errc{} &&
                    std::from_chars(line.data() + comma + 1, end, gpu).ptr == end &&
                    id == static_cast<std::int64_t>(pl.assign.size());
    if (!ok) throw std::runtime_error("placement parse error at line " + std::to_string(no));
    pl.assign.push_back(gpu);
  }
  return pl;
}

}  // namespace gimbal::placement
