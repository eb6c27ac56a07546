// Simulator driver — TEST INFRASTRUCTURE ONLY.
//
// Runs the reference's own discrete-event simulator (proj/src/sim.cpp, gimbal::run) on fixed
// synthetic workloads and prints report_to_json (proj/src/report.cpp, byte-stable).  Linked
// twice: against the reference's moe.cpp/placement.cpp (oracle/_ref/sim_report_ref) and against
// this repo's GPU shim (oracle/_ref/sim_report_shim).  Identical output = the GPU expert layer
// is a drop-in for MoeHook/MoeSubsystem (sim.cpp:76-218): routing, per-iteration stats,
// crossings, bottleneck excess, calibration, relocation cadence and anchors all agree.
#include <cstdio>
#include <string>
#include <vector>

#include "gimbal/report.hpp"
#include "gimbal/rng.hpp"
#include "gimbal/sim.hpp"
#include "gimbal/workload.hpp"

using namespace gimbal;

static std::vector<Request> workload_for(int n, double rps, std::uint64_t seed) {
  std::vector<TraceRecord> records;
  Rng rng(seed);
  for (int i = 0; i < n; ++i) {
    TraceRecord rec;
    rec.prefill_tokens = 1 + rng.uniform_int(2000);
    rec.output_tokens = 1 + rng.uniform_int(80);
    if (i % 4 == 0) rec.user_id = "u" + std::to_string(rng.uniform_int(16));
    records.push_back(rec);
  }
  return workload::gen_arrivals(records, rps, seed + 7);
}

int main(int argc, char** argv) {
  const int scenario = argc > 1 ? std::atoi(argv[1]) : 0;
  SimConfig cfg;
  cfg.n_engines = 2;
  cfg.seed = 11 + static_cast<std::uint64_t>(scenario);
  cfg.record_placements = true;
  cfg.cost.moe_imbalance_slowdown = 0.3;     // expert-layer load feeds the iteration time
  cfg.cost.comm_time_per_transition = 1e-7;  // and so do cross-GPU transitions
  switch (scenario) {
    case 0:  // gimbal policy, small topology, frequent relocations
      cfg.policy = Policy::kGimbal;
      cfg.topo = moe::MoeTopology{4, 8, 2, 2};
      cfg.placement.tau = 40;
      cfg.placement.offline_tokens = 3000;
      break;
    case 1:  // EDR only, wider layer
      cfg.policy = Policy::kEdrOnly;
      cfg.topo = moe::MoeTopology{6, 16, 4, 4};
      cfg.placement.tau = 25;
      cfg.placement.top_e = 6;
      cfg.placement.migration_stall = 1e-4;
      cfg.placement.offline_tokens = 4000;
      break;
    default:  // static placement baseline through the same hook
      cfg.policy = Policy::kBaselineRrFcfs;
      cfg.topo = moe::MoeTopology{3, 8, 2, 4};
      break;
  }
  const auto reqs = workload_for(120, 30.0, 100 + static_cast<std::uint64_t>(scenario));
  const auto report = run(cfg, reqs);
  std::fputs(report_to_json(report).c_str(), stdout);
  std::fputc('\n', stdout);
  return 0;
}
