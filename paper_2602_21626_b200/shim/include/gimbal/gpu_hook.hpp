// GpuMoeSubsystem: the serving simulator's expert-layer hook (the reference's MoeSubsystem,
// proj/src/sim.cpp:76-218, behind MoeHook, proj/include/gimbal/engine.hpp:56-68) with its
// per-iteration work on the GPU.
//
// Routing stays on the host (RoutingModel::route_token with the engine's Rng stream, so the token
// stream is the reference's, draw for draw).  Everything the reference then does per token runs
// as one CUDA graph per engine iteration (gimbal_online_iteration): the window statistics
// (add_token), the layer x GPU load histogram under the current placement, the cross-GPU
// transitions and the bottleneck excess, plus the per-GPU activation totals on the device.
// Relocation (maybe_relocate every tau forward steps) runs greedy_place on the device's window
// statistics.  The lifetime statistics are the closed windows folded together at each reset plus
// the open window (lifetime_stats()), instead of a second count of every token.
//
// A drop-in for MoeSubsystem in gimbal::run: same constructor arguments and the accessors run()
// reads for its MetricsReport.
#pragma once

#include <cstdint>
#include <vector>

#include "gimbal/engine.hpp"
#include "gimbal/moe.hpp"
#include "gimbal/placement.hpp"
#include "gimbal/rng.hpp"
#include "gimbal/sim.hpp"

struct gimbal_online_s;  // include/gimbal_gpu.h

namespace gimbal {

class GpuMoeSubsystem final : public MoeHook {
 public:
  GpuMoeSubsystem(const SimConfig& cfg, bool edr_enabled);
  ~GpuMoeSubsystem() override;
  GpuMoeSubsystem(const GpuMoeSubsystem&) = delete;
  GpuMoeSubsystem& operator=(const GpuMoeSubsystem&) = delete;

  double iteration_cost(std::int64_t n_tokens, double base_duration, const CostModel& cost) override;
  void on_forward_step(double now) override;
  double take_pending_stall(int engine_id) override;

  std::vector<std::int64_t> gpu_activation_totals() const;
  std::int64_t migrations() const { return migrations_; }
  std::int64_t global_step() const { return global_step_; }
  const std::vector<RelocationEvent>& relocations() const { return relocations_; }
  const placement::AffinitySet& affinity() const { return affinity_; }
  const std::vector<std::vector<int>>& snapshots() const { return snapshots_; }
  const moe::RoutingStats& lifetime_stats() const;

  // Last iteration's raw outputs (the excess sum over layers and the transition count).
  double last_excess_sum() const { return last_excess_; }
  std::int64_t last_crossings() const { return last_crossings_; }

 private:
  void upload_placement();

  moe::MoeTopology topo_;
  moe::RoutingModel model_;
  Rng rng_;
  moe::RoutingStats window_;     // counted on the device by the online hook
  moe::RoutingStats closed_;     // windows closed by relocations, folded together
  mutable moe::RoutingStats lifetime_view_;
  PlacementConfig pcfg_;
  bool edr_ = false;
  bool record_placements_ = false;
  placement::AffinitySet affinity_;
  placement::Placement placement_;
  std::vector<double> pending_stall_;
  std::vector<int> batch_;  // routed ids of one iteration, [n][L][k]
  gimbal_online_s* online_ = nullptr;
  std::int64_t global_step_ = 0;
  std::int64_t migrations_ = 0;
  std::vector<RelocationEvent> relocations_;
  std::vector<std::vector<int>> snapshots_;
  double last_excess_ = 0.0;
  std::int64_t last_crossings_ = 0;
};

}  // namespace gimbal
