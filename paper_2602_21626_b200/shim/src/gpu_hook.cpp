// GpuMoeSubsystem (gimbal/gpu_hook.hpp): MoeHook semantics of the reference's MoeSubsystem
// (proj/src/sim.cpp:76-218) with the per-iteration work on the GPU through include/gimbal_gpu.h.
#include "gimbal/gpu_hook.hpp"

#include <optional>
#include <span>
#include <stdexcept>

#include "gimbal_gpu.h"
#include "status.hpp"

namespace gimbal {

using gpu_shim::check;

namespace {

// Adds `from`'s counts into `to` on the device (both handles on the same device).
void fold(moe::RoutingStats& to, moe::RoutingStats& from) {
  gimbal_stats_s* src = from.gpu_handle();
  check(gimbal_stats_sync(src), "fold");
  std::uint64_t *E = nullptr, *A = nullptr;
  void* stream = nullptr;
  check(gimbal_stats_device_buffers(src, &E, &A, &stream), "fold");
  check(gimbal_stats_merge(to.gpu_handle(), E ? E : A, from.tokens(), GIMBAL_MEM_DEVICE), "fold");
}

}  // namespace

GpuMoeSubsystem::GpuMoeSubsystem(const SimConfig& cfg, bool edr_enabled)
    : topo_(cfg.topo),
      model_(cfg.topo, cfg.routing, mix_seed(cfg.seed, 0x70ce)),  // the reference's streams (sim.cpp:80-81)
      rng_(mix_seed(cfg.seed, 0x707e)),
      window_(cfg.topo),
      closed_(cfg.topo),
      lifetime_view_(cfg.topo),
      pcfg_(cfg.placement),
      edr_(edr_enabled),
      record_placements_(cfg.record_placements),
      pending_stall_(static_cast<std::size_t>(cfg.n_engines), 0.0) {
  if (edr_) {
    // offline calibration (sim.cpp:91-106): route offline_tokens on their own stream, take the
    // strong-pair set from their statistics and lay out the first placement around it
    Rng offline_rng(mix_seed(cfg.seed, 0x0ff1));
    const std::size_t per = static_cast<std::size_t>(topo_.n_layers * topo_.top_k);
    std::vector<int> ids(static_cast<std::size_t>(pcfg_.offline_tokens) * per);
    for (std::int64_t t = 0; t < pcfg_.offline_tokens; ++t)
      model_.route_token(std::nullopt, offline_rng, std::span<int>(ids.data() + t * per, per));
    moe::RoutingStats offline(topo_);
    if (pcfg_.offline_tokens > 0) offline.add_tokens(ids.data(), 4, pcfg_.offline_tokens, false);
    affinity_ = placement::build_affinity_set(offline.affinity(), topo_, pcfg_.affinity_threshold, pcfg_.top_e,
                                              topo_.total_experts() / topo_.n_gpus, pcfg_.anchor_gpu);
    placement_ = placement::greedy_place(offline.flat_activation(), affinity_, topo_.n_gpus);
    relocations_.push_back({0, 0.0, 0});
    if (record_placements_) snapshots_.push_back(placement_.assign);
  } else {
    affinity_.anchor_gpu = pcfg_.anchor_gpu;
    placement_ = placement::static_placement(topo_);
  }
  check(gimbal_online_create(window_.gpu_handle(), &online_), "GpuMoeSubsystem");
  upload_placement();
}

GpuMoeSubsystem::~GpuMoeSubsystem() {
  if (online_) gimbal_online_destroy(online_);
}

void GpuMoeSubsystem::upload_placement() {
  std::vector<std::int32_t> a(placement_.assign.begin(), placement_.assign.end());
  check(gimbal_online_set_placement(online_, a.data(), static_cast<std::int64_t>(a.size())), "placement");
}

double GpuMoeSubsystem::iteration_cost(std::int64_t n_tokens, double base_duration, const CostModel& cost) {
  if (n_tokens <= 0) return 0.0;
  const std::size_t per = static_cast<std::size_t>(topo_.n_layers * topo_.top_k);
  batch_.resize(static_cast<std::size_t>(n_tokens) * per);
  for (std::int64_t t = 0; t < n_tokens; ++t)  // the engine's routing stream, token by token
    model_.route_token(std::nullopt, rng_, std::span<int>(batch_.data() + t * per, per));
  check(gimbal_online_iteration(online_, batch_.data(), 4, n_tokens, &last_excess_, &last_crossings_), "iteration");
  // sim.cpp:132-146 on the device's excess sum and crossing count, in the reference's order
  double extra = 0.0;
  if (cost.moe_imbalance_slowdown > 0.0) {
    extra += base_duration * cost.moe_imbalance_slowdown * last_excess_ / static_cast<double>(topo_.n_layers);
  }
  extra += cost.comm_time_per_transition * static_cast<double>(last_crossings_);
  return extra;
}

void GpuMoeSubsystem::on_forward_step(double now) {
  ++global_step_;
  if (!edr_) return;
  // maybe_relocate is a no-op off the cadence (placement.cpp:305-307); the window's activation is
  // read back only when it can fire (tau < 1 still reaches it, for the reference's error)
  if (pcfg_.tau >= 1 && global_step_ % pcfg_.tau != 0) return;
  window_.gpu_handle();  // counts changed on the device since the last read
  auto reloc =
      placement::maybe_relocate(global_step_, pcfg_.tau, affinity_, window_.flat_activation(), topo_.n_gpus, placement_);
  if (!reloc) return;
  placement_ = std::move(reloc->placement);
  migrations_ += reloc->moved;
  relocations_.push_back({global_step_, now, reloc->moved});
  if (record_placements_) snapshots_.push_back(placement_.assign);
  fold(closed_, window_);
  window_.reset();
  upload_placement();
  if (pcfg_.migration_stall > 0.0 && reloc->moved > 0) {
    const double stall = pcfg_.migration_stall * static_cast<double>(reloc->moved);
    for (auto& s : pending_stall_) s += stall;
  }
}

double GpuMoeSubsystem::take_pending_stall(int engine_id) {
  double& s = pending_stall_.at(static_cast<std::size_t>(engine_id));
  const double out = s;
  s = 0.0;
  return out;
}

std::vector<std::int64_t> GpuMoeSubsystem::gpu_activation_totals() const {
  std::vector<std::int64_t> out(static_cast<std::size_t>(topo_.n_gpus));
  check(gimbal_online_gpu_totals(online_, out.data()), "gpu_activation_totals");
  return out;
}

const moe::RoutingStats& GpuMoeSubsystem::lifetime_stats() const {
  lifetime_view_ = closed_;
  fold(lifetime_view_, const_cast<moe::RoutingStats&>(window_));
  return lifetime_view_;
}

}  // namespace gimbal
