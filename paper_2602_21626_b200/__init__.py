"""B200-native (sm_100a) expert-statistics + placement hot path of Gimbal (arXiv 2602.21626).

Host mirror of the reference's ``gimbal::moe`` / ``gimbal::placement`` operator API
(/root/reference/proj/include/gimbal/{moe,placement}.hpp) over ``include/gimbal_gpu.h``.
All numeric work runs in ``lib/libgimbal_gpu.so``; there is no CPU fallback.
"""
from . import _native
from .moe import (AffinityTensor, MoeTopology, RoutedStream, RoutingParams, RoutingStats, comm_cost,
                  generate_trace, generator_tables, record_stats)
from .placement import (AffinitySet, Placement, PlacementCost, PlacementProblem, Relocation, build_affinity_set,
                        eval_cost, eval_costs, eval_excess, exact_solve, greedy_place, maybe_relocate, shuffled_candidates, static_placement)
from .pipeline import HotPath
from .hook import OnlineHook

__all__ = [
    "AffinityTensor", "MoeTopology", "RoutedStream", "RoutingParams", "RoutingStats", "comm_cost", "generate_trace",
    "generator_tables", "record_stats", "AffinitySet", "Placement", "PlacementCost", "PlacementProblem",
    "Relocation", "build_affinity_set", "eval_cost", "eval_costs", "eval_excess", "greedy_place", "maybe_relocate",
    "shuffled_candidates", "static_placement", "HotPath", "OnlineHook",
]
