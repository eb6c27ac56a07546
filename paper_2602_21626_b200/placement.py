"""Host mirror of the reference's ``gimbal::placement`` operator API over the sm_100a C ABI.

Reference: /root/reference/proj/include/gimbal/placement.hpp:14-85, proj/src/placement.cpp.
Two forms of every operator:

* the reference's general form (explicit ``PlacementProblem`` A / W, ``AffinityTensor``, dense
  activation) -> ``gimbal_*_dense`` entry points;
* the hot-path form over a device-resident ``RoutingStats`` (compact A / E, W never built) ->
  ``eval_costs`` / ``build_affinity_set(stats, ...)`` / ``greedy_place(stats, ...)``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .moe import AffinityTensor, MoeTopology, RoutingStats


@dataclass
class Placement:
    """placement::Placement (placement.hpp:14-17): expert id -> GPU id."""

    assign: List[int] = field(default_factory=list)


@dataclass
class PlacementProblem:
    """placement::PlacementProblem (placement.hpp:19-30)."""

    A: np.ndarray = None
    W: np.ndarray = None
    g: int = 2
    alpha: float = 1.0
    beta: float = 1.0

    def experts(self) -> int:
        return int(np.asarray(self.A).shape[1])


@dataclass
class PlacementCost:
    """placement::PlacementCost (placement.hpp:32-36)."""

    deviation: float = 0.0
    cut: float = 0.0
    objective: float = 0.0


@dataclass
class AffinitySet:
    """placement::AffinitySet (placement.hpp:38-42)."""

    experts: List[int] = field(default_factory=list)
    anchor_gpu: int = 0


@dataclass
class Relocation:
    placement: Placement
    moved: int = 0


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).astype(np.int32))


def eval_cost(problem: PlacementProblem, placement: Placement) -> PlacementCost:  # placement.cpp:58-85
    A = np.ascontiguousarray(np.atleast_2d(np.asarray(problem.A, np.float64)))
    W = np.ascontiguousarray(np.asarray(problem.W, np.float64))
    m = A.shape[1]
    if W.shape != (m, m):
        if m >= 1 and problem.g >= 1 and m % problem.g == 0:
            raise ValueError("PlacementProblem: W must be experts x experts")
    a = _i32(placement.assign)
    if a.size != m:
        if m >= 1 and problem.g >= 1 and m % problem.g == 0 and problem.alpha > 0 and problem.beta > 0:
            raise ValueError("placement: assignment size mismatch")
    D, c, o = C.c_double(), C.c_double(), C.c_double()
    N.check(N.lib().gimbal_eval_cost_dense(A.shape[0], m, A.ctypes.data, W.ctypes.data, problem.g, problem.alpha,
                                           problem.beta, a.ctypes.data if a.size == m else None, C.byref(D),
                                           C.byref(c), C.byref(o)), "eval_cost")
    return PlacementCost(D.value, c.value, o.value)


def exact_solve(problem: PlacementProblem):  # placement.cpp:87-184
    """placement::exact_solve: (Placement, PlacementCost) of the objective-minimal balanced placement
    (m <= 16 experts, g <= 4 GPUs; the lexicographically least among ties), every placement scored
    on the GPU.  A / W must be non-negative integer-valued (counts)."""
    A = np.ascontiguousarray(np.atleast_2d(np.asarray(problem.A, np.float64)))
    W = np.ascontiguousarray(np.asarray(problem.W, np.float64))
    m = A.shape[1]
    if W.shape != (m, m) and m >= 1 and problem.g >= 1 and m % problem.g == 0:
        raise ValueError("PlacementProblem: W must be experts x experts")
    a = np.zeros(max(m, 1), np.int32)
    D, c, o = C.c_double(), C.c_double(), C.c_double()
    N.check(N.lib().gimbal_exact_solve_dense(A.shape[0], m, A.ctypes.data, W.ctypes.data, problem.g, problem.alpha,
                                             problem.beta, a.ctypes.data, C.byref(D), C.byref(c), C.byref(o)),
            "exact_solve")
    return Placement([int(x) for x in a[:m]]), PlacementCost(D.value, c.value, o.value)


def eval_costs(stats: RoutingStats, candidates, alpha: float = 1.0, beta: float = 1.0, out=None):
    """Batch eval_cost of candidates [C][m] uint8 against the stats' flat A / W.

    ``candidates`` is a numpy array (host) or a CUDA tensor (device).  Returns (D, cut, objective,
    argmin) as numpy arrays, or — when ``out`` is a CUDA float64 tensor [3][C] — fills it and
    returns (out, argmin).
    """
    m = stats.topo.total_experts()
    if hasattr(candidates, "data_ptr"):
        cptr, cmem, n, keep = candidates.data_ptr(), (N.MEM_DEVICE if candidates.is_cuda else N.MEM_HOST), \
            candidates.shape[0], candidates
        if cmem == N.MEM_DEVICE:
            stats._after_torch(candidates)
    else:
        keep = np.ascontiguousarray(np.asarray(candidates, np.uint8))
        cptr, cmem, n = keep.ctypes.data, N.MEM_HOST, keep.shape[0]
    if n and int(np.prod(getattr(keep, "shape"))) != n * m:
        raise ValueError("placement: assignment size mismatch")
    am = C.c_int64(-1)
    if out is not None:
        base = out.data_ptr()
        N.check(N.lib().gimbal_eval_costs(stats.handle, C.c_void_p(cptr), n, cmem, alpha, beta, C.c_void_p(base),
                                          C.c_void_p(base + 8 * n), C.c_void_p(base + 16 * n), C.byref(am),
                                          N.MEM_DEVICE), "eval_costs")
        return out, am.value
    D, cut, obj = (np.zeros(n) for _ in range(3))
    N.check(N.lib().gimbal_eval_costs(stats.handle, C.c_void_p(cptr), n, cmem, alpha, beta, D.ctypes.data,
                                      cut.ctypes.data, obj.ctypes.data, C.byref(am), N.MEM_HOST), "eval_costs")
    return D, cut, obj, am.value


def eval_excess(stats: RoutingStats, candidates) -> np.ndarray:
    """Per-candidate bottleneck excess sum_l max(0, peak_l * g / (T * k) - 1) of the stats' A under
    each placement [C][m] uint8 (numpy or CUDA): the simulator's hotspot penalty (sim.cpp:132-144)
    over the counted trace."""
    m = stats.topo.total_experts()
    if hasattr(candidates, "data_ptr"):
        cptr, cmem, n, keep = candidates.data_ptr(), (N.MEM_DEVICE if candidates.is_cuda else N.MEM_HOST), \
            candidates.shape[0], candidates
        if cmem == N.MEM_DEVICE:
            stats._after_torch(candidates)
    else:
        keep = np.ascontiguousarray(np.asarray(candidates, np.uint8))
        cptr, cmem, n = keep.ctypes.data, N.MEM_HOST, keep.shape[0]
    if n and int(np.prod(getattr(keep, "shape"))) != n * m:
        raise ValueError("placement: assignment size mismatch")
    out = np.zeros(n)
    N.check(N.lib().gimbal_eval_excess(stats.handle, C.c_void_p(cptr), n, cmem, out.ctypes.data, N.MEM_HOST),
            "eval_excess")
    return out


def build_affinity_set(affinity, topo: MoeTopology, threshold: float, top_e: int, capacity: int,
                       anchor_gpu: int) -> AffinitySet:  # placement.cpp:186-238
    """``affinity`` is an AffinityTensor (reference form) or a RoutingStats (device E)."""
    cap_out = max(0, capacity) if top_e < 0 else min(max(0, capacity), 2 * max(top_e, 0))
    out = np.zeros(max(cap_out, topo.total_experts(), 1), np.int32)
    n = C.c_int32(0)
    if isinstance(affinity, RoutingStats):
        topo.validate()
        N.check(N.lib().gimbal_affinity_set(affinity.handle, float(threshold), int(top_e), int(capacity),
                                            int(anchor_gpu), out.ctypes.data, C.byref(n)), "build_affinity_set")
    else:
        E = np.ascontiguousarray(np.asarray(affinity.E, np.float64))
        nb = E.shape[0] if E.ndim == 3 else (len(affinity.E) if hasattr(affinity.E, "__len__") else 0)
        N.check(N.lib().gimbal_affinity_set_dense(C.byref(topo.c()), E.ctypes.data if E.size else None, nb,
                                                  float(threshold), int(top_e), int(capacity), int(anchor_gpu),
                                                  out.ctypes.data, C.byref(n)), "build_affinity_set")
    return AffinitySet(experts=[int(x) for x in out[: n.value]], anchor_gpu=anchor_gpu)


def greedy_place(activation, affinity: AffinitySet, g: int, out_u8_device=None) -> Placement:
    """placement.cpp:240-299.  ``activation`` is a dense [rows][m] matrix (reference form) or a
    RoutingStats (flat activation on the device).  ``out_u8_device`` optionally receives the
    result as uint8 (e.g. row 0 of a candidate batch)."""
    if isinstance(activation, RoutingStats):
        return Placement(assign=greedy_place_array(activation, affinity, g, out_u8_device).tolist())
    M = _i32(affinity.experts)
    A = np.ascontiguousarray(np.atleast_2d(np.asarray(activation, np.float64)))
    out = np.zeros(A.shape[1], np.int32)
    N.check(N.lib().gimbal_greedy_place_dense(A.shape[0], A.shape[1], A.ctypes.data,
                                              M.ctypes.data if M.size else None, M.size, affinity.anchor_gpu, g,
                                              out.ctypes.data), "greedy_place")
    return Placement(assign=[int(x) for x in out])


def greedy_place_array(stats: RoutingStats, affinity: AffinitySet, g: int, out_u8_device=None) -> np.ndarray:
    """greedy_place on device stats, returned as an int32 numpy array (no per-element Python
    objects: the streaming loop compares successive placements vectorised)."""
    if g != stats.topo.n_gpus:
        raise ValueError("greedy_place: g must equal the topology's n_gpus for device stats")
    M = _i32(affinity.experts)
    out = np.zeros(stats.topo.total_experts(), np.int32)
    N.check(N.lib().gimbal_greedy_place(stats.handle, M.ctypes.data if M.size else None, M.size,
                                        affinity.anchor_gpu, out.ctypes.data, N.MEM_HOST,
                                        C.c_void_p(out_u8_device.data_ptr()) if out_u8_device is not None
                                        else None), "greedy_place")
    return out


def maybe_relocate(step_count: int, tau: int, affinity: AffinitySet, recent_activation, g: int,
                   previous: Placement) -> Optional[Relocation]:  # placement.cpp:301-318
    if tau < 1:
        raise ValueError("maybe_relocate: tau must be >= 1")
    if step_count % tau != 0:
        return None
    pl = greedy_place(recent_activation, affinity, g)
    m = len(pl.assign)
    if len(previous.assign) == m:
        moved = int(sum(1 for a, b in zip(previous.assign, pl.assign) if a != b))
    else:
        moved = m
    return Relocation(placement=pl, moved=moved)


def static_placement(topo: MoeTopology) -> Placement:  # placement.cpp:320-331
    out = np.zeros(topo.total_experts(), np.int32)
    N.check(N.lib().gimbal_static_placement(C.byref(topo.c()), out.ctypes.data), "static_placement")
    return Placement(assign=[int(x) for x in out])


def shuffled_candidates(m: int, g: int, seed: int, n: int) -> np.ndarray:
    """Balanced random placements by the reference recipe (acceptance_main.cpp:344-351):
    assign[e] = e % g, then Rng(seed + c).shuffle, for c in [0, n).  [n][m] uint8."""
    out = np.zeros((n, m), np.uint8)
    N.check(N.lib().gimbal_shuffled_candidates(m, g, seed, n, out.ctypes.data), "shuffled_candidates")
    return out
