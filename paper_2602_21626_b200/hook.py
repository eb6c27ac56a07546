"""Host mirror of the online expert-layer hook (include/gimbal_gpu.h gimbal_online_*).

The reference's MoeSubsystem (proj/src/sim.cpp:76-218) implements MoeHook::iteration_cost by
looping over every routed token on the host (sim.cpp:113-147): statistics, the layer x GPU load
histogram under the current placement, cross-GPU transitions (sim.cpp:183-198) and the per-layer
bottleneck excess.  ``OnlineHook`` runs that loop as one CUDA graph per engine iteration, counting
into a window ``RoutingStats`` that stays on the device.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .moe import RoutingStats


class OnlineHook:
    """Per-iteration hook state over a window RoutingStats handle (same device and topology)."""

    def __init__(self, window: RoutingStats):
        self.window = window
        self.topo = window.topo
        h = C.c_void_p()
        N.check(N.lib().gimbal_online_create(window.handle, C.byref(h)), "OnlineHook")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().gimbal_online_destroy(h)
            except Exception:
                pass
            self._h = None

    def set_placement(self, assign) -> None:
        a = np.ascontiguousarray(np.asarray(assign, np.int32))
        N.check(N.lib().gimbal_online_set_placement(self._h, a.ctypes.data, a.size), "set_placement")

    def iteration(self, ids):
        """One engine iteration over n routed tokens ([n][L][k] ids, host uint8 or int32):
        returns (excess_sum, crossings) — sum over layers of max(0, peak * g / (n * k) - 1) and
        the cross-GPU transition count (sim.cpp:132-146 turns them into seconds)."""
        a = np.asarray(ids)
        a = np.ascontiguousarray(a if a.dtype == np.uint8 else a.astype(np.int32, copy=False))
        per = self.topo.n_layers * self.topo.top_k
        if a.size % per:
            raise ValueError("add_token: choice span size mismatch")
        ex, cr = C.c_double(), C.c_int64()
        N.check(N.lib().gimbal_online_iteration(self._h, a.ctypes.data, 1 if a.dtype == np.uint8 else 4, a.size // per,
                                                C.byref(ex), C.byref(cr)), "iteration")
        return ex.value, cr.value

    def gpu_totals(self) -> np.ndarray:
        out = np.zeros(self.topo.n_gpus, np.int64)
        N.check(N.lib().gimbal_online_gpu_totals(self._h, out.ctypes.data), "gpu_totals")
        return out
