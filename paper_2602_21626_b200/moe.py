"""Host mirror of the reference's ``gimbal::moe`` operator API over the sm_100a C ABI.

Reference: /root/reference/proj/include/gimbal/moe.hpp:14-118, proj/src/moe.cpp.  Names, argument
meaning and error behaviour follow the reference (``std::invalid_argument`` -> ``ValueError``).
Counts come back as ``numpy.uint64`` arrays (the reference keeps them as integer-valued doubles).
Traces may be numpy arrays (host) or CUDA tensors (device, consumed in place).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N


@dataclass
class MoeTopology:
    """moe::MoeTopology (moe.hpp:14-23)."""

    n_layers: int = 4
    n_experts: int = 8
    top_k: int = 2
    n_gpus: int = 2

    def validate(self) -> None:  # moe.cpp:12-24
        N.check(N.lib().gimbal_topology_validate(C.byref(self.c())), "MoeTopology")

    def total_experts(self) -> int:
        return self.n_layers * self.n_experts

    def flat_id(self, layer: int, expert: int) -> int:
        return layer * self.n_experts + expert

    def c(self) -> N.Topology:
        return N.Topology(self.n_layers, self.n_experts, self.top_k, self.n_gpus)


@dataclass
class RoutingParams:
    """moe::RoutingParams (moe.hpp:25-29)."""

    zipf_s: float = 1.2
    lambda_: float = 0.5
    affinity_peak: float = 0.8


@dataclass
class AffinityTensor:
    """moe::AffinityTensor (moe.hpp:38-41): E [(L-1)][n_e][n_e], W [n_e][n_e]."""

    E: np.ndarray
    W: np.ndarray


@dataclass
class RoutedStream:
    """moe::RoutedStream (moe.hpp:75-83): choices token-major [T][L][k] (numpy or CUDA tensor)."""

    topo: MoeTopology
    n_tokens: int = 0
    choices: object = None

    def token(self, t: int):
        stride = self.topo.n_layers * self.topo.top_k
        return np.asarray(self.choices).reshape(-1)[t * stride:(t + 1) * stride]


def _trace_arg(ids, topo: MoeTopology):
    """(pointer, id_bytes, n_tokens, mem, keepalive) for a numpy array or a CUDA tensor."""
    stride = topo.n_layers * topo.top_k
    if hasattr(ids, "data_ptr") and hasattr(ids, "is_cuda"):
        import torch

        t = ids
        if t.dtype not in (torch.uint8, torch.int32):
            raise TypeError("trace tensor must be uint8 or int32")
        if not t.is_contiguous():
            t = t.contiguous()
        n = t.numel()
        if n % stride:
            raise ValueError("add_token: choice span size mismatch")
        mem = N.MEM_DEVICE if t.is_cuda else N.MEM_HOST
        return t.data_ptr(), (1 if t.dtype == torch.uint8 else 4), n // stride, mem, t
    a = np.asarray(ids)
    if a.dtype == np.uint8:
        ib = 1
    else:
        if a.size and (a.min() < np.iinfo(np.int32).min or a.max() > np.iinfo(np.int32).max):
            raise ValueError("expert ids must fit int32")
        a = a.astype(np.int32, copy=False)
        ib = 4
    a = np.ascontiguousarray(a)
    if a.size % stride:
        raise ValueError("add_token: choice span size mismatch")
    return a.ctypes.data, ib, a.size // stride, N.MEM_HOST, a


class RoutingStats:
    """moe::RoutingStats (moe.hpp:86-105) backed by device counters on one B200.

    ``add_token`` keeps the reference's per-token signature (buffered on the host and flushed in
    one batch before the next read); ``add_tokens`` is the batch form for whole traces.
    """

    def __init__(self, topo: MoeTopology, device: int = 0):
        topo.validate()
        self.topo = topo
        self.device = device
        h = C.c_void_p()
        N.check(N.lib().gimbal_stats_create(C.byref(topo.c()), device, C.byref(h)), "RoutingStats")
        self._h = h
        self._pending: list = []
        self._inflight: list = []  # pinned host inputs whose asynchronous copies may be in flight

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().gimbal_stats_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- ingest ----
    def add_token(self, choices) -> None:  # moe.cpp:169-191
        c = np.asarray(choices).reshape(-1)
        if c.size != self.topo.n_layers * self.topo.top_k:
            raise ValueError("add_token: choice span size mismatch")
        self._pending.append(c.astype(np.int32))

    def add_tokens(self, ids) -> None:
        self._flush()
        ptr, ib, n, mem, keep = _trace_arg(ids, self.topo)
        if mem == N.MEM_DEVICE:
            self._after_torch(keep)
        N.check(N.lib().gimbal_stats_add_tokens(self._h, C.c_void_p(ptr), ib, n, mem), "add_tokens")
        self._keep_until_done(keep, mem)
        del keep

    def _keep_until_done(self, tensor, mem) -> None:
        """The count queued on the handle's stream may still read ``tensor`` after this call returns.
        Device tensor (possibly a temporary made by ``.contiguous()``): torch's current stream is
        made to wait for the handle's stream (an event, no host sync), so memory torch's caching
        allocator hands out again after the tensor dies is only written behind the count.  (Not
        ``record_stream``: the handle's stream can be destroyed before the tensor is freed, and the
        allocator would then record an event on a dead stream.)  Pinned host torch tensor (copied
        asynchronously, gimbal_gpu.h): held until the next synchronising call.  numpy inputs are
        pageable (copied through the library's own bounce buffers)."""
        if not hasattr(tensor, "data_ptr"):
            return
        if mem == N.MEM_DEVICE:
            import torch

            torch.cuda.current_stream(tensor.device).wait_stream(self._ext_stream)
        else:
            self._inflight.append(tensor)

    def _after_torch(self, tensor) -> None:
        """Orders the handle's stream after torch's current stream (device inputs produced by
        torch), without a host synchronisation."""
        import torch

        ours = getattr(self, "_ext_stream", None)
        if ours is None or ours.device != tensor.device:
            s = C.c_void_p()
            N.check(N.lib().gimbal_stats_device_buffers(self._h, None, None, C.byref(s)), "buffers")
            ours = self._ext_stream = torch.cuda.ExternalStream(s.value, device=tensor.device)
        cur = torch.cuda.current_stream(tensor.device)
        if cur.cuda_stream != ours.cuda_stream:
            ours.wait_stream(cur)

    def _flush(self) -> None:
        if self._pending:
            batch = np.stack(self._pending)
            self._pending = []
            ptr, ib, n, mem, keep = _trace_arg(batch, self.topo)
            N.check(N.lib().gimbal_stats_add_tokens(self._h, C.c_void_p(ptr), ib, n, mem), "add_token")

    def reset(self) -> None:  # moe.cpp:193-197
        self._pending = []
        N.check(N.lib().gimbal_stats_reset(self._h), "reset")

    # ---- readback ----
    def tokens(self) -> int:
        self._flush()
        t = C.c_int64()
        N.check(N.lib().gimbal_stats_tokens(self._h, C.byref(t)), "tokens")
        return t.value

    def read(self):
        """(A [L][n_e], E [(L-1)][n_e][n_e], W [n_e][n_e]) as uint64."""
        self._flush()
        L, ne = self.topo.n_layers, self.topo.n_experts
        A = np.zeros((L, ne), np.uint64)
        E = np.zeros((max(L - 1, 0), ne, ne), np.uint64)
        W = np.zeros((ne, ne), np.uint64)
        N.check(N.lib().gimbal_stats_read(self._h, A.ctypes.data, E.ctypes.data if E.size else None,
                                          W.ctypes.data, N.MEM_HOST), "read")
        self._inflight.clear()
        return A, E, W

    def activation(self) -> np.ndarray:  # moe.hpp:91
        return self.read()[0]

    def affinity(self) -> AffinityTensor:  # moe.cpp:199-205
        _, E, W = self.read()
        return AffinityTensor(E=E, W=W)

    def flat_activation(self) -> np.ndarray:  # moe.cpp:207-215
        self._flush()
        L, m = self.topo.n_layers, self.topo.total_experts()
        out = np.zeros((L, m), np.float64)
        N.check(N.lib().gimbal_stats_flat(self._h, out.ctypes.data, None, N.MEM_HOST), "flat_activation")
        return out

    def flat_pair_weights(self) -> np.ndarray:  # moe.cpp:217-231
        self._flush()
        m = self.topo.total_experts()
        out = np.zeros((m, m), np.float64)
        N.check(N.lib().gimbal_stats_flat(self._h, None, out.ctypes.data, N.MEM_HOST), "flat_pair_weights")
        return out

    # ---- multi-GPU plumbing ----
    def device_buffers(self):
        """(E pointer, A pointer, cudaStream_t) for in-place collectives over token shards."""
        self._flush()
        e, a, s = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.check(N.lib().gimbal_stats_device_buffers(self._h, C.byref(e), C.byref(a), C.byref(s)), "buffers")
        return e.value, a.value, s.value

    def count_timing(self, enable: bool = True):
        """(device ms, launches) of the counting kernels since the last call; keeps recording
        while ``enable``."""
        ms, n = C.c_double(0.0), C.c_int64(0)
        N.check(N.lib().gimbal_stats_count_timing(self._h, int(enable), C.byref(ms), C.byref(n)), "timing")
        return ms.value, n.value

    def merge(self, counts, tokens: int) -> None:
        """Adds a snapshot of counts (E, or A when L == 1; host uint64) and its token total."""
        a = np.ascontiguousarray(counts, np.uint64)
        N.check(N.lib().gimbal_stats_merge(self._h, a.ctypes.data, int(tokens), N.MEM_HOST), "merge")

    def mark_reduced(self, global_tokens: int) -> None:
        N.check(N.lib().gimbal_stats_mark_reduced(self._h, int(global_tokens)), "mark_reduced")

    def set_count_sms(self, n_sms: int) -> None:
        """Counting kernels use n_sms SMs (the rest stay free for another stream's kernels)."""
        N.check(N.lib().gimbal_stats_set_count_sms(self._h, int(n_sms)), "set_count_sms")

    def sync(self) -> None:
        self._flush()
        N.check(N.lib().gimbal_stats_sync(self._h), "sync")
        self._inflight.clear()

    @property
    def handle(self):
        self._flush()
        return self._h


def record_stats(stream: RoutedStream, device: int = 0) -> RoutingStats:  # moe.cpp:233-239
    stats = RoutingStats(stream.topo, device)
    if stream.n_tokens:
        stats.add_tokens(stream.choices)
    return stats


def comm_cost(stream: RoutedStream, expert_to_gpu, device: int = 0) -> int:  # moe.cpp:241-267
    topo = stream.topo
    a = np.ascontiguousarray(np.asarray(expert_to_gpu, dtype=np.int64))
    if a.size != topo.total_experts():
        raise ValueError("comm_cost: assignment size mismatch")
    if (a < 0).any():
        raise ValueError("comm_cost: unplaced expert")
    a32 = a.astype(np.int32)
    out = C.c_int64()
    if stream.n_tokens == 0:
        ptr, ib, n, mem, keep = 0, 1, 0, N.MEM_HOST, None
    else:
        ptr, ib, n, mem, keep = _trace_arg(stream.choices, topo)
    N.check(N.lib().gimbal_comm_cost(C.byref(topo.c()), C.c_void_p(ptr), ib, n, mem, a32.ctypes.data, a32.size,
                                     device, C.byref(out)), "comm_cost")
    return out.value


def generate_trace(topo: MoeTopology, n_tokens: int, params: Optional[RoutingParams] = None,
                   model_seed: int = 1, stream_seed: int = 2, first_token: int = 0, drift: float = 0.0,
                   drift_epoch: int = 0, device: int = 0, out=None):
    """Synthetic [T][L][k] uint8 routing trace on the GPU (RoutingModel semantics, moe.cpp:43-160)."""
    import torch

    p = params or RoutingParams()
    if out is None:
        out = torch.empty((n_tokens, topo.n_layers, topo.top_k), dtype=torch.uint8, device=f"cuda:{device}")
    N.check(N.lib().gimbal_generate_trace(C.byref(topo.c()), p.zipf_s, p.lambda_, p.affinity_peak, model_seed,
                                          stream_seed, drift, drift_epoch, first_token, n_tokens,
                                          C.c_void_p(out.data_ptr()), device), "generate_trace")
    return out


def generator_tables(topo: MoeTopology, params: Optional[RoutingParams] = None, model_seed: int = 1,
                     drift: float = 0.0, drift_epoch: int = 0):
    """(cdf [L][n_e] uint32, thresholds [2] uint64) used by the generator kernel."""
    p = params or RoutingParams()
    cdf = np.zeros((topo.n_layers, topo.n_experts), np.uint32)
    thr = np.zeros(2, np.uint64)
    N.check(N.lib().gimbal_generator_tables(C.byref(topo.c()), p.zipf_s, p.lambda_, p.affinity_peak, model_seed,
                                            drift, drift_epoch, cdf.ctypes.data, thr.ctypes.data), "tables")
    return cdf, thr
