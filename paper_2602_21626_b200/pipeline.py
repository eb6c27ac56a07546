"""The north-star pass: trace -> A/E/W -> strong-pair set M -> greedy -> C-candidate scoring ->
argmin, on one B200 or sharded over ranks.

Single GPU (``HotPath.run``): every stage is a kernel on the stats handle's stream; the only host
round trips are the strong-pair set (<= 2*top_e ids, validated on the host like the reference)
and the argmin / error flags.

Multi-GPU (``HotPath.run_distributed``): trace tokens shard into contiguous ranges per rank (A/E
are sums over tokens); partial u64 E is all-reduced in place (``torch.distributed``, NCCL over
NVLink; int64 SUM is bit-identical to u64 addition), M and greedy are recomputed identically on
every rank, candidates split into contiguous slices per rank and the per-candidate objectives
are all-gathered for a global argmin with the lowest index winning ties.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .moe import MoeTopology, RoutingStats
from .placement import AffinitySet, build_affinity_set, eval_costs, greedy_place, greedy_place_array


def shard_range(n: int, rank: int, world: int):
    """Contiguous [lo, hi) slice of n items for rank (the same split the oracle uses)."""
    return n * rank // world, n * (rank + 1) // world


def merge_argmin(objectives: np.ndarray) -> int:
    """Lowest index among the minimal objectives (placement argmin tie rule)."""
    if objectives.size == 0:
        return -1
    return int(np.flatnonzero(objectives == objectives.min())[0])


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def nccl_comm(group=None, device: int = 0):
    """The ncclComm_t (as an int) behind a torch NCCL process group, for the library's own
    collectives (gimbal_stats_allreduce, gimbal_pass_distributed_async); None when the group is
    not NCCL or torch does not expose it."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) != "nccl":
        return None
    try:
        pg = group if group is not None else dist.distributed_c10d._get_default_group()
        ptr = pg._get_backend(torch.device("cuda", device))._comm_ptr()
        return int(ptr) or None
    except Exception:  # noqa: BLE001 - older torch / lazily initialised communicator
        return None


def allreduce_counts(stats: RoutingStats, group=None) -> None:
    """In-place SUM all-reduce of the handle's counted buffer over the process group.  NCCL: the
    library's gimbal_stats_allreduce on the group's communicator, queued on the handle's stream
    (no host round trip); other backends: through host memory."""
    import torch
    import torch.distributed as dist

    comm = nccl_comm(group, stats.device)
    if comm is not None:
        N.check(N.lib().gimbal_stats_allreduce(stats.handle, C.c_void_p(comm), -1), "allreduce")
        return
    topo = stats.topo
    e_ptr, a_ptr, _ = stats.device_buffers()
    if topo.n_layers > 1:
        n, ptr = (topo.n_layers - 1) * topo.n_experts * topo.n_experts, e_ptr
    else:
        n, ptr = topo.n_layers * topo.n_experts, a_ptr
    stats.sync()
    dev = torch.device("cuda", stats.device)
    view = torch.as_tensor(_CudaArray(ptr, n), device=dev)
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(view, op=dist.ReduceOp.SUM, group=group)
        torch.cuda.current_stream(dev).synchronize()
    else:
        host = view.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        view.copy_(host)
        torch.cuda.synchronize(dev)
    tok = torch.tensor([stats.tokens()], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        tok = tok.to(dev)
    dist.all_reduce(tok, op=dist.ReduceOp.SUM, group=group)
    stats.mark_reduced(int(tok.item()))


@dataclass
class HotPathResult:
    affinity: AffinitySet
    greedy: list
    argmin: int
    objective: Optional[float] = None


class PendingPass:
    """A queued pass (HotPath.run_async); result() waits for it and decodes its packed results
    (raising the pass's deferred device-side error, if any)."""

    def __init__(self, hp: "HotPath", host, event):
        self._hp, self._host, self._event = hp, host, event
        self._res, self._err = None, None

    def done(self) -> bool:
        return self._res is not None or self._err is not None or self._event.query()

    def _resolve(self) -> None:
        if self._res is not None or self._err is not None:
            return
        self._event.synchronize()
        h = self._host.copy()  # the slot is reused by a later pass
        if h[4] or h[5]:
            try:
                self._hp.stats.sync()  # raises (and clears) the deferred device-side error
            except Exception as ex:  # kept for result(); a later pass's run_async must not raise it
                self._err = ex
                return
        self._res = self._hp._decode_pk(h)

    def result(self) -> HotPathResult:
        self._resolve()
        if self._err is not None:
            raise self._err
        return self._res


class HotPath:
    """One stats handle + device scratch for repeated passes of the same topology."""

    def __init__(self, topo: MoeTopology, device: int = 0, threshold: float = 0.0, top_e: int = 4,
                 anchor_gpu: int = 0, alpha: float = 1.0, beta: float = 1.0):
        topo.validate()
        self.topo = topo
        self.device = device
        self.stats = RoutingStats(topo, device)
        self.threshold, self.top_e, self.anchor_gpu = threshold, top_e, anchor_gpu
        self.alpha, self.beta = alpha, beta
        self._out = None

    def _scores(self, C: int):
        import torch

        if self._out is None or self._out.shape[1] != C:
            self._out = torch.empty((3, C), dtype=torch.float64, device=f"cuda:{self.device}")
        return self._out

    def place(self, candidates, greedy_row: bool = True):
        """Stats already counted: M -> greedy (written into candidates[0] if greedy_row) ->
        scores -> argmin.  candidates: CUDA uint8 tensor [C][m]."""
        topo = self.topo
        if (greedy_row and getattr(candidates, "is_cuda", False) and candidates.shape[0] > 0
                and topo.n_gpus <= 255):
            return self._place_queued(candidates)
        M = build_affinity_set(self.stats, topo, self.threshold, self.top_e,
                               topo.total_experts() // topo.n_gpus, self.anchor_gpu)
        gp = greedy_place(self.stats, M, topo.n_gpus, out_u8_device=candidates[0] if greedy_row else None)
        out, am = eval_costs(self.stats, candidates, self.alpha, self.beta, out=self._scores(candidates.shape[0]))
        return HotPathResult(affinity=M, greedy=gp.assign, argmin=am)

    def _ensure_pk(self) -> None:
        import torch

        m = self.topo.total_experts()
        if getattr(self, "_pk", None) is None:
            dev = torch.device("cuda", self.device)
            # int32 words: [0:2] argmin (int64), [2] |M|, [3] pad, [4:6] error flags, [6:6+m] M,
            # [6+m:6+2m] greedy
            self._pk = torch.zeros(6 + 2 * m, dtype=torch.int32, device=dev)
            self._pk_host = torch.empty(6 + 2 * m, dtype=torch.int32).pin_memory()
            self._hstream = torch.cuda.ExternalStream(self.stats.device_buffers()[2], device=dev)

    def _read_pk(self, extra=None):
        """One read-back of the packed results (plus an optional (device, pinned host) pair) behind
        the handle's stream, one sync; raises a deferred device-side error."""
        import torch

        # the read-back runs on torch's stream behind the handle's (a pinned block used on the
        # handle's own stream would outlive it in torch's host allocator)
        cur = torch.cuda.current_stream(torch.device("cuda", self.device))
        cur.wait_stream(self._hstream)
        self._pk_host.copy_(self._pk, non_blocking=True)
        if extra is not None:
            extra[1].copy_(extra[0], non_blocking=True)
        cur.synchronize()
        h = self._pk_host.numpy()
        if h[4] or h[5]:
            self.stats.sync()  # raises (and clears) the deferred device-side error
        return h

    def _place_queued(self, candidates) -> HotPathResult:
        """place() as one queued device chain (gimbal_pass_async: strong-pair set, greedy, scores,
        argmin), then a single read-back of [argmin | |M| | M | greedy] and one stream sync."""
        import torch

        topo = self.topo
        m, C_ = topo.total_experts(), int(candidates.shape[0])
        self._ensure_pk()
        scores = self._scores(C_)
        self.stats._after_torch(candidates)
        base = self._pk.data_ptr()
        N.check(N.lib().gimbal_pass_async(
            self.stats.handle, self.threshold, self.top_e, m // topo.n_gpus, self.anchor_gpu,
            C.c_void_p(candidates.data_ptr()), C_, self.alpha, self.beta, C.c_void_p(scores.data_ptr()),
            C.c_void_p(base), C.c_void_p(base + 24 + 4 * m), C.c_void_p(base + 24), C.c_void_p(base + 8),
            C.c_void_p(base + 16)), "pass")
        h = self._read_pk()
        n = int(h[2])
        return HotPathResult(affinity=AffinitySet(experts=h[6:6 + n].tolist(), anchor_gpu=self.anchor_gpu),
                             greedy=h[6 + m:6 + 2 * m].tolist(), argmin=int(h[0:2].view(np.int64)[0]))

    def place_with(self, M: AffinitySet, candidates, greedy_row: bool = True) -> HotPathResult:
        """Stats already counted, strong-pair set fixed (sim.cpp:94-104 computes M once from a
        calibration pass and keeps it): greedy -> scores -> argmin."""
        gp = greedy_place(self.stats, M, self.topo.n_gpus, out_u8_device=candidates[0] if greedy_row else None)
        out, am = eval_costs(self.stats, candidates, self.alpha, self.beta, out=self._scores(candidates.shape[0]))
        return HotPathResult(affinity=M, greedy=gp.assign, argmin=am)

    def run(self, trace, candidates, greedy_row: bool = True, graph: bool = True) -> HotPathResult:
        """One full pass over a trace (CUDA uint8 [T][L][k] or host array).  With a device trace and
        device candidates the step goes through gimbal_pass_graph: recorded once as a CUDA graph
        and replayed while the buffers stay the same (their contents may change)."""
        if (graph and greedy_row and getattr(trace, "is_cuda", False) and getattr(candidates, "is_cuda", False)
                and candidates.shape[0] > 0 and self.topo.n_gpus <= 255 and trace.is_contiguous()
                and str(trace.dtype) in ("torch.uint8", "torch.int32") and trace.numel() > 0):
            return self._run_graph(trace, candidates)
        self.stats.reset()
        self.stats.add_tokens(trace)
        return self.place(candidates, greedy_row)

    def _queue_graph(self, trace, candidates) -> None:
        import torch

        topo = self.topo
        m, C_ = topo.total_experts(), int(candidates.shape[0])
        per = topo.n_layers * topo.top_k
        if trace.numel() % per:
            raise ValueError("add_token: choice span size mismatch")
        self._ensure_pk()
        scores = self._scores(C_)
        st = self.stats
        st._after_torch(trace)
        st._after_torch(candidates)
        base = self._pk.data_ptr()
        N.check(N.lib().gimbal_pass_graph(
            st.handle, C.c_void_p(trace.data_ptr()), 1 if trace.dtype == torch.uint8 else 4, trace.numel() // per,
            self.threshold, self.top_e, m // topo.n_gpus, self.anchor_gpu, C.c_void_p(candidates.data_ptr()), C_,
            self.alpha, self.beta, C.c_void_p(scores.data_ptr()), C.c_void_p(base), C.c_void_p(base + 24 + 4 * m),
            C.c_void_p(base + 24), C.c_void_p(base + 8), C.c_void_p(base + 16)), "pass_graph")
        st._keep_until_done(trace, N.MEM_DEVICE)

    def _decode_pk(self, h) -> HotPathResult:
        m = self.topo.total_experts()
        n = int(h[2])
        return HotPathResult(affinity=AffinitySet(experts=h[6:6 + n].tolist(), anchor_gpu=self.anchor_gpu),
                             greedy=h[6 + m:6 + 2 * m].tolist(), argmin=int(h[0:2].view(np.int64)[0]))

    def _run_graph(self, trace, candidates) -> HotPathResult:
        self._queue_graph(trace, candidates)
        return self._decode_pk(self._read_pk())

    def run_async(self, trace, candidates) -> "PendingPass":
        """run() without waiting (gimbal_pass_enqueue): the pass joins torch's current stream both
        ways, replays as a graph, and its packed results ([argmin | |M| | error words | M | greedy])
        reach host memory (a copy into one of a ring of registered slots owned by this object, or,
        for the fused small-shape pass, the handle's mapped result ring written by the kernel); the
        host returns at once and PendingPass.result() waits for that pass only (at most 8 are kept
        in flight: the ninth call reads the oldest out).  Back-to-back passes therefore
        keep the GPU busy instead of paying a host round trip each (the scores stay in `self._out`,
        which the next pass overwrites).  Device trace and candidates only."""
        import torch

        if not (getattr(trace, "is_cuda", False) and getattr(candidates, "is_cuda", False)
                and candidates.shape[0] > 0 and self.topo.n_gpus <= 255 and trace.is_contiguous()
                and trace.dtype in (torch.uint8, torch.int32) and trace.numel() > 0):
            raise ValueError("run_async: needs a contiguous CUDA uint8/int32 trace and CUDA candidates")
        topo = self.topo
        per = topo.n_layers * topo.top_k
        if trace.numel() % per:
            raise ValueError("add_token: choice span size mismatch")
        self._ensure_pk()
        if getattr(self, "_ring", None) is None:
            ring = np.zeros((8, self._pk.numel()), np.int32)
            torch.cuda.cudart().cudaHostRegister(ring.ctypes.data, ring.nbytes, 0)
            self._ring, self._ring_ev, self._ring_next = ring, [None] * 8, 0
            import weakref

            def _unregister(ptr=ring.ctypes.data, keep=ring):
                try:
                    torch.cuda.cudart().cudaHostUnregister(ptr)
                except Exception:
                    pass

            weakref.finalize(self, _unregister)
        i = self._ring_next
        self._ring_next = (i + 1) % 8
        prev = self._ring_ev[i]
        if prev is not None:  # at most 8 passes in flight: the slot's previous pass is read out first
            prev._resolve()
        m, C_ = topo.total_experts(), int(candidates.shape[0])
        scores = self._scores(C_)
        cur = torch.cuda.current_stream(torch.device("cuda", self.device))
        where = C.c_void_p()
        N.check(N.lib().gimbal_pass_enqueue(
            self.stats.handle, trace.data_ptr(), 1 if trace.dtype == torch.uint8 else 4, trace.numel() // per,
            self.threshold, self.top_e, m // topo.n_gpus, self.anchor_gpu, candidates.data_ptr(), C_, self.alpha,
            self.beta, scores.data_ptr(), self._pk.data_ptr(), self._ring[i].ctypes.data, cur.cuda_stream,
            C.byref(where)), "pass_enqueue")
        ev = torch.cuda.Event()
        ev.record(cur)
        host = np.ctypeslib.as_array(C.cast(where.value, C.POINTER(C.c_int32)), shape=(6 + 2 * m,))
        pp = PendingPass(self, host, ev)
        self._ring_ev[i] = pp
        return pp

    def calibrate(self, trace) -> AffinitySet:
        """Offline calibration (sim.cpp:91-106): stats over a calibration trace -> strong-pair set."""
        self.stats.reset()
        self.stats.add_tokens(trace)
        topo = self.topo
        return build_affinity_set(self.stats, topo, self.threshold, self.top_e,
                                  topo.total_experts() // topo.n_gpus, self.anchor_gpu)

    def stream(self, windows, candidates, M: AffinitySet, previous=None, reserve_sms: int = 2):
        """Tumbling-window re-placement (config 5; sim.cpp:149-165 semantics per window: the window
        is counted from zero, greedy re-places with the fixed anchor set, all candidates are
        scored, and `moved` counts experts whose GPU changed against the previous choice).
        ``windows``: sequence of CUDA uint8 [T_w][L][k] traces; ``candidates``: CUDA uint8 [C][m]
        (row 0 is replaced by each window's greedy placement).  Returns per-window
        (argmin, moved, greedy placement as an int32 numpy array).

        The whole stream is queued without host synchronisation.  Windows alternate between this
        handle and a twin (own counts, own stream, own copy of the candidate batch), so window
        w+1 is counted while window w is placed and scored; counting leaves ``reserve_sms`` SMs
        free, where window w's latency-bound greedy walk runs alongside.  Each window's greedy
        placement, scores and argmin stay on the device until the end
        (gimbal_window_place_async); device-side errors surface at the final sync."""
        import torch

        windows = list(windows)
        if not windows:
            return []
        n, (n_c, m) = len(windows), tuple(candidates.shape)
        dev = torch.device("cuda", self.device)
        pair = (self, self._twin())
        scores = torch.empty((n, 3, n_c), dtype=torch.float64, device=dev)
        argmins = torch.empty((n,), dtype=torch.int64, device=dev)
        places = torch.empty((n, m), dtype=torch.int32, device=dev)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        for hp in pair:
            if getattr(hp, "_wcands", None) is None or tuple(hp._wcands.shape) != (n_c, m):
                hp._wcands = torch.empty_like(candidates)
            hp._wcands.copy_(candidates)
            hp.stats._after_torch(places)  # outputs and candidate copies are ready before use
            hp.stats.set_count_sms(max(1, sms - max(0, reserve_sms)))
        Mi = np.ascontiguousarray(np.asarray(M.experts, np.int32))
        lib = N.lib()
        try:
            pair[0].stats.reset()
            pair[0].stats.add_tokens(windows[0])
            for i in range(n):
                cur = pair[i % 2]
                if i + 1 < n:
                    nxt = pair[(i + 1) % 2]
                    nxt.stats.reset()
                    nxt.stats.add_tokens(windows[i + 1])
                N.check(lib.gimbal_window_place_async(
                    cur.stats.handle, Mi.ctypes.data if Mi.size else None, Mi.size, M.anchor_gpu,
                    C.c_void_p(cur._wcands.data_ptr()), int(n_c), self.alpha, self.beta,
                    C.c_void_p(scores[i].data_ptr()), C.c_void_p(argmins[i].data_ptr()),
                    C.c_void_p(places[i].data_ptr())), "window_place")
        finally:
            for hp in pair:
                hp.stats.set_count_sms(sms)
        errors = []
        for hp in pair:  # every handle's deferred flags are read (and cleared) before raising
            try:
                hp.stats.sync()
            except Exception as e:  # noqa: BLE001
                errors.append(e)
        if errors:
            raise errors[0]
        candidates[0].copy_(pair[(n - 1) % 2]._wcands[0])
        self._window_scores = scores
        am = argmins.cpu().numpy()
        pl = places.cpu().numpy()
        prev = None if previous is None else np.asarray(previous, np.int32)
        out = []
        for i in range(n):
            gp = pl[i]
            moved = int(np.count_nonzero(prev != gp)) if prev is not None and prev.shape == gp.shape else len(gp)
            out.append((int(am[i]), moved, gp))
            prev = gp
        return out

    def _twin(self) -> "HotPath":
        """A second handle with the same topology and parameters (stream double-buffering)."""
        if getattr(self, "_twin_hp", None) is None:
            self._twin_hp = HotPath(self.topo, device=self.device, alpha=self.alpha, beta=self.beta,
                                    threshold=self.threshold, top_e=self.top_e, anchor_gpu=self.anchor_gpu)
        return self._twin_hp

    def stream_distributed(self, window_shards, candidates_shard, cand_offset: int, n_candidates: int,
                           M: AffinitySet, group=None, previous=None, reserve_sms: int = 2):
        """stream() with each window's tokens sharded over ranks: count the shard, all-reduce E,
        re-place with the fixed M, score this rank's candidate slice, merge the argmin.

        Over NCCL the whole stream is queued like stream(): window w+1's shard is counted on the
        twin handle while window w's E is all-reduced on its handle's stream (the collective is
        ordered behind the counting and ahead of the placement without a host round trip) and
        placed with gimbal_window_place_async.  Objectives land in one [windows][C] buffer that a
        single MIN all-reduce merges at the end (lowest global index wins ties).  Global candidate
        0 is the greedy placement (rank 0's first row); other ranks score their slice behind a
        scratch greedy row."""
        import torch
        import torch.distributed as dist

        windows = list(window_shards)
        if not windows:
            return []
        if dist.get_backend(group) != "nccl":
            return self._stream_distributed_sync(windows, candidates_shard, cand_offset, n_candidates, M, group,
                                                 previous)
        n, m = len(windows), self.topo.total_experts()
        dev = torch.device("cuda", self.device)
        c_loc = int(candidates_shard.shape[0])
        # scratch greedy row ahead of a non-leading (or empty) slice: with C < world some ranks hold
        # no candidates, and their window placement still needs row 0 to receive the greedy row
        lead = 0 if (cand_offset == 0 and c_loc > 0) else 1
        tok = torch.tensor([int(w.shape[0]) for w in windows], dtype=torch.int64, device=dev)
        dist.all_reduce(tok, op=dist.ReduceOp.SUM, group=group)
        glob = tok.tolist()
        pair = (self, self._twin())
        rows = c_loc + lead
        scores = torch.empty((n, 3, max(rows, 1)), dtype=torch.float64, device=dev)
        argmins = torch.empty((n,), dtype=torch.int64, device=dev)
        places = torch.empty((n, m), dtype=torch.int32, device=dev)
        objs = torch.full((n, n_candidates), float("inf"), dtype=torch.float64, device=dev)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        exts = []
        for hp in pair:
            if getattr(hp, "_wcands", None) is None or tuple(hp._wcands.shape) != (rows, m):
                hp._wcands = torch.empty((rows, m), dtype=torch.uint8, device=dev)
            if c_loc:
                hp._wcands[lead:].copy_(candidates_shard)
            if lead:
                hp._wcands[0].copy_(hp._wcands[1] if c_loc else torch.zeros(m, dtype=torch.uint8, device=dev))
            hp.stats._after_torch(objs)
            hp.stats.set_count_sms(max(1, sms - max(0, reserve_sms)))
            exts.append(torch.cuda.ExternalStream(hp.stats.device_buffers()[2], device=dev))
        Mi = np.ascontiguousarray(np.asarray(M.experts, np.int32))
        lib = N.lib()
        topo = self.topo
        comm = nccl_comm(group, self.device)
        n_cells = (topo.n_layers - 1) * topo.n_experts * topo.n_experts if topo.n_layers > 1 else m
        try:
            pair[0].stats.reset()
            pair[0].stats.add_tokens(windows[0])
            for i in range(n):
                cur, ext = pair[i % 2], exts[i % 2]
                if i + 1 < n:
                    nxt = pair[(i + 1) % 2]
                    nxt.stats.reset()
                    nxt.stats.add_tokens(windows[i + 1])
                if comm is not None:  # the library's NCCL SUM on the handle's stream
                    N.check(lib.gimbal_stats_allreduce(cur.stats.handle, C.c_void_p(comm), int(glob[i])),
                            "allreduce")
                else:
                    e_ptr, a_ptr, _ = cur.stats.device_buffers()
                    view = torch.as_tensor(_CudaArray(e_ptr if topo.n_layers > 1 else a_ptr, n_cells), device=dev)
                    with torch.cuda.stream(ext):  # behind this window's counting, ahead of its placement
                        dist.all_reduce(view, op=dist.ReduceOp.SUM, group=group)
                    cur.stats.mark_reduced(int(glob[i]))
                if rows:
                    N.check(lib.gimbal_window_place_async(
                        cur.stats.handle, Mi.ctypes.data if Mi.size else None, Mi.size, M.anchor_gpu,
                        C.c_void_p(cur._wcands.data_ptr()), rows, self.alpha, self.beta,
                        C.c_void_p(scores[i].data_ptr()), C.c_void_p(argmins[i].data_ptr()),
                        C.c_void_p(places[i].data_ptr())), "window_place")
                    if c_loc:
                        with torch.cuda.stream(ext):
                            objs[i, cand_offset:cand_offset + c_loc].copy_(scores[i, 2, lead:lead + c_loc])
        finally:
            for hp in pair:
                hp.stats.set_count_sms(sms)
        errors = []
        for hp in pair:
            try:
                hp.stats.sync()
            except Exception as e:  # noqa: BLE001
                errors.append(e)
        if errors:
            raise errors[0]
        dist.all_reduce(objs, op=dist.ReduceOp.MIN, group=group)
        allobj = objs.cpu().numpy()
        pl = places.cpu().numpy()
        prev = None if previous is None else np.asarray(previous, np.int32)
        out = []
        for i in range(n):
            gp = pl[i]
            moved = int(np.count_nonzero(prev != gp)) if prev is not None and prev.shape == gp.shape else len(gp)
            out.append((merge_argmin(allobj[i]), moved, gp))
            prev = gp
        return out

    def _stream_distributed_sync(self, windows, candidates_shard, cand_offset: int, n_candidates: int,
                                 M: AffinitySet, group=None, previous=None):
        """Per-window synchronous form (any backend): count, all-reduce, place, merge."""
        out = []
        prev = previous
        for w in windows:
            res = self._distributed_pass(w, candidates_shard, cand_offset, n_candidates, group, M)
            moved = (sum(1 for a, b in zip(prev, res.greedy) if a != b) if prev is not None
                     and len(prev) == len(res.greedy) else len(res.greedy))
            out.append((res.argmin, moved, res.greedy))
            prev = res.greedy
        return out

    def run_distributed(self, trace_shard, candidates_shard, cand_offset: int, n_candidates: int,
                        group=None) -> HotPathResult:
        """This rank's token shard and candidate slice; returns the global argmin."""
        return self._distributed_pass(trace_shard, candidates_shard, cand_offset, n_candidates, group, None)

    def _distributed_queued(self, trace_shard, candidates_shard, cand_offset: int, n_candidates: int, comm):
        """One rank's pass as one queued device chain (gimbal_pass_distributed_async): count the shard,
        NCCL SUM of the counts, strong-pair set, greedy, scores of this slice, NCCL MIN merge of the
        objectives and the global argmin; then one read-back and one sync."""
        import torch

        topo = self.topo
        m = topo.total_experts()
        dev = torch.device("cuda", self.device)
        n_local = int(candidates_shard.shape[0])
        lead = 0 if (cand_offset == 0 and n_local > 0) else 1
        if lead:
            if getattr(self, "_dcands", None) is None or tuple(self._dcands.shape) != (n_local + 1, m):
                self._dcands = torch.zeros((n_local + 1, m), dtype=torch.uint8, device=dev)
            if n_local:
                self._dcands[1:].copy_(candidates_shard)
            buf = self._dcands
        else:
            buf = candidates_shard
        rows = n_local + lead
        scores = self._scores(rows)
        if getattr(self, "_gobj", None) is None or self._gobj.numel() != n_candidates:
            self._gobj = torch.empty(n_candidates, dtype=torch.float64, device=dev)
            self._gobj_host = torch.empty(n_candidates, dtype=torch.float64).pin_memory()
        self._ensure_pk()
        self.stats.reset()
        self.stats.add_tokens(trace_shard)
        self.stats._after_torch(buf)
        base = self._pk.data_ptr()
        N.check(N.lib().gimbal_pass_distributed_async(
            self.stats.handle, C.c_void_p(comm), self.threshold, self.top_e, m // topo.n_gpus, self.anchor_gpu,
            C.c_void_p(buf.data_ptr()), n_local, cand_offset, n_candidates, self.alpha, self.beta,
            C.c_void_p(scores.data_ptr()), C.c_void_p(self._gobj.data_ptr()), C.c_void_p(base),
            C.c_void_p(base + 24 + 4 * m), C.c_void_p(base + 24), C.c_void_p(base + 8), C.c_void_p(base + 16)),
            "pass_distributed")
        h = self._read_pk(extra=(self._gobj, self._gobj_host))
        n = int(h[2])
        objs = self._gobj_host.numpy()
        am = int(h[0:2].view(np.int64)[0])
        return HotPathResult(affinity=AffinitySet(experts=h[6:6 + n].tolist(), anchor_gpu=self.anchor_gpu),
                             greedy=h[6 + m:6 + 2 * m].tolist(), argmin=am,
                             objective=float(objs[am]) if am >= 0 else None)

    def _distributed_pass(self, trace_shard, candidates_shard, cand_offset: int, n_candidates: int,
                          group=None, M_fixed=None) -> HotPathResult:
        import torch
        import torch.distributed as dist

        topo = self.topo
        n_local = candidates_shard.shape[0]
        comm = nccl_comm(group, self.device)
        if (M_fixed is None and comm is not None and getattr(candidates_shard, "is_cuda", False)
                and topo.n_gpus <= 255):
            return self._distributed_queued(trace_shard, candidates_shard, cand_offset, n_candidates, comm)
        self.stats.reset()
        self.stats.add_tokens(trace_shard)
        allreduce_counts(self.stats, group)
        M = M_fixed if M_fixed is not None else build_affinity_set(
            self.stats, topo, self.threshold, self.top_e, topo.total_experts() // topo.n_gpus, self.anchor_gpu)
        # global candidate 0 is the greedy placement: written into the slice that holds it
        gp = greedy_place(self.stats, M, topo.n_gpus,
                          out_u8_device=candidates_shard[0] if (cand_offset == 0 and n_local > 0) else None)
        dev = torch.device("cuda", self.device)
        local = torch.full((n_candidates,), float("inf"), dtype=torch.float64, device=dev)
        if n_local:
            out, _ = eval_costs(self.stats, candidates_shard, self.alpha, self.beta, out=self._scores(n_local))
            local[cand_offset:cand_offset + n_local] = out[2]
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(local, op=dist.ReduceOp.MIN, group=group)
            objs = local.cpu().numpy()
        else:
            host = local.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.MIN, group=group)
            objs = host.numpy()
        return HotPathResult(affinity=M, greedy=gp.assign, argmin=merge_argmin(objs),
                             objective=float(objs.min()) if objs.size else None)
