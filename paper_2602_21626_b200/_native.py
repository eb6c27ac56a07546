"""ctypes binding of libgimbal_gpu.so (include/gimbal_gpu.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C paper_2602_21626_b200/csrc``).
There is no fallback: if the shared library is missing every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# GIMBAL_LIB selects another build of the same library (A/B kernel experiments on the GPU box)
LIB_PATH = os.environ.get("GIMBAL_LIB") or os.path.join(HERE, "lib", "libgimbal_gpu.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "gimbal_gpu.h")

ABI_VERSION = 4  # include/gimbal_gpu.h GIMBAL_ABI_VERSION
OK, INVALID_ARGUMENT, CUDA_ERROR, NCCL_ERROR, OVERFLOW, OUT_OF_RANGE, NOT_SUPPORTED = range(7)
MEM_HOST, MEM_DEVICE = 0, 1


class Topology(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("n_experts", C.c_int32), ("top_k", C.c_int32), ("n_gpus", C.c_int32)]


class GimbalError(RuntimeError):
    """CUDA / internal failure inside libgimbal_gpu."""


class NotSupportedError(GimbalError):
    pass


_P = C.c_void_p
_i32, _i64, _u64, _d = C.c_int32, C.c_int64, C.c_uint64, C.c_double
_TP = C.POINTER(Topology)

# (name, restype, argtypes) for every symbol declared in include/gimbal_gpu.h
SIGNATURES = [
    ("gimbal_abi_version", C.c_int, []),
    ("gimbal_last_error", C.c_char_p, []),
    ("gimbal_topology_validate", C.c_int, [_TP]),
    ("gimbal_stats_create", C.c_int, [_TP, C.c_int, C.POINTER(_P)]),
    ("gimbal_stats_destroy", C.c_int, [_P]),
    ("gimbal_stats_reset", C.c_int, [_P]),
    ("gimbal_stats_add_tokens", C.c_int, [_P, _P, C.c_int, _i64, C.c_int]),
    ("gimbal_stats_tokens", C.c_int, [_P, C.POINTER(_i64)]),
    ("gimbal_stats_read", C.c_int, [_P, _P, _P, _P, C.c_int]),
    ("gimbal_stats_flat", C.c_int, [_P, _P, _P, C.c_int]),
    ("gimbal_stats_device_buffers", C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    ("gimbal_stats_mark_reduced", C.c_int, [_P, _i64]),
    ("gimbal_stats_sync", C.c_int, [_P]),
    ("gimbal_stats_merge", C.c_int, [_P, _P, _i64, C.c_int]),
    ("gimbal_stats_count_timing", C.c_int, [_P, C.c_int, C.POINTER(_d), C.POINTER(_i64)]),
    ("gimbal_eval_costs", C.c_int, [_P, _P, _i64, C.c_int, _d, _d, _P, _P, _P, C.POINTER(_i64), C.c_int]),
    ("gimbal_eval_excess", C.c_int, [_P, _P, _i64, C.c_int, _P, C.c_int]),
    ("gimbal_affinity_set", C.c_int, [_P, _d, _i32, _i32, _i32, _P, C.POINTER(_i32)]),
    ("gimbal_greedy_place", C.c_int, [_P, _P, _i32, _i32, _P, C.c_int, _P]),
    ("gimbal_window_place_async", C.c_int, [_P, _P, _i32, _i32, _P, _i64, _d, _d, _P, _P, _P]),
    ("gimbal_stats_set_count_sms", C.c_int, [_P, C.c_int]),
    ("gimbal_pass_graph", C.c_int, [_P, _P, C.c_int, _i64, _d, _i32, _i32, _i32, _P, _i64, _d, _d, _P, _P, _P, _P, _P,
                                    _P]),
    ("gimbal_pass_async", C.c_int, [_P, _d, _i32, _i32, _i32, _P, _i64, _d, _d, _P, _P, _P, _P, _P, _P]),
    ("gimbal_pass_enqueue", C.c_int, [_P, _P, C.c_int, _i64, _d, _i32, _i32, _i32, _P, _i64, _d, _d, _P, _P, _P, _P,
                                      C.POINTER(_P)]),
    ("gimbal_dist_unique_id", C.c_int, [_P]),
    ("gimbal_dist_comm_init", C.c_int, [_i32, _i32, _P, C.c_int, C.POINTER(_P)]),
    ("gimbal_dist_comm_destroy", C.c_int, [_P]),
    ("gimbal_dist_comm_size", C.c_int, [_P, C.POINTER(_i32), C.POINTER(_i32)]),
    ("gimbal_stats_allreduce", C.c_int, [_P, _P, _i64]),
    ("gimbal_dist_merge_argmin", C.c_int, [_P, _P, _P, _i64, _i64, _i64, _P, _P]),
    ("gimbal_pass_distributed_async", C.c_int, [_P, _P, _d, _i32, _i32, _i32, _P, _i64, _i64, _i64, _d, _d, _P, _P, _P,
                                                _P, _P, _P, _P]),
    ("gimbal_online_create", C.c_int, [_P, C.POINTER(_P)]),
    ("gimbal_online_destroy", C.c_int, [_P]),
    ("gimbal_online_set_placement", C.c_int, [_P, _P, _i64]),
    ("gimbal_online_iteration", C.c_int, [_P, _P, C.c_int, _i64, C.POINTER(_d), C.POINTER(_i64)]),
    ("gimbal_online_gpu_totals", C.c_int, [_P, _P]),
    ("gimbal_exact_solve_dense", C.c_int, [_i32, _i32, _P, _P, _i32, _d, _d, _P, C.POINTER(_d), C.POINTER(_d),
                                           C.POINTER(_d)]),
    ("gimbal_eval_cost_dense", C.c_int, [_i32, _i32, _P, _P, _i32, _d, _d, _P, C.POINTER(_d), C.POINTER(_d),
                                         C.POINTER(_d)]),
    ("gimbal_affinity_set_dense", C.c_int, [_TP, _P, _i32, _d, _i32, _i32, _i32, _P, C.POINTER(_i32)]),
    ("gimbal_greedy_place_dense", C.c_int, [_i32, _i32, _P, _P, _i32, _i32, _i32, _P]),
    ("gimbal_static_placement", C.c_int, [_TP, _P]),
    ("gimbal_comm_cost", C.c_int, [_TP, _P, C.c_int, _i64, C.c_int, _P, _i32, C.c_int, C.POINTER(_i64)]),
    ("gimbal_generate_trace", C.c_int, [_TP, _d, _d, _d, _u64, _u64, _d, _u64, _i64, _i64, _P, C.c_int]),
    ("gimbal_generator_tables", C.c_int, [_TP, _d, _d, _d, _u64, _d, _u64, _P, _P]),
    ("gimbal_shuffled_candidates", C.c_int, [_i32, _i32, _u64, _i64, _P]),
]

_lock = threading.Lock()
_LIB = None


def lib() -> C.CDLL:
    """Loads libgimbal_gpu.so (raises if it was not built — there is no CPU fallback)."""
    global _LIB
    with _lock:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                                  f"g.build()'` (make -C paper_2602_21626_b200/csrc)")
            L = C.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            got = L.gimbal_abi_version()
            if got != ABI_VERSION:
                # an older build would ignore arguments this binding passes (e.g. ABI 2's flags_out
                # of gimbal_pass_async) and silently drop device-side errors
                raise ImportError(f"{LIB_PATH}: ABI version {got}, this binding needs {ABI_VERSION} "
                                  f"(include/gimbal_gpu.h GIMBAL_ABI_VERSION); rebuild the library")
            _LIB = L
        return _LIB


def last_error() -> str:
    msg = lib().gimbal_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    msg = last_error()
    text = msg or what
    if status == INVALID_ARGUMENT:
        raise ValueError(text)  # the reference raises std::invalid_argument
    if status == OUT_OF_RANGE:
        raise IndexError(text)
    if status == OVERFLOW:
        raise OverflowError(text)
    if status == NOT_SUPPORTED:
        raise NotSupportedError(text)
    raise GimbalError(f"{what}: status {status}: {text}")
