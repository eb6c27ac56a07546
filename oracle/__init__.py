"""CPU oracle for the expert-statistics + placement hot path — TEST INFRASTRUCTURE ONLY.

Two layers:

* ``Ref``    — the reference's own ``proj/src/moe.cpp`` + ``proj/src/placement.cpp`` compiled
               unchanged (Eigen subset in ``oracle/eigen_subset``) into ``oracle/_ref/libgimbal_ref.so``.
* ``Oracle`` — the restated plain-C oracle ``oracle/gimbal_oracle.c`` (u64 counts, threaded),
               pinned against ``Ref`` and the reference's golden KATs; used at full sizes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "libgimbal_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgimbal_ref.so")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def build(quiet: bool = True) -> None:
    """make -C oracle (C oracle always; the reference build only where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def _ids(ids: np.ndarray):
    ids = np.ascontiguousarray(ids)
    if ids.dtype == np.uint8:
        return ids, 1
    if ids.dtype == np.int32:
        return ids, 4
    raise TypeError("ids must be uint8 or int32")


class OracleError(RuntimeError):
    pass


class Oracle:
    """ctypes view of oracle/lib/libgimbal_oracle.so (restated C oracle)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.go_stats.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, _i64, C.c_int, _u64p, _u64p]
        L.go_w_from_e.argtypes = [C.c_int, C.c_int, _u64p, _u64p]
        L.go_w_from_e.restype = None
        L.go_comm_cost.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, _i64, _i32p, C.c_int,
                                   C.c_int, _i64p]
        L.go_eval_cost.argtypes = [C.c_int, C.c_int, C.c_int, _u64p, _u64p, _i32p, C.c_double, C.c_double,
                                   _dp, _dp, _dp]
        L.go_eval_costs.argtypes = [C.c_int, C.c_int, C.c_int, _u64p, _u64p, _u8p, _i64, C.c_double,
                                    C.c_double, _f64p, _f64p, _f64p, _i64p]
        L.go_eval_cost_dense.argtypes = [C.c_int, C.c_int, _f64p, _f64p, C.c_int, C.c_double, C.c_double,
                                         _i32p, _dp, _dp, _dp]
        L.go_affinity_set.argtypes = [C.c_int, C.c_int, C.c_int, _u64p, C.c_double, C.c_int, C.c_int,
                                      C.c_int, _i32p, C.POINTER(C.c_int)]
        L.go_greedy_place.argtypes = [C.c_int, C.c_int, C.c_int, _u64p, _i32p, C.c_int, C.c_int, _i32p]
        L.go_static_placement.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        L.go_generate_trace.argtypes = [C.c_int, C.c_int, C.c_int, _u32p, C.c_uint64, C.c_uint64,
                                        C.c_uint64, _i64, _i64, _u8p]
        L.go_check_feasible.argtypes = [C.c_int, C.c_int, _i32p]
        L.go_eval_costs_mt.argtypes = [C.c_int, C.c_int, C.c_int, _u64p, _u64p, _u8p, _i64, C.c_double,
                                       C.c_double, _f64p, _f64p, _f64p, _i64p, C.c_int]
        L.go_eval_excess.argtypes = [C.c_int, C.c_int, C.c_int, _u64p, _u8p, _i64, _f64p]
        L.go_generate_trace_mt.argtypes = [C.c_int, C.c_int, C.c_int, _u32p, C.c_uint64, C.c_uint64,
                                           C.c_uint64, _i64, _i64, _u8p, C.c_int]

    @staticmethod
    def _ok(st: int, what: str):
        if st == 1:
            raise ValueError(f"{what}: invalid argument")
        if st == 5:
            raise ValueError(f"{what}: expert id out of range")
        if st != 0:
            raise OracleError(f"{what}: status {st}")

    def stats(self, L, ne, k, ids, n_threads: int = 8):
        ids, ib = _ids(ids)
        T = ids.size // (L * k)
        A = np.zeros(L * ne, np.uint64)
        E = np.zeros(max(L - 1, 0) * ne * ne if L > 1 else 1, np.uint64)
        self._ok(self.lib.go_stats(L, ne, k, ids.ctypes.data, ib, T, n_threads, A, E), "stats")
        A = A.reshape(L, ne)
        E = E[: (L - 1) * ne * ne].reshape(L - 1, ne, ne)
        W = E.sum(axis=0, dtype=np.uint64) if L > 1 else np.zeros((ne, ne), np.uint64)
        return A, E, W

    def comm_cost(self, L, ne, k, ids, assign, n_threads: int = 8) -> int:
        ids, ib = _ids(ids)
        T = ids.size // (L * k)
        a = np.ascontiguousarray(assign, np.int32)
        out = C.c_int64(0)
        self._ok(self.lib.go_comm_cost(L, ne, k, ids.ctypes.data, ib, T, a, a.size, n_threads, C.byref(out)),
                 "comm_cost")
        return out.value

    def eval_cost(self, L, ne, g, A, E, assign, alpha=1.0, beta=1.0):
        A = np.ascontiguousarray(A, np.uint64).ravel()
        E = np.ascontiguousarray(E, np.uint64).ravel()
        if E.size == 0:
            E = np.zeros(1, np.uint64)
        a = np.ascontiguousarray(assign, np.int32)
        D, c, o = C.c_double(), C.c_double(), C.c_double()
        self._ok(self.lib.go_eval_cost(L, ne, g, A, E, a, alpha, beta, C.byref(D), C.byref(c), C.byref(o)),
                 "eval_cost")
        return D.value, c.value, o.value

    def eval_costs(self, L, ne, g, A, E, cands, alpha=1.0, beta=1.0, n_threads: int = 1):
        A = np.ascontiguousarray(A, np.uint64).ravel()
        E = np.ascontiguousarray(E, np.uint64).ravel()
        if E.size == 0:
            E = np.zeros(1, np.uint64)
        cands = np.ascontiguousarray(cands, np.uint8)
        Cn = cands.shape[0]
        D, cut, obj = (np.zeros(Cn) for _ in range(3))
        am = C.c_int64(-1)
        if n_threads > 1:
            self._ok(self.lib.go_eval_costs_mt(L, ne, g, A, E, cands, Cn, alpha, beta, D, cut, obj, C.byref(am),
                                               n_threads), "eval_costs")
        else:
            self._ok(self.lib.go_eval_costs(L, ne, g, A, E, cands, Cn, alpha, beta, D, cut, obj, C.byref(am)),
                     "eval_costs")
        return D, cut, obj, am.value

    def eval_excess(self, L, ne, g, A, cands):
        A = np.ascontiguousarray(A, np.uint64).ravel()
        cands = np.ascontiguousarray(cands, np.uint8)
        out = np.zeros(cands.shape[0])
        self._ok(self.lib.go_eval_excess(L, ne, g, A, cands, cands.shape[0], out), "eval_excess")
        return out

    def eval_cost_dense(self, A, W, g, assign, alpha=1.0, beta=1.0):
        A = np.ascontiguousarray(A, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        a = np.ascontiguousarray(assign, np.int32)
        D, c, o = C.c_double(), C.c_double(), C.c_double()
        self._ok(self.lib.go_eval_cost_dense(A.shape[0], A.shape[1], A, W, g, alpha, beta, a, C.byref(D),
                                             C.byref(c), C.byref(o)), "eval_cost_dense")
        return D.value, c.value, o.value

    def affinity_set(self, L, ne, g, E, threshold=0.0, top_e=4, capacity=None, anchor=0):
        E = np.ascontiguousarray(E, np.uint64).ravel()
        if E.size == 0:
            E = np.zeros(1, np.uint64)
        if capacity is None:
            capacity = L * ne // g
        n_out = C.c_int(0)
        out = np.zeros(max(1, 2 * max(top_e, 0) if top_e >= 0 else 2 * E.size), np.int32)
        if top_e < 0:
            out = np.zeros(L * ne, np.int32)
        self._ok(self.lib.go_affinity_set(L, ne, g, E, threshold, top_e, capacity, anchor, out, C.byref(n_out)),
                 "affinity_set")
        return out[: n_out.value].copy()

    def greedy_place(self, L, ne, g, A, M=(), anchor=0):
        A = np.ascontiguousarray(A, np.uint64).ravel()
        Mv = np.ascontiguousarray(np.asarray(M, np.int32).ravel())
        if Mv.size == 0:
            Mv = np.zeros(1, np.int32)
            nM = 0
        else:
            nM = Mv.size
        out = np.zeros(L * ne, np.int32)
        self._ok(self.lib.go_greedy_place(L, ne, g, A, Mv, nM, anchor, out), "greedy_place")
        return out

    def static_placement(self, L, ne, k, g):
        out = np.zeros(L * ne, np.int32)
        self._ok(self.lib.go_static_placement(L, ne, k, g, out), "static_placement")
        return out

    def generate_trace(self, L, ne, k, cdf, thr_base, thr_unif, seed, t0, T, n_threads: int = 1):
        out = np.zeros(T * L * k, np.uint8)
        cdf = np.ascontiguousarray(cdf, np.uint32).ravel()
        self._ok(self.lib.go_generate_trace_mt(L, ne, k, cdf, thr_base, thr_unif, seed, t0, T, out, n_threads),
                 "generate_trace")
        return out.reshape(T, L, k)

    def stats_accumulate(self, L, ne, k, ids, A, E, n_threads: int = 8) -> None:
        """Adds a trace chunk's counts into A [L][n_e] / E [(L-1)][n_e][n_e] (uint64, C-contiguous,
        updated in place): the incremental form of RoutingStats::add_token used to check
        BASELINE-size GPU counts chunk by chunk."""
        ids, ib = _ids(ids)
        T = ids.size // (L * k)
        assert A.dtype == np.uint64 and E.dtype == np.uint64 and A.flags.c_contiguous and E.flags.c_contiguous
        self._ok(self.lib.go_stats(L, ne, k, ids.ctypes.data, ib, T, n_threads, A.reshape(-1),
                                   E.reshape(-1) if E.size else np.zeros(1, np.uint64)), "stats")


class Ref:
    """ctypes view of oracle/_ref/libgimbal_ref.so (the reference's own sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (build with `make -C oracle` where /root/reference exists)")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_record_stats.argtypes = [C.c_int] * 4 + [C.c_void_p, C.c_int, _i64, _f64p, _f64p, _f64p, _i64p]
        L.ref_flat_forms.argtypes = [C.c_int] * 4 + [C.c_void_p, C.c_int, _i64, _f64p, _f64p]
        L.ref_comm_cost.argtypes = [C.c_int] * 4 + [C.c_void_p, C.c_int, _i64, _i32p, C.c_int, _i64p]
        L.ref_eval_cost.argtypes = [C.c_int, C.c_int, _f64p, _f64p, C.c_int, C.c_double, C.c_double, _i32p,
                                    C.c_int, _dp, _dp, _dp]
        L.ref_exact_solve.argtypes = [C.c_int, C.c_int, _f64p, _f64p, C.c_int, C.c_double, C.c_double, _i32p,
                                      _dp, _dp, _dp]
        L.ref_build_affinity_set.argtypes = [C.c_int] * 4 + [_f64p, C.c_int, C.c_double, C.c_int, C.c_int,
                                                              C.c_int, _i32p, C.POINTER(C.c_int)]
        L.ref_greedy_place.argtypes = [C.c_int, C.c_int, _f64p, _i32p, C.c_int, C.c_int, C.c_int, _i32p]
        L.ref_maybe_relocate.argtypes = [_i64, _i64, _i32p, C.c_int, C.c_int, C.c_int, C.c_int, _f64p, C.c_int,
                                         _i32p, C.c_int, _i32p, _i64p, C.POINTER(C.c_int)]
        L.ref_static_placement.argtypes = [C.c_int] * 4 + [_i32p]
        L.ref_route_tokens.argtypes = [C.c_int] * 4 + [C.c_double] * 3 + [C.c_uint64, C.c_uint64, _i64, _i32p]
        L.ref_model_weights.argtypes = [C.c_int] * 4 + [C.c_double] * 3 + [C.c_uint64, _f64p, _f64p]
        L.ref_pipeline.argtypes = [C.c_int] * 4 + [_u8p, _i64, C.c_int, _u8p, C.c_int, C.c_double, C.c_int,
                                                    C.c_int, C.c_double, C.c_double, _f64p, _i64p, _i32p, _f64p]
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_shuffled_balanced.argtypes = [C.c_int, C.c_int, C.c_uint64, _i32p]
        L.ref_shuffled_balanced.restype = None
        L.ref_hook_create.argtypes = [C.c_int] * 4 + [_i32p]
        L.ref_hook_create.restype = C.c_void_p
        L.ref_hook_destroy.argtypes = [C.c_void_p]
        L.ref_hook_destroy.restype = None
        L.ref_hook_set_placement.argtypes = [C.c_void_p, _i32p]
        L.ref_hook_set_placement.restype = None
        L.ref_hook_reset_window.argtypes = [C.c_void_p]
        L.ref_hook_reset_window.restype = None
        L.ref_hook_iteration.argtypes = [C.c_void_p, _i32p, _i64, _dp, _i64p]
        L.ref_hook_stats.argtypes = [C.c_void_p, _f64p, _f64p, _i64p]

    def _ok(self, st):
        if st != 0:
            raise ValueError(self.lib.ref_last_error().decode())

    def record_stats(self, L, ne, k, g, ids):
        ids, ib = _ids(ids)
        T = ids.size // (L * k)
        A = np.zeros(L * ne)
        E = np.zeros(max(L - 1, 1) * ne * ne)
        W = np.zeros(ne * ne)
        tok = C.c_int64(0)
        self._ok(self.lib.ref_record_stats(L, ne, k, g, ids.ctypes.data, ib, T, A, E, W, C.byref(tok)))
        return A.reshape(L, ne), E[: (L - 1) * ne * ne].reshape(L - 1, ne, ne), W.reshape(ne, ne), tok.value

    def flat_forms(self, L, ne, k, g, ids):
        ids, ib = _ids(ids)
        T = ids.size // (L * k)
        m = L * ne
        fA = np.zeros(L * m)
        fW = np.zeros(m * m)
        self._ok(self.lib.ref_flat_forms(L, ne, k, g, ids.ctypes.data, ib, T, fA, fW))
        return fA.reshape(L, m), fW.reshape(m, m)

    def comm_cost(self, L, ne, k, g, ids, assign):
        ids, ib = _ids(ids)
        T = ids.size // (L * k)
        a = np.ascontiguousarray(assign, np.int32)
        out = C.c_int64(0)
        self._ok(self.lib.ref_comm_cost(L, ne, k, g, ids.ctypes.data, ib, T, a, a.size, C.byref(out)))
        return out.value

    def eval_cost(self, A, W, g, assign, alpha=1.0, beta=1.0):
        A = np.ascontiguousarray(A, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        a = np.ascontiguousarray(assign, np.int32)
        D, c, o = C.c_double(), C.c_double(), C.c_double()
        self._ok(self.lib.ref_eval_cost(A.shape[0], A.shape[1], A, W, g, alpha, beta, a, a.size, C.byref(D),
                                        C.byref(c), C.byref(o)))
        return D.value, c.value, o.value

    def exact_solve(self, A, W, g, alpha=1.0, beta=1.0):
        """placement::exact_solve -> (assign, (D, cut, objective))."""
        A = np.ascontiguousarray(np.atleast_2d(A), np.float64)
        W = np.ascontiguousarray(W, np.float64)
        a = np.zeros(A.shape[1], np.int32)
        D, c, o = C.c_double(), C.c_double(), C.c_double()
        self._ok(self.lib.ref_exact_solve(A.shape[0], A.shape[1], A, W, g, alpha, beta, a, C.byref(D), C.byref(c),
                                          C.byref(o)))
        return a, (D.value, c.value, o.value)

    def build_affinity_set(self, L, ne, k, g, E, threshold=0.0, top_e=4, capacity=None, anchor=0):
        E = np.ascontiguousarray(E, np.float64).ravel()
        nb = E.size // (ne * ne)
        if E.size == 0:
            E = np.zeros(1)
        if capacity is None:
            capacity = L * ne // g
        out = np.zeros(L * ne + 2 * max(top_e, 0) + 2, np.int32)
        n = C.c_int(0)
        self._ok(self.lib.ref_build_affinity_set(L, ne, k, g, E, nb, threshold, top_e, capacity, anchor, out,
                                                 C.byref(n)))
        return out[: n.value].copy()

    def greedy_place(self, act, g, M=(), anchor=0):
        act = np.ascontiguousarray(act, np.float64)
        Mv = np.ascontiguousarray(np.asarray(M, np.int32).ravel())
        nM = Mv.size
        if nM == 0:
            Mv = np.zeros(1, np.int32)
        out = np.zeros(act.shape[1], np.int32)
        self._ok(self.lib.ref_greedy_place(act.shape[0], act.shape[1], act, Mv, nM, anchor, g, out))
        return out

    def maybe_relocate(self, step, tau, M, anchor, act, g, prev):
        act = np.ascontiguousarray(act, np.float64)
        Mv = np.ascontiguousarray(np.asarray(M, np.int32).ravel())
        nM = Mv.size
        if nM == 0:
            Mv = np.zeros(1, np.int32)
        pv = np.ascontiguousarray(np.asarray(prev, np.int32).ravel())
        npv = pv.size
        if npv == 0:
            pv = np.zeros(1, np.int32)
        out = np.zeros(act.shape[1], np.int32)
        moved = C.c_int64(0)
        fired = C.c_int(0)
        self._ok(self.lib.ref_maybe_relocate(step, tau, Mv, nM, anchor, act.shape[0], act.shape[1], act, g, pv,
                                             npv, out, C.byref(moved), C.byref(fired)))
        return (out, moved.value) if fired.value else None

    def static_placement(self, L, ne, k, g):
        out = np.zeros(L * ne, np.int32)
        self._ok(self.lib.ref_static_placement(L, ne, k, g, out))
        return out

    def route_tokens(self, L, ne, k, g, T, model_seed, rng_seed, zipf_s=1.2, lam=0.5, peak=0.8):
        out = np.zeros(T * L * k, np.int32)
        self._ok(self.lib.ref_route_tokens(L, ne, k, g, zipf_s, lam, peak, model_seed, rng_seed, T, out))
        return out.reshape(T, L, k)

    def model_weights(self, L, ne, k, g, model_seed, zipf_s=1.2, lam=0.5, peak=0.8):
        base = np.zeros(L * ne)
        kern = np.zeros(ne * ne)
        self._ok(self.lib.ref_model_weights(L, ne, k, g, zipf_s, lam, peak, model_seed, base, kern))
        return base.reshape(L, ne), kern.reshape(ne, ne)

    def pipeline(self, L, ne, k, g, ids, cands, n_threads=1, threshold=0.0, top_e=4, anchor=0, alpha=1.0,
                 beta=1.0):
        ids = np.ascontiguousarray(ids, np.uint8)
        T = ids.size // (L * k)
        cands = np.ascontiguousarray(cands, np.uint8)
        Cn = cands.shape[0]
        obj = np.zeros(max(Cn, 1))
        am = C.c_int64(-1)
        gr = np.zeros(L * ne, np.int32)
        t = np.zeros(4)
        self._ok(self.lib.ref_pipeline(L, ne, k, g, ids, T, n_threads, cands if Cn else np.zeros(1, np.uint8), Cn,
                                       threshold, top_e, anchor, alpha, beta, obj, C.byref(am), gr, t))
        return {"objectives": obj[:Cn], "argmin": am.value, "greedy": gr, "t_stats": t[0], "t_place": t[1],
                "t_eval": t[2], "t_total": t[3]}

    # ---- MoeSubsystem::iteration_cost's per-token work (sim.cpp:113-147) over the reference's
    # RoutingStats: oracle and host-timing baseline of the GPU hook (ref_capi.cpp ref_hook_*)
    def hook_create(self, L, ne, k, g, assign):
        a = np.ascontiguousarray(np.asarray(assign, np.int32))
        return C.c_void_p(self.lib.ref_hook_create(L, ne, k, g, a))

    def hook_destroy(self, h):
        self.lib.ref_hook_destroy(h)

    def hook_set_placement(self, h, assign):
        self.lib.ref_hook_set_placement(h, np.ascontiguousarray(np.asarray(assign, np.int32)))

    def hook_iteration(self, h, ids):
        a = np.ascontiguousarray(np.asarray(ids, np.int32))
        ex, cr = C.c_double(), C.c_int64()
        self._ok(self.lib.ref_hook_iteration(h, a, a.shape[0] if a.ndim > 1 else 0, C.byref(ex), C.byref(cr)))
        return ex.value, cr.value

    def hook_stats(self, h, L, ne, g):
        A = np.zeros(L * ne)
        E = np.zeros(max(L - 1, 1) * ne * ne)
        t = np.zeros(g, np.int64)
        self._ok(self.lib.ref_hook_stats(h, A, E, t.ctypes.data_as(_i64p)))
        return A.reshape(L, ne), E[: (L - 1) * ne * ne].reshape(L - 1, ne, ne), t

    def hook_reset_window(self, h):
        self.lib.ref_hook_reset_window(h)

    def mix_seed(self, seed, stream):
        return self.lib.ref_mix_seed(seed, stream)

    def shuffled_balanced(self, m, g, seed):
        out = np.zeros(m, np.int32)
        self.lib.ref_shuffled_balanced(m, g, seed, out)
        return out


def generator_tables_from_ref(ref: "Ref", L, ne, k, g, model_seed=1, zipf_s=1.2, lam=0.5, peak=0.8):
    """The trace generator's tables (cdf [L][n_e] u32, thresholds [2] u64; gimbal_gpu.h
    gimbal_generator_tables, drift 0) restated from the REFERENCE's RoutingModel weights
    (moe.cpp:43-78 via ref_model_weights): cdf = floor(2^32 x running sum of the normalised base
    row), the last entry saturated; thr = the base / uniform / successor component boundaries
    (1 - lambda, + lambda x rest x n_e) scaled to 2^32.  Lets the --impl reference leg build its
    inputs from the reference alone (no product library in that process)."""
    base, _ = ref.model_weights(L, ne, k, g, model_seed, zipf_s, lam, peak)
    two32 = 4294967296.0
    cdf = np.zeros((L, ne), np.uint32)
    for l in range(L):
        cum = 0.0
        for e in range(ne):
            cum += float(base[l, e])
            q = np.floor(cum * two32)
            cdf[l, e] = 0xFFFFFFFF if (e == ne - 1 or q >= 4294967295.0) else int(q)
    rest = (1.0 - peak) / (ne - 1) if ne > 1 else 0.0
    pb = 1.0 - lam
    pu = lam * rest * ne
    thr = np.array([min(two32, np.floor(pb * two32 + 0.5)), min(two32, np.floor((pb + pu) * two32 + 0.5))],
                   np.float64).astype(np.uint64)
    if lam == 0.0:
        thr[:] = np.uint64(1 << 32)
    return cdf, thr


def ref_available() -> bool:
    return os.path.exists(REF_SO)
