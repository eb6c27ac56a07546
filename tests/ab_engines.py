"""Engine-specific parity cases for the alternate kernels that only the test/tool build
``lib/libgimbal_gpu_ab.so`` can select (experiment knobs, ``internal.cuh`` GIMBAL_KNOB).

The shipped ``libgimbal_gpu.so`` has no knobs: its kernel choice depends on the inputs alone.
``tests/test_gpu_engines.py`` runs each case below in a fresh process with
``GIMBAL_LIB=lib/libgimbal_gpu_ab.so`` and the case's knob set, and compares against the CPU
oracle like the rest of the parity suite.

    python tests/ab_engines.py <case> [args...]      # exit 0 = parity holds
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _setup():
    import torch

    import oracle
    import paper_2602_21626_b200 as G

    assert os.environ.get("GIMBAL_LIB", "").endswith("libgimbal_gpu_ab.so"), "run with the AB build"
    G._native.lib()
    return G, oracle.Oracle(), torch


def case_fp4(L: str, T: str, dup: str) -> None:
    """GIMBAL_COUNT_PATH=fp4: the block-scaled FP4 tensor-core counter, repeated ids included."""
    G, orc, torch = _setup()
    L, T, dup = int(L), int(T), dup == "1"
    ne, k = 256, 8
    topo = G.MoeTopology(L, ne, k, 8)
    rng = np.random.default_rng(T + L)
    ids = rng.integers(0, ne, size=(T, L, k), dtype=np.uint8)
    if dup:
        ids[::3, :, 1] = ids[::3, :, 0]
    s = G.RoutingStats(topo, 0)
    s.add_tokens(torch.from_numpy(ids).cuda())
    A, E, W = s.read()
    oA, oE, oW = orc.stats(L, ne, k, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


def case_eval(L: str, ne: str, k: str, g: str, C: str, alpha: str, beta: str) -> None:
    """GIMBAL_EVAL_ALU / GIMBAL_EVAL_NO_SMALL: the integer-ALU / generic evaluators agree with the
    oracle exactly (placement.cpp:58-85)."""
    G, orc, torch = _setup()
    L, ne, k, g, C = int(L), int(ne), int(k), int(g), int(C)
    alpha, beta = float(alpha), float(beta)
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 20011, model_seed=2, stream_seed=5, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    cands = G.shuffled_candidates(L * ne, g, 31, C)
    want = orc.eval_costs(L, ne, g, oA, oE, cands, alpha, beta)
    got = G.eval_costs(s, torch.from_numpy(cands).cuda(), alpha, beta)
    for a, b in zip(got[:3], want[:3]):
        assert np.array_equal(a, b)
    assert got[3] == want[3]


def case_count(L: str, ne: str, k: str, T: str) -> None:
    """Any counting-engine knob (GIMBAL_COUNT_PATH=atomic|lm8|split, GIMBAL_NO_DIRECT, GIMBAL_NO_TMA,
    GIMBAL_NO_SMALL, GIMBAL_TMA_MODE=u15, GIMBAL_TMA_AGG=...): bit-exact A / E / W."""
    G, orc, torch = _setup()
    L, ne, k, T = int(L), int(ne), int(k), int(T)
    topo = G.MoeTopology(L, ne, k, 8 if ne % 8 == 0 else 1)
    trace = G.generate_trace(topo, T, model_seed=7, stream_seed=3, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    A, E, W = s.read()
    oA, oE, oW = orc.stats(L, ne, k, trace.cpu().numpy(), n_threads=os.cpu_count() or 8)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


def case_pass(L: str, ne: str, k: str, g: str, C: str) -> None:
    """GIMBAL_NO_TINY_PASS: small shapes through the multi-launch pass (topk, select, greedy keys,
    sort, walk, evaluator, finish) instead of the fused kernel: same answers as the oracle."""
    G, orc, torch = _setup()
    L, ne, k, g, C = int(L), int(ne), int(k), int(g), int(C)
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 20011, model_seed=4, stream_seed=2, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 41, C)).cuda()
    hp = G.HotPath(topo, 0)
    res = hp.run(trace, cands)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    M = list(orc.affinity_set(L, ne, g, oE, 0.0, 4, L * ne // g, 0))
    greedy = orc.greedy_place(L, ne, g, oA, M, 0)
    want = cands.cpu().numpy()
    assert np.array_equal(want[0], greedy.astype(np.uint8))
    D, cut, obj, am = orc.eval_costs(L, ne, g, oA, oE, want)
    sc = hp._out.cpu().numpy()
    assert res.affinity.experts == M and res.greedy == list(greedy) and res.argmin == am
    assert np.array_equal(sc[0], D) and np.array_equal(sc[1], cut) and np.array_equal(sc[2], obj)


if __name__ == "__main__":
    globals()["case_" + sys.argv[1]](*sys.argv[2:])
    print("ok")
