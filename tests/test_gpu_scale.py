"""Bit-exact parity at BASELINE token counts.

Every production scheduling path is compared cell by cell against the multi-threaded C oracle
(oracle/gimbal_oracle.c, pinned to the reference by tests/test_oracle.py) at the sizes the bench
runs: the DS-V3 counter past its whole-unit-round threshold (16 Mi tokens: 32 chunks x 57 pairs =
12 full rounds of 148 CTAs + the stream-K tail), the Qwen3 tensor-core counter at 32 Mi, the
DS-V2-Lite stacked tensor-core counter at 16 Mi, Mixtral at 1 Mi with C = 4096, and whole 1 Mi-token
streaming windows.  Compared: A, E, W, the strong-pair set M, the greedy placement, D / cut /
objective of every candidate and the argmin (reference: moe.cpp:169-231, placement.cpp:58-85,
186-299).  The trace is generated on the GPU and copied to the host chunk by chunk for the oracle.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8
CHUNK = 1 << 20


def oracle_counts(orc, trace, L, ne, k):
    """A, E, W of a device trace, counted by the oracle over host chunks."""
    A = np.zeros((L, ne), np.uint64)
    E = np.zeros((max(L - 1, 0), ne, ne), np.uint64)
    for lo in range(0, trace.shape[0], CHUNK):
        orc.stats_accumulate(L, ne, k, trace[lo:lo + CHUNK].cpu().numpy(), A, E, n_threads=THREADS)
    return A, E, E.sum(axis=0, dtype=np.uint64)


def oracle_pass(orc, L, ne, k, g, A, E, cands, top_e=4, M=None):
    """The reference pass on oracle counts: strong-pair set (threshold 0, top_e, capacity m/g,
    anchor 0: sim.hpp:37-38, sim.cpp:100-102), greedy as candidate 0, every candidate scored."""
    if M is None:
        M = orc.affinity_set(L, ne, g, E, 0.0, top_e, L * ne // g, 0)
    greedy = orc.greedy_place(L, ne, g, A, M, 0)
    c = cands.copy()
    c[0] = greedy
    D, cut, obj, am = orc.eval_costs(L, ne, g, A, E, c, n_threads=THREADS)
    return list(M), list(greedy), (D, cut, obj), am


@pytest.mark.parametrize("name,L,ne,k,g,T,C", [
    ("dsv3", 58, 256, 8, 8, 16 << 20, 4096),
    ("qwen3", 48, 128, 8, 8, 32 << 20, 1024),
    ("dsv2lite", 26, 64, 6, 8, 16 << 20, 4096),
    ("mixtral", 32, 8, 2, 8, 1 << 20, 4096),
])
def test_baseline_size_pass_bit_exact(G, orc, name, L, ne, k, g, T, C):
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, T, model_seed=1, stream_seed=2, device=0)
    cands_np = G.shuffled_candidates(L * ne, g, 1000, C)
    cands = torch.from_numpy(cands_np).cuda()
    hp = G.HotPath(topo, 0)
    res = hp.run(trace, cands)
    A, E, W = hp.stats.read()
    scores = hp._out.cpu().numpy()
    assert hp.stats.tokens() == T

    oA, oE, oW = oracle_counts(orc, trace, L, ne, k)
    assert np.array_equal(A, oA), f"{name}: A differs"
    assert np.array_equal(E, oE), f"{name}: E differs in {(E != oE).sum()} cells"
    assert np.array_equal(W, oW)
    M, greedy, (D, cut, obj), am = oracle_pass(orc, L, ne, k, g, oA, oE, cands_np)
    assert res.affinity.experts == M
    assert res.greedy == greedy
    assert np.array_equal(cands[0].cpu().numpy(), np.asarray(greedy, np.uint8))
    assert np.array_equal(scores[0], D) and np.array_equal(scores[1], cut) and np.array_equal(scores[2], obj)
    assert res.argmin == am


def test_stream_full_windows_bit_exact(G, orc):
    """Two whole 1 Mi-token DS-V3 windows with drift (config 5), M fixed from a calibration window:
    each window's greedy, all 256 scores and the argmin, queued through HotPath.stream."""
    L, ne, k, g, C = 58, 256, 8, 8, 256
    topo = G.MoeTopology(L, ne, k, g)
    win = 1 << 20
    windows = [G.generate_trace(topo, win, model_seed=1, stream_seed=2, first_token=w * win, drift=0.05,
                                drift_epoch=w + 1, device=0) for w in range(2)]
    calib = G.generate_trace(topo, 20000, model_seed=1, stream_seed=3, drift=0.05, drift_epoch=0, device=0)
    cands_np = G.shuffled_candidates(L * ne, g, 1000, C)
    hp = G.HotPath(topo, 0)
    Mset = hp.calibrate(calib)
    cA, cE, _ = oracle_counts(orc, calib, L, ne, k)
    assert Mset.experts == list(orc.affinity_set(L, ne, g, cE, 0.0, 4, L * ne // g, 0))
    out = hp.stream(windows, torch.from_numpy(cands_np).cuda(), Mset)
    scores = hp._window_scores.cpu().numpy()
    prev = None
    for w in range(2):
        oA, oE, _ = oracle_counts(orc, windows[w], L, ne, k)
        _, greedy, (D, cut, obj), am = oracle_pass(orc, L, ne, k, g, oA, oE, cands_np, M=Mset.experts)
        argmin, moved, gp = out[w]
        assert list(gp) == greedy
        assert np.array_equal(scores[w, 0], D) and np.array_equal(scores[w, 1], cut)
        assert np.array_equal(scores[w, 2], obj)
        assert argmin == am
        want_moved = len(greedy) if prev is None else int(np.count_nonzero(np.asarray(prev) != np.asarray(greedy)))
        assert moved == want_moved
        prev = greedy
