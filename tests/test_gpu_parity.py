"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on the same inputs.

Bar: bit-exact for counts, sets, placements and argmin; placement costs exact (integer-valued
doubles; the north_star tolerance is 1e-6 relative, asserted where inputs are non-integer).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = {
    # name: (L, n_e, k, g)
    "mixtral": (32, 8, 2, 8),
    "dsv2lite": (26, 64, 6, 8),
    "qwen3": (48, 128, 8, 8),
    "dsv3": (58, 256, 8, 8),
}


def _stats_gpu(G, topo, trace):
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    return s, s.read()


@pytest.mark.parametrize("shape", list(SHAPES))
def test_stats_generated_trace_matches_oracle(G, orc, shape):
    L, ne, k, g = SHAPES[shape]
    topo = G.MoeTopology(L, ne, k, g)
    T = 20000 + 37  # ragged: not a multiple of any tile
    trace = G.generate_trace(topo, T, model_seed=3, stream_seed=5, device=0)
    _, (A, E, W) = _stats_gpu(G, topo, trace)
    oA, oE, oW = orc.stats(L, ne, k, trace.cpu().numpy())
    assert np.array_equal(A, oA)
    assert np.array_equal(E, oE)
    assert np.array_equal(W, oW)


def test_stats_host_pageable_pinned_int32_agree(G, orc):
    L, ne, k, g = SHAPES["qwen3"]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 5000, model_seed=9, stream_seed=1, device=0)
    host = trace.cpu().numpy()
    oA, oE, _ = orc.stats(L, ne, k, host)
    for ids in (host, host.astype(np.int32), torch.from_numpy(host).pin_memory(), trace.to(torch.int32)):
        s = G.RoutingStats(topo, 0)
        s.add_tokens(ids)
        A, E, _ = s.read()
        assert np.array_equal(A, oA) and np.array_equal(E, oE)
        assert s.tokens() == 5000


def test_stats_incremental_equals_one_shot_and_reset(G, orc):
    L, ne, k, g = SHAPES["dsv2lite"]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 9000, model_seed=2, stream_seed=2, device=0)
    s = G.RoutingStats(topo, 0)
    for lo, hi in ((0, 1), (1, 4000), (4000, 4000), (4000, 9000)):
        s.add_tokens(trace[lo:hi])
    A, E, W = s.read()
    oA, oE, oW = orc.stats(L, ne, k, trace.cpu().numpy())
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)
    s.reset()
    A, E, W = s.read()
    assert A.sum() == 0 and E.sum() == 0 and W.sum() == 0 and s.tokens() == 0


def test_duplicates_counted_with_multiplicity(G, orc):
    # the reference counts every k x k pairing, repeated ids included (moe.cpp:176-187)
    topo = G.MoeTopology(3, 16, 4, 2)
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 3, size=(3000, 3, 4), dtype=np.uint8)  # heavy repetition
    _, (A, E, W) = _stats_gpu(G, topo, ids)
    oA, oE, oW = orc.stats(3, 16, 4, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


@pytest.mark.parametrize("L,ne,k", [(1, 8, 2), (2, 4, 1), (5, 6, 3), (7, 300, 5), (4, 24, 11)])
def test_stats_odd_shapes(G, orc, L, ne, k):
    topo = G.MoeTopology(L, ne, k, 2 if ne % 2 == 0 else 1)
    rng = np.random.default_rng(L * 1000 + ne)
    ids = rng.integers(0, ne, size=(4099, L, k)).astype(np.int32 if ne > 256 else np.uint8)
    _, (A, E, W) = _stats_gpu(G, topo, ids)
    oA, oE, oW = orc.stats(L, ne, k, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


def test_zero_tokens(G):
    topo = G.MoeTopology(3, 4, 2, 2)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(np.zeros((0, 3, 2), np.uint8))
    A, E, W = s.read()
    assert A.sum() == 0 and W.sum() == 0 and s.tokens() == 0


def test_out_of_range_id_is_an_error(G):
    topo = G.MoeTopology(2, 4, 1, 2)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(np.array([[[0], [4]]], np.uint8))
    with pytest.raises(IndexError):
        s.read()
    s2 = G.RoutingStats(topo, 0)
    s2.add_tokens(np.array([[[0], [-1]]], np.int32))
    with pytest.raises(IndexError):
        s2.read()


@pytest.mark.parametrize("shape", list(SHAPES))
def test_placement_pipeline_matches_oracle(G, orc, shape):
    L, ne, k, g = SHAPES[shape]
    topo = G.MoeTopology(L, ne, k, g)
    T, C = 30000, 70
    trace = G.generate_trace(topo, T, model_seed=4, stream_seed=8, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 123, C)).cuda()
    hp = G.HotPath(topo, 0)
    res = hp.run(trace, cands)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    M = orc.affinity_set(L, ne, g, oE, 0.0, 4)
    assert res.affinity.experts == list(M)
    gp = orc.greedy_place(L, ne, g, oA, M, 0)
    assert res.greedy == list(gp)
    hc = cands.cpu().numpy()
    D, cut, obj, am = orc.eval_costs(L, ne, g, oA, oE, hc)
    got = hp._out.cpu().numpy()
    assert np.array_equal(got[0], D) and np.array_equal(got[1], cut) and np.array_equal(got[2], obj)
    assert res.argmin == am


@pytest.mark.parametrize("threshold,top_e,cap", [(0.0, 4, None), (0.0, -1, None), (50.0, 16, 7), (1e12, 4, None),
                                                 (0.0, 0, None), (0.0, 64, 3), (3.0, 1000, None)])
def test_affinity_set_variants(G, orc, threshold, top_e, cap):
    L, ne, k, g = SHAPES["dsv2lite"]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 3000, model_seed=6, stream_seed=6, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    _, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    capacity = L * ne // g if cap is None else cap
    got = G.build_affinity_set(s, topo, threshold, top_e, capacity, 1).experts
    want = orc.affinity_set(L, ne, g, oE, threshold, top_e, capacity, 1)
    assert got == list(want)


def test_greedy_with_anchor_and_eval_alpha_beta(G, orc):
    L, ne, k, g = SHAPES["qwen3"]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 8000, model_seed=12, stream_seed=3, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    M = [3, 200, 517, 4000]
    gp = G.greedy_place(s, G.AffinitySet(M, 5), g)
    assert gp.assign == list(orc.greedy_place(L, ne, g, oA, M, 5))
    cands = G.shuffled_candidates(L * ne, g, 5, 9)
    D, cut, obj, am = G.eval_costs(s, cands, alpha=2.5, beta=0.75)
    oD, ocut, oobj, oam = orc.eval_costs(L, ne, g, oA, oE, cands, 2.5, 0.75)
    assert np.array_equal(D, oD) and np.array_equal(cut, ocut) and np.array_equal(obj, oobj) and am == oam


def test_eval_rejects_infeasible_candidate(G):
    topo = G.MoeTopology(2, 4, 1, 2)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(np.array([[[0], [1]]], np.uint8))
    bad = np.array([[0, 0, 0, 1, 1, 1, 1, 1]], np.uint8)
    with pytest.raises(ValueError):
        G.eval_costs(s, bad)
    ok = np.array([[0, 0, 1, 1, 0, 0, 1, 1]], np.uint8)
    D, cut, obj, am = G.eval_costs(s, ok)  # the handle stays usable
    assert am == 0


def test_comm_cost_matches_oracle_and_cut(G, orc):
    L, ne, k, g = SHAPES["dsv3"]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 4000, model_seed=1, stream_seed=9, device=0)
    host = trace.cpu().numpy()
    assign = G.static_placement(topo).assign
    stream = G.RoutedStream(topo, 4000, trace)
    got = G.comm_cost(stream, assign)
    assert got == orc.comm_cost(L, ne, k, host, assign)
    # acceptance c4: cut == comm_cost (acceptance_main.cpp:317-359)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    _, cut, _, _ = G.eval_costs(s, np.asarray([assign], np.uint8))
    assert cut[0] == float(got)


def test_generator_bit_exact_with_cpu_twin(G, orc):
    for (L, ne, k, g), drift, epoch in ((SHAPES["dsv3"], 0.0, 0), (SHAPES["mixtral"], 0.0, 0),
                                        (SHAPES["qwen3"], 0.25, 3)):
        topo = G.MoeTopology(L, ne, k, g)
        cdf, thr = G.generator_tables(topo, model_seed=5, drift=drift, drift_epoch=epoch)
        tr = G.generate_trace(topo, 3000, model_seed=5, stream_seed=17, first_token=1000, drift=drift,
                              drift_epoch=epoch, device=0)
        twin = orc.generate_trace(L, ne, k, cdf.ravel(), int(thr[0]), int(thr[1]), 17, 1000, 3000)
        assert np.array_equal(tr.cpu().numpy(), twin)
