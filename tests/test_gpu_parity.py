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


@pytest.mark.parametrize("L,T,offset", [(58, 70001, 0), (58, 700, 0), (58, 3000, 8), (7, 5000, 0), (2, 1025, 0)])
def test_direct_count_layouts(G, orc, L, T, offset):
    """n_e = 256, top-8 uint8 traces are counted straight from the token-major rows: TMA-staged
    when the row pitch and base are 16-byte aligned (L even), plain loads otherwise."""
    ne, k = 256, 8
    topo = G.MoeTopology(L, ne, k, 8)
    rng = np.random.default_rng(T + L)
    ids = rng.integers(0, ne, size=(T, L, k), dtype=np.uint8)
    buf = torch.empty(T * L * k + offset, dtype=torch.uint8, device="cuda")
    dev = buf[offset:].view(T, L, k)
    dev.copy_(torch.from_numpy(ids))
    _, (A, E, W) = _stats_gpu(G, topo, dev)
    oA, oE, oW = orc.stats(L, ne, k, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


@pytest.mark.parametrize("L,ne,T,offset,dup", [(48, 128, 70001, 0, False), (48, 128, 3000, 8, False),
                                               (48, 128, 5000, 0, True), (10, 100, 9000, 0, True),
                                               (9, 128, 4000, 0, False)])
def test_mma_count_layouts(G, orc, L, ne, T, offset, dup):
    """n_e in (64, 128], top-8 uint8 traces go through the tcgen05 contraction: straight from the
    token-major rows by TMA when L is even and the base 16-byte aligned (ids range-checked and
    repeats detected per row in the kernel), through the layer-major transposition otherwise."""
    k = 8
    topo = G.MoeTopology(L, ne, k, 4)
    rng = np.random.default_rng(T + ne)
    ids = rng.integers(0, ne, size=(T, L, k), dtype=np.uint8)
    if dup:
        ids[::7, :, 1] = ids[::7, :, 0]  # every 7th token repeats its first id
    buf = torch.empty(T * L * k + offset, dtype=torch.uint8, device="cuda")
    dev = buf[offset:].view(T, L, k)
    dev.copy_(torch.from_numpy(ids))
    _, (A, E, W) = _stats_gpu(G, topo, dev)
    oA, oE, oW = orc.stats(L, ne, k, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


@pytest.mark.parametrize("L,k,T,offset,dup", [(26, 6, 70001, 0, False), (26, 6, 1, 0, False), (26, 6, 65, 0, True),
                                              (2, 8, 5000, 0, False), (3, 1, 4097, 0, False), (17, 6, 3000, 0, False),
                                              (18, 5, 3000, 0, True), (34, 3, 9000, 0, False),
                                              (64, 8, 2000, 0, False), (26, 6, 3000, 8, False)])
def test_mma_stack_layouts(G, orc, L, k, T, offset, dup):
    """64-expert uint8 traces go through the stacked tcgen05 contraction (two layers per 128-row
    operand, rows bulk-copied from the token-major trace): odd and even pair counts per group,
    several groups, ragged tails shorter than one 16-byte copy unit, repeated ids; a base that is
    not 16-byte aligned falls back to the shared-memory counters."""
    ne = 64
    topo = G.MoeTopology(L, ne, k, 8)
    rng = np.random.default_rng(T * 7 + L)
    ids = rng.integers(0, ne, size=(T, L, k), dtype=np.uint8)
    if dup and k > 1:
        ids[::5, :, 1] = ids[::5, :, 0]
    buf = torch.empty(T * L * k + offset, dtype=torch.uint8, device="cuda")
    dev = buf[offset:].view(T, L, k)
    dev.copy_(torch.from_numpy(ids))
    _, (A, E, W) = _stats_gpu(G, topo, dev)
    oA, oE, oW = orc.stats(L, ne, k, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


@pytest.mark.parametrize("bad", [64, 255])
def test_mma_stack_out_of_range(G, bad):
    L, ne, k = 26, 64, 6
    topo = G.MoeTopology(L, ne, k, 8)
    ids = np.zeros((3000, L, k), np.uint8)
    ids[:, :, :] = np.arange(k, dtype=np.uint8)
    ids[2999, 25, 5] = bad
    s = G.RoutingStats(topo, 0)
    s.add_tokens(torch.from_numpy(ids).cuda())
    with pytest.raises(IndexError):
        s.read()


@pytest.mark.parametrize("L,ne,T,offset,dup,bad", [(32, 8, 70001, 0, False, None), (32, 8, 1, 0, False, None),
                                                  (32, 8, 5000, 0, True, None), (16, 16, 9001, 0, True, None),
                                                  (32, 8, 3000, 0, False, (2999, 31, 1, 8)),
                                                  (32, 16, 3000, 0, False, (5, 0, 0, 200)),
                                                  (32, 8, 3000, 8, False, None), (30, 8, 3000, 0, False, None),
                                                  # the event-histogram counter's other row widths (L = 8, 16, 24)
                                                  (8, 8, 4099, 0, True, None), (8, 8, 1, 0, False, None),
                                                  (16, 8, 70001, 0, False, None), (24, 8, 3000, 0, True, None),
                                                  (24, 8, 3000, 0, False, (1234, 23, 1, 9)),
                                                  (16, 8, 2000, 0, False, (0, 0, 0, 255))])
def test_small2_count_layouts(G, orc, L, ne, T, offset, dup, bad):
    """Top-2 traces of 8 / 16 experts are counted word-wise (small_count.cu small_count_row2):
    ragged blocks, one token, repeated ids, an out-of-range id (that row falls back to the
    byte-wise loop and the call reports the error), an unaligned base and L = 30 (even row stride:
    the byte-wise kernel)."""
    k = 2
    topo = G.MoeTopology(L, ne, k, 8)
    rng = np.random.default_rng(T + 7 * L + ne)
    ids = rng.integers(0, ne, size=(T, L, k), dtype=np.uint8)
    if dup:
        ids[::3, :, 1] = ids[::3, :, 0]
    if bad is not None:
        ids[bad[0], bad[1], bad[2]] = bad[3]
    buf = torch.empty(T * L * k + offset, dtype=torch.uint8, device="cuda")
    dev = buf[offset:].view(T, L, k)
    dev.copy_(torch.from_numpy(ids))
    s = G.RoutingStats(topo, 0)
    s.add_tokens(dev)
    if bad is not None:
        with pytest.raises(IndexError):
            s.read()
        return
    A, E, W = s.read()
    oA, oE, oW = orc.stats(L, ne, k, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


def test_events8_bin_bound(G, orc):
    """Top-2 over 8 experts counts token-pair events in 16-bit bins: 10.5 Mi tokens of one repeated
    id per layer put every token into the same bin of every pair, so the launcher must split the
    trace over more CTAs than SMs (<= 63 blocks of 1024 tokens each); E_l(0, 0) = 4 T (the pair
    (0, 0) counted with multiplicity 2 x 2)."""
    L, ne, k, T = 32, 8, 2, 10_500_000
    topo = G.MoeTopology(L, ne, k, 8)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(torch.zeros((T, L, k), dtype=torch.uint8, device="cuda"))
    A, E, W = s.read()
    assert (E[:, 0, 0] == 4 * T).all() and E.sum() == (L - 1) * 4 * T
    assert (A[:, 0] == 2 * T).all() and A.sum() == L * 2 * T


@pytest.mark.parametrize("ne,bad", [(128, 128), (128, 255), (100, 100)])
def test_mma_direct_out_of_range(G, ne, bad):
    L, k = 6, 8
    topo = G.MoeTopology(L, ne, k, 4)
    ids = np.zeros((1000, L, k), np.uint8)
    ids[:, :, :] = np.arange(k, dtype=np.uint8)
    ids[777, 3, 5] = bad
    s = G.RoutingStats(topo, 0)
    s.add_tokens(torch.from_numpy(ids).cuda())
    with pytest.raises(IndexError):
        s.read()


@pytest.mark.parametrize("dup", [False, True])
def test_counter_overflow_paths(G, dup):
    """Hot cells far beyond 2^15 / 2^16 per work unit (guarded 15-bit counters at n_e = 256,
    s32 tensor-core accumulators at n_e = 128): 1 Mi identical tokens, with and without
    repeated ids (multiplicity 64 per token-pair)."""
    for (L, ne, k, g) in (SHAPES["dsv3"], SHAPES["qwen3"]):
        topo = G.MoeTopology(L, ne, k, g)
        T = 1 << 20
        row = np.full((L, k), 3, np.uint8) if dup else np.tile(np.arange(k, dtype=np.uint8) * 5, (L, 1))
        trace = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(row, (T, L, k)))).cuda()
        s = G.RoutingStats(topo, 0)
        s.add_tokens(trace)
        A, E, W = s.read()
        want = np.zeros((L - 1, ne, ne), np.uint64)
        for a in range(k):
            for b in range(k):
                want[:, row[0, a], row[1, b]] += T
        assert np.array_equal(E, want)
        assert (A.sum(axis=1) == T * k).all()


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


@pytest.mark.parametrize("shape", ["dsv2lite", "dsv3"])
def test_stream_windows_match_oracle(G, orc, shape):
    """Config 5 (tumbling windows, sim.cpp:149-165): M fixed from a calibration window, each window
    counted from zero, greedy with M, all candidates scored; the two-handle overlapped loop gives
    the oracle's greedy placement, argmin and moved count for every window."""
    L, ne, k, g = SHAPES[shape]
    topo = G.MoeTopology(L, ne, k, g)
    C, T_w = 40, 6001
    calib = G.generate_trace(topo, 20000, model_seed=1, stream_seed=3, drift=0.05, drift_epoch=0, device=0)
    wins = [G.generate_trace(topo, T_w, model_seed=1, stream_seed=2, first_token=w * T_w, drift=0.05,
                             drift_epoch=w + 1, device=0) for w in range(5)]
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 77, C)).cuda()
    hp = G.HotPath(topo, 0)
    M = hp.calibrate(calib)
    cA, cE, _ = orc.stats(L, ne, k, calib.cpu().numpy())
    assert M.experts == list(orc.affinity_set(L, ne, g, cE, 0.0, 4))
    out = hp.stream(wins, cands, M)
    scores = hp._window_scores.cpu().numpy()
    prev = None
    for i, (w, (am, moved, gp)) in enumerate(zip(wins, out)):
        oA, oE, _ = orc.stats(L, ne, k, w.cpu().numpy())
        ogp = np.asarray(orc.greedy_place(L, ne, g, oA, M.experts, 0), np.int32)
        assert np.array_equal(gp, ogp)
        hc = cands.cpu().numpy()
        hc[0] = ogp.astype(np.uint8)  # the loop scores the window's greedy as candidate 0
        D, cut, obj, oam = orc.eval_costs(L, ne, g, oA, oE, hc)
        assert am == oam
        assert np.array_equal(scores[i][0], D) and np.array_equal(scores[i][1], cut)
        assert np.array_equal(scores[i][2], obj)
        assert moved == (len(ogp) if prev is None else int(np.count_nonzero(prev != ogp)))
        prev = ogp
    # the queued path leaves the handles usable by the synchronous API
    hp.stats.reset()
    hp.stats.add_tokens(wins[-1])
    res = hp.place_with(M, cands)
    assert res.greedy == list(out[-1][2])


def test_stream_infeasible_candidate_reported_at_sync(G):
    """gimbal_window_place_async defers device-side errors: an infeasible candidate row in the
    queued windows raises (like check_feasible, placement.cpp:30-50) when the stream syncs, and
    the flag is cleared afterwards."""
    L, ne, k, g = SHAPES["dsv2lite"]
    topo = G.MoeTopology(L, ne, k, g)
    wins = [G.generate_trace(topo, 3000, model_seed=1, stream_seed=2, first_token=w * 3000, device=0)
            for w in range(3)]
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 5, 8)).cuda()
    cands[5, 3] = (int(cands[5, 3]) + 1) % g  # one GPU over, one under its m/g share
    hp = G.HotPath(topo, 0)
    M = hp.calibrate(wins[0])
    with pytest.raises(ValueError, match="infeasible"):
        hp.stream(wins, cands, M)
    cands[5, 3] = (int(cands[5, 3]) - 1) % g
    out = hp.stream(wins, cands, M)
    assert len(out) == 3


@pytest.mark.parametrize("threshold,top_e,cap", [(0.0, 4, None), (0.0, -1, None), (50.0, 16, 7), (1e12, 4, None),
                                                 (0.0, 0, None), (0.0, 64, 3), (3.0, 1000, None), (0.0, 1, None),
                                                 (0.0, 8, None), (50.0, 8, 7), (0.0, 9, None)])
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


# ---- the reference's KATs and golden fixtures through the GPU path ----

def test_kats_through_gpu(G):
    import kat_util as K

    k = K.kats()
    for c in k["stats"]:
        s = G.RoutingStats(G.MoeTopology(c["L"], c["ne"], c["k"], 2), 0)
        s.add_tokens(K.trace(c))
        A, E, W = s.read()
        assert np.array_equal(A, np.asarray(c["A"], np.uint64)) and s.tokens() == c["tokens"], c["src"]
        assert np.array_equal(E, K.expected_e(c)) and np.array_equal(W, K.expected_w(c)), c["src"]
    for c in k["comm_cost"]:
        topo = G.MoeTopology(c["L"], c["ne"], c["k"], 2)
        st = G.RoutedStream(topo, len(c["choices"]), K.trace(c))
        if c.get("error"):
            with pytest.raises(ValueError):
                G.comm_cost(st, c["assign"])
        else:
            assert G.comm_cost(st, c["assign"]) == c["expected"], c["src"]
    for c in k["eval_cost"]:
        A = np.asarray(c["A"], np.float64)
        p = G.PlacementProblem(A=A, W=K.dense_w(c["W"], A.shape[1]), g=c["g"], alpha=c.get("alpha", 1.0),
                               beta=c.get("beta", 1.0))
        if c.get("error"):
            with pytest.raises(ValueError):
                G.eval_cost(p, G.Placement(c["assign"]))
            continue
        cost = G.eval_cost(p, G.Placement(c["assign"]))
        for key, attr in (("D", "deviation"), ("cut", "cut"), ("objective", "objective")):
            if key in c:
                assert getattr(cost, attr) == c[key], c["src"]
    for c in k["affinity_set"]:
        topo = G.MoeTopology(c["L"], c["ne"], 1, c["g"])
        E = K.e_from_nonzero(c).astype(np.float64)
        got = G.build_affinity_set(G.AffinityTensor(E=E, W=E.sum(0)), topo, c["threshold"], c["top_e"],
                                   c["capacity"], c["anchor"])
        assert got.experts == c["expected"] and got.anchor_gpu == c["anchor"], c["src"]
    for c in k["greedy"]:
        A = np.asarray(c["A"], np.float64)
        if c.get("error"):
            with pytest.raises(ValueError):
                G.greedy_place(A, G.AffinitySet(c["M"], c["anchor"]), c["g"])
            continue
        pl = G.greedy_place(A, G.AffinitySet(c["M"], c["anchor"]), c["g"])
        if "expected" in c:
            assert pl.assign == c["expected"], c["src"]
        if "deviation" in c:
            p = G.PlacementProblem(A=A, W=np.zeros((A.shape[1],) * 2), g=c["g"])
            assert G.eval_cost(p, pl).deviation == c["deviation"]
    for c in k["maybe_relocate"]:
        A = np.asarray(c["A"], np.float64)
        r = G.maybe_relocate(c["step"], c["tau"], G.AffinitySet(), A, c["g"], G.Placement(c["prev"]))
        assert (r is not None) == c["fires"]
        if r is not None:
            again = G.maybe_relocate(2 * c["step"], c["tau"], G.AffinitySet(), A, c["g"], r.placement)
            assert again.moved == c["again_moved"] and again.placement.assign == r.placement.assign


def test_golden_fixtures_through_gpu(G):
    import kat_util as K

    for c in K.golden_cases():
        L, ne, k, g = (int(x) for x in c["topo"])
        thr, top = float(c["params"][3]), int(c["params"][4])
        topo = G.MoeTopology(L, ne, k, g)
        s = G.RoutingStats(topo, 0)
        s.add_tokens(c["ids"])
        A, E, W = s.read()
        assert np.array_equal(A, c["A"]) and np.array_equal(E, c["E"]) and np.array_equal(W, c["W"])
        assert s.tokens() == int(c["tokens"])
        # flat forms (moe.cpp:207-231) as the reference builds them
        fA, fW = s.flat_activation(), s.flat_pair_weights()
        assert fA.shape == (L, L * ne) and fW.shape == (L * ne, L * ne)
        assert np.array_equal(fA.sum(0), np.concatenate(list(c["A"])).astype(np.float64))
        assert G.comm_cost(G.RoutedStream(topo, int(c["tokens"]), c["ids"]), c["assign"]) == int(c["comm_cost"])
        D, cut, obj, _ = G.eval_costs(s, np.asarray([c["assign"]], np.uint8))
        assert (D[0], cut[0], obj[0]) == tuple(c["cost"])
        D, cut, obj, _ = G.eval_costs(s, np.asarray([c["assign"]], np.uint8), 2.5, 0.75)
        assert (D[0], cut[0], obj[0]) == tuple(c["cost_ab"])
        # dense reference form on the flat matrices agrees too
        dense = G.eval_cost(G.PlacementProblem(A=fA, W=fW, g=g), G.Placement(list(c["assign"])))
        assert (dense.deviation, dense.cut, dense.objective) == tuple(c["cost"])
        M = G.build_affinity_set(s, topo, thr, top, L * ne // g, g - 1)
        assert M.experts == list(c["M"])
        gp = G.greedy_place(s, M, g)
        assert gp.assign == list(c["greedy"])
        assert G.greedy_place(fA, M, g).assign == list(c["greedy"])


def test_bench_scale_properties(G):
    """Size-independent identities at a BASELINE-scale token count (DS-V3 shape, 4M tokens):
    A row sums = T*k, sum E_l = T*k^2, W = sum_l E_l, and cut == comm_cost for two placements."""
    L, ne, k, g = SHAPES["dsv3"]
    topo = G.MoeTopology(L, ne, k, g)
    T = 1 << 22
    trace = G.generate_trace(topo, T, model_seed=1, stream_seed=2, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    A, E, W = s.read()
    assert (A.sum(axis=1) == T * k).all()
    assert (E.reshape(L - 1, -1).sum(axis=1) == T * k * k).all()
    assert np.array_equal(W, E.sum(axis=0, dtype=np.uint64))
    # A counted independently of our kernels (A is derived from E inside the library): torch's
    # bincount over each layer's ids on the device
    offs = (torch.arange(L, device=trace.device, dtype=torch.int64) * ne).view(1, L, 1)
    tA = torch.bincount((trace.to(torch.int64) + offs).view(-1), minlength=L * ne).view(L, ne).cpu().numpy()
    assert np.array_equal(A, tA.astype(np.uint64))
    assert (E.sum(axis=2) == A[:-1] * k).all() and (E[-1].sum(axis=0) == A[-1] * k).all()
    stream = G.RoutedStream(topo, T, trace)
    for assign in (G.static_placement(topo).assign, list(G.shuffled_candidates(L * ne, g, 5, 1)[0])):
        _, cut, _, _ = G.eval_costs(s, np.asarray([assign], np.uint8))
        assert cut[0] == float(G.comm_cost(stream, assign))


@pytest.mark.parametrize("L,ne,k,g,C", [(58, 256, 8, 8, 70), (48, 128, 8, 8, 33), (12, 256, 8, 4, 41),
                                        (9, 128, 4, 16, 17), (58, 256, 8, 16, 129), (3, 128, 8, 4, 9), (3, 128, 8, 4, 1),
                                        (26, 64, 6, 8, 70), (25, 64, 6, 4, 33), (9, 64, 4, 16, 17), (2, 64, 6, 8, 11)])
def test_eval_tensor_core_path_matches_oracle(G, orc, L, ne, k, g, C):
    """eval_mma.cu (E byte planes x one-hot assignment on tcgen05 kind::i8) gives exactly the
    oracle's D / cut / objective / argmin (placement.cpp:58-85), like the integer-ALU evaluator,
    on ragged candidate counts (partial groups), every supported g, and the stacked two-pairs-per-
    operand mode at 64 experts (odd and even pair counts)."""
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 20011, model_seed=2, stream_seed=5, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    cands = G.shuffled_candidates(L * ne, g, 31, C)
    want = orc.eval_costs(L, ne, g, oA, oE, cands, 2.0, 0.5)
    got = G.eval_costs(s, torch.from_numpy(cands).cuda(), 2.0, 0.5)
    for a, b in zip(got[:3], want[:3]):
        assert np.array_equal(a, b)
    assert got[3] == want[3]


def test_queued_pass_argument_errors(G):
    """gimbal_pass_async / gimbal_window_place_async validate like the synchronous API: the
    reference's messages for a bad anchor and an oversized strong-pair set, and alpha/beta > 0."""
    import ctypes as C

    from paper_2602_21626_b200 import _native as N

    L, ne, k, g = SHAPES["dsv2lite"]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 2000, model_seed=1, stream_seed=2, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    m = L * ne
    cands = torch.from_numpy(G.shuffled_candidates(m, g, 3, 4)).cuda()
    buf = torch.zeros(4 + 2 * m + 3 * 4 * 2, dtype=torch.int32, device="cuda")
    p = buf.data_ptr()
    lib = N.lib()
    with pytest.raises(ValueError, match="anchor_gpu out of range"):
        N.check(lib.gimbal_pass_async(s.handle, 0.0, 4, m // g, g, C.c_void_p(cands.data_ptr()), 4, 1.0, 1.0,
                                      C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), None))
    with pytest.raises(ValueError, match="capacity"):
        N.check(lib.gimbal_pass_async(s.handle, 0.0, 4, m // g + 1, 0, C.c_void_p(cands.data_ptr()), 4, 1.0, 1.0,
                                      C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), None))
    with pytest.raises(ValueError, match="alpha and beta"):
        N.check(lib.gimbal_pass_async(s.handle, 0.0, 4, m // g, 0, C.c_void_p(cands.data_ptr()), 4, 0.0, 1.0,
                                      C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), C.c_void_p(p), None))
    big = np.arange(m // g + 1, dtype=np.int32)
    with pytest.raises(ValueError, match="exceeds anchor capacity"):
        N.check(lib.gimbal_window_place_async(s.handle, big.ctypes.data, big.size, 0, C.c_void_p(cands.data_ptr()), 4,
                                              1.0, 1.0, C.c_void_p(p), C.c_void_p(p), C.c_void_p(p)))
    dup = np.array([3, 3], dtype=np.int32)
    with pytest.raises(ValueError, match="duplicate"):
        N.check(lib.gimbal_window_place_async(s.handle, dup.ctypes.data, dup.size, 0, C.c_void_p(cands.data_ptr()), 4,
                                              1.0, 1.0, C.c_void_p(p), C.c_void_p(p), C.c_void_p(p)))
    s.sync()  # nothing deferred


def test_stream_distributed_single_rank_matches_stream(G):
    """The queued multi-GPU streaming loop (NCCL all-reduce of E on the handle stream per window,
    candidate slices, one MIN all-reduce of the objectives) run as a one-rank NCCL group gives the
    single-GPU loop's per-window argmin, moved count and greedy placement."""
    import socket

    import torch.distributed as dist

    L, ne, k, g = SHAPES["dsv3"]
    topo = G.MoeTopology(L, ne, k, g)
    wins = [G.generate_trace(topo, 5003, model_seed=1, stream_seed=2, first_token=w * 5003, drift=0.05,
                             drift_epoch=w + 1, device=0) for w in range(4)]
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 77, 24)).cuda()
    hp = G.HotPath(topo, 0)
    M = hp.calibrate(wins[0])
    want = hp.stream(wins, cands.clone(), M)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        hp2 = G.HotPath(topo, 0)
        got = hp2.stream_distributed(wins, cands.clone(), 0, cands.shape[0], M)
    finally:
        dist.destroy_process_group()
    assert len(got) == len(want)
    for (am1, mv1, gp1), (am2, mv2, gp2) in zip(want, got):
        assert am1 == am2 and mv1 == mv2 and np.array_equal(np.asarray(gp1), np.asarray(gp2))


def test_stream_from_pinned_host_windows(G):
    """The end-to-end streaming path (windows in pinned host memory, copied on the handles' copy
    streams while counted) gives the device-resident loop's results."""
    L, ne, k, g = SHAPES["qwen3"]
    topo = G.MoeTopology(L, ne, k, g)
    wins = [G.generate_trace(topo, 3001, model_seed=3, stream_seed=4, first_token=w * 3001, drift=0.1,
                             drift_epoch=w + 1, device=0) for w in range(3)]
    host = [w.cpu().pin_memory() for w in wins]
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 9, 20)).cuda()
    hp = G.HotPath(topo, 0)
    M = hp.calibrate(wins[0])
    want = hp.stream(wins, cands.clone(), M)
    got = G.HotPath(topo, 0).stream(host, cands.clone(), M)
    for (am1, mv1, gp1), (am2, mv2, gp2) in zip(want, got):
        assert am1 == am2 and mv1 == mv2 and np.array_equal(gp1, gp2)


@pytest.mark.parametrize("shape", ["dsv2lite", "mixtral"])
def test_queued_pass_reports_infeasible_candidate(G, shape):
    """HotPath.run (gimbal_pass_async, greedy walk overlapped with the scoring of candidates 1..C-1
    where m >= 1024) raises like check_feasible for an infeasible candidate, then runs clean."""
    L, ne, k, g = SHAPES[shape]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 4000, model_seed=1, stream_seed=3, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 8, 12)).cuda()
    cands[7, 5] = (int(cands[7, 5]) + 1) % g
    hp = G.HotPath(topo, 0)
    with pytest.raises(ValueError, match="infeasible"):
        hp.run(trace, cands)
    cands[7, 5] = (int(cands[7, 5]) - 1) % g
    res = hp.run(trace, cands)
    assert 0 <= res.argmin < 12


@pytest.mark.parametrize("L,ne,k,g,C", [(32, 8, 2, 8, 4096), (5, 8, 3, 4, 9), (7, 16, 4, 8, 33), (3, 16, 2, 16, 5),
                                        (40, 8, 2, 2, 17), (2, 8, 8, 8, 3)])
def test_eval_small_shapes_match_oracle(G, orc, L, ne, k, g, C):
    """eval_small_kernel (warp per candidate, lane per layer, E and A in shared memory) gives the
    oracle's D / cut / objective / argmin exactly, as does the generic evaluator it replaces."""
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 30011, model_seed=4, stream_seed=6, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    cands = G.shuffled_candidates(L * ne, g, 13, C)
    want = orc.eval_costs(L, ne, g, oA, oE, cands, 1.5, 0.25)
    got = G.eval_costs(s, torch.from_numpy(cands).cuda(), 1.5, 0.25)
    for a, b in zip(got[:3], want[:3]):
        assert np.array_equal(a, b)
    assert got[3] == want[3]
    bad = cands.copy()
    bad[C // 2, 0] = (int(bad[C // 2, 0]) + 1) % g
    with pytest.raises(ValueError, match=f"candidate {C // 2} is infeasible"):
        G.eval_costs(s, torch.from_numpy(bad).cuda())


def test_run_distributed_single_rank_matches_run(G, orc):
    """run_distributed over NCCL (one rank) uses the queued pass: the first rank's slice carries the
    greedy row, a later slice is scored behind a scratch row; both give the oracle's answers."""
    import socket

    import torch.distributed as dist

    L, ne, k, g = SHAPES["qwen3"]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 9001, model_seed=2, stream_seed=4, device=0)
    C = 20
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 21, C)).cuda()
    want = G.HotPath(topo, 0).run(trace, cands.clone())
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        hp = G.HotPath(topo, 0)
        got = hp.run_distributed(trace, cands.clone(), 0, C)
        assert got.argmin == want.argmin and got.greedy == want.greedy
        assert got.affinity.experts == want.affinity.experts
        part = cands[5:].clone()
        got2 = hp.run_distributed(trace, part, 5, C)
        _, _, obj, am = orc.eval_costs(L, ne, g, oA, oE, part.cpu().numpy())
        assert got2.argmin == 5 + am and got2.objective == obj.min()
        assert got2.greedy == want.greedy
        assert torch.equal(part, cands[5:])  # the caller's slice is not overwritten
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,T,C", [("dsv3", 30011, 70), ("qwen3", 20011, 33), ("mixtral", 9001, 300),
                                       ("dsv2lite", 5000, 17)])
def test_eval_excess_matches_oracle(G, orc, shape, T, C):
    """gimbal_eval_excess: the simulator's bottleneck excess (sim.cpp:132-144) per candidate over the
    counted trace, bit-exact against the oracle (itself pinned to the reference hook loop)."""
    L, ne, k, g = SHAPES[shape]
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, T, model_seed=6, stream_seed=1, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    oA, _, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    cands = G.shuffled_candidates(L * ne, g, 17, C)
    cands[0] = np.asarray(G.static_placement(topo).assign, np.uint8)
    want = orc.eval_excess(L, ne, g, oA, cands)
    assert np.array_equal(G.eval_excess(s, cands), want)
    assert np.array_equal(G.eval_excess(s, torch.from_numpy(cands).cuda()), want)
    bad = cands.copy()
    bad[1, 3] = g
    with pytest.raises(ValueError):
        G.eval_excess(s, bad)


@pytest.mark.parametrize("shape", ["mixtral", "dsv2lite", "dsv3"])
def test_graph_replayed_pass_matches_oracle(G, orc, shape):
    """HotPath.run's graph path (gimbal_pass_graph): eager on the first call, recorded on the second,
    replayed after; new trace / candidate contents in the same buffers give the oracle's answers on
    every call, and the counting kernel stays timed through the replays."""
    L, ne, k, g = SHAPES[shape]
    topo = G.MoeTopology(L, ne, k, g)
    T, C = 12001, 40
    trace = torch.empty((T, L, k), dtype=torch.uint8, device="cuda")
    cands = torch.empty((C, L * ne), dtype=torch.uint8, device="cuda")
    hp = G.HotPath(topo, 0)
    hp.stats.count_timing(True)
    for it in range(4):
        trace.copy_(G.generate_trace(topo, T, model_seed=1, stream_seed=10 + it, device=0))
        cands.copy_(torch.from_numpy(G.shuffled_candidates(L * ne, g, 50 + it, C)))
        want_cands = cands.cpu().numpy()
        res = hp.run(trace, cands)
        oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
        M = list(orc.affinity_set(L, ne, g, oE, 0.0, 4, L * ne // g, 0))
        greedy = orc.greedy_place(L, ne, g, oA, M, 0)
        want_cands[0] = greedy
        D, cut, obj, am = orc.eval_costs(L, ne, g, oA, oE, want_cands)
        assert res.affinity.experts == M and res.greedy == list(greedy) and res.argmin == am, f"call {it}"
        sc = hp._out.cpu().numpy()
        assert np.array_equal(sc[0], D) and np.array_equal(sc[1], cut) and np.array_equal(sc[2], obj)
        A, E, _ = hp.stats.read()
        assert np.array_equal(A, oA) and np.array_equal(E, oE) and hp.stats.tokens() == T
    ms, launches = hp.stats.count_timing(False)
    assert launches == 4 and ms > 0
