"""The fused small-shape placement pass (placement.cu tiny_pass_kernel): one launch does the
derived activation, the strong-pair set, the greedy walk into candidate row 0, the scoring of every
candidate and the argmin.  Checked against the CPU oracle (placement.cpp:13-85, 186-299) over the
shapes and pass arguments it accepts, eager and graph-replayed, plus the fallback conditions."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(32, 8, 2, 8, 4096), (5, 8, 3, 4, 9), (7, 16, 4, 8, 33), (3, 16, 2, 16, 5), (40, 8, 2, 2, 17),
          (2, 8, 8, 8, 3), (33, 16, 2, 4, 1), (8, 8, 2, 8, 2), (16, 16, 6, 8, 700)]


def _check(G, orc, hp, trace, cands, threshold, top_e, anchor, alpha, beta, graph):
    topo = hp.topo
    L, ne, k, g = topo.n_layers, topo.n_experts, topo.top_k, topo.n_gpus
    m = L * ne
    res = hp.run(trace, cands, graph=graph)
    oA, oE, oW = orc.stats(L, ne, k, trace.cpu().numpy())
    M = list(orc.affinity_set(L, ne, g, oE, threshold, top_e, m // g, anchor))
    greedy = orc.greedy_place(L, ne, g, oA, M, anchor)
    want = cands.cpu().numpy()
    assert np.array_equal(want[0], greedy.astype(np.uint8))
    D, cut, obj, am = orc.eval_costs(L, ne, g, oA, oE, want, alpha, beta)
    assert res.affinity.experts == M
    assert res.greedy == list(greedy)
    assert res.argmin == am
    sc = hp._out.cpu().numpy()
    assert np.array_equal(sc[0], D) and np.array_equal(sc[1], cut) and np.array_equal(sc[2], obj)
    A, E, W = hp.stats.read()  # A as the fused pass wrote it, W derived afterwards
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW)


@pytest.mark.parametrize("L,ne,k,g,C", SHAPES)
def test_tiny_pass_matches_oracle(G, orc, L, ne, k, g, C):
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 20011, model_seed=6, stream_seed=L, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 77, C)).cuda()
    hp = G.HotPath(topo, 0)
    _check(G, orc, hp, trace, cands, 0.0, 4, 0, 1.0, 1.0, graph=False)


@pytest.mark.parametrize("threshold,top_e,anchor,alpha,beta", [
    (0.0, 0, 0, 1.0, 1.0), (0.0, 1, 3, 2.0, 0.5), (0.0, 6, 1, 1.0, 1.0), (0.0, 8, 7, 0.25, 3.0),
    (700.0, 4, 2, 1.0, 1.0), (1e12, 4, 0, 1.0, 1.0), (0.0, 5, 5, 1.5, 1.5)])
def test_tiny_pass_arguments(G, orc, threshold, top_e, anchor, alpha, beta):
    """Thresholds above every pair weight, top_e from 0 to 8 (4- and 8-key register lists), anchors
    other than GPU 0, alpha / beta != 1."""
    L, ne, k, g = 32, 8, 2, 8
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 30001, model_seed=2, stream_seed=9, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 5, 300)).cuda()
    hp = G.HotPath(topo, 0, threshold=threshold, top_e=top_e, anchor_gpu=anchor, alpha=alpha, beta=beta)
    _check(G, orc, hp, trace, cands, threshold, top_e, anchor, alpha, beta, graph=False)


def test_tiny_pass_graph_replays(G, orc):
    """gimbal_pass_graph records the fused pass (memset of the ticket / bad index + one kernel) and
    replays it with new buffer contents: every replay matches the oracle."""
    L, ne, k, g = 32, 8, 2, 8
    topo = G.MoeTopology(L, ne, k, g)
    T, C = 9001, 1000
    trace = torch.empty((T, L, k), dtype=torch.uint8, device="cuda")
    cands = torch.empty((C, L * ne), dtype=torch.uint8, device="cuda")
    hp = G.HotPath(topo, 0)
    for it in range(4):
        trace.copy_(G.generate_trace(topo, T, model_seed=3, stream_seed=20 + it, device=0))
        cands.copy_(torch.from_numpy(G.shuffled_candidates(L * ne, g, 60 + it, C)))
        _check(G, orc, hp, trace, cands, 0.0, 4, 0, 1.0, 1.0, graph=True)


def test_tiny_pass_infeasible_candidate(G):
    """Infeasible candidates are reported like check_feasible (placement.cpp:30-50) when the queued
    pass is read back, and the next pass on the same handle runs clean."""
    L, ne, k, g = 32, 8, 2, 8
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 4000, model_seed=1, stream_seed=3, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 8, 600)).cuda()
    for bad in (513, 77):
        cands[bad, 9] = (int(cands[bad, 9]) + 1) % g
    hp = G.HotPath(topo, 0)
    with pytest.raises(ValueError, match="infeasible"):
        hp.run(trace, cands)
    for bad in (513, 77):
        cands[bad, 9] = (int(cands[bad, 9]) - 1) % g
    assert 0 <= hp.run(trace, cands).argmin < 600


def test_tiny_pass_after_other_evaluator_calls(G, orc):
    """The fused pass keeps its completion ticket in the evaluator scratch between passes; an
    eval_costs call with more candidates on the same handle overwrites that scratch, and the next
    fused pass must notice (it re-initialises) and still match the oracle."""
    L, ne, k, g = 32, 8, 2, 8
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 7001, model_seed=5, stream_seed=1, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 3, 100)).cuda()
    many = torch.from_numpy(G.shuffled_candidates(L * ne, g, 4, 900)).cuda()
    hp = G.HotPath(topo, 0)
    for graph in (False, True, True):
        _check(G, orc, hp, trace, cands, 0.0, 4, 0, 1.0, 1.0, graph=graph)
        G.eval_costs(hp.stats, many, 1.0, 1.0)
    _check(G, orc, hp, trace, cands, 0.0, 4, 0, 1.0, 1.0, graph=True)


@pytest.mark.parametrize("shape", [(32, 8, 2, 8, 4096), (26, 64, 6, 8, 64)])
def test_run_async_matches_run(G, orc, shape):
    """HotPath.run_async (gimbal_pass_enqueue): 100 passes queued back to back without reading
    them, then read in order -- the fused pass's results come from the mapped ring (64 slots, at
    most 8 passes in flight), the multi-kernel pass's from copies into the registered slots; every
    one equals the synchronous run() and the oracle, and an error surfaces from result()."""
    L, ne, k, g, C = shape
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 6001, model_seed=2, stream_seed=4, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 9, C)).cuda()
    hp = G.HotPath(topo, 0)
    want = hp.run(trace, cands)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    M = list(orc.affinity_set(L, ne, g, oE, 0.0, 4, L * ne // g, 0))
    assert want.affinity.experts == M and want.greedy == list(orc.greedy_place(L, ne, g, oA, M, 0))
    pend = [hp.run_async(trace, cands) for _ in range(100)]
    for p in pend:
        r = p.result()
        assert r.argmin == want.argmin and r.greedy == want.greedy and r.affinity.experts == want.affinity.experts
    bad_cands = cands.clone()
    bad_cands[C // 2, 3] = (int(bad_cands[C // 2, 3]) + 1) % g
    bad = hp.run_async(trace, bad_cands)
    later = [hp.run_async(trace, cands) for _ in range(12)]  # the ninth call reads `bad` out
    for p in later:  # the bad pass's error stays with it
        assert p.result().argmin == want.argmin
    with pytest.raises(ValueError, match="infeasible"):
        bad.result()


def test_run_async_on_the_handle_stream(G, orc):
    """gimbal_pass_enqueue with the caller's stream = the handle's own stream (no joins): same answers."""
    L, ne, k, g, C = 32, 8, 2, 8, 200
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 5001, model_seed=8, stream_seed=1, device=0)
    cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 12, C)).cuda()
    hp = G.HotPath(topo, 0)
    want = hp.run(trace, cands)
    hs = torch.cuda.ExternalStream(hp.stats.device_buffers()[2], device=torch.device("cuda", 0))
    with torch.cuda.stream(hs):
        pend = [hp.run_async(trace, cands) for _ in range(20)]
    for p in pend:
        r = p.result()
        assert r.argmin == want.argmin and r.greedy == want.greedy and r.affinity.experts == want.affinity.experts
