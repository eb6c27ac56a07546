#!/usr/bin/env python3
"""Randomised parity sweep of the whole pass against the CPU oracle (not part of the test suite;
run on a GPU box with a time budget).  Each case draws a topology (layers, experts, top-k, GPUs),
a token count, a candidate count and pass arguments (threshold, top_e, anchor, alpha, beta), runs
HotPath.run (graph path, eager and replayed) or HotPath.run_async, and compares counts, strong-pair
set, greedy placement, every candidate's scores and the argmin with the oracle.

  python tools/fuzz_parity.py [--seconds 600] [--seed 1]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2602_21626_b200 as G  # noqa: E402


def draw(rng):
    ne = int(rng.choice([4, 8, 8, 16, 16, 24, 32, 64, 64, 100, 128, 256]))
    k = int(rng.integers(1, min(8, ne) + 1))
    divisors = [d for d in (1, 2, 4, 8, 16) if ne % d == 0 and d <= ne]
    g = int(rng.choice(divisors))
    L = int(rng.integers(1, 60 if ne <= 64 else 20))
    T = int(rng.choice([1, 7, 255, 1024, 4097, 20011, 70001]))
    C = int(rng.choice([1, 2, 9, 33, 300, 1025]))
    top_e = int(rng.choice([0, 1, 2, 4, 4, 6, 8]))
    threshold = float(rng.choice([0.0, 0.0, 3.0, 50.0]))
    anchor = int(rng.integers(0, g))
    alpha, beta = float(rng.choice([1.0, 0.5, 2.0])), float(rng.choice([1.0, 0.25, 3.0]))
    return L, ne, k, g, T, C, top_e, threshold, anchor, alpha, beta


def one(orc, rng, case):
    L, ne, k, g, T, C, top_e, threshold, anchor, alpha, beta = case
    topo = G.MoeTopology(L, ne, k, g)
    m = L * ne
    ids = rng.integers(0, ne, size=(T, L, k), dtype=np.uint8)
    if rng.random() < 0.3 and k > 1:  # repeated ids (counted with multiplicity)
        step = int(rng.integers(2, 9))
        ids[::step, :, 1] = ids[::step, :, 0]
    trace = torch.from_numpy(ids).cuda()
    cands = torch.from_numpy(G.shuffled_candidates(m, g, int(rng.integers(1, 1 << 30)), C)).cuda()
    hp = G.HotPath(topo, 0, threshold=threshold, top_e=top_e, anchor_gpu=anchor, alpha=alpha, beta=beta)
    mode = int(rng.integers(0, 3))
    if mode == 0:
        res = hp.run(trace, cands, graph=False)
    elif mode == 1:
        for _ in range(3):  # eager, recorded, replayed
            res = hp.run(trace, cands)
    else:
        res = hp.run_async(trace, cands).result()
    oA, oE, oW = orc.stats(L, ne, k, ids)
    A, E, W = hp.stats.read()
    assert np.array_equal(A, oA) and np.array_equal(E, oE) and np.array_equal(W, oW), "counts"
    if L < 2:
        M = []
    else:
        M = list(orc.affinity_set(L, ne, g, oE, threshold, top_e, m // g, anchor))
    assert res.affinity.experts == M, ("strong pairs", res.affinity.experts, M)
    greedy = orc.greedy_place(L, ne, g, oA, M, anchor)
    assert res.greedy == list(greedy), "greedy"
    want = cands.cpu().numpy()
    D, cut, obj, am = orc.eval_costs(L, ne, g, oA, oE, want, alpha, beta)
    sc = hp._out.cpu().numpy()
    assert np.array_equal(sc[0], D) and np.array_equal(sc[1], cut) and np.array_equal(sc[2], obj), "scores"
    assert res.argmin == am, ("argmin", res.argmin, am)
    return mode


def one_hook(ref, rng, case):
    """The online hook (gimbal_online_iteration, both graph variants) against the reference's
    per-token loop of MoeSubsystem::iteration_cost over random batch sizes and relocations."""
    L, ne, k, g = case[:4]
    if ne > 256:
        return
    topo = G.MoeTopology(L, ne, k, g)
    window = G.RoutingStats(topo, 0)
    hook = G.OnlineHook(window)
    place = list(G.shuffled_candidates(L * ne, g, int(rng.integers(1, 1 << 30)), 1)[0])
    hook.set_placement(place)
    rh = ref.hook_create(L, ne, k, g, place)
    try:
        for i in range(int(rng.integers(1, 6))):
            if rng.random() < 0.3:  # relocation: new placement, window closed and reset
                place = list(G.shuffled_candidates(L * ne, g, int(rng.integers(1, 1 << 30)), 1)[0])
                hook.set_placement(place)
                ref.hook_set_placement(rh, place)
                window.reset()
                ref.hook_reset_window(rh)
            n = int(rng.choice([1, 3, 64, 255, 256, 1000, 4096]))
            ids = rng.integers(0, ne, size=(n, L, k), dtype=np.uint8)
            if rng.random() < 0.3 and k > 1:
                ids[::2, :, 1] = ids[::2, :, 0]
            got = hook.iteration(ids.astype(np.int32) if rng.random() < 0.5 else ids)
            want = ref.hook_iteration(rh, ids.astype(np.int32))
            assert got[1] == want[1] and got[0] == want[0], ("iteration", i, got, want)
        A, E, W = window.read()
        rA, rE, rT = ref.hook_stats(rh, L, ne, g)
        assert np.array_equal(A, rA.astype(np.uint64)) and np.array_equal(E, rE.astype(np.uint64)), "window stats"
        assert np.array_equal(hook.gpu_totals(), rT), "gpu totals"
    finally:
        ref.hook_destroy(rh)


def one_stream(orc, rng, case):
    """Tumbling windows (HotPath.stream: two handles, queued per-window greedy / scores / argmin):
    every window's greedy placement, scores, argmin and moved count against the oracle."""
    L, ne, k, g, T, C = case[:6]
    if L < 2 or ne > 256:
        return
    topo = G.MoeTopology(L, ne, k, g)
    m = L * ne
    calib = torch.from_numpy(rng.integers(0, ne, size=(int(rng.integers(1, 5000)), L, k), dtype=np.uint8)).cuda()
    wins = [torch.from_numpy(rng.integers(0, ne, size=(int(rng.choice([1, 100, 4097, 20011])), L, k),
                                          dtype=np.uint8)).cuda() for _ in range(int(rng.integers(1, 5)))]
    cands = torch.from_numpy(G.shuffled_candidates(m, g, int(rng.integers(1, 1 << 30)), max(C, 2))).cuda()
    hp = G.HotPath(topo, 0)
    M = hp.calibrate(calib)
    cA, cE, _ = orc.stats(L, ne, k, calib.cpu().numpy())
    assert M.experts == list(orc.affinity_set(L, ne, g, cE, 0.0, 4, m // g, 0)), "calibration set"
    out = hp.stream(wins, cands, M)
    scores = hp._window_scores.cpu().numpy()
    prev = None
    for i, (w, (am, moved, gp)) in enumerate(zip(wins, out)):
        oA, oE, _ = orc.stats(L, ne, k, w.cpu().numpy())
        ogp = np.asarray(orc.greedy_place(L, ne, g, oA, M.experts, 0), np.int32)
        assert np.array_equal(gp, ogp), ("window greedy", i)
        hc = cands.cpu().numpy()
        hc[0] = ogp.astype(np.uint8)
        D, cut, obj, oam = orc.eval_costs(L, ne, g, oA, oE, hc)
        assert am == oam, ("window argmin", i)
        assert np.array_equal(scores[i][0], D) and np.array_equal(scores[i][1], cut), ("window scores", i)
        assert np.array_equal(scores[i][2], obj), ("window objective", i)
        assert moved == (len(ogp) if prev is None else int(np.count_nonzero(prev != ogp))), ("moved", i)
        prev = ogp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--what", default="pass", choices=["pass", "hook", "stream"])
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    orc = oracle.Oracle()
    ref = oracle.Ref() if args.what == "hook" else None
    t0, n, fails = time.time(), 0, 0
    while time.time() - t0 < args.seconds:
        case = draw(rng)
        try:
            if args.what == "hook":
                one_hook(ref, rng, case)
            elif args.what == "stream":
                one_stream(orc, rng, case)
            else:
                one(orc, rng, case)
        except Exception as ex:  # report and go on
            fails += 1
            print("FAIL", case, repr(ex)[:300], flush=True)
        n += 1
    print(f"fuzz {args.what}: {n} cases, {fails} failures, {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
