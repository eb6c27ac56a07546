#!/usr/bin/env python3
"""Generates tests/golden/ref_cases.npz from the REFERENCE's own code (oracle/_ref, built from
/root/reference/proj/src/{moe,placement}.cpp).  Run here (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Each case: a trace routed by the reference RoutingModel (moe.cpp:43-153, Rng streams seeded as
listed), and the reference's record_stats A/E/W, flat forms, comm_cost under a balanced shuffled
placement (acceptance_main.cpp:344-351), eval_cost of that placement and of the greedy placement,
build_affinity_set and greedy_place outputs.  The GPU box has no /root/reference: the fixtures
carry the reference's answers there.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

# (L, n_e, k, g, T, model_seed, rng_seed, zipf_s, lambda, peak, threshold, top_e)
CASES = [
    (2, 4, 1, 2, 64, 1, 2, 1.2, 0.5, 0.8, 0.0, 4),
    (4, 8, 2, 2, 300, 3, 5, 1.2, 0.5, 0.8, 0.0, 4),
    (5, 6, 2, 3, 500, 21, 22, 1.2, 0.7, 0.8, 2.0, 6),
    (3, 16, 4, 4, 400, 9, 10, 1.0, 0.3, 0.6, 0.0, -1),
    (6, 32, 3, 8, 256, 7, 8, 1.5, 0.5, 0.8, 5.0, 16),
    (8, 64, 6, 8, 200, 4, 4, 1.2, 0.5, 0.8, 0.0, 4),
    (4, 128, 8, 8, 128, 11, 12, 1.2, 0.5, 0.8, 0.0, 4),
    (3, 256, 8, 8, 96, 13, 14, 1.2, 0.5, 0.8, 0.0, 4),
]


def main():
    ref = oracle.Ref()
    out = {"n_cases": np.int64(len(CASES))}
    for i, (L, ne, k, g, T, ms, rs, s, lam, peak, thr, top) in enumerate(CASES):
        ids = ref.route_tokens(L, ne, k, g, T, ms, rs, zipf_s=s, lam=lam, peak=peak)
        A, E, W, tok = ref.record_stats(L, ne, k, g, ids)
        fA, fW = ref.flat_forms(L, ne, k, g, ids)
        m = L * ne
        assign = ref.shuffled_balanced(m, g, ref.mix_seed(rs, 0x51))
        cc = ref.comm_cost(L, ne, k, g, ids, assign)
        D, cut, obj = ref.eval_cost(fA, fW, g, assign, alpha=1.0, beta=1.0)
        D2, cut2, obj2 = ref.eval_cost(fA, fW, g, assign, alpha=2.5, beta=0.75)
        M = ref.build_affinity_set(L, ne, k, g, E, threshold=thr, top_e=top, capacity=m // g, anchor=g - 1)
        greedy = ref.greedy_place(fA, g, M, g - 1)
        gD, gcut, gobj = ref.eval_cost(fA, fW, g, greedy)
        p = f"c{i}_"
        out.update({
            p + "topo": np.array([L, ne, k, g], np.int64), p + "params": np.array([s, lam, peak, thr, float(top)]),
            p + "ids": ids.astype(np.uint8 if ne <= 256 else np.int32), p + "A": A.astype(np.uint64),
            p + "E": E.astype(np.uint64), p + "W": W.astype(np.uint64), p + "tokens": np.int64(tok),
            p + "assign": assign, p + "comm_cost": np.int64(cc), p + "cost": np.array([D, cut, obj]),
            p + "cost_ab": np.array([D2, cut2, obj2]), p + "M": np.asarray(M, np.int32),
            p + "greedy": greedy, p + "greedy_cost": np.array([gD, gcut, gobj]),
        })
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_cases.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(CASES)} cases, {os.path.getsize(path)} bytes")
    # byte-stable simulator reports of the reference over its own expert layer
    # (oracle/sim_report_main.cpp linked with proj/src/{sim,moe,placement,...}.cpp)
    import subprocess

    sim = os.path.join(oracle.HERE, "_ref", "sim_report_ref")
    for s in (0, 1, 2):
        rep = subprocess.run([sim, str(s)], capture_output=True, text=True, check=True).stdout
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"sim_report_{s}.json")
        with open(p, "w") as f:
            f.write(rep)
        print(f"wrote {p}: {len(rep)} bytes")


if __name__ == "__main__":
    main()
