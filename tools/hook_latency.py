#!/usr/bin/env python3
"""Per-iteration latency of the online expert-layer hook (gimbal_online_iteration: one CUDA graph
per engine iteration) next to the reference's host loop for the same work (MoeSubsystem::
iteration_cost's per-token loop, sim.cpp:113-147, restated over the reference's own RoutingStats in
oracle/_ref ref_hook_iteration; lifetime + window add_token, load histogram, crossings, excess).
Routing (RoutingModel::route_token) is excluded from both: the hook receives routed ids.

  python tools/hook_latency.py [--iters 200] > profiles/r2_online_hook_latency.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    import oracle
    import paper_2602_21626_b200 as G

    ref = oracle.Ref()
    rows = []
    for name, (L, ne, k, g) in {"sim-test (6,16,4,4)": (6, 16, 4, 4), "mixtral": (32, 8, 2, 8),
                                "dsv2lite": (26, 64, 6, 8), "dsv3": (58, 256, 8, 8)}.items():
        topo = G.MoeTopology(L, ne, k, g)
        assign = list(G.shuffled_candidates(L * ne, g, 5, 1)[0])
        for n in (64, 4096):  # a decode batch / max_batch_tokens (sim.hpp:47)
            batches = [G.generate_trace(topo, n, model_seed=1, stream_seed=2, first_token=i * n, device=0).cpu().numpy()
                       for i in range(8)]
            window = G.RoutingStats(topo, 0)
            hook = G.OnlineHook(window)
            hook.set_placement(assign)
            for b in batches[:3]:
                hook.iteration(b)
            t0 = time.perf_counter()
            for i in range(args.iters):
                hook.iteration(batches[i % 8])
            gpu_us = (time.perf_counter() - t0) / args.iters * 1e6
            b32 = [b.astype(np.int32) for b in batches]  # RoutedStream::choices as the engine passes them
            t0 = time.perf_counter()
            for i in range(args.iters):
                hook.iteration(b32[i % 8])
            gpu32_us = (time.perf_counter() - t0) / args.iters * 1e6
            rh = ref.hook_create(L, ne, k, g, assign)
            ref.hook_iteration(rh, b32[0])
            iters = max(3, min(args.iters, int(2.0 / max(1e-6, 1e-7 * n * L * k * k))))
            t0 = time.perf_counter()
            for i in range(iters):
                ref.hook_iteration(rh, b32[i % 8])
            cpu_us = (time.perf_counter() - t0) / iters * 1e6
            ref.hook_destroy(rh)
            rows.append({"shape": name, "L": L, "n_e": ne, "k": k, "g": g, "tokens_per_iteration": n,
                         "gpu_hook_us": gpu_us, "gpu_hook_int32_ids_us": gpu32_us, "reference_host_loop_us": cpu_us, "speedup": cpu_us / gpu_us,
                         "gpu_iters": args.iters, "host_iters": iters})
            print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
