#!/usr/bin/env python3
"""Device time per queued pass at the Mixtral bench shape, broken down: the graph replay alone
(gimbal_pass_graph), plus the packed read-back, plus the stream joins of gimbal_pass_enqueue with
torch's default stream; and the host cost per call.  Shows where a step's time beyond its two
kernels goes."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21626_b200 as G  # noqa: E402

L, ne, k, g, T, C = 32, 8, 2, 8, 1 << 20, 4096
topo = G.MoeTopology(L, ne, k, g)
trace = G.generate_trace(topo, T, model_seed=1, stream_seed=2, device=0)
cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 1000, C)).cuda()
hp = G.HotPath(topo, 0)
hs = torch.cuda.ExternalStream(hp.stats.device_buffers()[2], device=torch.device("cuda", 0))
n = 300


def timed(label, fn, stream):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    out = [fn() for _ in range(n)]
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{label:44s} device {1e3 * e0.elapsed_time(e1) / n:7.1f} us/step   host {1e6 * (t1 - t0) / n:6.1f} us/call")
    return out


hp.run(trace, cands)
hp.run(trace, cands)
timed("graph replay only (gimbal_pass_graph)", lambda: hp._queue_graph(trace, cands), hs)
timed("run_async, caller = torch default stream", lambda: hp.run_async(trace, cands), hs)
with torch.cuda.stream(hs):
    timed("run_async, caller = the handle's stream", lambda: hp.run_async(trace, cands), hs)
t0 = time.perf_counter()
for _ in range(200):
    hp.run(trace, cands)
print(f"{'synchronous run()':44s} wall {1e6 * (time.perf_counter() - t0) / 200:7.1f} us/step")
