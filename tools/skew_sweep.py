"""Sensitivity of one full pass (count, strong-pair set, greedy, C = 4096 scores, argmin) to the
routing skew: Zipf s in {0.8, 1.0, 1.2, 1.5, 2.0} (SURVEY.md §8d suggests sweeping the hotspot
strength) and to the trace length, on the DS-V3 shape.  Device time per pass with CUDA events on the
handle's stream.  python tools/skew_sweep.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_21626_b200 as G  # noqa: E402

topo = G.MoeTopology(58, 256, 8, 8)
C = 4096
cands = torch.from_numpy(G.shuffled_candidates(topo.total_experts(), 8, 1000, C)).cuda()


def timed(trace, reps=3):
    hp = G.HotPath(topo, 0)
    stream = torch.cuda.ExternalStream(hp.stats.device_buffers()[2], device=torch.device("cuda", 0))
    hp.stats.count_timing(True)
    hp.run(trace, cands)
    torch.cuda.synchronize()
    hp.stats.count_timing(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        hp.run(trace, cands)
    b.record(stream)
    torch.cuda.synchronize()
    cms, n = hp.stats.count_timing(False)
    return a.elapsed_time(b) / reps, cms / max(n, 1)


print("zipf_s  tokens    pass_ms  count_ms  Mtokens/s  E-updates/s(T)")
for s in (0.8, 1.0, 1.2, 1.5, 2.0):
    T = 16 << 20
    tr = G.generate_trace(topo, T, G.RoutingParams(zipf_s=s), model_seed=1, stream_seed=2, device=0)
    ms, cms = timed(tr)
    print(f"{s:6.1f}  {T:9d}  {ms:8.2f}  {cms:8.2f}  {T / ms / 1e3:9.1f}  {T * 57 * 64 / cms / 1e9:8.2f}")
    del tr
for T in (1 << 20, 4 << 20, 16 << 20, 64 << 20):
    tr = G.generate_trace(topo, T, model_seed=1, stream_seed=2, device=0)
    ms, cms = timed(tr, reps=2 if T > (16 << 20) else 3)
    print(f"{1.2:6.1f}  {T:9d}  {ms:8.2f}  {cms:8.2f}  {T / ms / 1e3:9.1f}  {T * 57 * 64 / cms / 1e9:8.2f}")
    del tr
