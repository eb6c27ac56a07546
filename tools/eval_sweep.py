"""Candidate-scoring cost vs the number of candidates C on the DS-V3 shape (16 Mi counted tokens):
tensor-core evaluator (eval_mma.cu) against the integer-ALU one (GIMBAL_EVAL_ALU=1), device time of
gimbal_eval_costs with CUDA events.  python tools/eval_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_21626_b200 as G  # noqa: E402

topo = G.MoeTopology(58, 256, 8, 8)
tr = G.generate_trace(topo, 16 << 20, model_seed=1, stream_seed=2, device=0)
s = G.RoutingStats(topo, 0)
s.add_tokens(tr)
stream = torch.cuda.ExternalStream(s.device_buffers()[2], device=torch.device("cuda", 0))
print("     C   tensor_ms   alu_ms   speed-up")
for C in (256, 1024, 4096, 16384):
    cands = torch.from_numpy(G.shuffled_candidates(topo.total_experts(), 8, 7, C)).cuda()
    out = torch.empty((3, C), dtype=torch.float64, device="cuda")
    res = {}
    for mode in ("tensor", "alu"):
        if mode == "alu":
            os.environ["GIMBAL_EVAL_ALU"] = "1"
        else:
            os.environ.pop("GIMBAL_EVAL_ALU", None)
        G.eval_costs(s, cands, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(5):
            G.eval_costs(s, cands, out=out)
        b.record(stream)
        torch.cuda.synchronize()
        res[mode] = a.elapsed_time(b) / 5
    print(f"{C:6d}   {res['tensor']:8.3f}   {res['alu']:7.3f}   {res['alu'] / res['tensor']:6.2f}x")
