import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2602_21626_b200 as G
topo = G.MoeTopology(32, 8, 2, 8)
trace = G.generate_trace(topo, 30000, model_seed=4, stream_seed=8, device=0)
cands = torch.from_numpy(G.shuffled_candidates(256, 8, 123, 70)).cuda()
hp = G.HotPath(topo, 0)
print("run", flush=True)
res = hp.run(trace, cands)
print("ok", res.argmin, len(res.affinity.experts), flush=True)
del hp
print("deleted", flush=True)
