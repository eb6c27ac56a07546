import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2602_21626_b200 as G
topo = G.MoeTopology(58, 256, 8, 8)
T = int(sys.argv[1]) if len(sys.argv) > 1 else (64 << 20)
tr = G.generate_trace(topo, T, model_seed=1, stream_seed=2, device=0)
cands = torch.from_numpy(G.shuffled_candidates(topo.total_experts(), 8, 1000, 64)).cuda()
hp = G.HotPath(topo, device=0)
res = hp.run(tr, cands)
torch.cuda.synchronize()
print("argmin", res.argmin)
