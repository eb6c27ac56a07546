import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2602_21626_b200 as G
topo = G.MoeTopology(58, 256, 8, 8)
tr = G.generate_trace(topo, 16 << 20, model_seed=1, stream_seed=7, device=0)
s = G.RoutingStats(topo, 0)
for i in range(2):
    s.reset(); s.add_tokens(tr); torch.cuda.synchronize()
print("ok")
