import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_21626_b200 as G
from oracle import Oracle
L, ne, k = 58, 256, 8
topo = G.MoeTopology(L, ne, k, 8)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 20037
trace = G.generate_trace(topo, T, model_seed=3, stream_seed=5, device=0)
s = G.RoutingStats(topo, 0)
s.add_tokens(trace)
A, E, W = s.read()
oA, oE, oW = Oracle().stats(L, ne, k, trace.cpu().numpy())
print("match", np.array_equal(E, oE), np.array_equal(A, oA))
