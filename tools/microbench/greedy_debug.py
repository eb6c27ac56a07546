# Debug helper: runs the DS-V3 pass with a printf-instrumented greedy kernel and times greedy.
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2602_21626_b200._native as N
N.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgimbal_gpu_dbg.so")
import torch, paper_2602_21626_b200 as G
for (L, ne, k, g, T) in ((58, 256, 8, 8, 1 << 24), (58, 256, 8, 8, 1 << 20)):
    topo = G.MoeTopology(L, ne, k, g)
    tr = G.generate_trace(topo, T, model_seed=1, stream_seed=2)
    s = G.RoutingStats(topo, 0); s.add_tokens(tr); s.sync()
    M = G.build_affinity_set(s, topo, 0.0, 4, L * ne // g, 0)
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); G.greedy_place(s, M, g); torch.cuda.synchronize()
        print("greedy ms", (time.perf_counter() - t) * 1e3, flush=True)
