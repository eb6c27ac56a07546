"""Quick correctness/timing check of the DS-V3 counting path against the oracle (small T), then
a timing comparison of the FP4 tensor-core path and the u15 atomic path at 64 Mi tokens."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import oracle
import paper_2602_21626_b200 as G

topo = G.MoeTopology(58, 256, 8, 8)
o = oracle.Oracle()
for T in (1, 127, 128, 129, 4096 + 3, 70001):
    tr = G.generate_trace(topo, T, model_seed=1, stream_seed=T, device=0)
    s = G.RoutingStats(topo, 0)
    s.add_tokens(tr)
    A, E, W = s.read()
    oA, oE, oW = o.stats(58, 256, 8, tr.cpu().numpy())
    print("T", T, "A", np.array_equal(A, oA), "E", np.array_equal(E, oE), "W", np.array_equal(W, oW),
          "maxdiff", int(np.abs(E.astype(np.int64) - oE.astype(np.int64)).max()), flush=True)
# duplicates
rng = np.random.default_rng(0)
ids = rng.integers(0, 256, size=(5000, 58, 8), dtype=np.uint8)
ids[::3, :, 1] = ids[::3, :, 0]
s = G.RoutingStats(topo, 0)
s.add_tokens(torch.from_numpy(ids).cuda())
A, E, W = s.read()
oA, oE, oW = o.stats(58, 256, 8, ids)
print("dups E", np.array_equal(E, oE), flush=True)
T = 64 << 20
tr = G.generate_trace(topo, T, model_seed=1, stream_seed=7, device=0)
for path in ("fp4", "u15"):
    os.environ["GIMBAL_COUNT_PATH"] = path
    s = G.RoutingStats(topo, 0)
    for i in range(4):
        torch.cuda.synchronize(); t0 = time.time()
        s.reset(); s.add_tokens(tr); torch.cuda.synchronize()
        dt = time.time() - t0
    A, E, W = s.read()
    print(path, "ms", round(dt * 1e3, 2), "E sum", int(E.sum()), flush=True)
