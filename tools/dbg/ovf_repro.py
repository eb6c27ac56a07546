import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_21626_b200 as G
L, ne, k = 58, 256, 8
topo = G.MoeTopology(L, ne, k, 8)
for T in (1 << 20, 100000, 1 << 20, 100000):
    row = np.full((L, k), 3, np.uint8)
    trace = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(row, (T, L, k)))).cuda()
    s = G.RoutingStats(topo, 0)
    s.add_tokens(trace)
    A, E, W = s.read()
    want = T * 64
    got = E[:, 3, 3].astype(np.int64)
    bad = np.nonzero(got != want)[0]
    print(T, "bad pairs", bad[:10], "diff", (got[bad] - want)[:10], "other nonzero", int((E.sum() - E[:, 3, 3].sum())))
    for p in bad[:2]:
        nz = np.argwhere(E[p] != 0)
        print(" pair", p, [(int(a), int(b), int(E[p, a, b])) for a, b in nz[:8]])
