"""A/B: streaming-window loop (bench config 5) with different numbers of SMs left free by the
counting kernels.  python tools/stream_reserve.py [reserve ...]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21626_b200 as G  # noqa: E402

topo = G.MoeTopology(58, 256, 8, 8)
W, n_win, C = 1 << 20, int(sys.argv[1]) if len(sys.argv) > 1 else 16, 256
wins = [G.generate_trace(topo, W, model_seed=1, stream_seed=2, first_token=w * W, drift=0.05, drift_epoch=w + 1,
                         device=0) for w in range(n_win)]
calib = G.generate_trace(topo, 20000, model_seed=1, stream_seed=3, drift=0.05, drift_epoch=0, device=0)
cands = torch.from_numpy(G.shuffled_candidates(topo.total_experts(), 8, 1000, C)).cuda()
hp = G.HotPath(topo, 0)
M = hp.calibrate(calib)
for r in [int(x) for x in sys.argv[2:]] or [0, 1, 2, 4]:
    for _ in range(2):
        hp.stream(wins, cands, M, reserve_sms=r)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        hp.stream(wins, cands, M, reserve_sms=r)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 3 * 1e3
    print(f"reserve {r}: {ms:.2f} ms / {n_win} windows = {ms / n_win:.3f} ms/window, {n_win * W / ms / 1e3:.1f} M tokens/s")
