#!/usr/bin/env python3
"""Phase timestamps of the fused small-shape pass (AB build only: GIMBAL_LIB=lib/libgimbal_gpu_ab.so).
CTA 0: E load + A derive | top-K + select | greedy keys + sort | greedy walk | row-0 score; then the
last CTA's finish.  Prints microseconds per phase for the Mixtral bench shape."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21626_b200 as G  # noqa: E402

L, ne, k, g, T, C = 32, 8, 2, 8, 1 << 20, int(sys.argv[1]) if len(sys.argv) > 1 else 4096
topo = G.MoeTopology(L, ne, k, g)
trace = G.generate_trace(topo, T, model_seed=1, stream_seed=2, device=0)
cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 1000, C)).cuda()
hp = G.HotPath(topo, 0)
lib = G._native.lib()
fn = lib.gimbal_debug_tiny_profile
fn.argtypes = [ctypes.c_void_p]
names = ["E+A", "topK+select", "keys+sort", "walk", "score row 0", "-> last CTA start", "finish"]
acc = []
for it in range(12):
    hp.run(trace, cands)
    torch.cuda.synchronize()
    buf = np.zeros(16, np.uint64)
    fn(buf.ctypes.data)
    if it >= 2:
        acc.append(np.diff(buf[:8].astype(np.int64)) / 1e3)
a = np.median(np.array(acc), axis=0)
for n, v in zip(names, a):
    print(f"{n:20s} {v:8.2f} us")
print(f"{'total (mark 0..7)':20s} {a.sum():8.2f} us")
