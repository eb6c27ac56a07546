#!/usr/bin/env python3
"""exact_solve: GPU enumeration (gimbal_exact_solve_dense) vs the reference's branch and bound
(oracle/_ref), same instances, wall time per call (best of 5 after a warm-up), answers compared."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2602_21626_b200 as G  # noqa: E402


def best_of(f, n=5):
    f()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t)
    return min(ts), r


def main():
    ref = oracle.Ref()
    rng = np.random.default_rng(5)
    for (m, g, rows) in [(8, 2, 2), (12, 3, 2), (12, 4, 2), (16, 2, 2), (16, 4, 1), (16, 4, 3), (16, 4, 16)]:
        A = rng.integers(0, 100, size=(rows, m)).astype(np.float64)
        W = np.triu(rng.integers(0, 30, size=(m, m)) * (rng.random((m, m)) < 0.3), 1).astype(np.float64)
        P = G.PlacementProblem(A=A, W=W, g=g)
        tg, (pl, c) = best_of(lambda: G.exact_solve(P))
        tr, (ra, rc) = best_of(lambda: ref.exact_solve(A, W, g))
        same = pl.assign == ra.tolist() and (c.deviation, c.cut, c.objective) == rc
        print(f"m={m:2d} g={g} rows={rows:2d}: gpu {tg * 1e3:8.2f} ms  reference {tr * 1e3:8.2f} ms  same={same}")


if __name__ == "__main__":
    main()
