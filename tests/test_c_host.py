"""A plain-C host (tools/c_host_pass.c, built as lib/c_host_pass) runs the pass through the C ABI only
-- host ids counted from host memory, strong-pair set, greedy placement, every candidate scored -- and
its outputs match the CPU oracle (moe.cpp:169-191, placement.cpp:58-85, 186-299)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2602_21626_b200", "lib", "c_host_pass")


@pytest.mark.parametrize("L,ne,k,g,T,C", [(26, 64, 6, 8, 30001, 70), (32, 8, 2, 8, 9001, 33), (58, 256, 8, 8, 4099, 9),
                                          (48, 128, 8, 8, 5000, 17)])
def test_c_host_pass_matches_oracle(G, orc, tmp_path, L, ne, k, g, T, C):
    topo = G.MoeTopology(L, ne, k, g)
    ids = G.generate_trace(topo, T, model_seed=5, stream_seed=L, device=0).cpu().numpy()
    cands = G.shuffled_candidates(L * ne, g, 19, C)
    ids.tofile(tmp_path / "ids.bin")
    cands.tofile(tmp_path / "cands.bin")
    out = subprocess.run([EXE, str(L), str(ne), str(k), str(g), str(T), str(C), str(tmp_path / "ids.bin"),
                          str(tmp_path / "cands.bin"), str(tmp_path / "out.bin")], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    raw = (tmp_path / "out.bin").read_bytes()
    m = L * ne
    off = 0

    def take(dtype, n):
        nonlocal off
        a = np.frombuffer(raw, dtype=dtype, count=n, offset=off)
        off += a.nbytes
        return a

    A = take(np.uint64, m).reshape(L, ne)
    E = take(np.uint64, (L - 1) * ne * ne).reshape(L - 1, ne, ne)
    nM = int(take(np.int32, 1)[0])
    M = take(np.int32, nM).tolist()
    greedy = take(np.int32, m)
    D, cut, obj = take(np.float64, C), take(np.float64, C), take(np.float64, C)
    argmin = int(take(np.int64, 1)[0])
    assert off == len(raw)
    oA, oE, _ = orc.stats(L, ne, k, ids)
    assert np.array_equal(A, oA) and np.array_equal(E, oE)
    oM = list(orc.affinity_set(L, ne, g, oE, 0.0, 4, m // g, 0))
    assert M == oM
    assert np.array_equal(greedy, orc.greedy_place(L, ne, g, oA, oM, 0))
    oD, ocut, oobj, oam = orc.eval_costs(L, ne, g, oA, oE, cands)
    assert np.array_equal(D, oD) and np.array_equal(cut, ocut) and np.array_equal(obj, oobj) and argmin == oam
