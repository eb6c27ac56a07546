"""bench.py contract checks that need no GPU: the --impl reference arm runs the reference's own code
(oracle/_ref) without loading the product library, and prints the same config keys as our arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, sys
sys.path.insert(0, {root!r})
import bench
bench.sample_size = lambda config: (4096, 2048, 4)
bench.single_thread_figure = lambda *a, **k: {{"value": 0.0}}
sys.argv = ["bench.py", "--impl", "reference", "--config", "mixtral", "--steps", "1", "--warmup", "3"]
bench.main()
maps = open("/proc/self/maps").read()
print(json.dumps({{"modules": sorted(m for m in sys.modules if m.startswith("paper_2602_21626_b200")),
                  "gpu_lib": "libgimbal_gpu" in maps, "ref_lib": "libgimbal_ref" in maps}}))
"""


def test_reference_arm_loads_only_the_reference():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "-c", PROBE.format(root=ROOT)], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.strip().splitlines()]
    line, probe = lines[0], lines[1]
    assert probe == {"modules": [], "gpu_lib": False, "ref_lib": True}
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert set(line["config"]) == {"workload", "tokens", "candidates", "g", "scaling", "parallelism", "l2"}
    assert line["config"] == __import__("bench").bench_config("mixtral", 1, 1 << 20, 4096, "strong")


def test_reference_sample_matches_gpu_arm_inputs():
    """The reference arm's tables / candidates are the product's (same bytes), built from the
    reference alone: generator tables from RoutingModel weights, candidates by the reference recipe."""
    import numpy as np

    import oracle
    import paper_2602_21626_b200 as G

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle.Ref()
    for L, ne, k, g in [(58, 256, 8, 8), (32, 8, 2, 8), (26, 64, 6, 8), (48, 128, 8, 8)]:
        cdf, thr = oracle.generator_tables_from_ref(ref, L, ne, k, g, model_seed=1)
        gc, gt = G.generator_tables(G.MoeTopology(L, ne, k, g), model_seed=1)
        assert np.array_equal(cdf, gc) and np.array_equal(thr, gt)
        m = L * ne
        want = G.shuffled_candidates(m, g, 1000, 3)
        got = np.stack([ref.shuffled_balanced(m, g, 1000 + c) for c in range(3)]).astype(np.uint8)
        assert np.array_equal(got, want)
