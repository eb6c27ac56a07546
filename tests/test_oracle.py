"""Pins the CPU oracle (CPU-only): reference KATs, reference golden fixtures, and live
comparison with the reference's own compiled sources (oracle/_ref) where they were built."""
import os
import subprocess

import numpy as np
import pytest

import kat_util as K


# ---- KATs transcribed from the reference unit tests ----

def test_kat_stats(orc):
    for c in K.kats()["stats"]:
        A, E, W = orc.stats(c["L"], c["ne"], c["k"], K.trace(c))
        assert np.array_equal(A, np.asarray(c["A"], np.uint64)), c["src"]
        assert np.array_equal(E, K.expected_e(c)), c["src"]
        assert np.array_equal(W, K.expected_w(c)), c["src"]


def test_kat_comm_cost(orc):
    for c in K.kats()["comm_cost"]:
        if c.get("error"):
            with pytest.raises(ValueError):
                orc.comm_cost(c["L"], c["ne"], c["k"], K.trace(c), c["assign"])
        else:
            assert orc.comm_cost(c["L"], c["ne"], c["k"], K.trace(c), c["assign"]) == c["expected"], c["src"]


def _check_cost(c, D, cut, obj):
    if "D" in c:
        assert D == c["D"], c["src"]
    if "cut" in c:
        assert cut == c["cut"], c["src"]
    if "objective" in c:
        assert obj == c["objective"], c["src"]


def test_kat_eval_cost_dense(orc):
    for c in K.kats()["eval_cost"]:
        A = np.asarray(c["A"], np.float64)
        W = K.dense_w(c["W"], A.shape[1])
        args = (A, W, c["g"], np.asarray(c["assign"], np.int32), c.get("alpha", 1.0), c.get("beta", 1.0))
        if c.get("error"):
            if len(c["assign"]) != A.shape[1]:
                continue  # the C oracle takes a fixed-size array; size errors are checked via Ref/GPU
            with pytest.raises(ValueError):
                orc.eval_cost_dense(*args)
        else:
            _check_cost(c, *orc.eval_cost_dense(*args))


def test_kat_eval_cost_compact_matches_dense(orc):
    # a 1 x m activation is a single-layer flat problem; W only on consecutive layers -> use L=1
    c = K.kats()["eval_cost"][5]
    A = np.asarray(c["A"], np.uint64)
    D, cut, obj = orc.eval_cost(1, A.shape[1], c["g"], A, np.zeros(1, np.uint64), c["assign"])
    assert (D, cut, obj) == (4.0, 0.0, 4.0)


def test_kat_affinity_set(orc):
    for c in K.kats()["affinity_set"]:
        E = K.e_from_nonzero(c)
        got = orc.affinity_set(c["L"], c["ne"], c["g"], E, c["threshold"], c["top_e"], c["capacity"], c["anchor"])
        assert list(got) == c["expected"], c["src"]


def test_kat_greedy(orc):
    for c in K.kats()["greedy"]:
        A = np.asarray(c["A"], np.uint64)
        if c.get("error"):
            with pytest.raises(ValueError):
                orc.greedy_place(1, A.shape[1], c["g"], A, c["M"], c["anchor"])
            continue
        out = orc.greedy_place(1, A.shape[1], c["g"], A, c["M"], c["anchor"])
        if "expected" in c:
            assert list(out) == c["expected"], c["src"]
        if "deviation" in c:
            D, _, _ = orc.eval_cost(1, A.shape[1], c["g"], A, np.zeros(1, np.uint64), out)
            assert D == c["deviation"], c["src"]


def test_kat_static_placement(orc):
    for c in K.kats()["static_placement"]:
        assert list(orc.static_placement(c["L"], c["ne"], c["k"], c["g"])) == c["expected"]


# ---- the KATs hold for the reference itself (proves the transcription) ----

def test_kats_against_reference(ref):
    k = K.kats()
    for c in k["stats"]:
        A, E, W, tok = ref.record_stats(c["L"], c["ne"], c["k"], 2, K.trace(c))
        assert np.array_equal(A, np.asarray(c["A"], np.float64)) and tok == c["tokens"]
        assert np.array_equal(E, K.expected_e(c).astype(np.float64))
    for c in k["comm_cost"]:
        if c.get("error"):
            with pytest.raises(ValueError):
                ref.comm_cost(c["L"], c["ne"], c["k"], 2, K.trace(c), c["assign"])
        else:
            assert ref.comm_cost(c["L"], c["ne"], c["k"], 2, K.trace(c), c["assign"]) == c["expected"]
    for c in k["eval_cost"]:
        A = np.asarray(c["A"], np.float64)
        W = K.dense_w(c["W"], A.shape[1])
        if c.get("error"):
            with pytest.raises(ValueError):
                ref.eval_cost(A, W, c["g"], c["assign"], c.get("alpha", 1.0), c.get("beta", 1.0))
        else:
            _check_cost(c, *ref.eval_cost(A, W, c["g"], c["assign"], c.get("alpha", 1.0), c.get("beta", 1.0)))
    for c in k["affinity_set"]:
        got = ref.build_affinity_set(c["L"], c["ne"], 1, c["g"], K.e_from_nonzero(c).astype(np.float64),
                                     c["threshold"], c["top_e"], c["capacity"], c["anchor"])
        assert list(got) == c["expected"], c["src"]
    for c in k["greedy"]:
        A = np.asarray(c["A"], np.float64)
        if c.get("error"):
            with pytest.raises(ValueError):
                ref.greedy_place(A, c["g"], c["M"], c["anchor"])
        elif "expected" in c:
            assert list(ref.greedy_place(A, c["g"], c["M"], c["anchor"])) == c["expected"]
    for c in k["maybe_relocate"]:
        A = np.asarray(c["A"], np.float64)
        r = ref.maybe_relocate(c["step"], c["tau"], [], 0, A, c["g"], c["prev"])
        assert (r is not None) == c["fires"]
        if r is not None and "again_moved" in c:
            r2 = ref.maybe_relocate(c["step"] * 2, c["tau"], [], 0, A, c["g"], r[0])
            assert r2[1] == c["again_moved"]


# ---- golden fixtures produced by the reference (tests/golden/make_golden.py) ----

def test_golden_fixtures_oracle(orc):
    for c in K.golden_cases():
        L, ne, k, g = (int(x) for x in c["topo"])
        thr, top = float(c["params"][3]), int(c["params"][4])
        A, E, W = orc.stats(L, ne, k, c["ids"])
        assert np.array_equal(A, c["A"]) and np.array_equal(E, c["E"]) and np.array_equal(W, c["W"])
        assert orc.comm_cost(L, ne, k, c["ids"], c["assign"]) == int(c["comm_cost"])
        assert orc.eval_cost(L, ne, g, A, E, c["assign"]) == tuple(c["cost"])
        assert orc.eval_cost(L, ne, g, A, E, c["assign"], 2.5, 0.75) == tuple(c["cost_ab"])
        M = orc.affinity_set(L, ne, g, E, thr, top, L * ne // g, g - 1)
        assert np.array_equal(M, c["M"])
        gp = orc.greedy_place(L, ne, g, A, M, g - 1)
        assert np.array_equal(gp, c["greedy"])
        assert orc.eval_cost(L, ne, g, A, E, gp) == tuple(c["greedy_cost"])


# ---- live cross-check against the reference's compiled sources ----

def test_oracle_vs_reference_random(orc, ref):
    rng = np.random.default_rng(7)
    for trial in range(60):
        g = int(rng.choice([1, 2, 4]))
        ne = g * int(rng.integers(1, 5))
        L = int(rng.integers(1, 6))
        k = int(rng.integers(1, ne + 1))
        T = int(rng.integers(0, 300))
        # duplicates within a layer are allowed by the reference (counted with multiplicity)
        ids = rng.integers(0, ne, size=(T, L, k)).astype(np.int32)
        A, E, W = orc.stats(L, ne, k, ids)
        rA, rE, rW, tok = ref.record_stats(L, ne, k, g, ids)
        assert np.array_equal(A, rA) and np.array_equal(E, rE) and np.array_equal(W, rW) and tok == T
        fA, fW = ref.flat_forms(L, ne, k, g, ids)
        assign = ref.shuffled_balanced(L * ne, g, trial)
        assert orc.comm_cost(L, ne, k, ids, assign) == ref.comm_cost(L, ne, k, g, ids, assign)
        a, b = float(rng.uniform(0.1, 3)), float(rng.uniform(0.1, 3))
        assert orc.eval_cost(L, ne, g, A, E, assign, a, b) == ref.eval_cost(fA, fW, g, assign, a, b)
        assert orc.eval_cost_dense(fA, fW, g, assign, a, b) == ref.eval_cost(fA, fW, g, assign, a, b)
        thr = float(rng.choice([0.0, 1.0, 3.0]))
        top = int(rng.choice([-1, 0, 2, 4, 9]))
        cap = int(rng.integers(-1, L * ne // g + 2))
        anc = int(rng.integers(0, g))
        if L > 1:
            M = orc.affinity_set(L, ne, g, E, thr, top, cap, anc)
            assert list(M) == list(ref.build_affinity_set(L, ne, k, g, rE, thr, top, cap, anc))
        else:
            M = np.zeros(0, np.int32)
        if len(M) <= L * ne // g:
            assert list(orc.greedy_place(L, ne, g, A, M, anc)) == list(ref.greedy_place(fA, g, M, anc))


def test_reference_unit_tests_pass_with_eigen_subset():
    """The reference's own test_moe.cpp + test_placement.cpp (32 TEST_CASEs) compiled against
    its own sources with oracle/eigen_subset and oracle/doctest_lite."""
    import oracle

    binary = os.path.join(oracle.HERE, "_ref", "ref_unit_tests")
    if not os.path.exists(binary):
        pytest.skip("oracle/_ref/ref_unit_tests not built")
    out = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "| 0 failed" in out.stdout


def test_generator_twin_is_deterministic_and_distinct(orc):
    import paper_2602_21626_b200 as G

    topo = G.MoeTopology(6, 32, 4, 4)
    cdf, thr = G.generator_tables(topo, model_seed=3)
    a = orc.generate_trace(6, 32, 4, cdf.ravel(), int(thr[0]), int(thr[1]), 9, 100, 500)
    b = orc.generate_trace(6, 32, 4, cdf.ravel(), int(thr[0]), int(thr[1]), 9, 100, 500)
    assert np.array_equal(a, b)
    # any token range is reproducible (counter-based stream)
    c = orc.generate_trace(6, 32, 4, cdf.ravel(), int(thr[0]), int(thr[1]), 9, 300, 100)
    assert np.array_equal(a[200:300], c)
    # top_k draws without replacement: distinct ids per layer
    assert all(len(set(a[t, l])) == 4 for t in range(500) for l in range(6))


def test_eval_excess_restatement_matches_reference_hook_loop(ref, orc):
    """The per-candidate bottleneck excess oracle (go_eval_excess) over a batch's counts equals the
    reference simulator's per-iteration excess (sim.cpp:132-144 via ref_hook_iteration) for that
    batch under the same placement."""
    import numpy as np

    for L, ne, k, g, n in [(4, 8, 2, 2, 333), (6, 16, 4, 4, 4096), (32, 8, 2, 8, 77), (5, 64, 6, 8, 1000)]:
        rng = np.random.default_rng(n)
        ids = rng.integers(0, ne, size=(n, L, k)).astype(np.int32)
        cands = np.stack([np.random.default_rng(c).permutation(np.arange(L * ne) % g) for c in range(5)]).astype(np.uint8)
        A, _, _ = orc.stats(L, ne, k, ids)
        got = orc.eval_excess(L, ne, g, A, cands)
        for c in range(5):
            h = ref.hook_create(L, ne, k, g, cands[c].astype(np.int32))
            try:
                want, _ = ref.hook_iteration(h, ids)
            finally:
                ref.hook_destroy(h)
            assert got[c] == want
