"""exact_solve on the GPU (csrc/exact.cu, gimbal_exact_solve_dense) against the reference's own branch
and bound (placement.cpp:87-184, compiled in oracle/_ref): the same placement (the lexicographically
least optimum) and the same cost, bit for bit, on the reference's unit-test cases
(test_placement.cpp:106-160) and on random instances up to the size limit (16 experts, 4 GPUs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def problem(G, A, W, g, alpha=1.0, beta=1.0):
    return G.PlacementProblem(A=np.atleast_2d(np.asarray(A, np.float64)), W=np.asarray(W, np.float64), g=g,
                              alpha=alpha, beta=beta)


def test_reference_cases(G):
    # test_placement.cpp:106-115: the forced two-expert split
    W = np.zeros((2, 2))
    W[0, 1] = 5.0
    pl, c = G.exact_solve(problem(G, [[1, 1]], W, 2))
    assert pl.assign == [0, 1] and (c.cut, c.deviation, c.objective) == (5.0, 0.0, 5.0)
    # :117-123: both {0,1}|{2,3} and {0,3}|{1,2} give D = 0; the lexicographically smaller wins
    pl, c = G.exact_solve(problem(G, [[8, 2, 6, 4]], np.zeros((4, 4)), 2))
    assert c.deviation == 0.0 and pl.assign == [0, 0, 1, 1]
    # :125-132: a dominant pair is co-located
    W = np.zeros((4, 4))
    W[0, 1] = 100.0
    pl, c = G.exact_solve(problem(G, [[1, 1, 1, 1]], W, 2))
    assert pl.assign[0] == pl.assign[1] and c.cut == 0.0


def test_validation(G):
    # test_placement.cpp:134-140
    with pytest.raises(ValueError):
        G.exact_solve(problem(G, [[1, 1, 1]], np.zeros((3, 3)), 2))
    with pytest.raises(ValueError, match="greedy_place"):
        G.exact_solve(problem(G, np.ones((1, 20)), np.zeros((20, 20)), 2))
    with pytest.raises(ValueError, match="greedy_place"):
        G.exact_solve(problem(G, np.ones((1, 10)), np.zeros((10, 10)), 5))
    with pytest.raises(ValueError):
        G.exact_solve(problem(G, [[1, 1]], np.zeros((2, 2)), 2, alpha=0.0))
    # outside the exact domain (non-integer counts): refused, not approximated
    with pytest.raises(Exception, match="integer"):
        G.exact_solve(problem(G, [[1.5, 1]], np.zeros((2, 2)), 2))


def random_instance(rng, m, g, rows, w_density=0.3, a_max=50, w_max=20):
    A = rng.integers(0, a_max, size=(rows, m)).astype(np.float64)
    W = np.triu(rng.integers(0, w_max, size=(m, m)) * (rng.random((m, m)) < w_density), 1).astype(np.float64)
    if rng.random() < 0.3:  # both triangles
        W += np.tril(rng.integers(0, w_max, size=(m, m)) * (rng.random((m, m)) < w_density), -1)
    return A, W


def check_against_reference(G, ref, A, W, g, alpha=1.0, beta=1.0):
    pl, c = G.exact_solve(problem(G, A, W, g, alpha, beta))
    ra, (rD, rc, ro) = ref.exact_solve(A, W, g, alpha, beta)
    assert pl.assign == ra.tolist(), (pl.assign, ra.tolist())
    assert (c.deviation, c.cut, c.objective) == (rD, rc, ro)


def test_random_small_like_reference(G, ref):
    # test_placement.cpp:142-160's generator: g in {2, 3}, m in {2g, 3g}, 1-2 layers
    rng = np.random.default_rng(2024)
    for _ in range(60):
        g = 2 + int(rng.integers(2))
        m = g * (2 + int(rng.integers(2)))
        A, W = random_instance(rng, m, g, 1 + int(rng.integers(2)))
        check_against_reference(G, ref, A, W, g)


@pytest.mark.parametrize("m,g,rows,seed", [(16, 4, 1, 1), (16, 4, 3, 2), (16, 2, 2, 3), (12, 3, 2, 4), (12, 4, 4, 5),
                                           (15, 3, 1, 6), (16, 1, 2, 7), (1, 1, 1, 8), (4, 4, 2, 9), (14, 2, 5, 10)])
def test_random_up_to_the_limit(G, ref, m, g, rows, seed):
    rng = np.random.default_rng(seed)
    for trial in range(3):
        A, W = random_instance(rng, m, g, rows, w_density=0.3 + 0.2 * trial)
        check_against_reference(G, ref, A, W, g)


def test_ties_and_weights(G, ref):
    rng = np.random.default_rng(11)
    # many ties: all-equal activations, sparse tiny weights; alpha / beta away from 1
    for (m, g) in ((8, 2), (12, 4), (16, 4), (9, 3)):
        A = np.ones((2, m))
        W = np.triu((rng.random((m, m)) < 0.1).astype(np.float64), 1)
        check_against_reference(G, ref, A, W, g)
        check_against_reference(G, ref, A, np.zeros((m, m)), g)
        A, W = random_instance(rng, m, g, 2)
        check_against_reference(G, ref, A, W, g, alpha=0.75, beta=2.5)
