"""The online expert-layer hook (gimbal_online_*) against the
reference's per-token loop of MoeSubsystem::iteration_cost (sim.cpp:113-147, token_crossings
sim.cpp:183-198) restated over the reference's own RoutingStats (oracle/_ref ref_hook_*):
every iteration's bottleneck-excess sum (bit-exact double) and crossing count, the window
statistics and the per-GPU activation totals, through placement changes and window resets."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,ne,k,g,batches,dup", [
    (4, 8, 2, 2, (1, 37, 4096, 5, 999), False),
    (6, 16, 4, 4, (4096, 3, 250, 4096), True),
    (32, 8, 2, 8, (4096, 17, 1), False),
    (26, 64, 6, 8, (1000, 4096), False),
    (58, 256, 8, 8, (4096, 129), False),
    (1, 8, 3, 2, (64, 7), False),
])
def test_online_iteration_matches_reference_loop(G, ref, L, ne, k, g, batches, dup):
    topo = G.MoeTopology(L, ne, k, g)
    window = G.RoutingStats(topo, 0)
    hook = G.OnlineHook(window)
    rng = np.random.default_rng(L * 1000 + ne)
    places = [G.static_placement(topo).assign] + [list(G.shuffled_candidates(L * ne, g, 70 + i, 1)[0]) for i in range(2)]
    hook.set_placement(places[0])
    rh = ref.hook_create(L, ne, k, g, places[0])
    try:
        t0 = 0
        for i, n in enumerate(batches):
            if i == 2:  # a relocation: new placement, the window is closed and reset
                hook.set_placement(places[1])
                ref.hook_set_placement(rh, places[1])
                window.reset()
                ref.hook_reset_window(rh)
            trace = G.generate_trace(topo, n, model_seed=3, stream_seed=9, first_token=t0, device=0).cpu().numpy()
            t0 += n
            if dup:
                trace[::3, :, -1] = trace[::3, :, 0]  # repeated ids: multiplicity, as add_token counts them
            ids = trace.astype(np.int32) if i % 2 else trace
            got = hook.iteration(ids)
            want = ref.hook_iteration(rh, trace.astype(np.int32))
            assert got[1] == want[1], f"iteration {i}: crossings"
            assert got[0] == want[0], f"iteration {i}: excess sum {got[0]!r} vs {want[0]!r}"
        A, E, W = window.read()
        rA, rE, rT = ref.hook_stats(rh, L, ne, g)
        assert np.array_equal(A, rA.astype(np.uint64))
        assert np.array_equal(E, rE.astype(np.uint64))
        assert np.array_equal(hook.gpu_totals(), rT)
        assert window.tokens() == (sum(batches[2:]) if len(batches) > 2 else sum(batches))
    finally:
        ref.hook_destroy(rh)


def test_online_iteration_errors(G):
    topo = G.MoeTopology(4, 8, 2, 2)
    window = G.RoutingStats(topo, 0)
    hook = G.OnlineHook(window)
    with pytest.raises(ValueError, match="no placement"):
        hook.iteration(np.zeros((3, 4, 2), np.uint8))
    with pytest.raises(ValueError, match="placement GPU id out of range"):
        hook.set_placement([5] * 32)
    hook.set_placement(G.static_placement(topo).assign)
    bad = np.zeros((3, 4, 2), np.int32)
    bad[1, 2, 1] = 8
    with pytest.raises(IndexError):
        hook.iteration(bad)
    assert hook.iteration(np.zeros((0, 4, 2), np.uint8)) == (0.0, 0)
