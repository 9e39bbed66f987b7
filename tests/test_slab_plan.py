"""z-slab decomposition plan (host-only, include/treemg_b200.h tmg_slab_plan):
every fine z-chunk, level L-1 plane and level L-2 plane has exactly one
owner, slabs are contiguous and in order, and the halo widths the exchange
schedule relies on hold."""
import pytest


@pytest.mark.parametrize("levels", [3, 4, 5, 6])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plan_partitions_every_level(tmg, levels, world):
    m, mc, m2 = 3 ** levels, 3 ** (levels - 1), 3 ** (levels - 2)
    try:
        plan = tmg.slab_plan(levels, world)
    except tmg.TreemgError:
        assert levels == 3 and world > 4  # 27^3 is too thin for 8 slabs
        return
    cb, ce, z0, z1, Zs, Ze, Ws, We = plan.T
    assert cb[0] == 0 and z0[0] == 1 and Zs[0] == 1 and Ws[0] == 1
    assert z1[-1] == m and Ze[-1] == mc and We[-1] == m2
    for r in range(world - 1):
        assert ce[r] == cb[r + 1] and z1[r] == z0[r + 1] and Ze[r] == Zs[r + 1] and We[r] == Ws[r + 1]
    for r in range(world):
        assert z0[r] % 3 == 1                      # chunk boundaries: restriction slots align
        assert Ze[r] - Zs[r] >= 2                  # two-plane r_C halo exists on the neighbour
        # level L-1 plane Z belongs to the owner of fine plane 3Z, L-2 plane W to the owner of 3W
        for Z in range(Zs[r], Ze[r]):
            assert z0[r] <= 3 * Z < z1[r] or 3 * Z == m
        for W in range(Ws[r], We[r]):
            assert Zs[r] <= 3 * W < Ze[r] or 3 * W == mc
        # the fused pass needs coarse planes [Zs-1, Ze] for its fine planes [z0-1, z1]
        assert min(z0[r] // 3, mc - 1) >= Zs[r] - 1 - 1e-9
        assert min(z1[r] // 3, mc - 1) + 1 <= Ze[r] + 1
