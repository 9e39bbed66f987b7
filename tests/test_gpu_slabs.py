"""z-slab execution on one GPU with K virtual slabs (the same code path as
the NCCL ranks, transfers as device copies): the fine-level iterate must be
bitwise identical to the unsharded run for every slab count, the norms equal
up to the summation order of the slab partials."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("levels,phi", [(4, 400 + 200j), (5, 400 + 200j)])
@pytest.mark.parametrize("kind", ["td-add", "td-bpx"])
@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_virtual_slabs_bitwise_equal_single(tmg, levels, phi, kind, k):
    pol = tmg.Policy("exponential", 0.6) if kind == "td-add" else tmg.Policy("undamped", 0.5, bpx=True)
    one = tmg.Hierarchy(3, levels, phi=phi, chi="seeded", precision="fast", max_vertices=10 ** 10)
    sl = tmg.Slabs(levels, phi, local=k)
    for n in range(1, 7):
        a = one.td_bpx(pol, n) if pol.bpx else one.td_add(pol, n)
        b = sl.cycle(pol, n)
        assert abs(a.h_norm - b.h_norm) <= 1e-13 * a.h_norm, n
        assert abs(a.max_norm - b.max_norm) <= 1e-15 * a.max_norm, n
    u1 = one.field(levels, "u")
    uk = sl.fine_u()
    assert np.array_equal(u1, uk)


def test_nccl_unique_id(tmg):
    uid = tmg.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
