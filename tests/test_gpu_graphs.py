"""CUDA graphs of back-to-back cycles (Hierarchy::time_cycles): a
run whose cycles are replayed from captured graphs must leave exactly the
state of the same cycles launched one by one (td_add / td_bpx with their norm
readback): every level's u / sc bitwise, and the next cycle's norms equal.
Regular 2D / 3D trees (fused fine passes, double-buffered fine level: both
buffer states are captured) and a static adaptive tree."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    dict(dim=2, level=5, phi=100 + 50j, bpx=False),
    dict(dim=2, level=6, phi=10000 + 5000j, bpx=True),
    dict(dim=3, level=4, phi=400 + 200j, bpx=False),
    dict(dim=3, level=4, phi=400 + 200j, bpx=True),
]


def _hier(tmg, c, **kw):
    return tmg.Hierarchy(c["dim"], c["level"], phi=c["phi"], chi="seeded", precision="fast", max_vertices=10 ** 10,
                         **kw)


def _pol(tmg, bpx):
    return tmg.Policy("undamped", 0.5, bpx=True) if bpx else tmg.Policy("exponential", 0.6)


@pytest.mark.parametrize("c", CASES, ids=lambda c: f"d{c['dim']}l{c['level']}{'bpx' if c['bpx'] else ''}")
def test_graph_replays_equal_launches(tmg, c):
    pol = _pol(tmg, c["bpx"])
    hg, hl = _hier(tmg, c), _hier(tmg, c)
    cycles = 7  # odd: ends on the other buffer state, both graphs replayed
    hg.time_cycles(pol, 1, cycles)
    for n in range(1, cycles + 1):
        hl.td_bpx(pol, n) if c["bpx"] else hl.td_add(pol, n)
    for lvl in range(1, c["level"] + 1):
        for f in ("u", "sc"):
            assert np.array_equal(hg.field(lvl, f), hl.field(lvl, f)), (lvl, f)
    sg = hg.td_bpx(pol, cycles + 1) if c["bpx"] else hg.td_add(pol, cycles + 1)
    sl = hl.td_bpx(pol, cycles + 1) if c["bpx"] else hl.td_add(pol, cycles + 1)
    assert (sg.max_norm, sg.euclid_norm) == (sl.max_norm, sl.euclid_norm)


@pytest.mark.parametrize("precision", ["fast", "exact"])
def test_graph_replays_equal_launches_adaptive(tmg, precision):
    kw = dict(phi=1600 + 800j, chi="seeded", rhs_seed=12345, rhs_sphere=True, precision=precision,
              max_vertices=10 ** 9, sphere_levels=2)
    hg, hl = tmg.Hierarchy(3, 2, **kw), tmg.Hierarchy(3, 2, **kw)
    pol = tmg.Policy("exponential", 0.6)
    hg.time_cycles(pol, 1, 5)
    for n in range(1, 6):
        hl.td_add(pol, n)
    for lvl in range(1, 5):
        for f in ("u", "sc", "rhat"):
            assert np.array_equal(hg.field(lvl, f), hl.field(lvl, f)), (lvl, f)
    assert hg.td_add(pol, 6).max_norm == hl.td_add(pol, 6).max_norm
