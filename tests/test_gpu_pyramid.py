"""The single-launch coarse phases against the launches they replace:
the pyramid top-down (fast::topdown_pyramid vs chain_down + topdown_coarse,
TMG_PYR=0), the bottom-up below level L-1 (fast::up_coop and the smoothing
folded into the restriction kernels vs restrict / smooth launches + the
cluster chain, TMG_UP=0), the parent-triple top-down of big coarse levels
(TMG_TRI_COARSE=0) and programmatic dependent launch (TMG_PDL=0).  Bitwise equal iterates and norms,
2D and 3D, additive / BPX / hb / ell_min, several tile-boundary alignments."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    (2, 3, 100 + 50j, "add"), (2, 5, 100 + 50j, "add"), (2, 6, 10000 + 5000j, "bpx"), (2, 7, 10000 + 5000j, "bpx"),
    (3, 2, 400 + 200j, "add"), (3, 3, 400 + 200j, "bpx"), (3, 4, 400 + 200j, "add"), (3, 4, 1600 + 800j, "hb"),
    (3, 5, 400 + 200j, "bpx"), (2, 5, 100 + 50j, "lgrid"), (3, 4, 400 + 200j, "bpx2"), (3, 6, 6400 + 3200j, "add"),
    (2, 8, 10000 + 5000j, "bpx"), (3, 3, 400 + 200j, "lgrid"),
]


def _run(tmg, dim, level, phi, kind, new, cycles=4):
    os.environ["TMG_PYR"] = os.environ["TMG_UP"] = os.environ["TMG_TRI_COARSE"] = os.environ["TMG_PDL"] = "1" if new else "0"
    try:
        pol = {"add": tmg.Policy("exponential", 0.6), "bpx": tmg.Policy("undamped", 0.5, bpx=True),
               "bpx2": tmg.Policy("undamped", 0.5, bpx=True), "lgrid": tmg.Policy("lgrid", 0.6, lgrid=1),
               "hb": tmg.Policy("exponential", 0.6, hb=True)}[kind]
        kw = {"ell_min": 2} if kind in ("lgrid", "bpx2") else {}
        h = tmg.Hierarchy(dim, level, phi=phi, chi="seeded", precision="fast", max_vertices=10 ** 10, **kw)
        norms = []
        for n in range(1, cycles + 1):
            st = h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
            norms.append((st.max_norm, st.h_norm))
        return norms, h.field(level, "u"), [h.field(l, "sc") for l in range(1, level)]
    finally:
        os.environ.pop("TMG_PYR", None)
        os.environ.pop("TMG_UP", None)
        os.environ.pop("TMG_TRI_COARSE", None)
        os.environ.pop("TMG_PDL", None)


@pytest.mark.parametrize("dim,level,phi,kind", CASES)
def test_single_launch_coarse_phases_bitwise_equal(tmg, dim, level, phi, kind):
    na, ua, sa = _run(tmg, dim, level, phi, kind, True)
    nb, ub, sb = _run(tmg, dim, level, phi, kind, False)
    assert na == nb
    assert np.array_equal(ua, ub)
    for x, y in zip(sa, sb):
        assert np.array_equal(x, y)
