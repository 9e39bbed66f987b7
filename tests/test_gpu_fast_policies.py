"""Fast precision (fused passes, v-form, cluster chains) against exact
precision (bit-identical to the reference) across the policy space the
BASELINE configs do not exercise: ell_min > 1, BPX, hb mask, l-grid,
jacobi-only, transition with two-phase schedule, theta != 0, 1D/2D/3D.
Gate: per-cycle norms within 1e-10 of max(first, current)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

POLICIES = {
    "ellmin2_exp": dict(kind="exponential", omega_s=0.6, ell_min=2),
    "ellmin3_bpx": dict(kind="undamped", omega_s=0.5, bpx=True, ell_min=3),
    "hb_undamped": dict(kind="undamped", omega_s=0.6, hb=True),
    "lgrid1": dict(kind="lgrid", omega_s=0.7, lgrid=1),
    "jacobi_only": dict(kind="jacobi-only", omega_s=0.8),
    "transition_2ph": dict(kind="transition", omega_s=0.6, two_phase=True),
}
GRIDS = [(3, 4, 0.0), (2, 5, 0.0), (1, 6, 0.0), (3, 3, 30.0)]


@pytest.mark.parametrize("pname", sorted(POLICIES))
@pytest.mark.parametrize("dim,level,theta", GRIDS)
def test_fast_matches_exact(tmg, pname, dim, level, theta):
    p = dict(POLICIES[pname])
    ell_min = p.pop("ell_min", 1)
    pol = tmg.Policy(p.pop("kind"), p.pop("omega_s"), lgrid=p.pop("lgrid", 2), hb=p.pop("hb", False),
                     bpx=p.pop("bpx", False), two_phase=p.pop("two_phase", False))
    phi = 100 + 50j if dim < 3 else 400 + 200j
    hs = [tmg.Hierarchy(dim, level, phi=phi, theta_deg=theta, chi="seeded", ell_min=ell_min, precision=prec,
                        max_vertices=10 ** 9) for prec in ("exact", "fast")]
    first = None
    for n in range(1, 9):
        a, b = [(h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)) for h in hs]
        ra = np.array([a.max_norm, a.euclid_norm, a.h_norm])
        rb = np.array([b.max_norm, b.euclid_norm, b.h_norm])
        first = ra if first is None else first
        assert np.all(np.abs(ra - rb) <= 1e-10 * np.maximum(ra, first)), (n, ra, rb)
    ue, uf = hs[0].field(level, "u"), hs[1].field(level, "u")
    assert np.max(np.abs(ue - uf)) <= 1e-10 * max(np.max(np.abs(ue)), 1e-300)
