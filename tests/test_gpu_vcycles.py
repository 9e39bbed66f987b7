"""Verification cycles through the cycle API (Hierarchy.bu_fas / textbook_add,
C-ABI tmg_bu_fas / tmg_textbook_add) against the live reference harness:
per-cycle norms and the finest iterate within the fast-path tolerance (the
reference sums these cycles in hash-map order, cycles.cpp:374-786)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "bufas_p2": dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50", cycle="bu-fas", omega="exponential",
                     omega_s=0.6, rhs="seeded", rhs_seed=12345),
    "bufas_p3_hb": dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", cycle="bu-fas", omega="undamped",
                        omega_s=0.6, hb=1, rhs="seeded", rhs_seed=12345),
    "bufas_p1_lgrid": dict(problem="poisson-sin", dim=1, level=5, cycle="bu-fas", omega="lgrid", lgrid=2,
                           omega_s=0.8),
    "textbook_p2": dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50", cycle="textbook", omega_s=0.6,
                        omega_cg=0.7, rhs="seeded", rhs_seed=12345),
    "textbook_p3": dict(problem="poisson-sin", dim=3, level=3, cycle="textbook", omega_s=0.8),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_cycle_api_matches_reference(tmg, ref_mod, name):
    cfg = CASES[name]
    ref = ref_mod.RefSession(cfg)
    assert ref.status == 0, ref.message
    phi = cfg.get("phi")
    if phi is None:
        phi = 0.0
    else:
        a = [float(x) for x in phi.split(",")]
        phi = complex(a[0], a[1] if len(a) > 1 else 0.0)
    chi = "seeded" if cfg.get("rhs") == "seeded" else "sin"
    h = tmg.Hierarchy(cfg["dim"], cfg["level"], phi=phi, chi=chi, rhs_seed=12345, precision="exact")
    pol = tmg.Policy(cfg.get("omega", "exponential"), float(cfg.get("omega_s", 0.8)), lgrid=int(cfg.get("lgrid", 2)),
                     hb=bool(int(cfg.get("hb", 0))))
    L = cfg["level"]
    first = None
    for n in range(1, 7):
        a = ref.sweep(n)
        if cfg["cycle"] == "bu-fas":
            st = h.bu_fas(pol, n)
        else:
            ws = float(cfg.get("omega_s", 0.8))
            st = h.textbook_add(ws, float(cfg.get("omega_cg", ws)))
        b = np.array([st.max_norm, st.euclid_norm, st.h_norm])
        first = a[:3] if first is None else first
        assert np.all(np.abs(b - a[:3]) <= 1e-10 * np.maximum(a[:3], first)), (n, a[:3], b)
        assert st.updated_fine_vertices == a[3]
    ur, ug = ref.field(L, "u"), h.field(L, "u")
    assert np.max(np.abs(ur - ug)) <= 1e-10 * np.max(np.abs(ur))
