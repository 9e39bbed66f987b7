"""GPU exact precision against the CPU restatement (itself pinned
bit-for-bit to the reference): every field of every level after every sweep
must be bit-identical; norms agree to summation order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

S = dict(rhs="seeded", rhs_seed=12345)
CASES = {
    "poisson_p2_l2": (dict(problem="poisson-sin", dim=2, level=2), 6),
    "helm_p2_l3_theta35": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", theta_deg=35), 6),
    "seeded_p2_l4": (dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50", **S), 6),
    "seeded_p3_l2": (dict(problem="helmholtz-sin", dim=3, level=2, phi="400,200", **S), 4),
    "seeded_p3_l3": (dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", **S), 3),
    "p1_l4_theta35": (dict(problem="helmholtz-sin", dim=1, level=4, phi="100,50", theta_deg=35), 6),
    "bpx_p2_l3": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", cycle="td-bpx", omega="undamped",
                       omega_s=0.5, **S), 6),
    "bpx_p3_l3": (dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", cycle="td-bpx", omega="undamped",
                       omega_s=0.5, **S), 3),
    "hb_p2_l3": (dict(problem="helmholtz-sin", dim=2, level=3, phi="-1000", hb=1, **S), 6),
    "transition_two_phase": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="transition",
                                  two_phase=1, **S), 6),
    "lgrid_ellmin2": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="lgrid", lgrid=1,
                           ell_min=2, **S), 6),
    "jacobi_only": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="jacobi-only", **S), 4),
    "random_init": (dict(problem="poisson-sin", dim=2, level=3, initial="random", seed=7), 5),
    "ball_p3_l3": (dict(problem="helmholtz-ball", dim=3, level=3), 3),
    "sphere_mask_p3": (dict(problem="helmholtz-sin", dim=3, level=3, phi="1600,800", rhs_mask="sphere", **S), 3),
}


def hierarchy_for(T, cfg, precision="exact"):
    phi = cfg.get("phi")
    if phi is None:
        phi = {"poisson-sin": 0.0, "helmholtz-sin": 2025.0, "helmholtz-ball": -1000.0}[cfg["problem"]]
    else:
        parts = [float(x) for x in str(phi).split(",")]
        phi = complex(parts[0], parts[1] if len(parts) > 1 else 0.0)
    chi = "seeded" if cfg.get("rhs") == "seeded" else ("ball" if cfg["problem"] == "helmholtz-ball" else "sin")
    h = T.Hierarchy(cfg["dim"], cfg["level"], phi=phi, theta_deg=float(cfg.get("theta_deg", 0)), chi=chi,
                    rhs_seed=int(cfg.get("rhs_seed", 12345)), rhs_sphere=cfg.get("rhs_mask") == "sphere",
                    ell_min=int(cfg.get("ell_min", 1)), precision=precision, max_vertices=10 ** 10)
    if cfg.get("initial") == "random":
        h.set_random_initial_guess(int(cfg.get("seed", 0)))
    ws = cfg.get("omega_s", 0.8)
    pol = T.Policy(kind=cfg.get("omega", "exponential"), omega_s=float(ws), lgrid=int(cfg.get("lgrid", 2)),
                   hb=bool(int(cfg.get("hb", 0))), bpx=cfg.get("cycle") == "td-bpx",
                   two_phase=bool(int(cfg.get("two_phase", 0))))
    return h, pol


@pytest.mark.parametrize("name", sorted(CASES))
def test_exact_bit_identical(tmg, oracle_mod, name):
    cfg, sweeps = CASES[name]
    o = oracle_mod.OracleSession(cfg)
    h, pol = hierarchy_for(tmg, cfg)
    L = cfg["level"]
    for n in range(1, sweeps + 1):
        a = o.sweep(n)
        st = h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
        b = np.array([st.max_norm, st.euclid_norm, st.h_norm])
        assert np.allclose(a[:3], b, rtol=1e-13, atol=0), (n, a, b)
        assert st.updated_fine_vertices == a[3]
        for level in range(1, L + 1):
            for f in ("u", "sc", "chi", "rhat", "uhat", "diag") + (("sf", "si") if level < L else ()):
                assert np.array_equal(o.field(level, f), h.field(level, f)), (n, level, f)


def test_many_vertices_per_thread_norms(tmg, oracle_mod):
    """3D level 4 (82^3 lattice) so grid-stride threads own several vertices."""
    cfg = dict(problem="helmholtz-sin", dim=3, level=4, phi="400,200", **S)
    o = oracle_mod.OracleSession(cfg)
    h, pol = hierarchy_for(tmg, cfg)
    for n in range(1, 4):
        a = o.sweep(n)
        st = h.td_add(pol, n)
        assert np.allclose(a[:3], [st.max_norm, st.euclid_norm, st.h_norm], rtol=1e-13, atol=0)
    assert np.array_equal(o.field(4, "u"), h.field(4, "u"))
    assert o.field_hash(4, "u") == h.field_hash(4, "u")
