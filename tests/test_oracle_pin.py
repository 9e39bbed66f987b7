"""Pins the CPU restatement bit-for-bit against the live reference
(oracle/_ref, the unmodified reference sources): every field of every level
after every sweep, for every cycle variant, omega kind and mask."""
import numpy as np
import pytest

FIELDS = ["u", "sc", "sf", "si", "chi", "r", "rhat", "uhat", "diag", "sinext"]
S = dict(rhs="seeded", rhs_seed=12345)
CASES = {
    "poisson_p2_l2": (dict(problem="poisson-sin", dim=2, level=2), 6),
    "helm_p2_l3_theta35": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", theta_deg=35), 6),
    "seeded_p2_l3": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", **S), 6),
    "seeded_p3_l2": (dict(problem="helmholtz-sin", dim=3, level=2, phi="400,200", **S), 4),
    "seeded_ball_p3_l3": (dict(problem="helmholtz-ball", dim=3, level=3, **S), 2),
    "p1_l4": (dict(problem="helmholtz-sin", dim=1, level=4, phi="100,50", theta_deg=35), 6),
    "bpx_p2_l3": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", cycle="td-bpx", omega="undamped",
                       omega_s=0.5, **S), 6),
    "bpx_p3_l2": (dict(problem="helmholtz-sin", dim=3, level=2, phi="400,200", cycle="td-bpx", omega="undamped",
                       omega_s=0.5, **S), 4),
    "hb_p2_l3": (dict(problem="helmholtz-sin", dim=2, level=3, phi="-1000", hb=1, **S), 6),
    "transition_two_phase": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="transition",
                                  two_phase=1, **S), 6),
    "lgrid_ellmin2": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="lgrid", lgrid=1,
                           ell_min=2, **S), 6),
    "jacobi_only": (dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="jacobi-only", **S), 4),
    "random_init": (dict(problem="poisson-sin", dim=2, level=3, initial="random", seed=7), 5),
    "sphere_mask_hb_sweeps": (dict(problem="helmholtz-sin", dim=3, level=2, phi="1600,800", rhs_mask="sphere",
                                   hb_sweeps=2, **S), 4),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_restatement_bit_identical_to_reference(ref_mod, oracle_mod, name):
    cfg, sweeps = CASES[name]
    r = ref_mod.RefSession(cfg)
    assert r.status == 0, r.message
    o = oracle_mod.OracleSession(cfg)
    for n in range(1, sweeps + 1):
        a, b = r.sweep(n), o.sweep(n)
        assert np.array_equal(a[:4], b[:4]), (n, a, b)  # norms summed in the same order
        for level in range(r.depth + 1):
            for f in FIELDS:
                assert np.array_equal(r.field(level, f), o.field(level, f)), (n, level, f)


def test_set_fine_interior_u_matches(ref_mod, oracle_mod):
    import dense
    cfg = dict(problem="helmholtz-sin", dim=2, level=2, phi="2025", theta_deg=35)
    u0 = dense.random_vector(64, 22)
    r, o = ref_mod.RefSession(cfg), oracle_mod.OracleSession(cfg)
    r.set_fine_interior_u(u0)
    o.set_fine_interior_u(u0)
    for n in range(1, 6):
        r.sweep(n)
        o.sweep(n)
        assert np.array_equal(r.field(2, "u"), o.field(2, "u"))


def test_omega_tables_match_reference(ref_mod, oracle_mod):
    for kind in range(5):
        for ws in (0.8 + 0j, 0.6 + 0j, 0.7 - 0.2j):
            for succ in range(5):
                for n in (1, 2, 3, 7):
                    for tp in (False, True):
                        a = ref_mod.omega(kind, ws, 2, False, False, tp, succ, False, n, masked=False)
                        b = oracle_mod.omega(kind, ws, 2, tp, succ, n)
                        assert a == b or (np.isnan(a) and np.isnan(b))
