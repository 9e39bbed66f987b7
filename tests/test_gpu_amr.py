"""Static adaptive tree (BASELINE cfg4) against the live
reference: the unmodified reference library (oracle/_ref) refines the same
sphere through Spacetree::refine_cell and runs td_add / td_bpx with its
hanging-vertex events; the GPU must reproduce every field of every level,
hanging vertices included, bit for bit after every sweep."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

S = dict(rhs="seeded", rhs_seed=12345)
CASES = {
    "p2_b2_k2": (dict(problem="helmholtz-sin", dim=2, level=2, sphere_levels=2, phi="100,50", **S), 6),
    "p2_b1_k3_jumps": (dict(problem="helmholtz-sin", dim=2, level=1, sphere_levels=3, phi="100,50", **S), 5),
    "p2_b3_k2_analytic": (dict(problem="helmholtz-sin", dim=2, level=3, sphere_levels=2, phi="2025"), 5),
    "p2_bpx": (dict(problem="helmholtz-sin", dim=2, level=2, sphere_levels=2, phi="100,50", cycle="td-bpx",
                    omega="undamped", omega_s=0.5, **S), 6),
    "p2_hb": (dict(problem="helmholtz-sin", dim=2, level=2, sphere_levels=2, phi="100,50", hb=1, **S), 5),
    "p2_random_init": (dict(problem="poisson-sin", dim=2, level=2, sphere_levels=2, initial="random", seed=7), 5),
    "p2_ellmin2_lgrid": (dict(problem="helmholtz-sin", dim=2, level=3, sphere_levels=1, phi="100,50",
                              omega="lgrid", lgrid=1, ell_min=2, **S), 5),
    "p2_transition": (dict(problem="helmholtz-sin", dim=2, level=2, sphere_levels=2, phi="100,50",
                           omega="transition", two_phase=1, **S), 5),
    "p3_b2_k2_cfg4op": (dict(problem="helmholtz-sin", dim=3, level=2, sphere_levels=2, phi="1600,800",
                             omega="exponential", omega_s=0.6, rhs_mask="sphere", hb=1, **S), 4),
    "p3_b1_k2_bpx": (dict(problem="helmholtz-sin", dim=3, level=1, sphere_levels=2, phi="400,200", cycle="td-bpx",
                          omega="undamped", omega_s=0.5, **S), 4),
    "p3_ball": (dict(problem="helmholtz-ball", dim=3, level=2, sphere_levels=1), 3),
}
FIELDS = ("u", "sc", "chi", "rhat", "uhat")


def hierarchy_for(T, cfg):
    phi = cfg.get("phi")
    if phi is None:
        phi = {"poisson-sin": 0.0, "helmholtz-sin": 2025.0, "helmholtz-ball": -1000.0}[cfg["problem"]]
    else:
        parts = [float(x) for x in str(phi).split(",")]
        phi = complex(parts[0], parts[1] if len(parts) > 1 else 0.0)
    chi = "seeded" if cfg.get("rhs") == "seeded" else ("ball" if cfg["problem"] == "helmholtz-ball" else "sin")
    h = T.Hierarchy(cfg["dim"], cfg["level"], phi=phi, chi=chi, rhs_seed=int(cfg.get("rhs_seed", 12345)),
                    rhs_sphere=cfg.get("rhs_mask") == "sphere", ell_min=int(cfg.get("ell_min", 1)),
                    precision=cfg.get("precision", "exact"), max_vertices=10 ** 9, sphere_levels=cfg["sphere_levels"])
    if cfg.get("initial") == "random":
        h.set_random_initial_guess(int(cfg.get("seed", 0)))
    pol = T.Policy(kind=cfg.get("omega", "exponential"), omega_s=float(cfg.get("omega_s", 0.8)),
                   lgrid=int(cfg.get("lgrid", 2)), hb=bool(int(cfg.get("hb", 0))), bpx=cfg.get("cycle") == "td-bpx",
                   two_phase=bool(int(cfg.get("two_phase", 0))))
    return h, pol


def ref_session(cfg):
    import refdriver as R
    s = R.RefSession(dict(cfg, max_vertices=10 ** 9))
    assert s.status == 0, s.message
    return s


@pytest.mark.parametrize("name", sorted(CASES))
def test_amr_bit_identical(tmg, name):
    cfg, sweeps = CASES[name]
    ref = ref_session(cfg)
    h, pol = hierarchy_for(tmg, cfg)
    L = cfg["level"] + cfg["sphere_levels"]
    assert h.leaf_vertices == ref.interior_count()
    for lvl in range(L + 1):
        fr, sr, cr = ref.flags(lvl)
        fm, sm, cm = h.flags(lvl)
        assert np.array_equal(fr, fm) and np.array_equal(sr, sm) and np.array_equal(cr, cm), lvl
    for n in range(1, sweeps + 1):
        a = ref.sweep(n)
        st = h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
        b = np.array([st.max_norm, st.euclid_norm, st.h_norm])
        assert np.allclose(a[:3], b, rtol=1e-12, atol=0), (n, a, b)
        assert st.updated_fine_vertices == a[3]
        for lvl in range(1, L + 1):
            for f in FIELDS + (("sf", "si") if lvl < L else ()):
                zr, mr = ref.field_all(lvl, f)
                zm = h.field(lvl, f + "@all")
                if f in ("sf", "si"):  # dead payload of hanging vertices is not kept
                    zr = np.where(mr == 1, zr, 0)
                    zm = np.where(mr == 1, zm, 0)
                bad = np.nonzero(zr != zm)[0]
                assert len(bad) == 0, (n, lvl, f, len(bad), bad[:4], zr[bad[:4]], zm[bad[:4]], mr[bad[:4]])


def test_amr_rejects_complex64_and_fmg(tmg):
    """precision = fast runs on static adaptive trees (test_gpu_amr_fast.py);
    complex64 storage and FMG unfolding do not."""
    with pytest.raises(Exception):
        tmg.Hierarchy(3, 2, phi=400 + 200j, chi="seeded", precision="fast-complex64", sphere_levels=1)
    with pytest.raises(Exception):
        tmg.run(dict(problem="helmholtz-sin", dim=3, level=2, sphere_levels=1, precision="fast-complex64",
                     max_sweeps=1))
    with pytest.raises(Exception):
        tmg.run(dict(problem="helmholtz-sin", dim=3, level=3, fmg_from=2, sphere_levels=1, max_sweeps=1))


@pytest.mark.parametrize("cfg", [
    dict(problem="helmholtz-sin", dim=3, level=4, sphere_levels=2, phi="1600,800", rhs="seeded", rhs_mask="sphere",
         omega_s=0.6),
    dict(problem="helmholtz-sin", dim=3, level=4, sphere_levels=2, phi="1600,800", rhs="seeded", cycle="td-bpx",
         omega="undamped", omega_s=0.5, initial="random", seed=3),
    dict(problem="helmholtz-sin", dim=2, level=6, sphere_levels=2, phi="10000,5000", rhs="seeded", omega_s=0.6),
], ids=["cfg4-tree", "cfg4-tree-bpx-random", "2d-base6"])
def test_direct_chi_gather_bitwise_equal_stored_lists(tmg, cfg):
    """Levels with >= 65536 listed vertices gather the chi of interior
    kRegularChi vertices from the per-permutation order table (amr.cu,
    kChiDirect) instead of a stored term list (TMG_CHI_DIRECT=0): the same terms
    in the same order, so chi, r-hat, u, u-hat and sc of every level are the
    same bits (BASELINE cfg4's tree: base 4 + 2 sphere levels; a 2D tree)."""
    import os

    def run(direct):
        os.environ["TMG_CHI_DIRECT"] = "1" if direct else "0"
        try:
            h, pol = hierarchy_for(tmg, cfg)
            norms = []
            for n in range(1, 4):
                st = h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
                norms.append((st.max_norm, st.h_norm))
            return norms, [h.field(l, f) for l in range(h.levels + 1) for f in ("u", "uhat", "sc", "chi", "rhat")]
        finally:
            os.environ.pop("TMG_CHI_DIRECT", None)

    na, fa = run(True)
    nb, fb = run(False)
    assert na == nb
    for x, y in zip(fa, fb):
        assert np.array_equal(x, y)
