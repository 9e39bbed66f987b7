"""precision = fast-complex64: the 3D fused fine pass with the finest level
stored and computed in complex64 (BASELINE.json north_star: "complex-double
(and complex-float) loads"), coarse levels, restriction partials and norm sums
in complex128 / double.

The reference is complex128 only (proj/include/treemg/types.hpp:11), so the
oracle for this mode is the complex128 path (itself pinned to the reference:
test_gpu_exact_parity.py, test_gpu_goldens.py, test_gpu_headline.py).  The
achievable gate is set by float rounding of the stored iterate and of the
fine residual (unit roundoff 6e-8, amplified by the cancellation in b - H u):
per-cycle norms within C64_NORM_TOL relative and the final fine u within
C64_U_TOL of max |u| on the BASELINE 3D configurations, same outcome and
sweep count through treemg_run.
"""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

C64_NORM_TOL = 3e-4  # cfg3 after 50 cycles: 9.7e-5 (B200, round 2)
C64_U_TOL = 3e-4


def _hist(tmg, level, phi, pol, precision, cycles):
    h = tmg.Hierarchy(3, level, phi=phi, chi="seeded", rhs_seed=12345, precision=precision, max_vertices=10 ** 10)
    try:
        out = []
        for n in range(1, cycles + 1):
            st = h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
            out.append([st.max_norm, st.euclid_norm, st.h_norm])
        return np.array(out), h.field(level, "u")
    finally:
        h.close()


CASES = [
    (3, 400 + 200j, "add", 12), (4, 400 + 200j, "add", 12), (4, 400 + 200j, "bpx", 10),
    (5, 400 + 200j, "add", 50),       # cfg3 at full size and cycle count
    (6, 6400 + 3200j, "add", 3),      # the headline workload (cfg5's final level)
]


@pytest.mark.parametrize("level,phi,kind,cycles", CASES)
def test_complex64_tracks_complex128(tmg, level, phi, kind, cycles):
    pol = tmg.Policy("exponential", 0.6) if kind == "add" else tmg.Policy("undamped", 0.5, bpx=True)
    hd, ud = _hist(tmg, level, phi, pol, "fast", cycles)
    hf, uf = _hist(tmg, level, phi, pol, "fast-complex64", cycles)
    rel = np.abs(hf - hd) / hd
    du = np.abs(uf - ud).max() / np.abs(ud).max()
    print(f"level {level} {kind}: complex64 vs complex128 per-cycle norms max rel {rel.max():.2e}, "
          f"final u {du:.2e}")
    assert np.all(rel <= C64_NORM_TOL), rel.max()
    assert du <= C64_U_TOL, du


def test_complex64_run_matches_golden_outcome(tmg):
    """treemg_run, precision = fast-complex64, on the cfg3 operator at 81^3
    (reference golden cfg3_l4): same outcome and sweep count, norms within
    the complex64 gate."""
    from conftest import parse_csv
    g = load_golden("cfg3_l4")
    cfg = dict(g["config"], precision="fast-complex64")
    r = tmg.run(cfg)
    assert (r.outcome, r.sweeps) == ({0: "converged", 1: "budget-exhausted", 2: "diverged"}[g["outcome"]],
                                     g["sweeps"])
    ref = np.array(parse_csv(g["csv"]))[:, 3:]
    rel = np.abs(r.history[:, 3:] - ref) / ref
    print(f"cfg3_l4 complex64 vs reference: max rel {rel.max():.2e}")
    assert np.all(rel <= C64_NORM_TOL)


@pytest.mark.parametrize("cfg", [
    dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50"),
    dict(problem="helmholtz-sin", dim=3, level=4, fmg_from=2, phi="400,200"),
    dict(problem="helmholtz-sin", dim=3, level=3, cycle="bu-fas", phi="400,200"),
])
def test_complex64_unsupported_modes_fail_loudly(tmg, cfg):
    with pytest.raises(tmg.TreemgError) as e:
        tmg.run(dict(cfg, precision="fast-complex64", max_sweeps=3))
    assert e.value.status == 1


def test_complex64_field_roundtrip(tmg):
    """set_field / field on the complex64 fine level: the stored u is the
    complex64 rounding of the input."""
    h = tmg.Hierarchy(3, 3, phi=400 + 200j, chi="seeded", precision="fast-complex64")
    try:
        n = h.lattice_size(3)
        rng = np.random.default_rng(3)
        u = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        h.set_field(3, "u", u)
        got = h.field(3, "u")
        assert np.array_equal(got, u.astype(np.complex64).astype(np.complex128) - 0)
    finally:
        h.close()
