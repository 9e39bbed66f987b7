"""Device-side building blocks against the host reference arithmetic."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_divdc3_matches_libgcc(tmg, oracle_mod):
    from test_divdc3 import cases
    v = [c for c in cases() if not (c[2] == 0.0 and c[3] == 0.0)]
    x = np.array([complex(a, b) for a, b, _, _ in v])
    y = np.array([complex(c, d) for _, _, c, d in v])
    ref = oracle_mod.cdiv(x, y)
    got = tmg.device_divide(x, y)
    same = (got.real == ref.real) | (np.isnan(got.real) & np.isnan(ref.real))
    same &= (got.imag == ref.imag) | (np.isnan(got.imag) & np.isnan(ref.imag))
    assert same.all(), np.nonzero(~same)[0][:10]


def test_seeded_rhs_matches_restatement(tmg, oracle_mod):
    """Seeded nodal f and its consistent-mass load, 3D."""
    cfg = dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", rhs="seeded", rhs_seed=99)
    o = oracle_mod.OracleSession(cfg)
    o.sweep(1)
    h = tmg.Hierarchy(3, 3, phi=400 + 200j, chi="seeded", rhs_seed=99)
    assert np.array_equal(o.field(3, "chi"), h.field(3, "chi"))


def test_fast_and_exact_agree_on_a_3d_run(tmg):
    h_e = tmg.Hierarchy(3, 4, phi=400 + 200j, chi="seeded", precision="exact")
    h_f = tmg.Hierarchy(3, 4, phi=400 + 200j, chi="seeded", precision="fast")
    pol = tmg.Policy("exponential", 0.6)
    for n in range(1, 16):
        a, b = h_e.td_add(pol, n), h_f.td_add(pol, n)
        assert abs(a.h_norm - b.h_norm) <= 1e-10 * a.h_norm
        assert abs(a.max_norm - b.max_norm) <= 1e-10 * a.max_norm
    ue, uf = h_e.field(4, "u"), h_f.field(4, "u")
    assert np.abs(ue - uf).max() <= 1e-10 * np.abs(ue).max()
