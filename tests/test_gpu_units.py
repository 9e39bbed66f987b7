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


def _fields_after(tmg, env, dim, level, phi, cycles, bpx=False):
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        h = tmg.Hierarchy(dim, level, phi=phi, chi="seeded", precision="fast", max_vertices=10 ** 10)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    pol = tmg.Policy("undamped", 0.5, bpx=True) if bpx else tmg.Policy("exponential", 0.6)
    norms = []
    for n in range(1, cycles + 1):
        st = h.td_bpx(pol, n) if bpx else h.td_add(pol, n)
        norms.append((st.max_norm, st.euclid_norm, st.h_norm))
    return np.array(norms), h.field(level, "u")


@pytest.mark.parametrize("dim,level,bpx", [(3, 5, False), (3, 4, True), (2, 6, False), (2, 5, True)])
def test_coarse_chain_bitwise_equals_per_level_launches(tmg, dim, level, bpx):
    """The cooperative coarse chain (fast.cu k_chain_*) computes the per-level
    kernels' values in the same order: identical iterates, norms equal up to
    the final reduction tree."""
    a_n, a_u = _fields_after(tmg, {"TMG_CHAIN": "1"}, dim, level, 400 + 200j, 5, bpx)
    b_n, b_u = _fields_after(tmg, {"TMG_CHAIN": "0"}, dim, level, 400 + 200j, 5, bpx)
    assert np.array_equal(a_u, b_u)
    np.testing.assert_allclose(a_n, b_n, rtol=1e-13)


@pytest.mark.parametrize("level,bpx", [(5, False), (6, True)])
def test_fused2_matches_unfused_2d(tmg, level, bpx):
    """2D fused fine pass vs the three-kernel path: same cycle, different
    rounding (FMA / summation grouping) -- agreement to ~1e-12."""
    a_n, a_u = _fields_after(tmg, {"TMG_FUSED2": "1"}, 2, level, 100 + 50j, 6, bpx)
    b_n, b_u = _fields_after(tmg, {"TMG_FUSED2": "0"}, 2, level, 100 + 50j, 6, bpx)
    np.testing.assert_allclose(a_n, b_n, rtol=1e-11)
    assert np.max(np.abs(a_u - b_u)) <= 1e-11 * np.max(np.abs(b_u))


@pytest.mark.parametrize("dim,level", [(3, 4), (2, 5)])
def test_vform_field_api_round_trip(tmg, dim, level):
    """The fused fast passes keep v = u + sc on the finest level; the field API
    must still read and write u and sc (u = v - sc, rounding only)."""
    h = tmg.Hierarchy(dim, level, phi=400 + 200j, chi="seeded", precision="fast", max_vertices=10 ** 10)
    pol = tmg.Policy("exponential", 0.6)
    for n in range(1, 4):
        h.td_add(pol, n)
    u0, sc0 = h.field(level, "u"), h.field(level, "sc")
    assert np.abs(sc0).max() > 0
    rng = np.random.default_rng(3)
    x = rng.standard_normal(u0.shape) + 1j * rng.standard_normal(u0.shape)
    h.set_field(level, "u", x)
    np.testing.assert_allclose(h.field(level, "u"), x, rtol=0, atol=1e-14 * np.abs(x).max())
    np.testing.assert_array_equal(h.field(level, "sc"), sc0)
    # the cycle continues from (u, sc): same as a hierarchy holding the original state
    h.set_field(level, "u", u0)
    a = h.td_add(pol, 4)
    b_h = tmg.Hierarchy(dim, level, phi=400 + 200j, chi="seeded", precision="fast", max_vertices=10 ** 10)
    for n in range(1, 4):
        b_h.td_add(pol, n)
    b = b_h.td_add(pol, 4)
    assert abs(a.h_norm - b.h_norm) <= 1e-12 * b.h_norm


def test_device_memory_exhaustion_is_a_capacity_error(tmg):
    """A problem past the device's 180 GB (3D depth 7: 10.5 G vertices per fine
    array) with the vertex cap lifted reports TREEMG_E_CAPACITY through the
    C-ABI (capi.cpp:28-43's mapping) and leaves the library usable."""
    with pytest.raises(tmg.TreemgError) as e:
        tmg.run(dict(problem="helmholtz-sin", dim=3, level=7, precision="fast", max_vertices=10 ** 12, max_sweeps=1))
    assert e.value.status == 2, e.value
    r = tmg.run(dict(problem="poisson-sin", dim=2, level=2, max_sweeps=60))
    assert r.outcome == "converged" and r.sweeps == 28
