"""Ports of the reference's own hot-path tests (proj/tests/test_kernels.cpp,
test_cycles.cpp, test_capi.cpp, test_runner.cpp) run against the B200
library, with the dense oracle (oracle/dense.py, restating
proj/src/oracle.cpp) as the trusted side -- in both precisions."""
import os
import subprocess

import numpy as np
import pytest

import dense
from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu

PRECISIONS = ["exact", "fast"]


def interior(field, p, level):
    m = 3 ** level
    a = field.reshape([m + 1] * p)  # axis 0 fastest -> reversed numpy order
    sl = tuple(slice(1, m) for _ in range(p))
    return a[sl].reshape(-1)


def chi_sin_fn(x):
    return dense.chi_sin(x)


@pytest.mark.parametrize("precision", ["exact"])
def test_discrete_delta_reproduces_stencil_centre(tmg, monkeypatch, precision):
    """test_kernels.cpp:57-75: r - chi at a unit delta = -8/3 (p=2, Poisson)."""
    monkeypatch.setenv("TMG_DEBUG_R", "1")
    h = tmg.Hierarchy(2, 1, phi=0.0, chi="sin", precision=precision)
    u = np.zeros(16, dtype=complex)
    u[1 + 4 * 1] = 1.0
    h.set_field(1, "u", u)
    h.td_add(tmg.Policy("jacobi-only"), 1)
    r, chi = h.field(1, "r"), h.field(1, "chi")
    assert abs((r - chi)[5] - (-8.0 / 3.0)) < 1e-13


RES_CASES = [(1, 2, 0.0, 0.0, 11), (1, 3, 35.0, 2025.0, 12), (2, 2, 0.0, -1000.0, 13), (2, 2, 35.0, 2025.0, 14),
             (3, 1, 35.0, -1000.0, 15), (3, 2, 0.0, 2025.0, 16)]


@pytest.mark.parametrize("p,level,theta_deg,phi,seed", RES_CASES)
def test_matrix_free_residual_equals_dense_oracle(tmg, monkeypatch, p, level, theta_deg, phi, seed):
    """test_kernels.cpp:104-146 (exact precision keeps r and r-hat)."""
    monkeypatch.setenv("TMG_DEBUG_R", "1")
    h = tmg.Hierarchy(p, level, phi=phi, theta_deg=theta_deg, chi="sin", precision="exact")
    u0 = dense.random_vector(dense.interior_count(p, level), seed)
    h.set_fine_interior_u(u0)
    h.td_add(tmg.Policy("exponential"), 1)
    theta = theta_deg * np.pi / 180.0
    b = dense.load_vector(p, level, theta, chi_sin_fn)
    r_or = dense.residual(p, level, theta, phi, b, u0)
    r_gpu = interior(h.field(level, "r"), p, level)
    assert np.abs(r_gpu - r_or).max() <= 1e-12 * max(1.0, np.abs(r_or).max())
    if level >= 2:
        P, I = dense.prolongation_matrix(p, level), dense.injection_matrix(p, level)
        rh_or = dense.residual(p, level, theta, phi, b, u0 - P @ (I @ u0))
        rh_gpu = interior(h.field(level, "rhat"), p, level)
        assert np.abs(rh_gpu - rh_or).max() <= 1e-12 * max(1.0, np.abs(rh_or).max())


def test_accumulated_diagonal_equals_dense(tmg):
    """test_kernels.cpp:148-159."""
    h = tmg.Hierarchy(2, 2, phi=2025.0, theta_deg=35.0, chi="sin")
    h.td_add(tmg.Policy(), 1)
    d = interior(h.field(2, "diag"), 2, 2)
    H = dense.dense_assemble(2, 2, 35.0 * np.pi / 180.0, 2025.0)
    assert np.all(np.abs(d - np.diag(H)) <= 1e-13 * np.abs(np.diag(H)))


@pytest.mark.parametrize("precision", PRECISIONS)
def test_first_traversal_leaves_u_unchanged(tmg, precision):
    """test_cycles.cpp:73-81."""
    h = tmg.Hierarchy(2, 2, phi=0.0, chi="sin", precision=precision)
    u0 = dense.random_vector(64, 5)
    h.set_fine_interior_u(u0)
    h.td_add(tmg.Policy(), 1)
    assert np.array_equal(interior(h.field(2, "u"), 2, 2), u0)


TRANSCRIPTION = [
    ("td-add", 1, 2, 0.0, 0.0, "exponential", 8, 21, 1e-13),
    ("td-add", 2, 2, 35.0, 2025.0, "exponential", 6, 22, 1e-12),
    ("td-bpx", 1, 2, 0.0, 0.0, "undamped", 10, 23, 1e-13),
    ("td-bpx", 2, 2, 35.0, 2025.0, "undamped", 6, 24, 1e-12),
    ("td-add", 2, 3, 0.0, -1000.0, "transition", 5, 25, 1e-12),
    ("td-add", 3, 2, 0.0, 400 + 200j, "exponential", 4, 26, 1e-12),
]


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("kind,p,levels,theta_deg,phi,omega,sweeps,seed,tol", TRANSCRIPTION)
def test_cycles_match_dense_transcription(tmg, precision, kind, p, levels, theta_deg, phi, omega, sweeps, seed, tol):
    """test_cycles.cpp:110-147: iterates vs the literal dense Alg. 2 / 3."""
    u0 = dense.random_vector(dense.interior_count(p, levels), seed)
    ref = dense.reference_cycles(kind, p, levels, theta_deg * np.pi / 180.0, phi, chi_sin_fn, omega, 0.8,
                                 sweeps, u0=u0)
    h = tmg.Hierarchy(p, levels, phi=phi, theta_deg=theta_deg, chi="sin", precision=precision)
    h.set_fine_interior_u(u0)
    pol = tmg.Policy(omega, 0.8, bpx=(kind == "td-bpx"))
    for n in range(1, sweeps + 1):
        h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
        got = interior(h.field(levels, "u"), p, levels)
        assert np.abs(got - ref[n - 1]).max() <= tol, n


def test_lemma2_coarse_rhs_realises_fas(tmg):
    """test_cycles.cpp:233-259: after one prelude traversal b_c = R r + H_c I u."""
    p, L = 2, 2
    u0 = dense.random_vector(64, 55)
    h = tmg.Hierarchy(p, L, phi=-1000.0, chi="sin", precision="exact")
    h.set_fine_interior_u(u0)
    h.td_add(tmg.Policy(), 1)
    bc = interior(h.field(1, "chi"), p, 1)
    Hf, Hc = dense.dense_assemble(p, L, 0.0, -1000.0), dense.dense_assemble(p, L - 1, 0.0, -1000.0)
    P, I = dense.prolongation_matrix(p, L), dense.injection_matrix(p, L)
    b = dense.load_vector(p, L, 0.0, chi_sin_fn)
    want = P.T @ (b - Hf @ u0) + Hc @ (I @ u0)
    assert np.abs(bc - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("precision", PRECISIONS)
def test_lemma1_injection_consistency(tmg, precision):
    """test_cycles.cpp:217-231: u_{l-1} = I u_l whenever residuals are evaluated (exact)."""
    h = tmg.Hierarchy(2, 3, phi=0.0, chi="sin", precision=precision)
    h.set_random_initial_guess(4242)
    for n in range(1, 11):
        h.td_add(tmg.Policy(), n)
    for lc in (1, 2):
        uc = h.field(lc, "u").reshape(3 ** lc + 1, -1)
        uf = h.field(lc + 1, "u").reshape(3 ** (lc + 1) + 1, -1)
        assert np.abs(uc - uf[::3, ::3]).max() <= 1e-12


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("p,levels,theta_deg,phi", [(2, 2, 0.0, 0.0), (1, 3, 35.0, 2025.0)])
def test_exact_solution_is_a_fixed_point(tmg, precision, p, levels, theta_deg, phi):
    """test_cycles.cpp:261-294."""
    theta = theta_deg * np.pi / 180.0
    H = dense.dense_assemble(p, levels, theta, phi)
    b = dense.load_vector(p, levels, theta, chi_sin_fn)
    ustar = np.linalg.solve(H, b)
    scale = max(1.0, np.abs(ustar).max())
    for kind in ("td-add", "td-bpx"):
        h = tmg.Hierarchy(p, levels, phi=phi, theta_deg=theta_deg, chi="sin", precision=precision)
        h.set_fine_interior_u(ustar)
        pol = tmg.Policy("undamped" if kind == "td-bpx" else "exponential", bpx=kind == "td-bpx")
        for n in (1, 2):
            h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
            assert np.abs(interior(h.field(levels, "u"), p, levels) - ustar).max() <= 1e-12 * scale


@pytest.mark.parametrize("precision", PRECISIONS)
def test_staged_corrections_vanish_at_cpoints(tmg, precision):
    """test_cycles.cpp:317-336: exact structural zeros under hb and BPX."""
    for variant in ("hb", "bpx"):
        h = tmg.Hierarchy(2, 2, phi=-1000.0, chi="sin", precision=precision)
        h.set_random_initial_guess(7)
        pol = tmg.Policy("exponential", hb=variant == "hb", bpx=variant == "bpx")
        for n in range(1, 6):
            h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
            for level in (1, 2):
                sc = h.field(level, "sc").reshape(3 ** level + 1, -1)
                assert np.all(sc[::3, ::3] == 0.0)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_singular_diagonal_is_detected(tmg, precision):
    """test_cycles.cpp:338-344: 1D, h=1/3, phi=27 -> vanishing diagonal."""
    h = tmg.Hierarchy(1, 1, phi=27.0, chi="sin", precision=precision)
    with pytest.raises(tmg.TreemgError) as e:
        h.td_add(tmg.Policy(), 1)
    assert e.value.status == 3 and "diagonal" in e.value.message
    r = tmg.run(dict(problem="helmholtz-sin", phi="27", dim=1, level=1, precision=precision))
    assert (r.outcome, r.sweeps, len(r.history)) == ("diverged", 1, 0)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_capi_small_solve(tmg, precision):
    """test_capi.cpp:8-28."""
    r = tmg.run(dict(problem="poisson-sin", dim=2, level=2, max_sweeps=60, precision=precision))
    assert r.outcome == "converged" and r.sweeps > 1 and r.vertex_count == 64
    assert r.final_norm["h"] > 0.0 and r.final_norm["max"] >= r.final_norm["h"]
    assert r.first_norm > r.final_norm["h"]
    assert abs(r.work_units - r.sweeps) < 1e-12


@pytest.mark.parametrize("precision", PRECISIONS)
def test_runner_outcomes(tmg, precision):
    """test_runner.cpp:460-505."""
    r = tmg.run(dict(level=2, dim=2, max_sweeps=1, target_drop=1e-30, precision=precision))
    assert (r.outcome, r.sweeps, r.work_units) == ("budget-exhausted", 1, 1.0)
    r = tmg.run(dict(problem="helmholtz-sin", phi=2025, level=3, dim=2, theta_deg=0, max_sweeps=300,
                     precision=precision))
    assert r.outcome == "diverged"


def test_reference_cli_runs_on_the_b200_library(tmg, tmp_path):
    """proj/tools/solve.cpp, unmodified, linked against libtreemg_b200.so
    (oracle/Makefile solve_b200): the reference's cli_smoke run."""
    exe = os.path.join(ROOT, "oracle", "_ref", "solve_b200")
    if not os.path.exists(exe):
        pytest.skip("solve_b200 not built (needs the reference sources at build time)")
    out = subprocess.run([exe, os.path.join(ROOT, "tests", "data", "poisson_smoke.cfg"), "--out",
                          str(tmp_path / "smoke"), "--norms", "host"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert (tmp_path / "smoke.csv").read_text() == load_golden("poisson_smoke")["csv"]


@pytest.mark.parametrize("cfg,sweeps", [
    (dict(problem="gaussian", dim=2, level=3), 5),
    (dict(problem="gaussian", dim=2, level=4, theta_deg=25, omega="transition"), 4),
    (dict(problem="gaussian", dim=2, level=3, cycle="td-bpx", omega="undamped", omega_s=0.3), 4),
])
def test_gaussian_scenario_bit_identical(tmg, ref_mod, cfg, sweeps):
    """Cell-varying phi and absorbing-layer theta (problems.cpp:20-24, 78-90;
    kernels.cpp:7-23): every field of every level bit-identical to the live
    reference after every sweep."""
    ref = ref_mod.RefSession(cfg)
    assert ref.status == 0, ref.message
    h = tmg.Hierarchy(2, cfg["level"], chi="gaussian", theta_deg=float(cfg.get("theta_deg", 0)), precision="exact")
    bpx = cfg.get("cycle") == "td-bpx"
    pol = tmg.Policy(cfg.get("omega", "exponential"), float(cfg.get("omega_s", 0.4)), bpx=bpx)
    L = cfg["level"]
    for n in range(1, sweeps + 1):
        a = ref.sweep(n)
        st = h.td_bpx(pol, n) if bpx else h.td_add(pol, n)
        assert np.allclose(a[:3], [st.max_norm, st.euclid_norm, st.h_norm], rtol=1e-12, atol=0), n
        for lvl in range(1, L + 1):
            for f in ("u", "sc", "chi", "rhat", "uhat") + (("sf", "si") if lvl < L else ()):
                assert np.array_equal(ref.field(lvl, f), h.field(lvl, f)), (n, lvl, f)
