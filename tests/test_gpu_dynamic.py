"""Dynamic adaptivity on the GPU against the REFERENCE:
  * goldens of h_max / h_min runs (tests/golden/dyn_*.json, make_goldens.py via
    oracle/_ref): identical outcome, sweep count, work units and vertex counts,
    norms within summation-order rounding (rel 1e-12), the per-sweep
    refine / erase / veto statistics of the log line by line, and the final
    fine u and sc bit-identical;
  * the live reference harness sweep by sweep: every field of every level
    (hanging vertices included), the structure and the mark statistics, under
    the reference's own marks and under random refine / erase marks;
  * the device restatement of libm hypot (mark features) against libm."""
import ctypes
import ctypes.util
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, parse_csv

pytestmark = pytest.mark.gpu

DYN = sorted(f[:-5] for f in os.listdir(GOLDEN) if f.startswith("dyn_") and f.endswith(".json"))
OUTCOME = {0: "converged", 1: "budget-exhausted", 2: "diverged"}


def test_dynamic_goldens_present():
    assert len(DYN) >= 5


@pytest.mark.parametrize("name", DYN)
def test_dynamic_run_matches_reference_golden(tmg, name, tmp_path):
    g = load_golden(name)
    cfg = dict(g["config"], precision="exact", fingerprint=1)
    r = tmg.run(cfg, out_prefix=str(tmp_path / "run"))
    assert (r.outcome, r.sweeps) == (OUTCOME[g["outcome"]], g["sweeps"])
    got, want = np.array(parse_csv((tmp_path / "run.csv").read_text())), np.array(parse_csv(g["csv"]))
    assert got.shape == want.shape
    assert np.array_equal(got[:, :3], want[:, :3])  # sweep, workUnits, vertexCount
    np.testing.assert_allclose(got[:, 3:], want[:, 3:], rtol=1e-12, atol=0)
    marks = [l for l in (tmp_path / "run.log").read_text().splitlines() if l.startswith("sweep ")]
    assert marks == [l for l in g["log"].splitlines() if l.startswith("sweep ")]
    assert f"{r.u_hash:016x}" == g["u_hash"] and f"{r.sc_hash:016x}" == g["sc_hash"]


CASES = {
    "h2d": (dict(problem="helmholtz-sin", dim=2, phi="100,50", h_max=0.04, h_min=0.004, omega="undamped",
                 omega_s=0.6), dict(dim=2, phi=100 + 50j, chi="sin"), dict(kind="undamped", omega_s=0.6)),
    "p2d_bpx": (dict(problem="poisson-sin", dim=2, h_max=0.04, h_min=0.002, cycle="td-bpx", omega="undamped",
                     omega_s=0.5), dict(dim=2, phi=0, chi="sin"), dict(kind="undamped", omega_s=0.5, bpx=True)),
    "p3d": (dict(problem="poisson-sin", dim=3, h_max=0.12, h_min=0.013, omega="undamped", omega_s=0.6),
            dict(dim=3, phi=0, chi="sin"), dict(kind="undamped", omega_s=0.6)),
    "p1d": (dict(problem="poisson-sin", dim=1, h_max=0.12, h_min=0.0005, omega="exponential", omega_s=0.8),
            dict(dim=1, phi=0, chi="sin"), dict(kind="exponential", omega_s=0.8)),
    "b2d_seeded": (dict(problem="helmholtz-ball", dim=2, h_max=0.12, h_min=0.0014, omega="exponential",
                        omega_s=0.8, rhs="seeded", rhs_seed=99, theta_deg=20),
                   dict(dim=2, phi=-1000, chi="seeded", rhs_seed=99, theta_deg=20),
                   dict(kind="exponential", omega_s=0.8)),
    "b2d_seeded_random": (dict(problem="helmholtz-ball", dim=2, h_max=0.12, h_min=0.0014, omega="exponential",
                               omega_s=0.8, rhs="seeded", rhs_seed=99, theta_deg=20, initial="random", seed=5),
                          dict(dim=2, phi=-1000, chi="seeded", rhs_seed=99, theta_deg=20),
                          dict(kind="exponential", omega_s=0.8)),
}
# sinext: the reference keeps siNext until the next touch-first zeroes it; the
# device zeroes it when it commits si = siNext (the same state for every cycle)
FIELDS = ["u", "sc", "uhat", "rhat", "sf", "si", "chi"]


def random_marks(ref, rng, dim):
    out = {}
    for level in range(ref.depth + 1):
        ce = ref.cell_marks(level)
        ex, refd = (ce & 1) > 0, (ce & 2) > 0
        m = np.zeros_like(ce)
        m[ex & ~refd & (rng.random(len(ce)) < 0.15)] |= 4
        # erase only where no neighbouring cell refines in the same traversal: a vertex erased and
        # re-created within one traversal is refused loudly by the device path
        n1 = 3 ** level + 1
        r4 = (m & 4).reshape((n1,) * dim)
        near = np.zeros_like(r4)
        for off in np.ndindex(*((3,) * dim)):
            near |= np.roll(r4, tuple(o - 1 for o in off), axis=tuple(range(dim)))
        m[refd & (near.reshape(-1) == 0) & (rng.random(len(ce)) < 0.35)] |= 8
        out[level] = m
    return out


def run_lockstep(tmg, ref_mod, case, sweeps, random_seed=None):
    rcfg, hkw, pkw = CASES[case]
    ref = ref_mod.RefSession(dict(rcfg, max_sweeps=sweeps))
    assert ref.status == 0, ref.message
    h = tmg.Hierarchy(levels=1, precision="exact", h_max=rcfg["h_max"], h_min=rcfg["h_min"], **hkw)
    if rcfg.get("initial") == "random":
        h.set_random_initial_guess(rcfg["seed"])
    pol = tmg.Policy(**pkw)
    rng = np.random.default_rng(random_seed) if random_seed is not None else None
    edits = 0
    for n in range(1, sweeps + 1):
        want = ref.sweep(n)
        got = h.td_bpx(pol, n) if pkw.get("bpx") else h.td_add(pol, n)
        rm, gm = ref.mark_stats(), h.mark()
        assert gm == rm, n
        assert got.updated_fine_vertices == int(want[3])
        np.testing.assert_allclose([got.max_norm, got.euclid_norm, got.h_norm], want[:3], rtol=1e-12, atol=0)
        assert h.depth() == ref.depth
        for level in range(ref.depth + 1):
            fl, sc, ce = ref.flags(level)
            gfl, gsc, gce = h.flags(level)
            assert np.array_equal(fl, gfl) and np.array_equal(sc, gsc) and np.array_equal(ce & 3, gce & 3)
            for fld in FIELDS:
                a, _ = ref.field_all(level, fld)
                assert np.array_equal(a, h.field(level, fld + "@all")), (n, level, fld)
        edits += gm["refined"] + gm["erased"]
        if rng is not None:
            for level, m in random_marks(ref, rng, rcfg["dim"]).items():
                ref.set_cell_marks(level, m)
                h.set_cell_marks(level, m)
    h.close()
    return edits


@pytest.mark.parametrize("case,sweeps", [("h2d", 9), ("p2d_bpx", 9), ("p3d", 7), ("p1d", 10), ("b2d_seeded", 10),
                                         ("b2d_seeded_random", 8)])
def test_dynamic_sweeps_bit_identical_to_live_reference(tmg, ref_mod, case, sweeps):
    edits = run_lockstep(tmg, ref_mod, case, sweeps)
    assert edits > 0 or case in ("p1d", "b2d_seeded_random")  # those two stay on their start grid


@pytest.mark.parametrize("case,sweeps,seed", [("h2d", 8, 1), ("p2d_bpx", 7, 2), ("p3d", 5, 3)])
def test_dynamic_random_refine_erase_bit_identical(tmg, ref_mod, case, sweeps, seed):
    assert run_lockstep(tmg, ref_mod, case, sweeps, seed) > 0


def test_device_hypot_matches_libm(tmg):
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(3)
    n = 200000
    x = rng.standard_normal(n) * np.exp(rng.uniform(-40, 40, n))
    y = x * (1 + rng.uniform(-1e-6, 1e-6, n))
    y[::3] = rng.standard_normal(len(y[::3])) * np.exp(rng.uniform(-40, 40, len(y[::3])))
    y[::7] *= 2.0 ** -600
    got = tmg.device_hypot(x, y)
    want = np.array([libm.hypot(a, b) for a, b in zip(x.tolist(), y.tolist())])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("extra", [dict(precision="fast"), dict(cycle="bu-fas"), dict(channels=2),
                                   dict(problem="gaussian"), dict(norms="host")])
def test_unsupported_dynamic_variants_fail_loudly(tmg, extra):
    cfg = dict(dict(problem="helmholtz-sin", phi="100,50", dim=2, h_max=0.04, h_min=0.004, max_sweeps=2), **extra)
    with pytest.raises(tmg.TreemgError):
        tmg.run(cfg)
