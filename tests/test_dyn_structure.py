"""Dynamic adaptivity, host side, against the REFERENCE
itself (oracle/_ref via the live harness):
  * the structural replay of a traversal with applyMarks (dyn.hpp, C-ABI
    tmg_dyn_*) leaves the reference's tree behind -- every cell, every vertex
    classification and succ, refined / erased counts and the touch-last
    update count -- under the reference's own marks (amr.cpp mark()) and under
    random refine / erase marks (erase coverage: natural runs rarely erase);
  * the restatement of the host libm's hypot that the device mark pass uses
    (glibc's Borges algorithm, non-FMA kernel) equals libm bit for bit;
  * the harness's adaptive run loop writes the reference runner's CSV.
No GPU: the structural replay is host code."""
import ctypes
import ctypes.util
import os

import numpy as np
import pytest

from conftest import load_golden


def level_for_h(h):
    level, m = 0, 1.0
    while m > h * (1 + 1e-12) and level < 12:
        m /= 3.0
        level += 1
    return level


def replay(tmg, ref_mod, cfg, sweeps, seed=None):
    rng = np.random.default_rng(seed) if seed is not None else None
    s = ref_mod.RefSession(cfg)
    assert s.status == 0, s.message
    dim = int(cfg["dim"])
    start = max(1, level_for_h(cfg["h_max"]))
    D = tmg.DynStructure(dim, start, min(level_for_h(cfg["h_min"]), 9), 1, cfg["h_min"])
    totals = dict(refined=0, erased=0, special=0)
    for n in range(1, sweeps + 1):
        if rng is None:  # the marks the reference's mark() left pending
            for level in range(s.depth + 1):
                D.set_cell_marks(level, s.cell_marks(level))
        c = D.sweep()
        want = s.sweep(n)
        ms = s.mark_stats()
        assert (c["refined"], c["erased"]) == (ms["refined"], ms["erased"]), n
        assert c["updated"] == int(want[3]), n
        for k in totals:
            totals[k] += c[k]
        assert D.depth == s.depth
        for level in range(s.depth + 1):
            fl, sc, ce = s.flags(level)
            gfl, gsc, gce = D.flags(level)
            assert np.array_equal(fl, gfl), (n, level)
            assert np.array_equal(sc, gsc), (n, level)
            assert np.array_equal(ce & 3, gce & 3), (n, level)
        assert D.interior_count() == s.interior_count()
        if rng is not None:  # random marks on both sides
            for level in range(s.depth + 1):
                ce = s.cell_marks(level)
                ex, refd = (ce & 1) > 0, (ce & 2) > 0
                m = np.zeros_like(ce)
                m[ex & ~refd & (rng.random(len(ce)) < 0.15)] |= 4
                m[refd & (rng.random(len(ce)) < 0.35)] |= 8
                s.set_cell_marks(level, m)
                D.set_cell_marks(level, m)
    return totals


CASES = {
    "h2d": dict(problem="helmholtz-sin", dim=2, phi="100,50", h_max=0.04, h_min=0.004, omega="undamped",
                omega_s=0.6, max_sweeps=99),
    "p3d": dict(problem="poisson-sin", dim=3, h_max=0.12, h_min=0.013, omega="undamped", omega_s=0.6, max_sweeps=99),
    "p1d": dict(problem="poisson-sin", dim=1, h_max=0.12, h_min=0.0005, omega="exponential", omega_s=0.8,
                max_sweeps=99),
}


@pytest.mark.parametrize("case,sweeps", [("h2d", 9), ("p3d", 6)])
def test_replay_matches_reference_marks(tmg, ref_mod, case, sweeps):
    t = replay(tmg, ref_mod, CASES[case], sweeps)
    assert t["refined"] > 0 and t["special"] > 0


@pytest.mark.parametrize("case,seed", [("h2d", 0), ("h2d", 1), ("p3d", 0), ("p1d", 2)])
def test_replay_matches_reference_random_marks(tmg, ref_mod, case, seed):
    sweeps = 5 if case == "p3d" else 8
    try:
        t = replay(tmg, ref_mod, CASES[case], sweeps, seed)
    except tmg.TreemgError as e:  # a vertex erased and re-created within one traversal: refused loudly
        assert "re-created" in str(e)
        return
    assert t["refined"] > 0 and (t["erased"] > 0 or case == "p1d")


def test_hypot_restatement_matches_libm():
    """std::abs(complex<double>) -> libm hypot (glibc 2.35+: Borges' algorithm,
    non-FMA correction); the device mark pass restates it (amr.cu host_hypot)."""
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]

    def kernel(ax, ay):
        h = np.sqrt(ax * ax + ay * ay)
        if h <= 2.0 * ay:
            delta = h - ay
            t1 = ax * (2.0 * delta - ax)
            t2 = (delta - 2.0 * (ax - ay)) * delta
        else:
            delta = h - ax
            t1 = 2.0 * delta * (ax - 2.0 * ay)
            t2 = (4.0 * delta - ay) * ay + delta * delta
        return h - (t1 + t2) / (2.0 * h)

    def hyp(x, y):
        x, y = abs(x), abs(y)
        ax, ay = (y, x) if x < y else (x, y)
        if ax > 2.0 ** 511:
            return ax + ay if ay <= ax * 2.0 ** -54 else kernel(ax * 2.0 ** -600, ay * 2.0 ** -600) / 2.0 ** -600
        if ay < 2.0 ** -511:
            return ax + ay if ax >= ay / 2.0 ** -54 else kernel(ax / 2.0 ** -600, ay / 2.0 ** -600) * 2.0 ** -600
        return ax + ay if ay <= ax * 2.0 ** -54 else kernel(ax, ay)

    rng = np.random.default_rng(7)
    x = rng.standard_normal(20000) * np.exp(rng.uniform(-30, 30, 20000))
    y = x * (1 + rng.uniform(-1e-6, 1e-6, 20000))
    y[::3] = rng.standard_normal(len(y[::3])) * np.exp(rng.uniform(-30, 30, len(y[::3])))
    for a, b in zip(x.tolist(), y.tolist()):
        assert hyp(float(np.float64(a)), float(np.float64(b))) == libm.hypot(a, b), (a, b)


def test_adaptive_loop_csv_equals_reference_runner(ref_mod, tmp_path):
    """The harness's adaptive run loop (goldens) writes the reference runner's CSV."""
    g = load_golden("dyn_p2d_transition")
    st, _ = ref_mod.capi_run(g["config"], str(tmp_path / "ref"))
    assert st == 0
    assert (tmp_path / "ref.csv").read_text() == g["csv"]
    log = (tmp_path / "ref.log").read_text().splitlines()
    assert [l for l in log if l.startswith("sweep ")] == [l for l in g["log"].splitlines() if l.startswith("sweep ")]
