"""Parity at the benchmark's own size and the strict north_star gate.

* The headline workload (bench.py's default: cfg5's final level, 729^3,
  k = 80, seeded rhs, exponential omega 0.6) in fast precision against exact
  precision for the first cycles.  Exact precision is bit-identical to the
  reference on every smaller configuration (tests/test_gpu_exact_parity.py,
  test_gpu_goldens.py) and at 729^3 itself to the reference golden
  tests/golden/cfg5_l6_head.json when present.  Gate (BASELINE.json
  north_star): per-cycle relative error of every norm <= 1e-10 and
  max |u_fast - u_exact| <= 1e-10 max |u_exact|.  Sizes past 2^31 bytes per
  array, the 16,744-block grid and the level-6 chunk geometry are exercised
  here and nowhere else.
* The fast path's final fine u against the exact path's at the full BASELINE
  sizes of cfg1 / cfg2 / cfg3 after the golden's full cycle count.

Reference semantics: td_add / td_bpx (proj/src/cycles.cpp:336-354), the
sweep loop of proj/src/runner.cpp:268-366.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, parse_csv

pytestmark = pytest.mark.gpu

STRICT = 1e-10
HEAD = dict(levels=6, phi=6400 + 3200j, cycles=3)


def _norms(st):
    return np.array([st.max_norm, st.euclid_norm, st.h_norm])


def _run(tmg, dim, level, phi, pol, precision, cycles, keep_u=True):
    h = tmg.Hierarchy(dim, level, phi=phi, chi="seeded", rhs_seed=12345, precision=precision, max_vertices=10 ** 10)
    try:
        hist = []
        for n in range(1, cycles + 1):
            st = h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
            hist.append(_norms(st))
        u = h.field(level, "u") if keep_u else None
        return np.array(hist), u
    finally:
        h.close()


def _max_rel_u(u_fast, u_exact):
    scale = np.abs(u_exact).max()
    return float(np.abs(u_fast - u_exact).max() / scale)


def test_headline_729_fast_matches_exact(tmg):
    pol = tmg.Policy("exponential", 0.6)
    he, ue = _run(tmg, 3, HEAD["levels"], HEAD["phi"], pol, "exact", HEAD["cycles"])
    hf, uf = _run(tmg, 3, HEAD["levels"], HEAD["phi"], pol, "fast", HEAD["cycles"])
    strict = np.abs(hf - he) / he
    du = _max_rel_u(uf, ue)
    print(f"729^3 fast vs exact: strict per-cycle relative error {strict.max():.2e}, max|du|/max|u| {du:.2e}")
    assert np.all(strict <= STRICT), strict
    assert du <= STRICT, du
    path = os.path.join(GOLDEN, "cfg5_l6_head.json")
    if os.path.exists(path):  # the reference itself at 729^3 (make_goldens.py cfg5_l6_head, run on the GPU host)
        g = load_golden("cfg5_l6_head")
        ref = np.array(parse_csv(g["csv"]))[:, 3:6]
        k = len(ref)
        np.testing.assert_allclose(he[:k], ref, rtol=1e-12, atol=0)
        assert np.all(np.abs(hf[:k] - ref) / ref <= STRICT)
        print(f"729^3 against the reference's first {k} cycles: exact max rel {(np.abs(he[:k] - ref) / ref).max():.2e}")


def test_headline_729_exact_bit_identical_to_reference(tmg):
    """Exact precision at 729^3 for the golden's cycle count: the fine u and sc
    bit patterns hash to the reference's (FNV-1a, tests/golden/make_goldens.py)."""
    path = os.path.join(GOLDEN, "cfg5_l6_head.json")
    if not os.path.exists(path):
        pytest.skip("cfg5_l6_head golden not generated")
    g = load_golden("cfg5_l6_head")
    pol = tmg.Policy("exponential", 0.6)
    h = tmg.Hierarchy(3, 6, phi=HEAD["phi"], chi="seeded", rhs_seed=12345, precision="exact", max_vertices=10 ** 10)
    try:
        for n in range(1, g["sweeps"] + 1):
            h.td_add(pol, n)
        assert f"{h.field_hash(6, 'u'):016x}" == g["u_hash"]
        assert f"{h.field_hash(6, 'sc'):016x}" == g["sc_hash"]
    finally:
        h.close()


def _golden_case(tmg, name):
    g = load_golden(name)
    c = g["config"]
    phi = [float(x) for x in c["phi"].split(",")]
    bpx = c["cycle"] == "td-bpx"
    pol = tmg.Policy(c["omega"], float(c["omega_s"]), bpx=bpx)
    return g, int(c["dim"]), int(c["level"]), complex(phi[0], phi[1]), pol


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_fast_final_u_matches_exact_full_size(tmg, name):
    """After the golden's full cycle count (cfg1 20, cfg2 200, cfg3 50) the fast
    fine u equals the exact one (bit-identical to the reference's: u_hash) to
    1e-10 of max |u|, and every cycle's norms to 1e-10 relative."""
    g, dim, level, phi, pol = _golden_case(tmg, name)
    cycles = g["sweeps"]
    he, ue = _run(tmg, dim, level, phi, pol, "exact", cycles)
    hf, uf = _run(tmg, dim, level, phi, pol, "fast", cycles)
    strict = np.abs(hf - he) / he
    du = _max_rel_u(uf, ue)
    print(f"{name}: fast vs exact over {cycles} cycles: strict {strict.max():.2e}, final max|du|/max|u| {du:.2e}")
    assert np.all(strict <= STRICT)
    assert du <= STRICT
