"""Several unknowns per vertex (RunConfig::channels and
couplingAij, runner.cpp:152-157; the coupled element kernel kernels.cpp:33-66)
on the GPU against golden runs of the REFERENCE itself (tests/golden/mc*.json,
make_goldens.py via oracle/_ref): identical outcome and sweep count, every
aggregate and per-channel CSV column within summation-order rounding
(rel 1e-12, device norms), and the final fine u of EVERY channel plus channel
0's sc bit-identical.  Also the reference's own multichannel consistency
cases (proj/tests/test_runner.cpp:120-155)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, parse_csv

pytestmark = pytest.mark.gpu

MC = sorted(f[:-5] for f in os.listdir(GOLDEN)
            if f.endswith(".json") and int(load_golden(f[:-5])["config"].get("channels", 1)) > 1)
OUTCOME = {0: "converged", 1: "budget-exhausted", 2: "diverged"}


def test_multichannel_goldens_present():
    assert len(MC) >= 4


@pytest.mark.parametrize("name", MC)
def test_multichannel_matches_reference_golden(tmg, name, tmp_path):
    g = load_golden(name)
    cfg = dict(g["config"], precision="exact", fingerprint=1)
    cfg.setdefault("max_vertices", 8388608)
    r = tmg.run(cfg, out_prefix=str(tmp_path / "run"))
    assert (r.outcome, r.sweeps) == (OUTCOME[g["outcome"]], g["sweeps"])
    text = (tmp_path / "run.csv").read_text()
    assert text.splitlines()[0] == g["csv"].splitlines()[0]  # per-channel header, runner.cpp:248-250
    got, want = np.array(parse_csv(text)), np.array(parse_csv(g["csv"]))
    assert got.shape == want.shape and got.shape[1] == 6 + 3 * int(cfg["channels"])
    assert np.array_equal(got[:, :3], want[:, :3])
    np.testing.assert_allclose(got[:, 3:], want[:, 3:], rtol=1e-12, atol=0)
    assert [f"{h:016x}" for h in r.channel_u_hashes] == g["channel_u_hashes"]
    assert f"{r.u_hash:016x}" == g["u_hash"] and f"{r.sc_hash:016x}" == g["sc_hash"]


def _hist(tmg, cfg, tmp_path, tag):
    tmg.run(cfg, out_prefix=str(tmp_path / tag))
    return np.array(parse_csv((tmp_path / f"{tag}.csv").read_text()))


def test_identical_uncoupled_channels_iterate_identically(tmg, tmp_path):
    """test_runner.cpp:121-135: per-channel h and max norms equal every sweep."""
    cfg = dict(problem="helmholtz-sin", phi="-1000", level=2, dim=2, channels=2, max_sweeps=10, target_drop=1e-30)
    h = _hist(tmg, cfg, tmp_path, "mc")
    assert h.shape == (10, 12)
    assert np.array_equal(h[:, 6:9], h[:, 9:12])


def test_zero_coupling_equals_independent_channels(tmg, tmp_path):
    """test_runner.cpp:136-154 (there to 1e-14; here bit-identical: the zero
    coupling adds no terms, as in the reference's empty coupling block)."""
    base = dict(problem="helmholtz-sin", phi="-1000", level=2, dim=2, max_sweeps=12, target_drop=1e-30)
    solo = _hist(tmg, base, tmp_path, "solo")
    both = _hist(tmg, dict(base, channels=2, coupling="0"), tmp_path, "both")
    assert solo.shape[0] == both.shape[0]
    assert np.array_equal(both[:, 8], solo[:, 5]) and np.array_equal(both[:, 11], solo[:, 5])


def test_coupling_changes_the_iteration(tmg, tmp_path):
    base = dict(problem="helmholtz-sin", phi="100,50", level=3, dim=2, channels=2, max_sweeps=6, target_drop=1e-30)
    a = _hist(tmg, base, tmp_path, "a")
    b = _hist(tmg, dict(base, coupling="30,10"), tmp_path, "b")
    assert not np.array_equal(a[:, 3:], b[:, 3:])


def test_hierarchy_api_channels(tmg):
    """The cycle-level API on the mc2_coupled_2d golden's configuration:
    per-channel norms of every sweep equal the reference's per-channel CSV
    columns, and the fields of both channels ("u", "u#1") match its hashes."""
    g = load_golden("mc2_coupled_2d")
    want = np.array(parse_csv(g["csv"]))
    H = tmg.Hierarchy(2, 4, phi=100 + 50j, chi="seeded", rhs_seed=12345, channels=2, coupling=30 + 10j)
    pol = tmg.Policy(kind="undamped", omega_s=0.6)
    for n in range(1, g["sweeps"] + 1):
        st = H.td_add(pol, n)
        cn = np.array(H.channel_norms())
        assert cn.shape == (2, 3)
        np.testing.assert_allclose(cn.ravel(), want[n - 1, 6:12], rtol=1e-12, atol=0)
        assert st.max_norm == cn[:, 0].max()
    assert f"{H.field_hash(4, 'u'):016x}" == g["channel_u_hashes"][0]
    assert f"{H.field_hash(4, 'u#1'):016x}" == g["channel_u_hashes"][1]
    assert not np.array_equal(H.field(4, "u"), H.field(4, "u#1"))
    with pytest.raises(tmg.TreemgError):
        H.field(4, "u#2")
    H.close()


@pytest.mark.parametrize("extra", [dict(precision="fast"), dict(sphere_levels=1), dict(cycle="bu-fas"),
                                   dict(norms="host")])
def test_unsupported_multichannel_variants_fail_loudly(tmg, extra):
    cfg = dict(problem="helmholtz-sin", phi="100,50", level=3, dim=2, channels=2, max_sweeps=2, **extra)
    with pytest.raises(tmg.TreemgError):
        tmg.run(cfg)
