"""The CPU restatement (oracle/treemg_oracle.cpp) against the golden fixtures
generated from the reference itself (tests/golden/make_goldens.py): CSV rows
byte-identical, outcome, sweep count and the fine-level u bit pattern."""
import pytest

from conftest import load_golden

CASES = ["cfg1", "cfg2_l5", "conv2d", "hb_then_add", "poisson_smoke", "runner_poisson_l3",
         "runner_helmholtz_diverges", "runner_budget_one", "capi_poisson_l2", "rotated_3d_bpx", "cfg3_l4"]


@pytest.mark.parametrize("name", CASES)
def test_restatement_matches_reference_golden(oracle_mod, name):
    g = load_golden(name)
    o = oracle_mod.OracleSession(g["config"])
    outcome, sweeps = o.run()
    assert (outcome, sweeps) == (g["outcome"], g["sweeps"])
    assert o.csv() == g["csv"]
    L = int(g["config"]["level"])
    assert f"{o.field_hash(L, 'u'):016x}" == g["u_hash"]
    assert f"{o.field_hash(L, 'sc'):016x}" == g["sc_hash"]
