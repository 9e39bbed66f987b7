import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def ref_mod():
    import refdriver as R
    if not R.available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return R


@pytest.fixture(scope="session")
def tmg():
    import paper_1508_03954_b200 as T
    T.lib()
    return T


def load_golden(name):
    import json
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def parse_csv(text):
    rows = [line.split(",") for line in text.strip().splitlines()[1:]]
    return [[float(x) for x in r] for r in rows]
