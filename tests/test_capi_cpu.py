"""The B200 library's C-ABI without a GPU: it loads, exports every symbol the
include/*.h headers declare, and maps configuration errors to the reference's
status codes (proj/tests/test_capi.cpp:30-53) before any device call."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def declared_functions():
    names = []
    for h in ("treemg.h", "treemg_b200.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"\b(treemg_\w+|tmg_\w+)\s*\(", text)
    return sorted(set(names))


def test_library_exports_every_declared_symbol(tmg):
    exported = set(tmg.exported_symbols())
    declared = declared_functions()
    assert len(declared) >= 14 + 16
    missing = [n for n in declared if n not in exported]
    assert not missing, missing
    for n in tmg.TREEMG_SYMBOLS + tmg.EXTENSION_SYMBOLS:
        assert n in exported


def test_version_and_error_codes(tmg):
    L = tmg.lib()
    assert L.treemg_version() == 100
    c = L.treemg_config_new()
    assert L.treemg_config_set(c, b"no_such_key", b"1") == 1
    assert len(L.treemg_last_error()) > 0
    assert L.treemg_config_load_file(c, b"missing_file.cfg") == 1
    res = ctypes.c_void_p()
    assert L.treemg_run(c, ctypes.byref(res)) == 1  # no grid selected
    assert res.value is None
    assert L.treemg_config_set(None, b"a", b"b") == 1
    assert L.treemg_run(c, None) == 1
    L.treemg_config_free(c)


@pytest.mark.parametrize("kv,status", [
    ({"dim": "4", "level": "6"}, 2),                      # test_capi.cpp:46-53: capacity first
    ({"dim": "3", "level": "5"}, 2),                      # 243^3 exceeds the default 8 Mi cap
    ({"level": "2", "max_vertices": "50"}, 2),
    ({"level": "2", "theta_deg": "60"}, 1),               # problems.cpp:326-327
    ({"level": "2", "max_sweeps": "0"}, 1),
    ({"level": "2", "h_max": "0.1", "h_min": "0.01"}, 1),  # level and adaptive bounds conflict
    ({"level": "2", "problem": "nope"}, 1),
    ({"level": "10"}, 1),                                 # kMaxLevel
    ({"level": "2", "cycle": "bu-fas", "sphere_levels": "1"}, 1),  # runner.cpp:232: adaptive needs td-*
    ({"level": "2", "channels": "2", "precision": "fast"}, 1),
    ({"level": "2", "channels": "2", "sphere_levels": "1"}, 1),
    ({"dim": "4", "level": "2"}, 1),
])
def test_run_config_errors_without_gpu(tmg, kv, status):
    L = tmg.lib()
    c = L.treemg_config_new()
    for k, v in kv.items():
        assert L.treemg_config_set(c, k.encode(), v.encode()) == 0
    res = ctypes.c_void_p()
    assert L.treemg_run(c, ctypes.byref(res)) == status, L.treemg_last_error()
    assert res.value is None
    L.treemg_config_free(c)


def test_config_file_parsing(tmg, tmp_path):
    L = tmg.lib()
    p = tmp_path / "c.cfg"
    p.write_text("# comment\nproblem = helmholtz-sin\nlevel = 2\ntheta_deg = 35\nphi = 2025\nmax_sweeps = 5\n"
                 "rhs = seeded\nprecision = fast\n")
    c = L.treemg_config_new()
    assert L.treemg_config_load_file(c, str(p).encode()) == 0
    p.write_text("level 2\n")
    assert L.treemg_config_load_file(c, str(p).encode()) == 1  # malformed line
    assert L.treemg_config_set(c, b"omega_s", b"0.8,-0.25") == 0
    assert L.treemg_config_set(c, b"hb", b"maybe") == 1
    assert L.treemg_config_set(c, b"precision", b"half") == 1
    L.treemg_config_free(c)
