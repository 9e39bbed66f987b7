"""ctypes wrapper of the oracle harness around the UNMODIFIED reference library.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product.

``oracle/_ref/libtreemg_ref.so`` is built by ``oracle/Makefile`` from the
reference sources under /root/reference/proj/src (the build only runs where
those sources exist; the built .so travels to the GPU box with the repo
snapshot).  See oracle/refdriver.cpp for what the harness adds.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REF_LIB = os.path.join(REF_DIR, "libtreemg_ref.so")
REF_SOURCES = "/root/reference/proj"

_lib = None


def build(quiet: bool = True) -> bool:
    """Build oracle/_ref from the reference sources when they are present."""
    import subprocess
    if not os.path.isdir(REF_SOURCES):
        return os.path.exists(REF_LIB)
    cmd = ["make", "-C", HERE, "-j8"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle/_ref build failed:\n" + out.stdout + out.stderr)
    return True


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError("oracle/_ref/libtreemg_ref.so is not built (run `make -C oracle`)")
        L = ctypes.CDLL(REF_LIB)
        vp, cp, ip, dp = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_double
        L.refd_new.restype = vp
        L.refd_new.argtypes = [cp]
        L.refd_free.argtypes = [vp]
        for name in ("refd_status", "refd_depth", "refd_run", "refd_outcome", "refd_sweeps",
                     "refd_history_rows", "refd_timed_sweeps"):
            getattr(L, name).restype = ip
            getattr(L, name).argtypes = [vp]
        for name in ("refd_message", "refd_csv", "refd_log"):
            getattr(L, name).restype = cp
            getattr(L, name).argtypes = [vp]
        for name in ("refd_first_norm", "refd_final_norm"):
            getattr(L, name).restype = dp
            getattr(L, name).argtypes = [vp]
        L.refd_history_row.argtypes = [vp, ip, ctypes.POINTER(dp)]
        L.refd_sweep_seconds.restype = dp
        L.refd_sweep_seconds.argtypes = [vp, ip]
        L.refd_sweep.restype = ip
        L.refd_sweep.argtypes = [vp, ip, ctypes.POINTER(dp)]
        L.refd_lattice_size.restype = ctypes.c_longlong
        L.refd_lattice_size.argtypes = [vp, ip]
        L.refd_field.argtypes = [vp, ip, cp, ip, ctypes.POINTER(dp), ctypes.POINTER(ctypes.c_ubyte)]
        L.refd_set_fine_interior_u.argtypes = [vp, ctypes.POINTER(dp)]
        L.refd_field_all.argtypes = [vp, ip, cp, ip, ctypes.POINTER(dp), ctypes.POINTER(ctypes.c_ubyte)]
        L.refd_flags.argtypes = [vp, ip, vp, vp, vp]
        L.refd_interior_count.restype = ctypes.c_longlong
        L.refd_interior_count.argtypes = [vp]
        L.refd_field_hash.restype = ctypes.c_ulonglong
        L.refd_field_hash.argtypes = [vp, ip, cp, ip]
        L.refd_vertex_succ.restype = ip
        L.refd_vertex_succ.argtypes = [vp, ip, ctypes.POINTER(ip)]
        L.refd_omega.argtypes = [ip, dp, dp, ip, ip, ip, ip, ip, ip, ip, ip, ctypes.POINTER(dp)]
        L.refd_mark_stats.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
        L.refd_cell_marks.argtypes = [vp, ip, vp]
        L.refd_set_cell_marks.argtypes = [vp, ip, vp]
        # the reference's own C-ABI (proj/src/capi.cpp), unmodified
        L.treemg_config_new.restype = vp
        L.treemg_config_free.argtypes = [vp]
        L.treemg_config_set.restype = ip
        L.treemg_config_set.argtypes = [vp, cp, cp]
        L.treemg_config_load_file.restype = ip
        L.treemg_config_load_file.argtypes = [vp, cp]
        L.treemg_run.restype = ip
        L.treemg_run.argtypes = [vp, ctypes.POINTER(vp)]
        L.treemg_result_free.argtypes = [vp]
        L.treemg_result_outcome.restype = ip
        L.treemg_result_outcome.argtypes = [vp]
        L.treemg_result_sweeps.restype = ip
        L.treemg_result_sweeps.argtypes = [vp]
        L.treemg_result_work_units.restype = dp
        L.treemg_result_work_units.argtypes = [vp]
        L.treemg_result_vertex_count.restype = ctypes.c_longlong
        L.treemg_result_vertex_count.argtypes = [vp]
        L.treemg_result_final_norm.restype = dp
        L.treemg_result_final_norm.argtypes = [vp, cp, ip]
        L.treemg_result_first_norm.restype = dp
        L.treemg_result_first_norm.argtypes = [vp]
        L.treemg_last_error.restype = cp
        _lib = L
    return _lib


def cfg_text(cfg: dict) -> str:
    return "".join(f"{k} = {v}\n" for k, v in cfg.items())


class RefSession:
    """One reference spacetree + problem + policy, built from config keys."""

    def __init__(self, cfg: dict):
        self.L = lib()
        self.h = self.L.refd_new(cfg_text(cfg).encode())
        self.cfg = dict(cfg)

    def close(self):
        if self.h:
            self.L.refd_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def status(self) -> int:
        return self.L.refd_status(self.h)

    @property
    def message(self) -> str:
        return self.L.refd_message(self.h).decode()

    @property
    def depth(self) -> int:
        return self.L.refd_depth(self.h)

    def run(self) -> int:
        return self.L.refd_run(self.h)

    def outcome(self) -> int:
        return self.L.refd_outcome(self.h)

    def sweeps(self) -> int:
        return self.L.refd_sweeps(self.h)

    def csv(self) -> str:
        return self.L.refd_csv(self.h).decode()

    def log(self) -> str:
        return self.L.refd_log(self.h).decode()

    def history(self) -> np.ndarray:
        rows = self.L.refd_history_rows(self.h)
        out = np.zeros((rows, 6))
        buf = (ctypes.c_double * 6)()
        for i in range(rows):
            self.L.refd_history_row(self.h, i, buf)
            out[i] = list(buf)
        return out

    def sweep_seconds(self) -> np.ndarray:
        n = self.L.refd_timed_sweeps(self.h)
        return np.array([self.L.refd_sweep_seconds(self.h, i) for i in range(n)])

    def sweep(self, n: int) -> np.ndarray:
        buf = (ctypes.c_double * 5)()
        st = self.L.refd_sweep(self.h, n, buf)
        if st != 0:
            raise RuntimeError(f"reference sweep failed ({st}): {self.message}")
        return np.array(list(buf))

    def field(self, level: int, name: str, channel: int = 0, with_mask: bool = False):
        n = self.L.refd_lattice_size(self.h, level)
        out = np.zeros(2 * n)
        mask = np.zeros(n, dtype=np.uint8)
        self.L.refd_field(self.h, level, name.encode(), channel,
                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                          mask.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)))
        z = out[0::2] + 1j * out[1::2]
        return (z, mask.astype(bool)) if with_mask else z

    def field_all(self, level: int, name: str, channel: int = 0):
        """Every vertex of the level incl. hanging ones; mask 1 regular, 2 hanging."""
        n = self.L.refd_lattice_size(self.h, level)
        out = np.zeros(2 * n)
        mask = np.zeros(n, dtype=np.uint8)
        self.L.refd_field_all(self.h, level, name.encode(), channel,
                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                              mask.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)))
        return out[0::2] + 1j * out[1::2], mask

    def flags(self, level: int):
        n = self.L.refd_lattice_size(self.h, level)
        fl = np.zeros(n, np.uint8)
        sc = np.zeros(n, np.int8)
        ce = np.zeros(n, np.uint8)
        self.L.refd_flags(self.h, level, fl.ctypes.data_as(ctypes.c_void_p), sc.ctypes.data_as(ctypes.c_void_p),
                          ce.ctypes.data_as(ctypes.c_void_p))
        return fl, sc, ce

    MARK_KEYS = ("refined", "erased", "refine_vertices", "erase_vertices", "refine_cells", "erase_cells",
                 "veto_conv", "veto_hmin", "veto_hmax")

    def mark_stats(self) -> dict:
        """h_max/h_min sessions: refined/erased cells of the last sweep() and the
        MarkStats of the mark() that followed it."""
        buf = (ctypes.c_longlong * 9)()
        self.L.refd_mark_stats(self.h, buf)
        return dict(zip(self.MARK_KEYS, list(buf)))

    def cell_marks(self, level: int) -> np.ndarray:
        """Per cell (lower corner): 1 exists | 2 refined | 4 refineMark | 8 eraseMark."""
        n = self.L.refd_lattice_size(self.h, level)
        ce = np.zeros(n, np.uint8)
        self.L.refd_cell_marks(self.h, level, ce.ctypes.data_as(ctypes.c_void_p))
        return ce

    def set_cell_marks(self, level: int, cells: np.ndarray):
        c = np.ascontiguousarray(cells, np.uint8)
        self.L.refd_set_cell_marks(self.h, level, c.ctypes.data_as(ctypes.c_void_p))

    def interior_count(self) -> int:
        return int(self.L.refd_interior_count(self.h))

    def field_hash(self, level: int, name: str, channel: int = 0) -> int:
        return int(self.L.refd_field_hash(self.h, level, name.encode(), channel))

    def set_fine_interior_u(self, u: np.ndarray):
        buf = np.empty(2 * len(u))
        buf[0::2] = u.real
        buf[1::2] = u.imag
        self.L.refd_set_fine_interior_u(self.h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))


def omega(kind: int, ws: complex, lgrid: int, hb: bool, bpx: bool, two_phase: bool, succ: int,
          cpoint: bool, n: int, masked: bool = True) -> complex:
    out = (ctypes.c_double * 2)()
    lib().refd_omega(kind, ws.real, ws.imag, lgrid, int(hb), int(bpx), int(two_phase), succ,
                     int(cpoint), n, int(masked), out)
    return complex(out[0], out[1])


def capi_run(cfg: dict, out_prefix: Optional[str] = None):
    """Run through the reference's own C-ABI (proj/src/capi.cpp) unchanged."""
    L = lib()
    c = L.treemg_config_new()
    try:
        for k, v in cfg.items():
            st = L.treemg_config_set(c, str(k).encode(), str(v).encode())
            if st != 0:
                return st, None
        if out_prefix:
            L.treemg_config_set(c, b"out", out_prefix.encode())
        res = ctypes.c_void_p()
        st = L.treemg_run(c, ctypes.byref(res))
        if st != 0:
            return st, L.treemg_last_error().decode()
        try:
            info = dict(outcome=L.treemg_result_outcome(res), sweeps=L.treemg_result_sweeps(res),
                        work_units=L.treemg_result_work_units(res),
                        vertex_count=L.treemg_result_vertex_count(res),
                        first_norm=L.treemg_result_first_norm(res),
                        final_h=L.treemg_result_final_norm(res, b"h", -1),
                        final_max=L.treemg_result_final_norm(res, b"max", -1),
                        final_euclid=L.treemg_result_final_norm(res, b"euclid", -1))
        finally:
            L.treemg_result_free(res)
        return 0, info
    finally:
        L.treemg_config_free(c)
