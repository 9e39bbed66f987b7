"""ctypes wrapper of the CPU restatement (oracle/treemg_oracle.cpp).

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke()).  Built by
``make -C oracle restatement``; needs no reference sources, so it also builds
on the GPU box.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libtreemg_oracle.so")
_lib = None

# OmegaKind numbering of proj/include/treemg/cycles.hpp:12
OMEGA_KINDS = {"jacobi-only": 0, "undamped": 1, "lgrid": 2, "exponential": 3, "transition": 4}


def build() -> None:
    out = subprocess.run(["make", "-C", HERE, "restatement"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle restatement build failed:\n" + out.stdout + out.stderr)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        vp, cp, ip, dp = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_double
        pd = ctypes.POINTER(dp)
        L.tmo_new.restype = vp
        L.tmo_new.argtypes = [cp]
        L.tmo_free.argtypes = [vp]
        for n in ("tmo_status", "tmo_run", "tmo_outcome", "tmo_sweeps", "tmo_history_rows"):
            getattr(L, n).restype = ip
            getattr(L, n).argtypes = [vp]
        L.tmo_message.restype = cp
        L.tmo_message.argtypes = [vp]
        L.tmo_sweep.restype = ip
        L.tmo_sweep.argtypes = [vp, ip, pd]
        L.tmo_history_row.argtypes = [vp, ip, pd]
        L.tmo_lattice_size.restype = ctypes.c_longlong
        L.tmo_lattice_size.argtypes = [vp, ip]
        L.tmo_field.restype = ip
        L.tmo_field.argtypes = [vp, ip, cp, pd]
        L.tmo_set_fine_interior_u.argtypes = [vp, pd]
        L.tmo_omega.argtypes = [ip, dp, dp, ip, ip, ip, ip, pd]
        L.tmo_cdiv.argtypes = [pd, pd, pd, ctypes.c_longlong]
        L.tmo_csv.restype = cp
        L.tmo_csv.argtypes = [vp]
        L.tmo_field_hash.restype = ctypes.c_ulonglong
        L.tmo_field_hash.argtypes = [vp, ip, cp]
        _lib = L
    return _lib


def _pd(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleSession:
    """Level-wise restatement of one reference run (regular grid, 1 channel)."""

    def __init__(self, cfg: dict):
        self.L = lib()
        text = "".join(f"{k} = {v}\n" for k, v in cfg.items())
        self.h = self.L.tmo_new(text.encode())
        if self.L.tmo_status(self.h) != 0:
            msg = self.L.tmo_message(self.h).decode()
            self.L.tmo_free(self.h)
            self.h = None
            raise ValueError(msg)

    def close(self):
        if self.h:
            self.L.tmo_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sweep(self, n: int) -> np.ndarray:
        out = np.zeros(5)
        st = self.L.tmo_sweep(self.h, n, _pd(out))
        if st != 0:
            raise ArithmeticError(self.L.tmo_message(self.h).decode())
        return out

    def run(self):
        self.L.tmo_run(self.h)
        return self.L.tmo_outcome(self.h), self.L.tmo_sweeps(self.h)

    def history(self) -> np.ndarray:
        rows = self.L.tmo_history_rows(self.h)
        out = np.zeros((rows, 6))
        buf = np.zeros(6)
        for i in range(rows):
            self.L.tmo_history_row(self.h, i, _pd(buf))
            out[i] = buf
        return out

    def csv(self) -> str:
        return self.L.tmo_csv(self.h).decode()

    def field_hash(self, level: int, name: str) -> int:
        return int(self.L.tmo_field_hash(self.h, level, name.encode()))

    def field(self, level: int, name: str) -> np.ndarray:
        n = self.L.tmo_lattice_size(self.h, level)
        out = np.zeros(2 * n)
        if self.L.tmo_field(self.h, level, name.encode(), _pd(out)) != 0:
            raise KeyError(name)
        return out[0::2] + 1j * out[1::2]

    def set_fine_interior_u(self, u: np.ndarray):
        buf = np.empty(2 * len(u))
        buf[0::2] = u.real
        buf[1::2] = u.imag
        self.L.tmo_set_fine_interior_u(self.h, _pd(buf))


def omega(kind, ws: complex, lgrid: int, two_phase: bool, succ: int, n: int) -> complex:
    out = np.zeros(2)
    k = OMEGA_KINDS[kind] if isinstance(kind, str) else int(kind)
    lib().tmo_omega(k, ws.real, ws.imag, lgrid, int(two_phase), succ, n, _pd(out))
    return complex(out[0], out[1])


def cdiv(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """x / y elementwise with libgcc's __divdc3 (the reference's division)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    y = np.ascontiguousarray(y, dtype=np.complex128)
    out = np.zeros_like(x)
    lib().tmo_cdiv(_pd(x.view(np.float64)), _pd(y.view(np.float64)), _pd(out.view(np.float64)), len(x))
    return out
