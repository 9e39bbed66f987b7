"""Dense-matrix oracle for small regular grids (numpy), restating the
reference's trusted side proj/src/oracle.cpp.

TEST INFRASTRUCTURE ONLY.  Unknowns are the interior vertices of one level,
lexicographic with axis 0 fastest (oracle.cpp:87-120).  Used by the ported
reference tests (tests/test_gpu_reference_ports.py) exactly where the
reference's own tests use oracle::dense_assemble / load_vector / residual /
prolongation_matrix / injection_matrix / reference_cycles.
"""
from __future__ import annotations

import itertools
from typing import Callable, List

import numpy as np

KW0 = [1.0, 2.0 / 3.0, 1.0 / 3.0, 0.0]  # proj/src/transfer.cpp:7
KW1 = [0.0, 1.0 / 3.0, 2.0 / 3.0, 1.0]  # proj/src/transfer.cpp:8


def reference_matrices(p: int):
    """proj/src/elemops.cpp:32-55 (tensor products, axis 0 = bit 0)."""
    lap1 = np.array([[1.0, -1.0], [-1.0, 1.0]])
    mas1 = np.array([[1.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 1.0 / 3.0]])
    n = 1 << p
    K = np.zeros((n, n))
    M = np.zeros((n, n))
    for a in range(n):
        for b in range(n):
            bits = [((a >> d) & 1, (b >> d) & 1) for d in range(p)]
            M[a, b] = np.prod([mas1[x, y] for x, y in bits])
            K[a, b] = sum(lap1[bits[d]] * np.prod([mas1[bits[i]] for i in range(p) if i != d]) for d in range(p))
    return K, M


def cell_operator(p: int, h: float, theta: float, phi: complex) -> np.ndarray:
    """proj/src/elemops.cpp:70-85: hElem^(p-2) K - phi hElem^p M."""
    K, M = reference_matrices(p)
    he = h * complex(np.cos(theta), np.sin(theta))
    return he ** (p - 2) * K - phi * he ** p * M


def interior_count(p: int, level: int) -> int:
    return (3 ** level - 1) ** p


def interior_flat(p: int, level: int, idx) -> int:  # oracle.cpp:93-101
    m = 3 ** level - 1
    return sum((idx[d] - 1) * m ** d for d in range(p))


def _interior(p, level, idx):
    m = 3 ** level
    return all(0 < idx[d] < m for d in range(p))


def _cells(p, level):
    m = 3 ** level
    for t in range(m ** p):
        yield tuple((t // m ** d) % m for d in range(p))


def _corner(ci, e, p):
    return tuple(ci[d] + ((e >> d) & 1) for d in range(p))


def dense_assemble(p: int, level: int, theta: float, phi: complex, cap: int = 10000) -> np.ndarray:
    """oracle.cpp:153-175 (constant phi)."""
    n = interior_count(p, level)
    if n > cap:
        raise ValueError("dense_assemble: too many unknowns")
    H = np.zeros((n, n), dtype=complex)
    A = cell_operator(p, 3.0 ** -level, theta, phi)
    nc = 1 << p
    for ci in _cells(p, level):
        for a in range(nc):
            va = _corner(ci, a, p)
            if not _interior(p, level, va):
                continue
            ia = interior_flat(p, level, va)
            for b in range(nc):
                vb = _corner(ci, b, p)
                if _interior(p, level, vb):
                    H[ia, interior_flat(p, level, vb)] += A[a, b]
    return H


def load_vector(p: int, level: int, theta: float, chi: Callable[[np.ndarray], complex]) -> np.ndarray:
    """oracle.cpp:177-202: sum over cells of hElem^p M chi(corners)."""
    n = interior_count(p, level)
    b = np.zeros(n, dtype=complex)
    h = 3.0 ** -level
    ms = (h * complex(np.cos(theta), np.sin(theta))) ** p
    _, M = reference_matrices(p)
    nc = 1 << p
    for ci in _cells(p, level):
        vals = [chi(np.array(_corner(ci, e, p)) * h) for e in range(nc)]
        for a in range(nc):
            va = _corner(ci, a, p)
            if _interior(p, level, va):
                b[interior_flat(p, level, va)] += ms * sum(M[a, e] * vals[e] for e in range(nc))
    return b


def residual(p, level, theta, phi, b, u) -> np.ndarray:
    """oracle.cpp:204-240 (row-wise b - H u, no size cap) via the assembled stencil."""
    H = dense_assemble(p, level, theta, phi, cap=10 ** 9)
    return b - H @ u


def prolongation_matrix(p: int, fine_level: int) -> np.ndarray:
    """oracle.cpp:242-268."""
    nf, ncoarse = interior_count(p, fine_level), interior_count(p, fine_level - 1)
    P = np.zeros((nf, ncoarse))
    mc = 3 ** (fine_level - 1)
    m = 3 ** fine_level
    for idx in itertools.product(range(1, m), repeat=p):
        idx = idx[::-1]
        q = [min(idx[d] // 3, mc - 1) for d in range(p)]
        rel = [idx[d] - 3 * q[d] for d in range(p)]
        f = interior_flat(p, fine_level, idx)
        for e in range(1 << p):
            w = 1.0
            vc = []
            for d in range(p):
                bit = (e >> d) & 1
                vc.append(q[d] + bit)
                w *= KW1[rel[d]] if bit else KW0[rel[d]]
            if w != 0.0 and _interior(p, fine_level - 1, vc):
                P[f, interior_flat(p, fine_level - 1, vc)] += w
    return P


def injection_matrix(p: int, fine_level: int) -> np.ndarray:
    """oracle.cpp:270-280."""
    nf, ncoarse = interior_count(p, fine_level), interior_count(p, fine_level - 1)
    I = np.zeros((ncoarse, nf))
    mc = 3 ** (fine_level - 1)
    for idx in itertools.product(range(1, mc), repeat=p):
        idx = idx[::-1]
        I[interior_flat(p, fine_level - 1, idx), interior_flat(p, fine_level, [3 * x for x in idx])] = 1.0
    return I


def omega_unmasked(kind: str, ws: complex, succ: int, n: int, lgrid: int = 2) -> complex:
    """proj/src/cycles.cpp:17-31 (no two-phase)."""
    if kind == "jacobi-only":
        return ws if succ == 0 else 0.0
    if kind == "undamped":
        return ws
    if kind == "lgrid":
        return ws if succ <= lgrid else 0.0
    if kind == "exponential":
        return ws ** (succ + 1)
    e = (1.0 - 1.0 / n) * (succ + 1)
    return 1.0 if e == 0.0 else complex(ws) ** e


def reference_cycles(kind: str, p: int, levels: int, theta: float, phi: complex, chi, omega_kind: str,
                     ws: complex, sweeps: int, u0=None, hb: bool = False) -> List[np.ndarray]:
    """Literal dense transcription of Alg. 2 / 3 (td-add / td-bpx), oracle.cpp:465-509."""
    L = levels
    H = {l: dense_assemble(p, l, theta, phi) for l in range(1, L + 1)}
    diag = {l: np.diag(H[l]).copy() for l in H}
    P = {l: prolongation_matrix(p, l) for l in range(2, L + 1)}
    Iop = {l: injection_matrix(p, l) for l in range(2, L + 1)}
    cp = {}
    for l in range(1, L + 1):
        m = 3 ** l
        flags = np.zeros(interior_count(p, l), dtype=bool)
        for idx in itertools.product(range(1, m), repeat=p):
            idx = idx[::-1]
            flags[interior_flat(p, l, idx)] = all(x % 3 == 0 for x in idx)
        cp[l] = flags
    u = {l: np.zeros(interior_count(p, l), dtype=complex) for l in range(1, L + 1)}
    b = {l: np.zeros(interior_count(p, l), dtype=complex) for l in range(1, L + 1)}
    sc = {l: np.zeros_like(u[l]) for l in u}
    sf = {l: np.zeros_like(u[l]) for l in u}
    si = {l: np.zeros_like(u[l]) for l in u}
    b[L] = load_vector(p, L, theta, chi)
    if u0 is not None:
        u[L] = np.array(u0, dtype=complex)
        for l in range(L, 1, -1):
            u[l - 1] = Iop[l] @ u[l]
    bpx = kind == "td-bpx"
    out = []
    for n in range(1, sweeps + 1):
        uhat = {}
        for l in range(1, L + 1):
            if l > 1:
                sc[l] = sc[l] + P[l] @ sc[l - 1]
                if bpx:
                    psi = P[l] @ si[l - 1]
                    sc[l] = np.where(cp[l], sc[l], sc[l] - psi)
            u[l] = u[l] + sc[l] + sf[l]
            sf[l] = np.zeros_like(sf[l])
            uhat[l] = u[l] - P[l] @ u[l - 1] if l > 1 else u[l].copy()
        for l in range(L, 0, -1):
            r = b[l] - H[l] @ u[l]
            rhat = b[l] - H[l] @ uhat[l]
            s = r / diag[l]
            w = omega_unmasked(omega_kind, ws, L - l, n)
            if bpx:
                sc[l] = np.where(cp[l], 0.0, w * s)
                if l > 1:
                    si[l - 1] = Iop[l] @ (w * s)
            else:
                wv = np.where(cp[l] & hb, 0.0, w)
                sc[l] = wv * s
            if l > 1:
                b[l - 1] = P[l].T @ rhat
                sf[l - 1] = Iop[l] @ (sf[l] + sc[l])
        out.append(u[L].copy())
    return out


def chi_sin(x: np.ndarray) -> complex:
    """proj/src/problems.cpp:7-12."""
    v = len(x) * np.pi * np.pi
    for xi in x:
        v *= np.sin(np.pi * xi)
    return v


def random_vector(n: int, seed: int) -> np.ndarray:
    """proj/tests/test_util.hpp:31-44 (splitmix sequence)."""
    mask = (1 << 64) - 1
    s = seed
    vals = []
    for _ in range(2 * n):
        s = (s + 0x9E3779B97F4A7C15) & mask
        x = s
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & mask
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & mask
        x = x ^ (x >> 31)
        vals.append(2.0 * float(x >> 11) / 9007199254740992.0 - 1.0)
    return np.array(vals[0::2]) + 1j * np.array(vals[1::2])
