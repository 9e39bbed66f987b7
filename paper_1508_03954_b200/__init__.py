"""treemg on B200: the additive multilevel Helmholtz cycle of Reps & Weinzierl
(arXiv 1508.03954) as hand-written sm_100a kernels behind the reference's
C interface.

This module is the Python-side mirror of the reference interface for the hot
path (ctypes over ``libtreemg_b200.so``):

* :func:`run` / :class:`RunResult` -- ``treemg_run`` (proj/include/treemg.h,
  proj/src/capi.cpp:67-112) with the per-sweep history extension;
* :class:`Hierarchy` -- the device-resident drop-in for the C++ cycle API
  ``td_add`` / ``td_bpx`` (proj/include/treemg/cycles.hpp:56-62) plus field
  import/export, so the reference's cycle tests read the same here.

There is no CPU fallback: importing works without a GPU (so the CPU test
suite can check the C-ABI exports), but every compute call fails loudly when
the CUDA library or the device is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TMG_LIB") or os.path.join(PKG, "libtreemg_b200.so")  # TMG_LIB: developer A/B of build variants

STATUS = {0: "TREEMG_OK", 1: "TREEMG_E_USAGE", 2: "TREEMG_E_CAPACITY", 3: "TREEMG_E_RUNTIME"}
OUTCOME = {0: "converged", 1: "budget-exhausted", 2: "diverged"}
OMEGA_KINDS = {"jacobi-only": 0, "undamped": 1, "lgrid": 2, "exponential": 3, "transition": 4}
CHI_KINDS = {"zero": 0, "sin": 1, "ball": 2, "seeded": 3, "gaussian": 4}
PRECISIONS = {"exact": 0, "fast": 1, "fast-complex64": 2}

# The 14 entry points of proj/include/treemg.h and the extensions of
# include/treemg_b200.h, all exported by libtreemg_b200.so.
TREEMG_SYMBOLS = [
    "treemg_version", "treemg_last_error", "treemg_config_new", "treemg_config_free",
    "treemg_config_load_file", "treemg_config_set", "treemg_run", "treemg_result_free",
    "treemg_result_outcome", "treemg_result_sweeps", "treemg_result_work_units",
    "treemg_result_vertex_count", "treemg_result_final_norm", "treemg_result_first_norm",
]
EXTENSION_SYMBOLS = [
    "treemg_result_history_rows", "treemg_result_history_row", "treemg_result_device_ms",
    "tmg_hierarchy_create", "tmg_hierarchy_destroy", "tmg_td_add", "tmg_td_bpx", "tmg_lattice_size",
    "tmg_get_field", "tmg_set_field", "tmg_set_fine_interior_u", "tmg_set_random_initial_guess",
    "tmg_set_fine_rhs", "tmg_field_hash", "tmg_time_cycles", "tmg_e2e_step", "tmg_last_error",
    "treemg_result_fingerprint", "tmg_test_divdc3", "tmg_test_hypot", "tmg_nccl_unique_id", "tmg_slabs_create", "tmg_slabs_destroy",
    "tmg_slabs_cycle", "tmg_slabs_get_fine_u", "tmg_slabs_time_cycles", "tmg_slabs_owned_planes", "tmg_slab_plan",
    "tmg_slabs_e2e_step", "tmg_get_flags", "tmg_hanging_vertices", "tmg_leaf_vertices", "tmg_sphere_tree",
    "tmg_bu_fas", "tmg_textbook_add", "tmg_channel_norms", "tmg_dyn_create", "tmg_dyn_destroy", "tmg_dyn_depth",
    "tmg_dyn_interior_count", "tmg_dyn_set_cell_marks", "tmg_dyn_sweep", "tmg_dyn_flags", "tmg_dyn_sweep_tables",
    "tmg_mark", "tmg_levels", "tmg_set_cell_marks", "tmg_dyn_phase_ms", "tmg_existing_vertices",
    "tmg_slabs_create_local", "tmg_slabs_get_field",
]

_lib = None


class TreemgError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


class _Problem(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("levels", ctypes.c_int), ("ell_min", ctypes.c_int),
                ("theta", ctypes.c_double), ("phi_re", ctypes.c_double), ("phi_im", ctypes.c_double),
                ("chi_kind", ctypes.c_int), ("rhs_seed", ctypes.c_ulonglong), ("rhs_sphere", ctypes.c_int),
                ("precision", ctypes.c_int), ("max_vertices", ctypes.c_longlong), ("device", ctypes.c_int),
                ("sphere_levels", ctypes.c_int), ("channels", ctypes.c_int),
                ("coupling_re", ctypes.c_double), ("coupling_im", ctypes.c_double),
                ("h_max", ctypes.c_double), ("h_min", ctypes.c_double)]


class _Policy(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("omega_re", ctypes.c_double), ("omega_im", ctypes.c_double),
                ("lgrid", ctypes.c_int), ("hb", ctypes.c_int), ("bpx", ctypes.c_int), ("two_phase", ctypes.c_int)]


class _Stats(ctypes.Structure):
    _fields_ = [("max_norm", ctypes.c_double), ("euclid_norm", ctypes.c_double), ("h_norm", ctypes.c_double),
                ("updated_fine_vertices", ctypes.c_longlong)]


def build(force: bool = False) -> str:
    from . import build as _b
    return _b.build(force=force)


def lib():
    """The loaded CUDA library; raises if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_1508_03954_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, cp, ip, dp, pd = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_double)
        L.treemg_version.restype = ctypes.c_uint
        L.treemg_last_error.restype = cp
        L.tmg_last_error.restype = cp
        L.treemg_config_new.restype = vp
        L.treemg_config_free.argtypes = [vp]
        L.treemg_config_set.restype = ip
        L.treemg_config_set.argtypes = [vp, cp, cp]
        L.treemg_config_load_file.restype = ip
        L.treemg_config_load_file.argtypes = [vp, cp]
        L.treemg_run.restype = ip
        L.treemg_run.argtypes = [vp, ctypes.POINTER(vp)]
        L.treemg_result_free.argtypes = [vp]
        for n, rt in (("treemg_result_outcome", ip), ("treemg_result_sweeps", ip),
                      ("treemg_result_work_units", dp), ("treemg_result_vertex_count", ctypes.c_longlong),
                      ("treemg_result_first_norm", dp), ("treemg_result_history_rows", ip),
                      ("treemg_result_device_ms", dp)):
            getattr(L, n).restype = rt
            getattr(L, n).argtypes = [vp]
        L.treemg_result_final_norm.restype = dp
        L.treemg_result_final_norm.argtypes = [vp, cp, ip]
        L.treemg_result_history_row.restype = ip
        L.treemg_result_history_row.argtypes = [vp, ip, pd]
        L.tmg_hierarchy_create.restype = ip
        L.tmg_hierarchy_create.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(vp)]
        L.tmg_hierarchy_destroy.argtypes = [vp]
        L.tmg_dyn_create.restype = ip
        L.tmg_dyn_create.argtypes = [ip, ip, ip, ip, dp, ctypes.c_longlong, ctypes.POINTER(vp)]
        L.tmg_dyn_destroy.argtypes = [vp]
        L.tmg_dyn_depth.restype = ip
        L.tmg_dyn_depth.argtypes = [vp]
        L.tmg_dyn_interior_count.restype = ctypes.c_longlong
        L.tmg_dyn_interior_count.argtypes = [vp]
        L.tmg_dyn_set_cell_marks.restype = ip
        L.tmg_dyn_set_cell_marks.argtypes = [vp, ip, vp]
        L.tmg_dyn_sweep.restype = ip
        L.tmg_dyn_sweep.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
        L.tmg_dyn_flags.restype = ip
        L.tmg_dyn_flags.argtypes = [vp, ip, vp, vp, vp]
        L.tmg_dyn_sweep_tables.restype = ip
        L.tmg_dyn_sweep_tables.argtypes = [vp, ip, vp, vp, vp, vp, vp, vp]
        L.tmg_mark.restype = ip
        L.tmg_mark.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
        L.tmg_dyn_phase_ms.restype = ip
        L.tmg_dyn_phase_ms.argtypes = [vp, pd]
        L.tmg_existing_vertices.restype = ctypes.c_longlong
        L.tmg_existing_vertices.argtypes = [vp]
        L.tmg_set_cell_marks.restype = ip
        L.tmg_set_cell_marks.argtypes = [vp, ip, vp]
        L.tmg_levels.restype = ip
        L.tmg_levels.argtypes = [vp]
        L.tmg_channel_norms.restype = ip
        L.tmg_channel_norms.argtypes = [vp, pd, pd, pd, ip]
        for n in ("tmg_td_add", "tmg_td_bpx"):
            getattr(L, n).restype = ip
            getattr(L, n).argtypes = [vp, ctypes.POINTER(_Policy), ip, ctypes.POINTER(_Stats)]
        L.tmg_get_flags.restype = ip
        L.tmg_get_flags.argtypes = [vp, ip, vp, vp, vp]
        L.tmg_sphere_tree.restype = ip
        L.tmg_sphere_tree.argtypes = [ip, ip, ip, ip, vp, vp, vp, vp]
        L.tmg_hanging_vertices.restype = ctypes.c_longlong
        L.tmg_hanging_vertices.argtypes = [vp]
        L.tmg_leaf_vertices.restype = ctypes.c_longlong
        L.tmg_leaf_vertices.argtypes = [vp]
        L.tmg_bu_fas.restype = ip
        L.tmg_bu_fas.argtypes = [vp, ctypes.POINTER(_Policy), ip, ctypes.POINTER(_Stats)]
        L.tmg_textbook_add.restype = ip
        L.tmg_textbook_add.argtypes = [vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.POINTER(_Stats)]
        L.tmg_lattice_size.restype = ctypes.c_longlong
        L.tmg_lattice_size.argtypes = [vp, ip]
        L.tmg_get_field.restype = ip
        L.tmg_get_field.argtypes = [vp, ip, cp, pd]
        L.tmg_set_field.restype = ip
        L.tmg_set_field.argtypes = [vp, ip, cp, pd]
        L.tmg_set_fine_interior_u.restype = ip
        L.tmg_set_fine_interior_u.argtypes = [vp, pd]
        L.tmg_set_random_initial_guess.restype = ip
        L.tmg_set_random_initial_guess.argtypes = [vp, ctypes.c_ulonglong]
        L.tmg_set_fine_rhs.restype = ip
        L.tmg_set_fine_rhs.argtypes = [vp, pd]
        L.tmg_field_hash.restype = ctypes.c_ulonglong
        L.tmg_field_hash.argtypes = [vp, ip, cp]
        L.tmg_time_cycles.restype = ip
        L.tmg_time_cycles.argtypes = [vp, ctypes.POINTER(_Policy), ip, ip, ip, pd]
        L.treemg_result_fingerprint.restype = ctypes.c_ulonglong
        L.treemg_result_fingerprint.argtypes = [vp, cp]
        L.tmg_test_hypot.restype = ip
        L.tmg_test_hypot.argtypes = [pd, pd, pd, ctypes.c_longlong]
        L.tmg_test_divdc3.restype = ip
        L.tmg_test_divdc3.argtypes = [pd, pd, pd, ctypes.c_longlong]
        L.tmg_nccl_unique_id.restype = ip
        L.tmg_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.tmg_slabs_create.restype = ip
        L.tmg_slabs_create.argtypes = [ctypes.POINTER(_Problem), ip, ip, ip, ctypes.c_char_p, ctypes.POINTER(vp)]
        L.tmg_slabs_destroy.argtypes = [vp]
        L.tmg_slabs_create_local.restype = ip
        L.tmg_slabs_create_local.argtypes = [ctypes.POINTER(_Problem), ip, ip, ctypes.POINTER(vp)]
        L.tmg_slabs_get_field.restype = ip
        L.tmg_slabs_get_field.argtypes = [vp, ip, cp, pd]
        L.tmg_slabs_cycle.restype = ip
        L.tmg_slabs_cycle.argtypes = [vp, ctypes.POINTER(_Policy), ip, ctypes.POINTER(_Stats)]
        L.tmg_slabs_get_fine_u.restype = ip
        L.tmg_slabs_get_fine_u.argtypes = [vp, pd]
        L.tmg_slabs_time_cycles.restype = ip
        L.tmg_slabs_time_cycles.argtypes = [vp, ctypes.POINTER(_Policy), ip, ip, pd]
        L.tmg_slabs_owned_planes.restype = ip
        L.tmg_slabs_owned_planes.argtypes = [vp, ctypes.POINTER(ip), ctypes.POINTER(ip)]
        L.tmg_slabs_e2e_step.restype = ip
        L.tmg_slabs_e2e_step.argtypes = [vp, ctypes.POINTER(_Policy), ip, pd, pd, ctypes.POINTER(ctypes.c_longlong)]
        L.tmg_slab_plan.restype = ip
        L.tmg_slab_plan.argtypes = [ip, ip, ctypes.POINTER(ip)]
        L.tmg_e2e_step.restype = ip
        L.tmg_e2e_step.argtypes = [vp, ctypes.POINTER(_Policy), ip, pd, pd]
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise TreemgError(st, lib().treemg_last_error().decode())


def _pd(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@dataclass
class RunResult:
    """RunResult of proj/include/treemg/runner.hpp:60-68 via the C-ABI."""
    outcome: str
    sweeps: int
    work_units: float
    vertex_count: int
    first_norm: float
    final_norm: Dict[str, float]
    history: np.ndarray = field(repr=False)
    device_ms: float = 0.0
    u_hash: int = 0
    sc_hash: int = 0
    channel_u_hashes: List[int] = field(default_factory=list)  # fingerprint: u of every channel


def run(cfg: Dict[str, object], out_prefix: Optional[str] = None) -> RunResult:
    """treemg_config_set for every key, then treemg_run (synchronous)."""
    L = lib()
    c = L.treemg_config_new()
    try:
        for k, v in cfg.items():
            _check(L.treemg_config_set(c, str(k).encode(), str(v).encode()))
        if out_prefix:
            _check(L.treemg_config_set(c, b"out", out_prefix.encode()))
        res = ctypes.c_void_p()
        _check(L.treemg_run(c, ctypes.byref(res)))
    finally:
        L.treemg_config_free(c)
    try:
        rows = L.treemg_result_history_rows(res)
        hist = np.zeros((rows, 6))
        buf = np.zeros(6)
        for i in range(rows):
            _check(L.treemg_result_history_row(res, i, _pd(buf)))
            hist[i] = buf
        return RunResult(
            outcome=OUTCOME[L.treemg_result_outcome(res)], sweeps=L.treemg_result_sweeps(res),
            work_units=L.treemg_result_work_units(res), vertex_count=L.treemg_result_vertex_count(res),
            first_norm=L.treemg_result_first_norm(res),
            final_norm={w: L.treemg_result_final_norm(res, w.encode(), -1) for w in ("max", "euclid", "h")},
            history=hist, device_ms=L.treemg_result_device_ms(res),
            u_hash=L.treemg_result_fingerprint(res, b"u"), sc_hash=L.treemg_result_fingerprint(res, b"sc"),
            channel_u_hashes=[L.treemg_result_fingerprint(res, f"u#{c}".encode())
                              for c in range(int(cfg.get("channels", 1)))])
    finally:
        L.treemg_result_free(res)


@dataclass
class Policy:
    """OmegaPolicy (proj/include/treemg/cycles.hpp:17-24)."""
    kind: str = "exponential"
    omega_s: complex = 0.8 + 0j
    lgrid: int = 2
    hb: bool = False
    bpx: bool = False
    two_phase: bool = False

    def c(self) -> _Policy:
        return _Policy(OMEGA_KINDS[self.kind], complex(self.omega_s).real, complex(self.omega_s).imag,
                       self.lgrid, int(self.hb), int(self.bpx), int(self.two_phase))


@dataclass
class SweepStats:
    max_norm: float
    euclid_norm: float
    h_norm: float
    updated_fine_vertices: int


class Hierarchy:
    """Device-resident regular 3^d hierarchy (the Spacetree drop-in of the cycle API)."""

    def __init__(self, dim: int, levels: int, phi: complex = 0.0, theta_deg: float = 0.0, chi: str = "sin",
                 rhs_seed: int = 12345, rhs_sphere: bool = False, ell_min: int = 1, precision: str = "exact",
                 max_vertices: int = 0, device: int = 0, sphere_levels: int = 0, channels: int = 1,
                 coupling: complex = 0.0, h_max: float = 0.0, h_min: float = 0.0):
        """levels: depth of the regular base tree; sphere_levels > 0 adds that many
        levels refined inside |x - 1/2|^2 < 0.04 (static adaptive tree, cfg4).
        channels > 1: that many unknowns per vertex with the same fields, coupled
        by A_ij = coupling (i != j) through the mass matrix (runner.cpp:152-157);
        exact precision, regular trees.  field(level, "u#1") reads channel 1."""
        self.L = lib()
        prob = _Problem(dim, levels, ell_min, np.deg2rad(theta_deg) if theta_deg else 0.0,
                        complex(phi).real, complex(phi).imag, CHI_KINDS[chi], rhs_seed, int(rhs_sphere),
                        PRECISIONS[precision], max_vertices, device, sphere_levels, channels,
                        complex(coupling).real, complex(coupling).imag, h_max, h_min)
        if theta_deg:
            prob.theta = theta_deg * np.pi / 180.0  # ProblemSpec::thetaGlobal = deg * M_PI / 180.0
        h = ctypes.c_void_p()
        _check(self.L.tmg_hierarchy_create(ctypes.byref(prob), ctypes.byref(h)))
        self.h = h
        self.dim, self.levels = dim, levels + sphere_levels
        self.dynamic = h_max > 0 and h_min > 0
        if self.dynamic:
            self.levels = self.L.tmg_levels(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.L.tmg_hierarchy_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _sweep(self, fn, pol: Policy, n: int) -> SweepStats:
        st = _Stats()
        pc = pol.c()
        _check(fn(self.h, ctypes.byref(pc), n, ctypes.byref(st)))
        return SweepStats(st.max_norm, st.euclid_norm, st.h_norm, st.updated_fine_vertices)

    def td_add(self, pol: Policy, n: int) -> SweepStats:
        return self._sweep(self.L.tmg_td_add, pol, n)

    def td_bpx(self, pol: Policy, n: int) -> SweepStats:
        return self._sweep(self.L.tmg_td_bpx, pol, n)

    MARK_KEYS = ("refined", "erased", "refine_vertices", "erase_vertices", "refine_cells", "erase_cells",
                 "veto_conv", "veto_hmin", "veto_hmax")

    def mark(self) -> dict:
        """Dynamic adaptivity: mark on the device after a sweep (amr.cpp:61-222);
        refined / erased are the structural edits of that sweep."""
        out = (ctypes.c_longlong * 9)()
        _check(self.L.tmg_mark(self.h, out))
        self.levels = self.L.tmg_levels(self.h)
        return dict(zip(self.MARK_KEYS, list(out)))

    def depth(self) -> int:
        return self.L.tmg_levels(self.h)

    def dyn_phase_ms(self) -> dict:
        """Cumulative ms: host replay, table upload, device sweep, final upload, mark."""
        out = np.zeros(6)
        _check(self.L.tmg_dyn_phase_ms(self.h, _pd(out)))
        return dict(zip(("replay", "tables", "device", "final", "mark", "launches"), out.tolist()))

    @property
    def existing_vertices(self) -> int:
        return int(self.L.tmg_existing_vertices(self.h))

    def set_cell_marks(self, level: int, cells: np.ndarray):
        """Overwrite the pending cell marks of `level` (4 refine, 8 erase per lattice cell)."""
        c = np.ascontiguousarray(cells, np.uint8)
        _check(self.L.tmg_set_cell_marks(self.h, level, c.ctypes.data_as(ctypes.c_void_p)))

    def channel_norms(self):
        """Per-channel (max, euclid, h) norms of the last td_add / td_bpx sweep
        (SweepStats per channel, cycles.hpp:27-31); empty for one channel."""
        cap = 16
        mx, eu, hn = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        n = self.L.tmg_channel_norms(self.h, _pd(mx), _pd(eu), _pd(hn), cap)
        return [(mx[c], eu[c], hn[c]) for c in range(max(n, 0))]

    def bu_fas(self, pol: Policy, n: int) -> SweepStats:
        """bu_fas + evaluate_residual_norms (cycles.cpp:374-603, 716-786); exact storage."""
        return self._sweep(self.L.tmg_bu_fas, pol, n)

    def textbook_add(self, omega_s: complex, omega_cg: complex) -> SweepStats:
        """textbook_add + evaluate_residual_norms (cycles.cpp:605-714, 716-786); exact storage."""
        st = _Stats()
        _check(self.L.tmg_textbook_add(self.h, complex(omega_s).real, complex(omega_s).imag,
                                       complex(omega_cg).real, complex(omega_cg).imag, ctypes.byref(st)))
        return SweepStats(st.max_norm, st.euclid_norm, st.h_norm, st.updated_fine_vertices)

    def lattice_size(self, level: int) -> int:
        return self.L.tmg_lattice_size(self.h, level)

    def field(self, level: int, name: str) -> np.ndarray:
        n = self.lattice_size(level)
        out = np.zeros(2 * n)
        _check(self.L.tmg_get_field(self.h, level, name.encode(), _pd(out)))
        return out[0::2] + 1j * out[1::2]

    def flags(self, level: int):
        """Adaptive trees: (flags, succ, cells) per lattice point of `level`
        (flags 1 exists | 2 hanging | 4 refined | 8 boundary | 16 cPoint;
        cells 1 exists | 2 refined, indexed by the lower corner)."""
        n = self.lattice_size(level)
        fl = np.zeros(n, np.uint8)
        sc = np.zeros(n, np.int8)
        ce = np.zeros(n, np.uint8)
        _check(self.L.tmg_get_flags(self.h, level, fl.ctypes.data_as(ctypes.c_void_p),
                                    sc.ctypes.data_as(ctypes.c_void_p), ce.ctypes.data_as(ctypes.c_void_p)))
        return fl, sc, ce

    @property
    def hanging_vertices(self) -> int:
        return int(self.L.tmg_hanging_vertices(self.h))

    @property
    def leaf_vertices(self) -> int:
        return int(self.L.tmg_leaf_vertices(self.h))

    def set_field(self, level: int, name: str, values: np.ndarray):
        buf = np.ascontiguousarray(np.asarray(values, dtype=np.complex128)).view(np.float64).copy()
        _check(self.L.tmg_set_field(self.h, level, name.encode(), _pd(buf)))

    def set_fine_interior_u(self, u: np.ndarray):
        buf = np.ascontiguousarray(np.asarray(u, dtype=np.complex128)).view(np.float64).copy()
        _check(self.L.tmg_set_fine_interior_u(self.h, _pd(buf)))

    def set_random_initial_guess(self, seed: int):
        _check(self.L.tmg_set_random_initial_guess(self.h, seed))

    def set_fine_rhs(self, chi: np.ndarray):
        buf = np.ascontiguousarray(np.asarray(chi, dtype=np.complex128)).view(np.float64).copy()
        _check(self.L.tmg_set_fine_rhs(self.h, _pd(buf)))

    def field_hash(self, level: int, name: str) -> int:
        return int(self.L.tmg_field_hash(self.h, level, name.encode()))

    def time_cycles(self, pol: Policy, n0: int, count: int, flush_l2: bool = True) -> np.ndarray:
        out = np.zeros(4)
        pc = pol.c()
        _check(self.L.tmg_time_cycles(self.h, ctypes.byref(pc), n0, count, int(flush_l2), _pd(out)))
        return out

    def e2e_step(self, pol: Policy, n: int, chi_host: np.ndarray) -> np.ndarray:
        out = np.zeros(3)
        pc = pol.c()
        buf = chi_host.view(np.float64) if chi_host.dtype == np.complex128 else chi_host
        _check(self.L.tmg_e2e_step(self.h, ctypes.byref(pc), n, _pd(buf), _pd(out)))
        return out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().tmg_nccl_unique_id(buf))
    return buf.raw


def slab_plan(levels: int, world: int) -> np.ndarray:
    """Per slab (cb, ce, z0, z1, Zs, Ze, Ws, We), host-only."""
    out = (ctypes.c_int * (8 * world))()
    _check(lib().tmg_slab_plan(levels, world, out))
    return np.array(list(out)).reshape(world, 8)


class Slabs:
    """z-slab decomposition of a 3D fast-precision hierarchy.

    nccl_id=None: `local` virtual slabs on this process's device (test mode);
    else one slab for `rank` of `world` over NCCL."""

    def __init__(self, levels: int, phi: complex, chi: str = "seeded", rhs_seed: int = 12345, ell_min: int = 1,
                 local: int = 1, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None, device: int = 0,
                 devices: int = 1):
        """devices > 1 (nccl_id None): the `local` slabs spread over that many GPUs of this process."""
        self.L = lib()
        prob = _Problem(3, levels, ell_min, 0.0, complex(phi).real, complex(phi).imag, CHI_KINDS[chi], rhs_seed, 0, 1,
                        10 ** 12, device)
        h = ctypes.c_void_p()
        if nccl_id is None:
            _check(self.L.tmg_slabs_create_local(ctypes.byref(prob), local, devices, ctypes.byref(h)))
        else:
            _check(self.L.tmg_slabs_create(ctypes.byref(prob), local, rank, world, nccl_id, ctypes.byref(h)))
        self.h = h
        self.levels = levels

    def close(self):
        if getattr(self, "h", None):
            self.L.tmg_slabs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def cycle(self, pol: "Policy", n: int) -> "SweepStats":
        st = _Stats()
        pc = pol.c()
        _check(self.L.tmg_slabs_cycle(self.h, ctypes.byref(pc), n, ctypes.byref(st)))
        return SweepStats(st.max_norm, st.euclid_norm, st.h_norm, st.updated_fine_vertices)

    def fine_u(self) -> np.ndarray:
        n = (3 ** self.levels + 1) ** 3
        out = np.zeros(2 * n)
        _check(self.L.tmg_slabs_get_fine_u(self.h, _pd(out)))
        return out[0::2] + 1j * out[1::2]

    def field(self, level: int, name: str) -> np.ndarray:
        """Whole-lattice u / sc of `level` gathered from the slabs (bitwise one GPU's field)."""
        n = (3 ** level + 1) ** 3
        out = np.zeros(2 * n)
        _check(self.L.tmg_slabs_get_field(self.h, level, name.encode(), _pd(out)))
        return out[0::2] + 1j * out[1::2]

    def owned_planes(self):
        z0, z1 = ctypes.c_int(), ctypes.c_int()
        self.L.tmg_slabs_owned_planes(self.h, ctypes.byref(z0), ctypes.byref(z1))
        return z0.value, z1.value

    def time_cycles(self, pol: "Policy", n0: int, count: int) -> np.ndarray:
        out = np.zeros(4)
        pc = pol.c()
        _check(self.L.tmg_slabs_time_cycles(self.h, ctypes.byref(pc), n0, count, _pd(out)))
        return out

    def e2e_step(self, pol: "Policy", n: int, chi_host: np.ndarray):
        out = np.zeros(3)
        nb = ctypes.c_longlong()
        pc = pol.c()
        buf = chi_host.view(np.float64) if chi_host.dtype == np.complex128 else chi_host
        _check(self.L.tmg_slabs_e2e_step(self.h, ctypes.byref(pc), n, _pd(buf), _pd(out), ctypes.byref(nb)))
        return out, nb.value


def device_divide(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """x / y on the device with the kernels' __divdc3 restatement (test hook)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    y = np.ascontiguousarray(y, dtype=np.complex128)
    out = np.zeros_like(x)
    _check(lib().tmg_test_divdc3(_pd(x.view(np.float64)), _pd(y.view(np.float64)), _pd(out.view(np.float64)), len(x)))
    return out


def device_hypot(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """hypot(x, y) on the device with the mark pass's libm restatement (test hook)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros_like(x)
    _check(lib().tmg_test_hypot(_pd(x), _pd(y), _pd(out), len(x)))
    return out


class DynStructure:
    """Host-only structural replay of dynamic adaptivity (tmg_dyn_*, dyn.hpp):
    the tree a td_add / td_bpx traversal with applyMarks leaves behind."""

    def __init__(self, dim: int, start: int, max_level: int, ell_min: int = 1, h_min: float = 1e-3,
                 max_vertices: int = 0):
        self.L = lib()
        h = ctypes.c_void_p()
        _check(self.L.tmg_dyn_create(dim, start, max_level, ell_min, h_min, max_vertices, ctypes.byref(h)))
        self.h, self.dim = h, dim

    def close(self):
        if getattr(self, "h", None):
            self.L.tmg_dyn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def depth(self) -> int:
        return self.L.tmg_dyn_depth(self.h)

    def interior_count(self) -> int:
        return int(self.L.tmg_dyn_interior_count(self.h))

    def _n(self, level: int) -> int:
        return (3 ** level + 1) ** self.dim

    def set_cell_marks(self, level: int, cells: np.ndarray):
        c = np.ascontiguousarray(cells, np.uint8)
        _check(self.L.tmg_dyn_set_cell_marks(self.h, level, c.ctypes.data_as(ctypes.c_void_p)))

    def sweep(self):
        out = (ctypes.c_longlong * 4)()
        _check(self.L.tmg_dyn_sweep(self.h, out))
        return dict(refined=out[0], erased=out[1], updated=out[2], special=out[3])

    def flags(self, level: int):
        n = self._n(level)
        fl, sc, ce = np.zeros(n, np.uint8), np.zeros(n, np.int8), np.zeros(n, np.uint8)
        _check(self.L.tmg_dyn_flags(self.h, level, fl.ctypes.data_as(ctypes.c_void_p),
                                    sc.ctypes.data_as(ctypes.c_void_p), ce.ctypes.data_as(ctypes.c_void_p)))
        return fl, sc, ce

    def sweep_tables(self, level: int):
        n = self._n(level)
        arrs = [np.zeros(n, np.uint8) for _ in range(4)] + [np.zeros(n, np.int8), np.zeros(n, np.uint8)]
        _check(self.L.tmg_dyn_sweep_tables(self.h, level, *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs]))
        return dict(zip(("role", "finish_corner", "finish_cells", "skip_cells", "succ", "cells"), arrs))


def sphere_tree(dim: int, base: int, sphere_levels: int, level: int):
    """Host-side structure of the static sphere tree (no GPU needed):
    (flags, succ, cells, finish_corner) per lattice point of `level`."""
    L = lib()
    n = (3 ** level + 1) ** dim
    fl, sc, ce, fc = np.zeros(n, np.uint8), np.zeros(n, np.int8), np.zeros(n, np.uint8), np.zeros(n, np.uint8)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(L.tmg_sphere_tree(dim, base, sphere_levels, level, ptr(fl), ptr(sc), ptr(ce), ptr(fc)))
    return fl, sc, ce, fc


def exported_symbols() -> List[str]:
    """Dynamic symbols of the built library (checked by the CPU test suite)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    return [line.split()[-1] for line in out.splitlines() if line.strip()]
