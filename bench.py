#!/usr/bin/env python
"""Benchmark of the additive multilevel Helmholtz cycle on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload cfg5|cfg3|cfg2|cfg1] [--precision fast|exact]

A "step" is one additive multigrid cycle (td_add / td_bpx) over
the whole hierarchy of the workload, inputs resident in HBM.  Metric
(BASELINE.json): complex DoF-updates/s per cycle = interior fine DoF x
cycles / device time, plus the fine-pass kernel's achieved HBM GB/s against
MEASURED_PEAKS.json.  Prints ONE JSON line on rank 0.

Workload: the BASELINE metric's target is quoted on the 243^3
and 729^3 configs; the 729^3 cycle (cfg5's final FMG level, k=80) fits one
GPU, so it is the N=1 workload.  Other configs are parity-test cases.

N>1 (torchrun, one process per GPU): 3D workloads run the z-slab
decomposition: each rank owns a slab of the fine level and of
level L-1, halos / restriction partials / the replicated level's residual
move over NCCL; the problem size is fixed ("scaling": "strong") and value =
DoF x cycles / max-over-ranks device time.  2D workloads run one replica
per GPU ("scaling": "weak").  --mode replicas forces replicas.

--impl reference: the reference CPU implementation (oracle/_ref, built from
the unmodified reference sources) on the host cores -- one single-threaded
reference process per core (the reference has no intra-solve parallelism;
capped by host RAM), rank 0 only.  The sample is the workload itself where
the reference can hold it in a few minutes (2D, 243^3) and otherwise the
243^3 tree with the workload's operator (cfg5: its own FMG stage 5; 729^3
needs ~130 GB and ~15 min per sweep); the line's cpu_baseline.sample says
which.  `config` is the workload, identical in both arms.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs -> solver settings: phi = k^2 (1 + 0.5 i)
WORKLOADS = {
    "cfg1": dict(dim=2, level=5, k=10, cycle="td-add", omega="exponential", omega_s=0.6,
                 desc="2D depth 5 (243^2), k=10, additive MG, exponential omega 0.6"),
    "cfg2": dict(dim=2, level=7, k=100, cycle="td-bpx", omega="undamped", omega_s=0.5,
                 desc="2D depth 7 (2187^2), k=100, BPX variant, undamped omega 0.5"),
    "cfg3": dict(dim=3, level=5, k=20, cycle="td-add", omega="exponential", omega_s=0.6,
                 desc="3D depth 5 (243^3), k=20, additive MG, exponential omega 0.6"),
    "cfg4": dict(dim=3, level=4, sphere_levels=2, k=40, cycle="td-add", omega="exponential", omega_s=0.6,
                 desc="3D adaptive: depth 4 refined to 6 inside |x-1/2|<0.2 (hanging vertices), k=40, f in the ball, "
                      "additive MG, exponential omega 0.6"),
    "cfg5": dict(dim=3, level=6, k=80, cycle="td-add", omega="exponential", omega_s=0.6,
                 desc="3D depth 6 (729^3), k=80, additive MG, exponential omega 0.6 (cfg5 final FMG level)"),
    # dynamic adaptivity: feature-based refine / erase marks after every sweep
    "dyn2d": dict(dim=2, level=3, dynamic=True, h_max=0.04, h_min=0.001, k=10, cycle="td-add", omega="undamped",
                  omega_s=0.6, desc="2D dynamic adaptivity h_max 0.04 -> h_min 0.001 (levels 3 -> 7), k=10, sin rhs, "
                                    "additive MG, undamped omega 0.6, marks after every sweep, exact precision"),
}
RHS_SEED = 12345


def workload_config(name, w):
    """The `config` object of the JSON line: the workload only, identical in the
    B200 arm and the reference arm (run settings are top-level keys)."""
    if w.get("sphere_levels") or w.get("dynamic"):
        return {"workload": name, "desc": w["desc"]}
    n_lat = lattice(w["level"], w["dim"])
    return {"workload": name, "desc": w["desc"], "dim": w["dim"], "level": w["level"],
            "interior_dof": interior(w), "cycle": w["cycle"],
            "l2": f"inputs larger than L2 (fine level arrays of {16 * n_lat / 1e9:.2f} GB each); no flush"}


def interior(w):
    return (3 ** w["level"] - 1) ** w["dim"]


def lattice(level, dim):
    return (3 ** level + 1) ** dim


def fine_bytes_per_vertex(w, precision):
    """Algorithmic HBM bytes per fine vertex of the fine pass, SURVEY §8(d):
    80 B (u, sc, b read; u, sc written) -- the basis of roofline.achieved.  The
    fused fast passes move less for the same work (v-form, fused3.cuh: v, b
    read, v written = 48 B); the exact pass is not fused (176 B)."""
    if precision == "exact":
        return 176
    if precision == "fast-complex64":  # complex64 halves B
        return 40
    return 80 if w["dim"] >= 2 else 128


def moved_bytes_per_vertex(w, precision):
    """Bytes per fine vertex the implementation's fine pass actually has to move:
    the fused 3D pass reads v and b and writes v (v-form, the write-only fine sc is
    re-derived on demand: fused3.cuh derive_u) -- 48 B, 24 B in complex64; the
    fused 2D pass also stores the fine sc -- 64 B, 32 B in complex64."""
    if precision == "exact":
        return 176
    if precision == "fast-complex64":
        return 24 if w["dim"] == 3 else 32
    return 48 if w["dim"] == 3 else 64 if w["dim"] == 2 else 128


def algorithmic_bytes(w, precision):
    """B = b_f N_L + 200 sum_{l<L} N_l (complex128 lattice sizes)."""
    NL = lattice(w["level"], w["dim"])
    coarse = sum(lattice(l, w["dim"]) for l in range(1, w["level"]))
    bf = fine_bytes_per_vertex(w, precision)
    return bf * NL + 200 * coarse, bf * NL


def fine_kernel_label(w, precision):
    if precision == "exact":
        return "exact fine pass (k_topdown + k_residual_exact + k_restrict_exact)"
    if w["dim"] == 3:
        return ("fused fine pass k_fused3<complex64> (TMA ring: top-down + residual + smooth + z/xy restriction)"
                if precision == "fast-complex64" else
                "fused fine pass k_fused3 (TMA ring: top-down + residual + smooth + z/xy restriction)")
    return ("fused fine pass k_fused2<complex64> (row-marching strips: top-down + residual + smooth + restriction)"
            if precision == "fast-complex64" else
            "fused fine pass k_fused2 (row-marching strips: top-down + residual + smooth + restriction)")


def ncu_traffic(workload: str, precision: str, mode: str):
    """DRAM bytes per launch of the fine-pass kernel from the committed ncu capture
    (profiles/traffic.json, written from a `ncu` run of the same workload), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(f"{workload}/{precision}/{mode}")
    except Exception:
        return None


def settle(h, pol, D=None, ctx=None, seconds=0.3, **kw):
    """Untimed cycles for ~`seconds` before the warm-up: brings SM / HBM clocks to
    their steady state so short timed regions are not measured on a ramp.  The
    cycle count is agreed over ranks (slab cycles exchange data collectively)."""
    ms = float(h.time_cycles(pol, 1, 1, **kw)[0])
    if D is not None and ctx is not None:
        ms = D.reduce_max(ctx, ms)
    count = int(min(2000, max(1, seconds * 1e3 / max(ms, 1e-3))))
    h.time_cycles(pol, 1, count, **kw)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"tmg_clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            # nvidia-smi needs ~0.1-0.5 s to start: wait for its first sample so the
            # (often short) timed region is actually covered
            t0 = time.time()
            while time.time() - t0 < 3.0:
                self.fh.flush()
                if os.path.getsize(self.path) > 0:
                    break
                time.sleep(0.01)
            self.start_lines = self._lines()
        except Exception:
            self.proc = None
        return self

    def _lines(self):
        try:
            with open(self.path) as f:
                return sum(1 for _ in f)
        except Exception:
            return 0

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            lines = open(self.path).read().splitlines()
            # samples taken while the timed region ran (plus the one just before it)
            lines = lines[max(0, getattr(self, "start_lines", 1) - 1):]
            for line in lines:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx = max(mx, float(f[1]))
                except ValueError:
                    continue
                for n, v in zip(names, f[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# reference CPU arm
def _ref_cfg(w, level):
    cfg = dict(problem="helmholtz-sin", dim=w["dim"], level=level,
               phi=f"{w['k'] ** 2},{0.5 * w['k'] ** 2}", cycle=w["cycle"], omega=w["omega"],
               omega_s=w["omega_s"], max_sweeps=10 ** 6, target_drop=1e-300, rhs="seeded", rhs_seed=RHS_SEED,
               max_vertices=10 ** 9)
    if w.get("sphere_levels"):
        cfg.update(sphere_levels=w["sphere_levels"], rhs_mask="sphere")
    return cfg


def _ref_worker(args):
    w, level, sweeps, warmup, bar, q = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refdriver as R
    s = R.RefSession(_ref_cfg(w, level))
    for n in range(1, warmup + 1):
        s.sweep(n)
    bar.wait()  # every process starts its timed sweeps together
    for n in range(warmup + 1, warmup + sweeps + 1):
        s.sweep(n)
    q.put(1)


def sample_level(w):
    """The reference sample of a workload.  3D regular: the 243^3 tree with the
    workload's operator (for cfg5 that is its own FMG stage 5; the reference's
    per-DoF rate does not depend on the size: 4.0e5 at 81^3, 4.2e5 at
    243^3, while 729^3 needs ~130 GB and ~15 min per sweep on one core).  2D and
    the adaptive tree: the workload itself (levels <= 7) or its base 3."""
    if w.get("sphere_levels"):
        return 3
    if w["dim"] == 3:
        return min(w["level"], 5)
    return min(w["level"], 7)


def host_ram_gb():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except (ValueError, OSError):
        return 16.0


def reference_sample(w, sweeps, warmup, procs):
    """`procs` concurrent single-threaded reference processes (the reference has
    no intra-solve parallelism), each `warmup` untimed + `sweeps` timed cycles of
    the sample; value = all timed DoF-updates / wall time of the timed region
    (from the barrier all processes pass after their warm-up to the last finish)."""
    level = sample_level(w)
    dof = (3 ** level - 1) ** w["dim"]
    if w.get("sphere_levels"):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import refdriver as R
        s = R.RefSession(dict(problem="helmholtz-sin", dim=w["dim"], level=level,
                              sphere_levels=w["sphere_levels"], max_vertices=10 ** 9))
        dof = s.interior_count()
        s.close()
    # ~350 B of reference RSS per DoF (4.87 GB at 243^3)
    procs = max(1, min(procs, int(0.7 * host_ram_gb() / max(350e-9 * dof, 1e-3))))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    bar = ctx.Barrier(procs + 1)
    ps = [ctx.Process(target=_ref_worker, args=((w, level, sweeps, warmup, bar, q),)) for _ in range(procs)]
    for p in ps:
        p.start()
    bar.wait()
    t0 = time.perf_counter()
    for _ in ps:
        q.get()
    wall = time.perf_counter() - t0
    for p in ps:
        p.join()
    value = procs * dof * sweeps / wall
    cells = f"{3 ** level}^{w['dim']}"
    what = (f"the level-{level} + {w['sphere_levels']} sphere-refined tree ({dof} leaf DoF)"
            if w.get("sphere_levels") else
            f"the {cells} tree ({dof} DoF) with the workload's operator" +
            ("" if level == w["level"] else f" (the workload is {3 ** w['level']}^{w['dim']}; {cells} is "
                                              f"{'its FMG stage ' + str(level) if w['dim'] == 3 else 'a sub-problem'})"))
    sample = (f"{procs} concurrent single-threaded reference processes (oracle/_ref, unmodified reference sources), "
              f"each {warmup} untimed + {sweeps} timed td cycles on {what}; value = {procs * sweeps} timed cycles x "
              f"DoF / wall time of the timed region")
    return value, wall / sweeps, sample, procs


def level_for_h(h):  # runner.cpp:165-174
    level, m = 0, 1.0
    while m > h * (1.0 + 1e-12) and level < 12:
        m /= 3.0
        level += 1
    return level


def dyn_cfg(w, sweeps):
    k = w["k"]
    return dict(problem="helmholtz-sin", dim=w["dim"], phi=f"{k * k},{0.5 * k * k}", h_max=w["h_max"],
                h_min=w["h_min"], cycle=w["cycle"], omega=w["omega"], omega_s=w["omega_s"], max_sweeps=sweeps,
                target_drop=1e-300)


def dyn_reference_sample(w, sweeps):
    """The reference's own adaptive run (one core), the first `sweeps` sweeps:
    DoF-updates/s over them (touch-last updates of unrefined interior vertices)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refdriver as R
    s = R.RefSession(dyn_cfg(w, sweeps))
    upd, t = 0.0, 0.0
    for n in range(1, sweeps + 1):
        t0 = time.perf_counter()
        out = s.sweep(n)  # sweep + mark, as the runner does
        t += time.perf_counter() - t0
        upd += out[3]
    sample = (f"the reference's adaptive run (oracle/_ref, one core), sweeps 1..{sweeps} of the same configuration "
              f"incl. mark() after each; {int(upd)} updates")
    return upd / t, t / sweeps, sample


def run_reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if w.get("dynamic"):
        value, sec, sample = dyn_reference_sample(w, min(args.steps, 16))
        print(json.dumps({
            "metric": "complex DoF-updates/s per additive MG cycle", "value": value, "unit": "DoF-updates/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": min(args.steps, 16), "warmup": 0,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "complex128 (f64)", "data": "synthetic (analytic sin rhs)",
            "config": workload_config(args.workload, w), "precision": "reference",
            "cpu_baseline": {"value": value, "unit": "DoF-updates/s", "cores": 1, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return 0
    procs = max(1, min(os.cpu_count() or 1, 64))
    try:
        import refdriver  # noqa: F401
    except Exception:
        pass
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libtreemg_ref.so")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtreemg_ref.so not built"}))
        return 0
    # every process the same number of timed cycles: the K steps spread over the cores
    sweeps = max(1, -(-args.steps // procs))
    value, sec_per_cycle, sample, procs = reference_sample(w, sweeps, 1, procs)
    line = {
        "metric": "complex DoF-updates/s per additive MG cycle", "value": value, "unit": "DoF-updates/s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": interior(w) / value * 1e3 if not w.get("sphere_levels") else sec_per_cycle * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "complex128 (f64)", "data": "synthetic (seeded uniform complex rhs, SURVEY §8d)",
        "config": workload_config(args.workload, w), "precision": "reference (bit-exact complex128)",
        "cpu_baseline": {"value": value, "unit": "DoF-updates/s", "cores": procs, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------
def run_amr(args, w):
    """cfg4: the static adaptive tree, one GPU (replicas for N > 1).  precision
    fast (default): the regular vertices' residual as the assembled stencil in
    FMAs; exact: every iterate bit-identical to the reference."""
    from paper_1508_03954_b200 import dist as D
    import paper_1508_03954_b200 as T
    ctx = D.init()
    k = w["k"]
    prec = "exact" if args.precision == "exact" else "fast"
    h = T.Hierarchy(w["dim"], w["level"], phi=complex(k * k, 0.5 * k * k), chi="seeded", rhs_seed=RHS_SEED,
                    rhs_sphere=True, precision=prec, max_vertices=10 ** 10, device=ctx.local,
                    sphere_levels=w["sphere_levels"])
    pol = T.Policy(kind=w["omega"], omega_s=w["omega_s"])
    settle(h, pol, D, ctx)
    h.time_cycles(pol, 1, args.warmup)
    D.barrier(ctx)
    with ClockSampler(ctx.local) as clk:
        out = h.time_cycles(pol, args.warmup + 1, args.steps)
    D.barrier(ctx)
    total_ms = D.reduce_max(ctx, float(out[0]))
    dof = h.leaf_vertices
    value = ctx.world * dof * args.steps / (total_ms / 1e3)
    existing = sum(int(((h.flags(l)[0] & 1) == 1).sum()) for l in range(w["level"] + w["sphere_levels"] + 1))
    B = 176 * existing
    peak, peak_kind = peaks()
    achieved = B / (total_ms / args.steps / 1e3) / 1e9
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        v, _, sample, _ = reference_sample(w, 3, 1, 1)
        cpu = {"value": v, "unit": "DoF-updates/s", "cores": 1, "kind": "reference", "sample": sample}
    # e2e through the public C-ABI: treemg_run of the same configuration (setup + cycles + norms to the host)
    t0 = time.perf_counter()
    r = T.run(dict(problem="helmholtz-sin", dim=w["dim"], level=w["level"], sphere_levels=w["sphere_levels"],
                   phi=f"{k * k},{0.5 * k * k}", omega=w["omega"], omega_s=w["omega_s"], rhs="seeded",
                   rhs_seed=RHS_SEED, rhs_mask="sphere", max_sweeps=args.steps, target_drop=1e-300,
                   max_vertices=10 ** 10, device=ctx.local, precision=prec))
    e2e_s = time.perf_counter() - t0
    if ctx.rank == 0:
        line = {
            "metric": "complex DoF-updates/s per additive MG cycle", "value": value, "unit": "DoF-updates/s",
            "n_gpus": ctx.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
            "data": "synthetic (seeded uniform complex rhs in the ball, SURVEY §8d)",
            "config": {"workload": args.workload, "desc": w["desc"], "leaf_dof": dof,
                       "hanging_vertices": h.hanging_vertices, "existing_vertices": existing,
                       "precision": prec, "parallelism": f"replicas x{ctx.world}" if ctx.world > 1 else "single GPU",
                       "l2": "level-6 box arrays of 0.4 GB each (> L2); no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "peak_kind": peak_kind,
                         "kernel": f"whole {prec} adaptive cycle (k_amr_topdown/chi/residual per level), 176 B per "
                                   "existing vertex" + ("; FP64-issue bound (element-by-element, reference order)"
                                                        if prec == "exact" else
                                                        "; regular vertices' residual as the assembled stencil (FMA)")},
            "cpu_baseline": cpu,
            "e2e": {"value": ctx.world * dof * r.sweeps / e2e_s, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 48, "note": f"treemg_run of {r.sweeps} cycles incl. tree setup "
                    f"(host classification + flag upload) and per-cycle norm readback, wall clock"},
            "clocks": clk.summary(), "gpu_launches": int(out[3]) * args.steps,
        }
        print(json.dumps(line))
    D.finalize(ctx)
    return 0


def run_dyn(args, w):
    """Dynamic adaptivity: K sweeps of the adaptive run from its start grid (mark
    after each), exact precision; replicas for N > 1.  The step includes the
    host replay of the traversal's structural edits (dyn.hpp) -- it is part of
    the algorithm -- so the step is wall-clock timed (each sweep ends in a
    synchronising norm read-back); the device share is reported beside it."""
    from paper_1508_03954_b200 import dist as D
    import paper_1508_03954_b200 as T
    ctx = D.init()
    k = w["k"]
    hkw = dict(dim=w["dim"], levels=1, phi=complex(k * k, 0.5 * k * k), chi="sin", precision="exact",
               h_max=w["h_max"], h_min=w["h_min"], device=ctx.local)
    pol = T.Policy(kind=w["omega"], omega_s=w["omega_s"])
    warm = T.Hierarchy(**hkw)  # warm-up: context, module load, first sweeps
    for n in range(1, args.warmup + 1):
        warm.td_add(pol, n)
        warm.mark()
    warm.close()
    h = T.Hierarchy(**hkw)
    D.barrier(ctx)
    updates, existing = 0, 0
    with ClockSampler(ctx.local) as clk:
        t0 = time.perf_counter()
        for n in range(1, args.steps + 1):
            st = h.td_add(pol, n)
            updates += st.updated_fine_vertices
            existing += h.existing_vertices  # after the sweep's edits
            h.mark()
        wall = time.perf_counter() - t0
    D.barrier(ctx)
    wall = D.reduce_max(ctx, wall)
    phases = h.dyn_phase_ms()
    value = ctx.world * updates / wall
    peak, peak_kind = peaks()
    achieved = 176 * existing / (phases["device"] / 1e3) / 1e9
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        v, _, sample = dyn_reference_sample(w, min(args.steps, 16))
        cpu = {"value": v, "unit": "DoF-updates/s", "cores": 1, "kind": "reference", "sample": sample}
    t0 = time.perf_counter()
    r = T.run(dict(dyn_cfg(w, args.steps), device=ctx.local))
    e2e_s = time.perf_counter() - t0
    if ctx.rank == 0:
        print(json.dumps({
            "metric": "complex DoF-updates/s per additive MG cycle", "value": value, "unit": "DoF-updates/s",
            "n_gpus": ctx.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
            "data": "synthetic (analytic sin rhs)",
            "config": {"workload": args.workload, "desc": w["desc"], "updates": updates, "depth": h.depth(),
                       "final_leaf_dof": h.leaf_vertices, "precision": "exact",
                       "phase_ms": {k2: round(v2, 2) for k2, v2 in phases.items() if k2 != "launches"},
                       "parallelism": f"replicas x{ctx.world}" if ctx.world > 1 else "single GPU",
                       "l2": "state of 4.8M-point level-7 lattices (> L2); no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "peak_kind": peak_kind,
                         "kernel": "device share of the sweeps (k_amr_topdown/chi/residual/k_dyn_special per level), "
                                   "176 B per stored vertex; the step is bound by the host replay and table "
                                   "transfers (phase_ms), not by the device"},
            "cpu_baseline": cpu,
            "e2e": {"value": ctx.world * r.work_units * (3 ** level_for_h(w["h_min"]) - 1) ** w["dim"] / e2e_s,
                    "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 24 + 72,
                    "note": f"treemg_run of {r.sweeps} sweeps incl. setup, host replay, marks and per-sweep norm / "
                            f"mark-statistics read-back, wall clock"},
            "clocks": clk.summary(), "gpu_launches": int(phases["launches"]),
        }))
    h.close()
    D.finalize(ctx)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=list(WORKLOADS))
    ap.add_argument("--precision", default=os.environ.get("TMG_PRECISION", "fast"),
                    choices=["fast", "exact", "fast-complex64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="developer A/B: skip the end-to-end leg")
    ap.add_argument("--mode", default=None, choices=["single", "slabs", "replicas"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference_arm(args, w)

    if w.get("sphere_levels"):
        return run_amr(args, w)
    if w.get("dynamic"):
        return run_dyn(args, w)

    from paper_1508_03954_b200 import dist as D
    ctx = D.init()
    world, rank, local, dist = ctx.world, ctx.rank, ctx.local, ctx.dist

    import numpy as np
    import paper_1508_03954_b200 as T

    k = w["k"]
    phi = complex(k * k, 0.5 * k * k)
    mode = args.mode or ("slabs" if (world > 1 and w["dim"] == 3 and args.precision == "fast") else
                         ("replicas" if world > 1 else "single"))
    pol = T.Policy(kind=w["omega"], omega_s=w["omega_s"], bpx=(w["cycle"] == "td-bpx"))
    if mode == "slabs":
        uid = D.broadcast_bytes(ctx, T.nccl_unique_id() if rank == 0 else None)
        h = T.Slabs(w["level"], phi, chi="seeded", rhs_seed=RHS_SEED, rank=rank, world=world, nccl_id=uid,
                    device=local)
        settle(h, pol, D, ctx)
        h.time_cycles(pol, 1, args.warmup)
    else:
        h = T.Hierarchy(w["dim"], w["level"], phi=phi, chi="seeded", rhs_seed=RHS_SEED, precision=args.precision,
                        max_vertices=10 ** 10, device=local)
        # warm-up cycles (untimed), then K timed cycles with CUDA events on the library stream
        settle(h, pol, D, ctx, flush_l2=False)
        h.time_cycles(pol, 1, args.warmup, flush_l2=False)

    def barrier():
        D.barrier(ctx)

    barrier()
    with ClockSampler(local) as clk:
        if mode == "slabs":
            out = h.time_cycles(pol, args.warmup + 1, args.steps)
        else:
            out = h.time_cycles(pol, args.warmup + 1, args.steps, flush_l2=False)
    barrier()
    total_ms, fine_ms, launches_per_cycle = float(out[0]), float(out[1]), int(out[3])
    total_ms = D.reduce_max(ctx, total_ms)
    dof = interior(w)
    ms_per_step = total_ms / args.steps
    copies = 1 if mode == "slabs" else world
    value = copies * dof * args.steps / (total_ms / 1e3)
    B_total, B_fine = algorithmic_bytes(w, args.precision)
    if mode == "slabs":  # this rank's share of the fine level
        z0, z1 = h.owned_planes()
        B_fine = fine_bytes_per_vertex(w, args.precision) * (z1 - z0) * (3 ** w["level"] + 1) ** 2
        B_total = B_total * (z1 - z0) / (3 ** w["level"] - 1)
        launches_per_cycle = int(out[3]) or (2 * w["level"] + 6)
    peak, peak_kind = peaks()
    achieved = B_fine / (fine_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "kernel": fine_kernel_label(w, args.precision) +
                f", {B_fine / 1e9:.2f} GB algorithmic per cycle "
                f"({fine_bytes_per_vertex(w, args.precision)} B per fine vertex)",
                "peak_kind": peak_kind, "whole_cycle_GBps": B_total / (ms_per_step / 1e3) / 1e9}

    moved = moved_bytes_per_vertex(w, args.precision)
    roofline["basis"] = (f"SURVEY §8(d) algorithmic bytes: {fine_bytes_per_vertex(w, args.precision)} B per fine "
                         f"lattice vertex x {B_fine // fine_bytes_per_vertex(w, args.precision)} vertices per launch")
    roofline["frac_moved_basis"] = roofline["frac"] * moved / fine_bytes_per_vertex(w, args.precision)
    roofline["moved_bytes_per_vertex"] = moved
    tr = ncu_traffic(args.workload, args.precision, mode) if mode != "slabs" or world == 1 else None
    if tr:
        roofline["traffic"] = tr["bytes_per_launch"]
        roofline["traffic_source"] = tr["source"]
        # the kernel's actual DRAM bytes (ncu) over its live event-timed duration
        roofline["frac_dram_actual"] = tr["bytes_per_launch"] / (fine_ms / 1e3) / 1e9 / peak

    e2e = None
    if not args.no_e2e:  # developer A/B runs skip the end-to-end leg
        # e2e through the boundary: host rhs (pinned) -> device -> one cycle -> host norms
        n_lat = lattice(w["level"], w["dim"])
        try:
            import torch
            chi_host = torch.empty(2 * n_lat, dtype=torch.float64, pin_memory=True).numpy()
        except Exception:
            chi_host = np.empty(2 * n_lat)
        rng = np.random.default_rng(RHS_SEED)
        chi_host[:] = rng.uniform(-1, 1, size=2 * n_lat)
        h2d = 16 * n_lat
        n0 = args.warmup + args.steps + 1
        one = (lambda n: h.cycle(pol, n)) if mode == "slabs" else (h.td_bpx if pol.bpx else h.td_add)
        if mode != "slabs":
            one = (lambda f: (lambda n: f(pol, n)))(one)
        # (a) a solve through the public API: the step's input (the rhs) uploaded
        #     from pinned host memory once, then K cycles, each returning its norms
        barrier()
        t0 = time.perf_counter()
        if mode == "slabs":
            _, h2d = h.e2e_step(pol, n0, chi_host)
        else:
            h.e2e_step(pol, n0, chi_host)
        for i in range(1, args.steps):
            one(n0 + i)
        solve_s = D.reduce_max(ctx, time.perf_counter() - t0)
        # (b) the pessimistic variant: a fresh rhs uploaded before every cycle
        reps = max(2, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for i in range(reps):
            h.e2e_step(pol, n0 + args.steps + i, chi_host)
        every_s = D.reduce_max(ctx, (time.perf_counter() - t0) / reps)
        # (c) the reference's own entry point: treemg_run of the workload's configuration
        #     (seeded rhs generated on the device, hierarchy setup, K cycles with the
        #     per-cycle norm readback, result to the host), wall clock incl. setup
        api = None
        if mode == "single" and args.precision != "fast-complex64":
            h.close()  # the timed hierarchy is done with: treemg_run allocates its own
            cfg = dict(problem="helmholtz-sin", dim=w["dim"], level=w["level"], phi=f"{phi.real},{phi.imag}",
                       cycle=w["cycle"], omega=w["omega"], omega_s=w["omega_s"], rhs="seeded", rhs_seed=RHS_SEED,
                       max_sweeps=args.steps, target_drop=1e-300, precision=args.precision,
                       max_vertices=10 ** 11, device=local)
            t0 = time.perf_counter()
            r = T.run(cfg)
            api_s = time.perf_counter() - t0
            api = {"value": dof * r.sweeps / api_s, "unit": "DoF-updates/s", "sweeps": r.sweeps,
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 24,
                   "note": "treemg_run (the reference's C-ABI entry point) of the workload's configuration: "
                           "hierarchy setup, seeded rhs and load vector built on the device, K cycles each reading "
                           "its norms back, wall clock including setup"}
        e2e = {"value": copies * dof * args.steps / solve_s, "unit": "DoF-updates/s",
               "h2d_bytes_per_step": int(h2d) // max(1, args.steps), "d2h_bytes_per_step": 24,
               "note": f"public-API solve of K={args.steps} cycles (wall clock, max over ranks): H2D of the nodal rhs "
                       "(16 B/vertex from pinned memory; slabs: the rank's planes) and the device load vector once, "
                       "then every cycle with D2H of its three residual norms",
               "rhs_every_cycle": {"value": copies * dof / every_s, "h2d_bytes_per_step": int(h2d),
                                   "note": "a fresh rhs uploaded before each cycle (PCIe-bound)"}}
        if api:
            e2e["treemg_run"] = api

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # one cycle of the 243^3 sample (~35 s of CPU work; 3D) without warm-up
            v, sps, sample, _ = reference_sample(w, 1, 0, 1)
            cpu = {"value": v, "unit": "DoF-updates/s", "cores": 1, "kind": "reference", "sample": sample}
        except Exception as exc:  # reported, never silently replaced
            cpu = {"value": None, "unit": "DoF-updates/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": "complex DoF-updates/s per additive MG cycle", "value": value, "unit": "DoF-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if mode == "slabs" else "weak", "vs_baseline": None,
            "dtype": "complex64 (f32)" if args.precision == "fast-complex64" else "complex128 (f64)",
            "data": "synthetic (seeded uniform complex rhs, SURVEY §8d)",
            "config": workload_config(args.workload, w), "precision": args.precision,
            "parallelism": {"slabs": f"z-slabs x{world} (NCCL)", "replicas": f"replicas x{world}",
                            "single": "single GPU"}[mode],
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": launches_per_cycle * args.steps, "fine_pass_ms": fine_ms,
        }
        print(json.dumps(line))
    D.finalize(ctx)
    return 0


if __name__ == "__main__":
    sys.exit(main())
