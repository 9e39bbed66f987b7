"""Generates the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref, built from
/root/reference/proj by oracle/Makefile) through the oracle harness
(oracle/refdriver.cpp) and records, per configuration:
  * the per-sweep CSV exactly as the reference runner writes it
    (runner.cpp:318-329, %.17g),
  * outcome / sweep count / first and final norm,
  * FNV-1a hashes of the finest-level u and sc bit patterns (sign of zero
    folded), which pin the iterates bit-for-bit at any size,
  * the reference's per-sweep wall time on this host (planning only; the
    CPU baseline proper is measured on the GPU box by bench.py).

Usage:  python tests/golden/make_goldens.py <name> [<name> ...]
Names:  see CONFIGS.  Only runnable where /root/reference exists.
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

SEEDED = dict(rhs="seeded", rhs_seed=12345, theta_deg=0, ell_min=1, norm="h")

# BASELINE.json configs (SURVEY §8d mapping) plus the reference's own
# test_runner / test_capi / cli_smoke runs.
CONFIGS = {
    # cfg1: 2D depth 5, k=10 -> phi = k^2(1+0.5i), exponential omega 0.6, 20 cycles
    "cfg1": dict(problem="helmholtz-sin", dim=2, level=5, phi="100,50", cycle="td-add", omega="exponential",
                 omega_s=0.6, max_sweeps=20, target_drop=1e-30, **SEEDED),
    # cfg2: 2D depth 7, k=100, BPX undamped 0.5, to 1e-8 or 200 cycles
    "cfg2": dict(problem="helmholtz-sin", dim=2, level=7, phi="10000,5000", cycle="td-bpx", omega="undamped",
                 omega_s=0.5, max_sweeps=200, target_drop=1e-8, **SEEDED),
    # cfg3: 3D depth 5, k=20, exponential 0.6, 50 cycles (vertex cap raised)
    "cfg3": dict(problem="helmholtz-sin", dim=3, level=5, phi="400,200", cycle="td-add", omega="exponential",
                 omega_s=0.6, max_sweeps=50, target_drop=1e-30, max_vertices=40000000, **SEEDED),
    # the headline workload itself (cfg5's final level, 729^3, k=80): the first 2 cycles (about 130 GB of host
    # RAM and ~15 min per sweep on one core -- generated on the GPU host, tests/golden/make_head_golden.sh)
    "cfg5_l6_head": dict(problem="helmholtz-sin", dim=3, level=6, phi="6400,3200", cycle="td-add",
                         omega="exponential", omega_s=0.6, max_sweeps=2, target_drop=1e-30, max_vertices=500000000,
                         **SEEDED),
    # cfg3 operator at 81^3 (fast to regenerate; used by the CPU suite's oracle pin)
    "cfg3_l4": dict(problem="helmholtz-sin", dim=3, level=4, phi="400,200", cycle="td-add", omega="exponential",
                    omega_s=0.6, max_sweeps=12, target_drop=1e-30, **SEEDED),
    # cfg2 operator at 243^2
    "cfg2_l5": dict(problem="helmholtz-sin", dim=2, level=5, phi="10000,5000", cycle="td-bpx", omega="undamped",
                    omega_s=0.5, max_sweeps=60, target_drop=1e-8, **SEEDED),
    # a converging seeded 2D case (k=10 undamped)
    "conv2d": dict(problem="helmholtz-sin", dim=2, level=5, phi="100,50", cycle="td-add", omega="undamped",
                   omega_s=0.6, max_sweeps=120, target_drop=1e-8, **SEEDED),
    # cfg4 schedule on a regular grid: hb for 5 sweeps then additive
    "hb_then_add": dict(problem="helmholtz-sin", dim=3, level=3, phi="1600,800", cycle="td-add",
                        omega="exponential", omega_s=0.6, max_sweeps=12, target_drop=1e-30, hb_sweeps=5,
                        rhs_mask="sphere", **SEEDED),
    # reference tests: cli_smoke (tests/data/poisson_smoke.cfg), test_runner.cpp:472-505, test_capi.cpp:8-28
    "poisson_smoke": dict(problem="poisson-sin", dim=2, cycle="td-add", omega="exponential", omega_s=0.8,
                          level=2, max_sweeps=60, target_drop=1e-6, norm="h"),
    "runner_poisson_l3": dict(problem="poisson-sin", dim=2, level=3, omega="exponential", max_sweeps=80),
    "runner_helmholtz_diverges": dict(problem="helmholtz-sin", phi="2025", dim=2, level=3, theta_deg=0,
                                      max_sweeps=300),
    "runner_budget_one": dict(problem="poisson-sin", dim=2, level=2, max_sweeps=1, target_drop=1e-30),
    "capi_poisson_l2": dict(problem="poisson-sin", dim=2, level=2, max_sweeps=60),
    # BASELINE cfg5 exactly as specified (FMG 3 -> 6, k = 80, to a drop of 1e-8 per level): the reference
    # diverges in its first (27^3) stage, so the golden is cheap
    "cfg5": dict(problem="helmholtz-sin", dim=3, level=6, fmg_from=3, phi="6400,3200", cycle="td-add",
                 omega="exponential", omega_s=0.6, max_sweeps=400, target_drop=1e-8, max_vertices=1000000000,
                 **SEEDED),
    # cfg5 schedule (FMG unfolding) at reduced depth: 3D 2 -> 4 with the cfg5 operator, and converging variants
    "fmg3d_cfg5op": dict(problem="helmholtz-sin", dim=3, level=4, fmg_from=2, phi="6400,3200", cycle="td-add",
                         omega="exponential", omega_s=0.6, max_sweeps=40, fmg_stage_cap=40, target_drop=1e-8,
                         **SEEDED),
    "fmg3d_k20": dict(problem="helmholtz-sin", dim=3, level=4, fmg_from=2, phi="400,200", cycle="td-add",
                      omega="undamped", omega_s=0.6, max_sweeps=60, fmg_stage_cap=60, target_drop=1e-6, **SEEDED),
    "fmg3d_poisson": dict(problem="poisson-sin", dim=3, level=4, fmg_from=2, cycle="td-add", omega="exponential",
                          omega_s=0.8, max_sweeps=60, fmg_stage_cap=60, target_drop=1e-6, norm="h"),
    "fmg3d_seeded_k3": dict(problem="helmholtz-sin", dim=3, level=4, fmg_from=2, phi="9,4.5", cycle="td-add",
                            omega="undamped", omega_s=0.6, max_sweeps=60, fmg_stage_cap=60, target_drop=1e-6,
                            **SEEDED),
    "fmg2d_k10": dict(problem="helmholtz-sin", dim=2, level=5, fmg_from=2, phi="100,50", cycle="td-add",
                      omega="undamped", omega_s=0.6, max_sweeps=80, fmg_stage_cap=80, target_drop=1e-8, **SEEDED),
    "fmg2d_bpx": dict(problem="helmholtz-sin", dim=2, level=4, fmg_from=2, phi="100,50", cycle="td-bpx",
                      omega="undamped", omega_s=0.5, max_sweeps=50, fmg_stage_cap=50, target_drop=1e-6, **SEEDED),
    # cfg4: static sphere refinement 4 -> 6, f masked to the ball, hb for 25 cycles then additive (SURVEY §8d pin)
    "cfg4": dict(problem="helmholtz-sin", dim=3, level=4, sphere_levels=2, phi="1600,800", cycle="td-add",
                 omega="exponential", omega_s=0.6, hb_sweeps=25, rhs_mask="sphere", max_sweeps=50,
                 target_drop=1e-30, max_vertices=100000000, **SEEDED),
    # cfg4 at reduced depth (2 -> 4, SURVEY §7.3 item 5 probe size) and 2D adaptive variants
    "cfg4_small": dict(problem="helmholtz-sin", dim=3, level=2, sphere_levels=2, phi="1600,800", cycle="td-add",
                       omega="exponential", omega_s=0.6, hb_sweeps=10, rhs_mask="sphere", max_sweeps=20,
                       target_drop=1e-30, **SEEDED),
    "amr2d_conv": dict(problem="helmholtz-sin", dim=2, level=3, sphere_levels=2, phi="100,50", cycle="td-add",
                       omega="undamped", omega_s=0.6, max_sweeps=150, target_drop=1e-8, **SEEDED),
    "amr2d_bpx": dict(problem="helmholtz-sin", dim=2, level=2, sphere_levels=3, phi="100,50", cycle="td-bpx",
                      omega="undamped", omega_s=0.5, max_sweeps=40, target_drop=1e-8, **SEEDED),
    # verification cycles: bottom-up FAS and textbook additive, regular trees
    "vc_bufas_2d": dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50", cycle="bu-fas", omega="exponential",
                        omega_s=0.6, max_sweeps=40, target_drop=1e-8, **SEEDED),
    "vc_bufas_3d_poisson": dict(problem="poisson-sin", dim=3, level=3, cycle="bu-fas", omega="undamped",
                                omega_s=0.8, max_sweeps=30, target_drop=1e-8, norm="h"),
    "vc_textbook_2d": dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50", cycle="textbook", omega_s=0.6,
                           max_sweeps=40, target_drop=1e-8, **SEEDED),
    "vc_textbook_3d_cg": dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", cycle="textbook", omega_s=0.6,
                              omega_cg=0.9, max_sweeps=25, target_drop=1e-8, **SEEDED),
    # gaussian scenario (problems.cpp:20-24, 78-90): cell-varying phi, absorbing-layer theta, reference omega 0.4
    "gaussian_l3": dict(problem="gaussian", dim=2, level=3, max_sweeps=40, target_drop=1e-8),
    "gaussian_l4_transition": dict(problem="gaussian", dim=2, level=4, theta_deg=25, omega="transition",
                                   max_sweeps=30, target_drop=1e-8),
    "gaussian_l4_bpx": dict(problem="gaussian", dim=2, level=4, cycle="td-bpx", omega="undamped", omega_s=0.3,
                            max_sweeps=30, target_drop=1e-8),
    "rotated_3d_bpx": dict(problem="helmholtz-sin", dim=3, level=3, phi="2025", theta_deg=35, cycle="td-bpx",
                           omega="transition", max_sweeps=15, target_drop=1e-30),
    # several channels: test_runner.cpp:120-155 cases, and coupled / random-start variants
    "mc2_identical": dict(problem="helmholtz-sin", phi="-1000", dim=2, level=2, channels=2, max_sweeps=10,
                          target_drop=1e-30),
    "mc2_coupled_2d": dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50", channels=2, coupling="30,10",
                           cycle="td-add", omega="undamped", omega_s=0.6, max_sweeps=40, target_drop=1e-8,
                           **SEEDED),
    "mc3_coupled_3d_bpx": dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", channels=3,
                               coupling="-20,5", cycle="td-bpx", omega="undamped", omega_s=0.5, max_sweeps=25,
                               target_drop=1e-8, **SEEDED),
    "mc2_random_2d": dict(problem="poisson-sin", dim=2, level=3, channels=2, coupling="4,0", initial="random",
                          seed=7, omega="exponential", omega_s=0.8, max_sweeps=30, target_drop=1e-8, norm="h"),
    # dynamic adaptivity: h_max / h_min runs, marks after every sweep
    "dyn_h2d": dict(problem="helmholtz-sin", dim=2, phi="100,50", h_max=0.04, h_min=0.004, cycle="td-add",
                    omega="undamped", omega_s=0.6, max_sweeps=14, target_drop=1e-8),
    "dyn_p2d_bpx": dict(problem="poisson-sin", dim=2, h_max=0.04, h_min=0.002, cycle="td-bpx", omega="undamped",
                        omega_s=0.5, max_sweeps=12, target_drop=1e-8),
    "dyn_p3d": dict(problem="poisson-sin", dim=3, h_max=0.12, h_min=0.013, cycle="td-add", omega="undamped",
                    omega_s=0.6, max_sweeps=12, target_drop=1e-8),
    "dyn_b2d_seeded": dict(problem="helmholtz-ball", dim=2, h_max=0.12, h_min=0.0014, theta_deg=20,
                           omega="exponential", omega_s=0.8, max_sweeps=12, target_drop=1e-8, rhs="seeded",
                           rhs_seed=99),
    # proj/tests/test_amr.cpp:172-190 (adaptive runs are deterministic)
    "dyn_p2d_transition": dict(problem="poisson-sin", dim=2, cycle="td-add", omega="transition", h_max=1.0 / 9.0,
                               h_min=1.0 / 81.0, max_sweeps=12, target_drop=1e-30),
}


def generate(name: str) -> dict:
    import refdriver as R
    cfg = CONFIGS[name]
    t0 = time.time()
    s = R.RefSession(cfg)
    if s.status != 0:
        raise RuntimeError(s.message)
    build_s = time.time() - t0
    s.run()
    L = s.depth
    secs = s.sweep_seconds()
    rec = dict(
        name=name, config={k: str(v) for k, v in cfg.items()}, outcome=s.outcome(), sweeps=s.sweeps(),
        csv=s.csv(), log=s.log(),
        u_hash=f"{s.field_hash(L, 'u'):016x}", sc_hash=f"{s.field_hash(L, 'sc'):016x}",
        coarse_u_hash=f"{s.field_hash(L - 1, 'u'):016x}" if L >= 1 else "",
        channel_u_hashes=[f"{s.field_hash(L, 'u', c):016x}" for c in range(int(cfg.get("channels", 1)))],
        reference_seconds_per_sweep=float(secs.mean()) if len(secs) else 0.0,
        reference_build_seconds=build_s, host=platform.node(), cpu=platform.processor() or platform.machine(),
        generator="tests/golden/make_goldens.py via oracle/_ref (unmodified reference sources)",
    )
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    return rec


if __name__ == "__main__":
    for n in sys.argv[1:] or [k for k in CONFIGS if k not in ("cfg2", "cfg3", "cfg4", "cfg5_l6_head")]:
        r = generate(n)
        print(n, r["outcome"], r["sweeps"], f"{r['reference_seconds_per_sweep']:.3f}s/sweep", flush=True)
