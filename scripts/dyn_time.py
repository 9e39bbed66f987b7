"""Wall clock of a dynamic-adaptivity run through treemg_run (the reference's
57 s CPU configuration: 2D helmholtz-sin, h_max 0.04 -> h_min 0.001, 30 sweeps),
plus the Hierarchy-API breakdown (setup, sweeps, marks)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1508_03954_b200 as T

cfg = dict(problem="helmholtz-sin", dim=2, phi="100,50", h_max=0.04, h_min=0.001, max_sweeps=30, target_drop=1e-8,
           omega="undamped", omega_s=0.6, precision="exact")
T.run(dict(cfg, max_sweeps=3))  # warm-up (context, module load)
for rep in range(2):
    t0 = time.perf_counter()
    r = T.run(cfg, out_prefix="gpurun_out/dyn_time" if rep else None)
    t1 = time.perf_counter()
    print(f"run {rep} ({'with' if rep else 'no'} artefacts): {t1 - t0:.3f} s, {r.sweeps} sweeps, vertices "
          f"{r.vertex_count}, final h {r.final_norm['h']:.6g}", flush=True)
t0 = time.perf_counter()
h = T.Hierarchy(2, 1, phi=100 + 50j, chi="sin", precision="exact", h_max=0.04, h_min=0.001)
t1 = time.perf_counter()
pol = T.Policy(kind="undamped", omega_s=0.6)
ts = tm = 0.0
for n in range(1, 31):
    a = time.perf_counter(); h.td_add(pol, n); b = time.perf_counter(); h.mark(); c = time.perf_counter()
    ts += b - a; tm += c - b
print(f"setup {t1 - t0:.3f} s, sweeps {ts:.3f} s, marks {tm:.3f} s, phases {h.dyn_phase_ms()}")
