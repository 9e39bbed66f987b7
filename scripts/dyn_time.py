"""Wall clock of a dynamic-adaptivity run through treemg_run (the reference's
57 s CPU configuration: 2D helmholtz-sin, h_max 0.04 -> h_min 0.001, 30 sweeps)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1508_03954_b200 as T

cfg = dict(problem="helmholtz-sin", dim=2, phi="100,50", h_max=0.04, h_min=0.001, max_sweeps=30, target_drop=1e-8,
           omega="undamped", omega_s=0.6, precision="exact")
T.run(dict(cfg, max_sweeps=3))  # warm-up (context, module load)
for rep in range(2):
    t0 = time.perf_counter()
    r = T.run(cfg, out_prefix="gpurun_out/dyn_time")
    t1 = time.perf_counter()
    print(f"run {rep}: {t1 - t0:.3f} s, {r.sweeps} sweeps, vertices {r.vertex_count}, final h {r.final_norm['h']:.6g}, "
          f"work units {r.work_units:.5f}", flush=True)
