"""cfg5 as BASELINE states it on one GPU: FMG unfolding 3 -> 6 with additive
cycles to a relative residual drop of 1e-8 per level, through treemg_run."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1508_03954_b200 as T
prec = sys.argv[1] if len(sys.argv) > 1 else "fast"
T.lib()
cfg = dict(problem="helmholtz-sin", dim=3, level=6, fmg_from=3, phi="6400,3200", omega="exponential", omega_s=0.6,
           rhs="seeded", rhs_seed=12345, target_drop=1e-8, max_sweeps=400, precision=prec, max_vertices=10 ** 11)
t0 = time.perf_counter()
r = T.run(cfg)
dt = time.perf_counter() - t0
print(f"{prec}: outcome {r.outcome}, sweeps {r.sweeps}, wall {dt:.3f} s, first {r.history[0][5]:.3e} final {r.history[-1][5]:.3e}")
import numpy as np
h = np.array(r.history)
print("vertex counts per stage:", sorted(set(int(v) for v in h[:, 2])))
