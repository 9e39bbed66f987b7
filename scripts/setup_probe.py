"""Where treemg_run's setup time goes at 729^3 (cfg5 level): hierarchy construction vs cycles."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1508_03954_b200 as T
level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
k = 80.0
T.lib()
for rep in range(2):
    t0 = time.perf_counter()
    h = T.Hierarchy(3, level, phi=complex(k * k, 0.5 * k * k), chi="seeded", rhs_seed=12345, precision="fast",
                    max_vertices=10 ** 11)
    t1 = time.perf_counter()
    pol = T.Policy("exponential", 0.6)
    h.td_add(pol, 1)
    t2 = time.perf_counter()
    h.close()
    t3 = time.perf_counter()
    print(f"construct {1e3*(t1-t0):.1f} ms, first cycle {1e3*(t2-t1):.1f} ms, close {1e3*(t3-t2):.1f} ms")
for sweeps in (1, 20):
    cfg = dict(problem="helmholtz-sin", dim=3, level=level, phi=f"{k*k},{0.5*k*k}", omega="exponential", omega_s=0.6,
               rhs="seeded", rhs_seed=12345, max_sweeps=sweeps, target_drop=1e-300, precision="fast",
               max_vertices=10 ** 11)
    t0 = time.perf_counter()
    r = T.run(cfg)
    print(f"treemg_run {sweeps} sweeps: {1e3*(time.perf_counter()-t0):.1f} ms")
