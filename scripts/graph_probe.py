"""Per-cycle wall time of public-API cycles (td_add with norms readback) after a
back-to-back time_cycles run, CUDA graph on / off (TMG_GRAPH)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1508_03954_b200 as T
dim, level, k = (2, 5, 10) if len(sys.argv) < 2 else tuple(int(x) for x in sys.argv[1:4])
h = T.Hierarchy(dim, level, phi=complex(k * k, 0.5 * k * k), chi="seeded", precision="fast", max_vertices=10**10)
pol = T.Policy("exponential", 0.6)
out = h.time_cycles(pol, 1, 3)
out = h.time_cycles(pol, 4, 20)
print("time_cycles us/cycle", out[0] / 20 * 1e3)
ts = []
for n in range(24, 54):
    t0 = time.perf_counter()
    h.td_add(pol, n)
    ts.append((time.perf_counter() - t0) * 1e6)
print(os.environ.get("TMG_GRAPH", "1"), " ".join(f"{t:.0f}" for t in ts))
import numpy as np
n_lat = (3 ** level + 1) ** dim
chi = np.random.default_rng(1).uniform(-1, 1, size=2 * n_lat)
for rep in range(4):
    t0 = time.perf_counter()
    h.e2e_step(pol, 100 + 40 * rep, chi)
    for i in range(1, 20):
        h.td_add(pol, 100 + 40 * rep + i)
    print("e2e solve us", round((time.perf_counter() - t0) * 1e6))
