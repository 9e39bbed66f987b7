"""cfg4 (static sphere 4 -> 6) on the GPU: setup time, ms per exact cycle, and
the first cycles' norms (compare with tests/golden/cfg4.json)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1508_03954_b200 as T

base, k = int(sys.argv[1]) if len(sys.argv) > 1 else 4, int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.time()
h = T.Hierarchy(3, base, phi=1600 + 800j, chi="seeded", rhs_seed=12345, rhs_sphere=True, precision="exact",
                max_vertices=10 ** 10, sphere_levels=k)
t1 = time.time()
print(f"setup {t1 - t0:.2f}s leaf {h.leaf_vertices} hanging {h.hanging_vertices}", flush=True)
pol = T.Policy(kind="exponential", omega_s=0.6, hb=True)
for n in range(1, 4):
    st = h.td_add(pol, n)
    print(n, st.max_norm, st.euclid_norm, st.h_norm, st.updated_fine_vertices, flush=True)
out = h.time_cycles(pol, 4, 5)
print(f"ms/cycle {out[0] / 5:.3f}  DoF/s {h.leaf_vertices * 5 / (out[0] / 1e3):.3e}")
