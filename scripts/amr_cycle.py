"""Minimal cfg4 driver for ncu: build the adaptive hierarchy, run a few exact cycles."""
import sys
sys.path.insert(0, ".")
import paper_1508_03954_b200 as T
base, k, cycles = 4, 2, int(sys.argv[1]) if len(sys.argv) > 1 else 2
prec = sys.argv[2] if len(sys.argv) > 2 else "exact"
h = T.Hierarchy(3, base, phi=1600 + 800j, chi="seeded", rhs_seed=12345, rhs_sphere=True, precision=prec,
                max_vertices=10 ** 10, sphere_levels=k)
pol = T.Policy(kind="exponential", omega_s=0.6)
for n in range(1, cycles + 1):
    st = h.td_add(pol, n)
print("ok", st)
