"""Wall time of the cfg4 adaptive hierarchy construction (tree build, classification, uploads, chi lists)."""
import sys, time
sys.path.insert(0, ".")
import paper_1508_03954_b200 as T
for rep in range(2):
    t0 = time.perf_counter()
    h = T.Hierarchy(3, 4, phi=1600 + 800j, chi="seeded", rhs_seed=12345, rhs_sphere=True, precision="exact",
                    max_vertices=10 ** 10, sphere_levels=2)
    t1 = time.perf_counter()
    st = h.td_add(T.Policy(kind="exponential", omega_s=0.6), 1)
    t2 = time.perf_counter()
    print(f"setup {t1 - t0:.3f} s, first cycle {1e3 * (t2 - t1):.1f} ms")
    del h
