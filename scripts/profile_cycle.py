"""Minimal driver for ncu: build one hierarchy, run a few cycles."""
import argparse, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1508_03954_b200 as T
ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=3); ap.add_argument("--level", type=int, default=5)
ap.add_argument("--k", type=float, default=20); ap.add_argument("--precision", default="fast")
ap.add_argument("--cycles", type=int, default=3); ap.add_argument("--bpx", action="store_true")
a = ap.parse_args()
h = T.Hierarchy(a.dim, a.level, phi=complex(a.k**2, 0.5*a.k**2), chi="seeded", precision=a.precision, max_vertices=10**10)
pol = T.Policy("undamped", 0.5, bpx=True) if a.bpx else T.Policy("exponential", 0.6)
for n in range(1, a.cycles + 1):
    st = h.td_bpx(pol, n) if a.bpx else h.td_add(pol, n)
print("ok", st)
