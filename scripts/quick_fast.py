"""Fast-precision vs exact-precision (bit-exact reference) on the same problem."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_1508_03954_b200 as T

def case(dim, level, phi, pol, sweeps, label, **kw):
    he = T.Hierarchy(dim, level, phi=phi, chi="seeded", precision="exact", max_vertices=10**10, **kw)
    hf = T.Hierarchy(dim, level, phi=phi, chi="seeded", precision="fast", max_vertices=10**10, **kw)
    first = None; worst_norm = 0; worst_strict = 0
    for n in range(1, sweeps + 1):
        a = he.td_bpx(pol, n) if pol.bpx else he.td_add(pol, n)
        b = hf.td_bpx(pol, n) if pol.bpx else hf.td_add(pol, n)
        if first is None: first = a.h_norm
        worst_norm = max(worst_norm, abs(a.h_norm - b.h_norm) / first)
        worst_strict = max(worst_strict, abs(a.h_norm - b.h_norm) / a.h_norm)
    ue = he.field(level, "u"); uf = hf.field(level, "u")
    du = np.abs(ue - uf).max() / max(np.abs(ue).max(), 1e-300)
    print(f"{label:28s} first={first:.4e} last={a.h_norm:.4e} drop={a.h_norm/first:.2e} "
          f"|dnorm|/first={worst_norm:.2e} strict={worst_strict:.2e} |du|/|u|={du:.2e}", flush=True)

case(2, 4, 100+50j, T.Policy("exponential", 0.6), 20, "2D L4 k10 exp")
case(2, 5, 100+50j, T.Policy("exponential", 0.6), 20, "cfg1 2D L5 k10 exp")
case(2, 5, 10000+5000j, T.Policy("undamped", 0.5, bpx=True), 60, "cfg2op 2D L5 bpx")
case(3, 3, 400+200j, T.Policy("exponential", 0.6), 20, "3D L3 exp")
case(3, 4, 400+200j, T.Policy("exponential", 0.6), 20, "3D L4 exp")
case(3, 5, 400+200j, T.Policy("exponential", 0.6), 50, "cfg3 3D L5 exp")
case(3, 4, 400+200j, T.Policy("undamped", 0.5, bpx=True), 20, "3D L4 bpx")
case(3, 4, 1600+800j, T.Policy("exponential", 0.6, hb=True), 10, "3D L4 hb")
case(2, 5, 100+50j, T.Policy("transition", 0.6, two_phase=True), 20, "2D transition 2phase")
case(2, 5, 100+50j, T.Policy("lgrid", 0.6, lgrid=1), 20, "2D lgrid ellmin2", ell_min=2)
