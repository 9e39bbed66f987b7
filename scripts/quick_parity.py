"""Ad-hoc exact-mode parity sweep: GPU hierarchy vs the CPU restatement."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import oracle as O
import paper_1508_03954_b200 as T

FIELDS = ["u", "sc", "sf", "si", "chi", "rhat", "uhat", "diag"]
def case(cfg, sweeps, label, init=None):
    o = O.OracleSession(cfg)
    kind = cfg.get("omega", "exponential")
    pol = T.Policy(kind=kind, omega_s=complex(*(float(x) for x in str(cfg.get("omega_s", "0.8")).split(","))) if "," in str(cfg.get("omega_s","0.8")) else float(cfg.get("omega_s", 0.8)),
                   lgrid=int(cfg.get("lgrid", 2)), hb=bool(int(cfg.get("hb", 0))), bpx=cfg.get("cycle") == "td-bpx",
                   two_phase=bool(int(cfg.get("two_phase", 0))))
    phi = cfg.get("phi", 0)
    if isinstance(phi, str):
        a = [float(x) for x in phi.split(",")]; phi = complex(a[0], a[1] if len(a) > 1 else 0)
    chi = "seeded" if cfg.get("rhs") == "seeded" else ("ball" if cfg.get("problem") == "helmholtz-ball" else "sin")
    if cfg.get("problem") == "helmholtz-sin" and "phi" not in cfg: phi = 2025.0
    if cfg.get("problem") == "helmholtz-ball" and "phi" not in cfg: phi = -1000.0
    h = T.Hierarchy(cfg["dim"], cfg["level"], phi=phi, theta_deg=float(cfg.get("theta_deg", 0)), chi=chi,
                    rhs_seed=int(cfg.get("rhs_seed", 12345)), ell_min=int(cfg.get("ell_min", 1)))
    if init is not None:
        o.set_fine_interior_u(init); h.set_fine_interior_u(init)
    if cfg.get("initial") == "random":
        h.set_random_initial_guess(int(cfg.get("seed", 0)))
    bad = []
    L = cfg["level"]
    for n in range(1, sweeps + 1):
        a = o.sweep(n)
        st = h.td_bpx(pol, n) if pol.bpx else h.td_add(pol, n)
        b = np.array([st.max_norm, st.euclid_norm, st.h_norm])
        rel = np.abs(a[:3] - b) / np.maximum(np.abs(a[:3]), 1e-300)
        if rel.max() > 1e-12: bad.append(("norms", n, rel))
        for l in range(1, L + 1):
            for f in FIELDS:
                if f in ("sf", "si") and l == L: continue
                x = o.field(l, f); y = h.field(l, f)
                if not np.array_equal(x, y):
                    bad.append((n, l, f, float(np.abs(x - y).max()), int((x != y).sum()), len(x)))
    print(f"{label:30s}", "OK" if not bad else bad[:5], flush=True)
    return not bad

ok = True
S = dict(rhs="seeded", rhs_seed=12345)
ok &= case(dict(problem="poisson-sin", dim=2, level=2), 6, "poisson p2 L2")
ok &= case(dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", theta_deg=35), 6, "helm p2 L3 th35")
ok &= case(dict(problem="helmholtz-sin", dim=2, level=4, phi="100,50", **S), 6, "seeded p2 L4")
ok &= case(dict(problem="helmholtz-sin", dim=3, level=2, phi="400,200", **S), 4, "seeded p3 L2")
ok &= case(dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", **S), 3, "seeded p3 L3")
ok &= case(dict(problem="helmholtz-sin", dim=1, level=4, phi="100,50", theta_deg=35), 6, "p1 L4")
ok &= case(dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", cycle="td-bpx", omega="undamped", omega_s=0.5, **S), 6, "bpx p2 L3")
ok &= case(dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", cycle="td-bpx", omega="undamped", omega_s=0.5, **S), 3, "bpx p3 L3")
ok &= case(dict(problem="helmholtz-sin", dim=2, level=3, phi="-1000", hb=1, **S), 6, "hb p2 L3")
ok &= case(dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="transition", two_phase=1, **S), 6, "transition twophase")
ok &= case(dict(problem="helmholtz-sin", dim=2, level=3, phi="100,50", omega="lgrid", lgrid=1, ell_min=2, **S), 6, "lgrid ellmin2")
ok &= case(dict(problem="poisson-sin", dim=2, level=3, initial="random", seed=7), 5, "random init")
ok &= case(dict(problem="helmholtz-ball", dim=3, level=3), 3, "ball p3 L3")
print("ALL OK" if ok else "FAILURES")
