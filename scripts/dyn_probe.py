"""Dynamic adaptivity (h_max / h_min) on the GPU against the live reference
harness, sweep by sweep: norms, mark statistics, structure and every field of
every level (hanging vertices included).  Prints the first mismatch."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_1508_03954_b200 as T
import refdriver as R

SWEEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 8
CASE = sys.argv[2] if len(sys.argv) > 2 else "h2d"
CASES = {
    "h2d": (dict(problem="helmholtz-sin", dim=2, phi="100,50", h_max=0.04, h_min=0.004, omega="undamped",
                 omega_s=0.6), dict(dim=2, phi=100 + 50j, chi="sin"), dict(kind="undamped", omega_s=0.6)),
    "p2d_bpx": (dict(problem="poisson-sin", dim=2, h_max=0.04, h_min=0.002, cycle="td-bpx", omega="undamped",
                     omega_s=0.5), dict(dim=2, phi=0, chi="sin"), dict(kind="undamped", omega_s=0.5, bpx=True)),
    "h3d": (dict(problem="helmholtz-sin", dim=3, phi="400,200", h_max=0.12, h_min=0.013, omega="exponential",
                 omega_s=0.6), dict(dim=3, phi=400 + 200j, chi="sin"), dict(kind="exponential", omega_s=0.6)),
    "p3d": (dict(problem="poisson-sin", dim=3, h_max=0.12, h_min=0.013, omega="undamped", omega_s=0.6),
            dict(dim=3, phi=0, chi="sin"), dict(kind="undamped", omega_s=0.6)),
    "b2d_seeded": (dict(problem="helmholtz-ball", dim=2, h_max=0.12, h_min=0.0014, omega="exponential",
                        omega_s=0.8, rhs="seeded", rhs_seed=99, theta_deg=20),
                   dict(dim=2, phi=-1000, chi="seeded", rhs_seed=99, theta_deg=20),
                   dict(kind="exponential", omega_s=0.8)),
}
rcfg, hkw, pkw = CASES[CASE]
ref = R.RefSession(dict(rcfg, max_sweeps=SWEEPS))
assert ref.status == 0, ref.message
h = T.Hierarchy(levels=1, precision="exact", h_max=rcfg["h_max"], h_min=rcfg["h_min"], **hkw)
pol = T.Policy(**pkw)
rng = np.random.default_rng(1)
# sinext: the reference keeps siNext until the next touch-first zeroes it, the
# device zeroes it when it commits si = siNext -- the same state for the cycle
FIELDS = ["u", "sc", "uhat", "rhat", "sf", "si", "chi"]
for n in range(1, SWEEPS + 1):
    want = ref.sweep(n)
    got = h.td_bpx(pol, n) if pkw.get("bpx") else h.td_add(pol, n)
    rm = ref.mark_stats()
    gm = h.mark()
    g = np.array([got.max_norm, got.euclid_norm, got.h_norm, got.updated_fine_vertices])
    rel = np.abs(g[:3] - want[:3]) / np.maximum(want[:3], 1e-300)
    print(f"sweep {n}: depth {h.depth()} / {ref.depth} updated {int(g[3])} / {int(want[3])} rel {rel.max():.2e}"
          f" marks r{gm['refine_cells']} e{gm['erase_cells']} refined {gm['refined']} erased {gm['erased']}")
    if rm != gm:
        print("  marks differ:\n   ref", rm, "\n   gpu", gm)
    bad = False
    for l in range(0, ref.depth + 1):
        fl, sc, ce = ref.flags(l)
        gfl, gsc, gce = h.flags(l)
        if not (np.array_equal(fl, gfl) and np.array_equal(sc, gsc) and np.array_equal(ce & 3, gce & 3)):
            print(f"  level {l}: structure differs ({int((fl != gfl).sum())} flags)")
            bad = True
            continue
        for fld in FIELDS:
            a, mask = ref.field_all(l, fld)
            b = h.field(l, fld + "@all")
            d = np.flatnonzero(a != b)
            if len(d):
                print(f"  level {l} field {fld}: {len(d)} differ of {int((mask > 0).sum())}; first idx {d[:4]}"
                      f" ref {a[d[:2]]} gpu {b[d[:2]]} mask {mask[d[:4]]}")
                bad = True
    if bad and "--keep" not in sys.argv:
        break
    if "--random" in sys.argv:  # replace the marks on both sides by the same random ones (erase coverage)
        for l in range(ref.depth + 1):
            ce = ref.cell_marks(l)
            ex, refd = (ce & 1) > 0, (ce & 2) > 0
            m = np.zeros_like(ce)
            m[ex & ~refd & (rng.random(len(ce)) < 0.15)] |= 4
            # erase only where no neighbouring cell refines in the same traversal (a vertex erased
            # and re-created within one traversal is refused by the device path)
            n1 = 3 ** l + 1
            r4 = (m & 4).reshape((n1,) * rcfg["dim"])
            near = np.zeros_like(r4)
            for off in np.ndindex(*((3,) * rcfg["dim"])):
                near |= np.roll(r4, tuple(o - 1 for o in off), axis=tuple(range(rcfg["dim"])))
            m[refd & (near.reshape(-1) == 0) & (rng.random(len(ce)) < 0.35)] |= 8
            ref.set_cell_marks(l, m)
            h.set_cell_marks(l, m)
