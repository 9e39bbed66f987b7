"""Host-only timing of the dynamic-adaptivity structural replay (dyn.cpp):
grow a 2D tree from level 3 with refine marks on every leaf cell up to
level `top`, then time sweeps without marks (the pure traversal replay)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1508_03954_b200 as T
top = int(sys.argv[1]) if len(sys.argv) > 1 else 6
D = T.DynStructure(2, 3, top, 1, 1e-9)
for l in range(3, top):
    D.set_cell_marks(l, np.full((3 ** l + 1) ** 2, 4, np.uint8))  # refineMark on every cell of level l
    D.sweep()
print("depth", D.depth, "interior", D.interior_count())
ts = []
for i in range(5):
    t0 = time.perf_counter()
    D.sweep()
    ts.append((time.perf_counter() - t0) * 1e3)
print("sweep ms", " ".join(f"{t:.1f}" for t in ts))
