import os, sys, subprocess, numpy as np
sys.path.insert(0, '.')
code = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1508_03954_b200 as T
L = int(sys.argv[1]); dim = int(sys.argv[2])
h = T.Hierarchy(dim, L, phi=400+200j, chi="seeded", precision="fast", max_vertices=10**10)
pol = T.Policy("exponential", 0.6)
out = {}
for n in range(1, 5):
    st = h.td_add(pol, n)
    out[f"norm{n}"] = np.array([st.max_norm, st.euclid_norm, st.h_norm])
    for l in range(1, L + 1):
        for f in ("u", "sc", "rhat", "si"):
            try: out[f"{n}_{l}_{f}"] = h.field(l, f)
            except Exception: pass
np.savez(sys.argv[3], **out)
'''
open('/tmp/cc.py', 'w').write(code)
for L, dim in ((5, 3), (4, 2)):
    for c in ("0", "1"):
        env = dict(os.environ, TMG_CHAIN=c)
        subprocess.run([sys.executable, '/tmp/cc.py', str(L), str(dim), f'/tmp/cc_{c}.npz'], env=env, check=True)
    a, b = np.load('/tmp/cc_0.npz'), np.load('/tmp/cc_1.npz')
    for k in a.files:
        if not np.array_equal(a[k], b[k]):
            d = np.abs(a[k] - b[k]); i = int(np.argmax(d))
            print(L, dim, k, "DIFF", int((d > 0).sum()), d.max(), i)
    print(L, dim, "done")
