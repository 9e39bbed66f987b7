"""The complex division the kernels restate (libgcc __divdc3, GCC >= 12 with
underflow/overflow scaling; exact_ops.cuh divdc3 + hierarchy.cu div_const)
transcribed to Python floats and checked bit-for-bit against the host
libgcc (through the restatement's std::complex division) on adversarial
inputs.  The device side is checked the same way in test_gpu_units.py."""
import math

import numpy as np

RBIG = 8.98846567431157953865e+307
RMIN = 2.22507385850720138309e-308
RMIN2 = 2.220446049250313080847e-16
RMINSCAL = 4503599627370496.0
RMAX2 = RBIG * RMIN2


def div_const(c, d):
    swap = not (abs(c) < abs(d))
    big = abs(c) if swap else abs(d)
    pre = 0
    if big >= RBIG:
        c, d, pre = c / 2, d / 2, 1
    big2 = abs(c) if swap else abs(d)
    if big2 < RMIN2:
        c, d = c * RMINSCAL, d * RMINSCAL
        pre = 1 if pre == 1 else 2
    if not swap:
        ratio = c / d
        denom = c * ratio + d
        tiny = (c * RMINSCAL) * ratio + d * RMINSCAL
    else:
        ratio = d / c
        denom = d * ratio + c
        tiny = (d * RMINSCAL) * ratio + c * RMINSCAL
    return dict(c=c, d=d, ratio=ratio, denom=denom, tiny=tiny, swap=swap, pre=pre, sub=not abs(ratio) > RMIN)


def divdc3(a, b, k):
    c, d, denom = k["c"], k["d"], k["denom"]
    if k["pre"] == 1:
        a, b = a * 0.5, b * 0.5
    if k["pre"] == 2:
        a, b = a * RMINSCAL, b * RMINSCAL
    else:
        big = abs(c) if k["swap"] else abs(d)
        if (abs(a) < RMIN and abs(b) < RMAX2 and big < RMAX2) or (abs(b) < RMIN and abs(a) < RMAX2 and big < RMAX2):
            a, b, c, d, denom = a * RMINSCAL, b * RMINSCAL, c * RMINSCAL, d * RMINSCAL, k["tiny"]
    r = k["ratio"]
    if not k["swap"]:
        if not k["sub"]:
            x, y = (a * r + b) / denom, (b * r - a) / denom
        else:
            x, y = (c * (a / d) + b) / denom, (c * (b / d) - a) / denom
    else:
        if not k["sub"]:
            x, y = (b * r + a) / denom, (b - a * r) / denom
        else:
            x, y = (a + d * (b / c)) / denom, (b - d * (a / c)) / denom
    return complex(x, y)


def cases():
    rng = np.random.default_rng(7)
    vals = []
    for _ in range(3000):
        e = rng.integers(-320, 300, size=4)
        m = rng.uniform(-1, 1, size=4)
        vals.append((m[0] * 10.0 ** e[0], m[1] * 10.0 ** e[1], m[2] * 10.0 ** e[2], m[3] * 10.0 ** e[3]))
    for _ in range(3000):
        vals.append(tuple(rng.uniform(-1, 1, size=4) * [1e-3, 1e-3, 4e-3, 2e-3]))
    vals += [(1.0, 0.0, 3.0, 0.0), (0.0, 0.0, 2.0, 1.0), (1e-310, 1e-320, 1e-3, 1e-3), (5e-324, 1.0, 1e-17, 1e-18),
             (1.0, 1.0, 1e308, 1e307), (3.0, -2.0, 0.0, 7.0), (2.5e-16, 1e-300, 1e-200, 3e-201)]
    return vals


def test_python_transcription_matches_libgcc(oracle_mod):
    v = cases()
    x = np.array([complex(a, b) for a, b, _, _ in v])
    y = np.array([complex(c, d) for _, _, c, d in v])
    ref = oracle_mod.cdiv(x, y)
    for (a, b, c, d), q in zip(v, ref):
        if c == 0.0 and d == 0.0:
            continue
        got = divdc3(a, b, div_const(c, d))
        for g, r in ((got.real, q.real), (got.imag, q.imag)):
            assert (math.isnan(g) and math.isnan(r)) or g == r, (a, b, c, d, got, q)
