"""The closed-form traversal-order rules the sm_100a kernels use instead of
sorting (paper_1508_03954_b200/csrc/exact_ops.cuh) against brute-force base-3
Morton (DFS) sorting of the reference traversal (spacetree.cpp:394-424)."""
import itertools

import pytest


def morton(l, c, p):
    key = 0
    for k in range(l - 1, -1, -1):
        slot, mul = 0, 1
        for d in range(p):
            slot += ((c[d] // 3 ** k) % 3) * mul
            mul *= 3
        key = key * 3 ** p + slot
    return key


def tz3(x):
    if x == 0:
        return 31
    t = 0
    while x % 3 == 0:
        x //= 3
        t += 1
    return t


# --- Python transcription of exact_ops.cuh perm_axis / perm_cell / perm_id ---
def perm_axis(P, pid, j):
    if P == 1:
        return 0
    if P == 2:
        return (1 if j == 0 else 0) if pid == 0 else (0 if j == 0 else 1)
    if j == 0:
        return pid // 2
    if j == 1:
        return ((1 if pid // 2 == 0 else 0) if pid % 2 == 0 else (1 if pid // 2 == 2 else 2))
    return ((1 if pid // 2 == 2 else 2) if pid % 2 == 0 else (1 if pid // 2 == 0 else 0))


def perm_cell(P, pid, i):
    e = 0
    for j in range(P):
        e |= ((i >> (P - 1 - j)) & 1) << perm_axis(P, pid, j)
    return e


def perm_id(P, idx):
    if P == 1:
        return 0
    if P == 2:
        return 0 if tz3(idx[1]) >= tz3(idx[0]) else 1
    k = [tz3(idx[d]) * 4 + d for d in range(3)]
    pr = sorted(range(3), key=lambda d: k[d], reverse=True)
    return 2 * pr[0] + (1 if pr[1] > pr[2] else 0)


def test_permutations_are_bijections():
    for P, n in ((1, 1), (2, 2), (3, 6)):
        seen = set()
        for pid in range(n):
            cells = tuple(perm_cell(P, pid, i) for i in range(1 << P))
            assert sorted(cells) == list(range(1 << P))
            seen.add(cells)
        assert len(seen) == n


@pytest.mark.parametrize("p,levels", [(1, 4), (2, 3), (3, 2)])
def test_cell_order_rule(p, levels):
    """Rule (1): cells around a vertex in DFS order."""
    for l in range(1, levels + 1):
        m = 3 ** l
        for v in itertools.product(range(m + 1), repeat=p):
            pid = perm_id(p, v)
            rule = []
            for i in range(1 << p):
                e = perm_cell(p, pid, i)
                c = tuple(v[d] - 1 + ((e >> d) & 1) for d in range(p))
                if all(0 <= c[d] <= m - 1 for d in range(p)):
                    rule.append(c)
            brute = sorted(rule, key=lambda c: morton(l, c, p))
            assert rule == brute, (l, v)


@pytest.mark.parametrize("p,levels", [(1, 4), (2, 3), (3, 2)])
def test_restriction_order_rule(p, levels):
    """Rule (2): interior fine vertices restricted into coarse W in touch-last order."""
    for l in range(2, levels + 1):
        m = 3 ** l
        for W in itertools.product(range(3 ** (l - 1) + 1), repeat=p):
            pid = perm_id(p, W)
            rule = []
            for gi in range(1 << p):
                f = perm_cell(p, pid, gi)
                ranges = [range(0, 3) if (f >> d) & 1 else range(-2, 0) for d in range(p)]
                for kk in itertools.product(*reversed(ranges)):
                    k = kk[::-1]
                    v = tuple(3 * W[d] + k[d] for d in range(p))
                    if all(1 <= v[d] <= m - 1 for d in range(p)):
                        rule.append(v)
            brute = sorted(rule, key=lambda v: morton(l, v, p))
            assert rule == brute, (l, W)
