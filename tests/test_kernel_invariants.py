"""Host-side invariants the new coarse-level kernels rely on, checked by
brute force on CPU (restatements of the index arithmetic in fast.cu /
fused2.cu; the GPU tests check the numerics):

* pyramid top-down (fast.cu k_topdown_pyr / pyramid_setup): the ancestor box
  a CTA builds at every level fits the shared-memory capacity the host
  reserves, for every tile position of every level size;
* 2D fused pass coarse-row ring (fused2.cu issueCoarse / computeV): every
  coarse row is copied in a ring group that has landed before its first use
  and its slot is not reused while a later fine row still reads it.
"""
import pytest

TX, TY = 32, 8


def pyramid_caps(P, T, n1s, k):
    ext = [TX, TY if P == 3 else TY * k, k][:P]
    sz, caps = list(ext), {}
    for l in range(T - 1, -1, -1):
        cap = 1
        for d in range(P):
            sz[d] = min((sz[d] - 1 + 2) // 3 + 2, n1s[l])
            cap *= sz[d]
        caps[l] = cap
    return caps


def pyramid_boxes(P, T, ms, tile, k):
    ext = [TX, TY if P == 3 else TY * k, k][:P]
    lo = [tile[d] * ext[d] for d in range(P)]
    hi = [min(lo[d] + ext[d] - 1, ms[T]) for d in range(P)]
    boxes = {}
    for l in range(T - 1, -1, -1):
        mp = ms[l]
        lo = [min(x // 3, mp - 1) for x in lo]
        hi = [min(x // 3, mp - 1) + 1 for x in hi]
        n = 1
        for d in range(P):
            assert 0 <= lo[d] <= hi[d] <= mp
            n *= hi[d] - lo[d] + 1
        boxes[l] = n
    return boxes


@pytest.mark.parametrize("P,Tmax,k", [(2, 7, 4), (3, 5, 8)])
def test_pyramid_boxes_fit_reserved_shared_memory(P, Tmax, k):
    for T in range(1, Tmax + 1):
        ms = [3 ** l for l in range(T + 1)]
        n1s = [m + 1 for m in ms]
        caps = pyramid_caps(P, T, n1s, k)
        ext = [TX, TY if P == 3 else TY * k, k][:P]
        ntiles = [(n1s[T] + ext[d] - 1) // ext[d] for d in range(P)]
        # every tile along each axis independently bounds the product
        worst = {l: 0 for l in range(T)}
        import itertools
        axes = [range(n) for n in ntiles]
        if P == 3 and ntiles[0] * ntiles[1] * ntiles[2] > 20000:  # sample the interior densely, edges fully
            axes = [sorted(set(list(range(min(n, 6))) + list(range(max(0, n - 6), n)))) for n in ntiles]
        for tile in itertools.product(*axes):
            for l, n in pyramid_boxes(P, T, ms, tile, k).items():
                assert n <= caps[l], (P, T, tile, l, n, caps[l])
                worst[l] = max(worst[l], n)
        assert all(worst[l] > 0 for l in range(T))


def ring_schedule(m, y0, yc, kring=4):
    """Replays k_fused2's issue order: fine row it2 (yy = y0 - 1 + it2) is
    issued at iteration it2 - (kring - 1) (the first kring - 1 in the prologue);
    coarse row (yy + 1) / 3 + 1 rides with fine row yy when yy % 3 == 2.
    Returns (issue iteration per coarse row, first use iteration per coarse row,
    last use iteration per coarse row)."""
    mc = m // 3
    y1 = min(y0 + yc, m)
    nrows = y1 - y0 + 2
    issued, first_use, last_use = {}, {}, {}
    q0 = min(max(y0 - 1, 0) // 3, mc - 1)
    issued[q0] = issued[q0 + 1] = -kring  # synchronous prologue copy
    for it2 in range(nrows):
        yy = y0 - 1 + it2
        at = max(it2 - (kring - 1), -1)  # iteration whose body issues fine row it2 (-1: prologue)
        if yy >= 2 and yy % 3 == 2 and (yy + 1) // 3 < mc:
            q = (yy + 1) // 3 + 1
            issued.setdefault(q, (at, it2))
    for it in range(nrows):  # computeV(yy) for row it runs in iteration it - 1 (prologue for it = 0)
        yy = y0 - 1 + it
        qy = min(max(yy, 0) // 3, mc - 1)
        for q in (qy, qy + 1):
            first_use.setdefault(q, it - 1)
            last_use[q] = it - 1
    return issued, first_use, last_use


@pytest.mark.parametrize("m", [27, 81, 243, 729, 2187])
@pytest.mark.parametrize("yc", [3, 6, 27, 48])
def test_fused2_coarse_ring_lands_before_use_and_is_not_overwritten(m, yc):
    for y0 in range(1, m, yc):
        issued, first_use, last_use = ring_schedule(m, y0, yc)
        for q, it_use in first_use.items():
            assert q in issued, (m, yc, y0, q)
            iss = issued[q]
            if isinstance(iss, tuple):
                # waited on in iteration it2 (wait_group before reading row it2): must precede computeV's use
                _, fine_row = iss
                assert fine_row <= it_use, (m, yc, y0, q, iss, it_use)
        # slot q % 4 is next written by coarse row q + 4; that copy is issued
        # after the last computeV reading q
        for q, it_last in last_use.items():
            nxt = issued.get(q + 4)
            if isinstance(nxt, tuple):
                issue_iter, _ = nxt
                assert issue_iter > it_last, (m, yc, y0, q, nxt, it_last)  # issueRow precedes computeV in an iteration
