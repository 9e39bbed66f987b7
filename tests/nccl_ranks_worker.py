"""Worker of tests/test_gpu_nccl_branch.py: the slab ranks of the NCCL branch
as THREADS of this process on one GPU, over the test double tests/fake_nccl.cpp
(TMG_NCCL_LIB).  Every rank builds its own SlabGroup through tmg_slabs_create
(rank, world, unique id) exactly as bench.py's ranks do under torchrun, runs
the cycles, and hands back its norms and its owned fine planes; the gathered
iterate must be bitwise the single-GPU one.

usage: nccl_ranks_worker.py LEVELS WORLD td-add|td-bpx CYCLES  ->  one JSON line
"""
import ctypes
import json
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03954_b200 as T  # noqa: E402


def main():
    levels, world, kind, cycles = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
    phi = 400 + 200j
    pol = T.Policy("exponential", 0.6) if kind == "td-add" else T.Policy("undamped", 0.5, bpx=True)
    one = T.Hierarchy(3, levels, phi=phi, chi="seeded", precision="fast", max_vertices=10 ** 10)
    ref = [one.td_bpx(pol, n) if pol.bpx else one.td_add(pol, n) for n in range(1, cycles + 1)]
    u1 = one.field(levels, "u")
    # then bench.py's sequence: device-timed back-to-back cycles, and an end-to-end step
    # (host rhs -> the rank's planes -> load vector -> cycle -> norms)
    n_lat = (3 ** levels + 1) ** 3
    chi_host = np.random.default_rng(7).uniform(-1, 1, size=2 * n_lat)
    one.time_cycles(pol, cycles + 1, 2, flush_l2=False)
    e1 = one.e2e_step(pol, cycles + 3, chi_host)
    u2 = one.field(levels, "u")
    one.close()

    uid = T.nccl_unique_id()
    assert uid.startswith(b"fake-nccl-"), "the test double is not the library's NCCL"
    out = [None] * world
    errs = []

    def rank_main(r):
        try:
            sl = T.Slabs(levels, phi, rank=r, world=world, nccl_id=uid)
            norms = [sl.cycle(pol, n) for n in range(1, cycles + 1)]
            z0, z1 = sl.owned_planes()
            u = sl.fine_u()
            sl.time_cycles(pol, cycles + 1, 2)
            e, h2d = sl.e2e_step(pol, cycles + 3, chi_host)
            out[r] = (norms, (z0, z1), u, np.array(e), h2d, sl.fine_u())
            sl.close()
        except Exception as e:  # noqa: BLE001
            errs.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs or any(o is None for o in out):
        print(json.dumps({"ok": False, "errors": errs}))
        return 1
    n1 = 3 ** levels + 1
    plan = T.slab_plan(levels, world)
    gathered = np.zeros(n1 ** 3, dtype=np.complex128)
    planes = []
    gathered2 = np.zeros(n1 ** 3, dtype=np.complex128)
    e2e_err, h2d_total = 0.0, 0
    for r, (norms, (z0, z1), u, e, h2d, ub) in enumerate(out):
        gathered2.reshape(n1, n1, n1)[z0:z1] = ub.reshape(n1, n1, n1)[z0:z1]
        e2e_err = max(e2e_err, float(np.max(np.abs(e - np.array(e1)) / np.abs(np.array(e1)))))
        h2d_total += h2d
        assert h2d == 16 * n1 * n1 * (z1 - z0 + 2), (r, h2d)
        assert (z0, z1) == (int(plan[r][2]), int(plan[r][3])), (r, z0, z1, plan[r])
        u3 = u.reshape(n1, n1, n1)  # [z][y][x]
        other = np.ones(n1, dtype=bool)
        other[z0:z1] = False
        assert not u3[other].any(), f"rank {r} returned planes it does not own"
        gathered.reshape(n1, n1, n1)[z0:z1] = u3[z0:z1]
        planes += list(range(z0, z1))
    assert planes == list(range(1, n1 - 1)), "owned planes do not partition the interior"
    bitwise = bool(np.array_equal(gathered, u1)) and bool(np.array_equal(gathered2, u2))
    same_across_ranks = True
    norm_err = e2e_err
    for n in range(cycles):
        a = ref[n]
        for r in range(world):
            b = out[r][0][n]
            norm_err = max(norm_err, abs(a.h_norm - b.h_norm) / a.h_norm, abs(a.max_norm - b.max_norm) / a.max_norm)
            same_across_ranks &= (b.h_norm == out[0][0][n].h_norm and b.max_norm == out[0][0][n].max_norm)
    st = (ctypes.c_ulonglong * 3)()
    ctypes.CDLL(os.environ["TMG_NCCL_LIB"]).fake_nccl_stats(st)
    print(json.dumps({"ok": True, "bitwise": bitwise, "norm_err": norm_err, "same_across_ranks": same_across_ranks,
                      "sends": int(st[0]), "bytes": int(st[1]), "groups": int(st[2])}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
