"""The N>1 host path on CPU with a world-size-2 gloo group: the control
plumbing bench.py uses (paper_1508_03954_b200/dist.py) and the slab plan
each rank derives independently must agree across ranks -- the NCCL id
broadcast reaches every rank, the owned fine / coarse planes of all ranks
partition the levels, and max-over-ranks timing reduces correctly."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
mp = torch.multiprocessing


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, levels, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import paper_1508_03954_b200 as T
    from paper_1508_03954_b200 import dist as D
    ctx = D.init("gloo")
    uid = D.broadcast_bytes(ctx, bytes(range(128)) if rank == 0 else None)
    plan = T.slab_plan(levels, world)           # every rank computes the plan on its own
    mine = tuple(int(v) for v in plan[rank])
    everyone = D.all_gather_obj(ctx, mine)
    slowest = D.reduce_max(ctx, float(rank + 1))
    D.barrier(ctx)
    q.put((rank, uid, everyone, slowest))
    D.finalize(ctx)


@pytest.mark.parametrize("levels", [5, 6])
def test_two_rank_gloo_plan_and_plumbing(levels):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, levels, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, mc = 3 ** levels, 3 ** (levels - 1)
    for rank, uid, everyone, slowest in res:
        assert uid == bytes(range(128))
        assert slowest == float(world)
        assert everyone == res[0][2]
    plans = res[0][2]
    fine = [z for (_, _, z0, z1, *_rest) in plans for z in range(z0, z1)]
    assert fine == list(range(1, m))           # interior fine planes, each exactly once
    coarse = [Z for (_, _, _, _, Zs, Ze, _, _) in plans for Z in range(Zs, Ze)]
    assert coarse == list(range(1, mc))
