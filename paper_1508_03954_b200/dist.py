"""Process-group plumbing for multi-GPU runs (one process per GPU).

torch.distributed carries only control traffic here -- barriers, the NCCL
unique id of the library's own communicator, and max-over-ranks timings;
the data path (halo planes, restriction partials, coarse all-gather) runs
inside libtreemg_b200.so on its own NCCL communicator.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional


@dataclass
class Ctx:
    rank: int = 0
    world: int = 1
    local: int = 0
    dist: Optional[object] = None
    cuda: bool = False


def init(backend: Optional[str] = None) -> Ctx:
    """Reads RANK / WORLD_SIZE / LOCAL_RANK (torchrun); world 1 needs no group."""
    ctx = Ctx(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
              int(os.environ.get("LOCAL_RANK", "0")))
    if ctx.world > 1:
        import torch
        import torch.distributed as dist
        ctx.cuda = torch.cuda.is_available() and backend != "gloo"
        if ctx.cuda:
            torch.cuda.set_device(ctx.local)
        dist.init_process_group(backend or ("nccl" if ctx.cuda else "gloo"))
        ctx.dist = dist
    return ctx


def barrier(ctx: Ctx) -> None:
    if ctx.dist is not None:
        ctx.dist.barrier()
    if ctx.cuda:
        import torch
        torch.cuda.synchronize()


def broadcast_bytes(ctx: Ctx, payload: Optional[bytes]) -> bytes:
    """rank 0's payload on every rank (the 128-byte NCCL unique id)."""
    if ctx.dist is None:
        return payload
    box = [payload]
    ctx.dist.broadcast_object_list(box, src=0)
    return box[0]


def reduce_max(ctx: Ctx, x: float) -> float:
    if ctx.dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{ctx.local}" if ctx.cuda else "cpu")
    ctx.dist.all_reduce(t, op=ctx.dist.ReduceOp.MAX)
    return float(t.item())


def all_gather_obj(ctx: Ctx, obj):
    if ctx.dist is None:
        return [obj]
    out = [None] * ctx.world
    ctx.dist.all_gather_object(out, obj)
    return out


def finalize(ctx: Ctx) -> None:
    if ctx.dist is not None:
        ctx.dist.destroy_process_group()
