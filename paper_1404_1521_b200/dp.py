"""Host-side plumbing of the data-parallel path (one process per GPU).

torch.distributed is used only for the bootstrap and for host-level
reductions: the gradient exchange itself runs inside libpg (ncclAllGather of
per-rank records on the model stream, see pg_attach_nccl / DESIGN.md).
"""
from __future__ import annotations

import numpy as np


def shard(idx, corr, rank: int, world: int):
    """Contiguous equal shards of a global batch."""
    B = corr.shape[0]
    if B % world:
        raise ValueError(f"global batch {B} is not divisible by world size {world}")
    b = B // world
    return idx[rank * b:(rank + 1) * b], corr[rank * b:(rank + 1) * b]


def broadcast_bytes(payload: bytes, rank: int, size: int, device=None) -> bytes:
    """Broadcast `size` bytes from rank 0 over the default process group."""
    import torch
    import torch.distributed as dist
    buf = bytearray(payload if rank == 0 else bytes(size))
    t = torch.frombuffer(buf, dtype=torch.uint8).clone()
    if device is not None:
        t = t.to(device)
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def attach(model, rank: int, world: int, device=None):
    """NCCL bootstrap: rank 0 creates the unique id, everyone joins."""
    import paper_1404_1521_b200 as pg
    uid = pg.pg_nccl_unique_id() if rank == 0 else bytes(128)
    uid = broadcast_bytes(uid, rank, 128, device)
    model.attach_nccl(rank, world, uid)


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(a: np.ndarray) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.numpy()
