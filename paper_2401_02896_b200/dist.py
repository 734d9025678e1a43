"""Image-tile sharding over ranks: one process per GPU, the
particle set and LUT replicated in every GPU's HBM, 8x8-pixel tiles interleaved
over ranks (tile t -> rank t % nranks), finished tiles gathered with NCCL over
NVLink inside the library (engine.cpp).  torch.distributed is plumbing only:
it carries the 128-byte NCCL unique id from rank 0 to the others.

tests/dist_layout.py restates the packed tile layout in numpy for the CPU
(gloo) tests.
"""
from __future__ import annotations

import numpy as np

TILE = 8  # render.cuh kTile


def tile_grid(width: int, height: int):
    tx = (width + TILE - 1) // TILE
    ty = (height + TILE - 1) // TILE
    return tx, ty, tx * ty


def owned_tiles(rank: int, nranks: int, ntiles: int) -> np.ndarray:
    """Global tile ids rank `rank` renders, in packed order."""
    return np.arange(rank, ntiles, nranks, dtype=np.int64)


def packed_tiles_per_rank(nranks: int, ntiles: int) -> int:
    return (ntiles + nranks - 1) // nranks


def init_comm(ctx, rank: int, world: int):
    """Create the library's NCCL communicator; the unique id travels over
    torch.distributed (any backend)."""
    import torch.distributed as dist

    if world <= 1:
        return
    obj = [ctx.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.init_comm(rank, world, obj[0])
