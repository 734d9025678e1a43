"""Image-tile sharding over ranks: one process per GPU, the
particle set and LUT replicated in every GPU's HBM, 8x8-pixel tiles interleaved
over ranks (tile t -> rank t % nranks), finished tiles gathered with NCCL over
NVLink inside the library (engine.cpp).  torch.distributed is plumbing only:
it carries the 128-byte NCCL unique id from rank 0 to the others.

The numpy functions here restate the tile layout the CUDA kernels implement
(k_render_rays' packed writes and k_unpack in render.cu) so the layout can be
tested on CPU with gloo.
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


def pack(image: np.ndarray, rank: int, nranks: int) -> np.ndarray:
    """The packed buffer rank `rank` produces for a full (H, W, 3) image."""
    H, W, _ = image.shape
    tx, ty, nt = tile_grid(W, H)
    per = packed_tiles_per_rank(nranks, nt)
    out = np.zeros((per, TILE, TILE, 3), dtype=image.dtype)
    for j, t in enumerate(owned_tiles(rank, nranks, nt)):
        y0, x0 = (t // tx) * TILE, (t % tx) * TILE
        blk = image[y0:y0 + TILE, x0:x0 + TILE]
        out[j, : blk.shape[0], : blk.shape[1]] = blk
    return out.reshape(-1)


def unpack(gathered: np.ndarray, nranks: int, width: int, height: int) -> np.ndarray:
    """k_unpack: rank-major concatenation of packed buffers -> (H, W, 3)."""
    tx, ty, nt = tile_grid(width, height)
    per = packed_tiles_per_rank(nranks, nt)
    g = gathered.reshape(nranks, per, TILE, TILE, 3)
    img = np.zeros((ty * TILE, tx * TILE, 3), dtype=gathered.dtype)
    for t in range(nt):
        r, j = t % nranks, t // nranks
        y0, x0 = (t // tx) * TILE, (t % tx) * TILE
        img[y0:y0 + TILE, x0:x0 + TILE] = g[r, j]
    return img[:height, :width]


def init_comm(ctx, rank: int, world: int):
    """Create the library's NCCL communicator; the unique id travels over
    torch.distributed (any backend)."""
    import torch.distributed as dist

    if world <= 1:
        return
    obj = [ctx.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.init_comm(rank, world, obj[0])
