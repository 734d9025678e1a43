"""Test helper: numpy restatement of the packed tile layout of the multi-GPU
path -- what k_render_rays writes when a rank renders its interleaved tiles
(render_kernel.cuh, packed output) and what k_unpack (render.cu) reads after
the NCCL all-gather -- so the layout can be checked on CPU with gloo."""
import numpy as np

from paper_2401_02896_b200.dist import TILE, owned_tiles, packed_tiles_per_rank, tile_grid


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
