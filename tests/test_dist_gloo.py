"""CPU, world_size 2 over gloo: the image-tile partition and gather contract of
the multi-GPU path.  Each rank packs its interleaved tiles
(tile t -> rank t % nranks, the layout k_render_rays writes when packed), the
packed buffers are all-gathered (NCCL on the GPU box, gloo here) and unpacked
(k_unpack's layout); the result must equal the single-rank image exactly, and
the NCCL unique-id broadcast plumbing must deliver rank 0's bytes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_02896_b200 import dist as D
from tests import dist_layout as DL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, H, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1234)
        full = rng.random((H, W, 3))
        packed = torch.from_numpy(DL.pack(full, rank, world))
        bufs = [torch.empty_like(packed) for _ in range(world)]
        dist.all_gather(bufs, packed)
        gathered = torch.cat(bufs).numpy()
        img = DL.unpack(gathered, world, W, H)
        ok_img = bool((img == full).all())
        # unique-id broadcast as dist.init_comm does it
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ok_id = obj[0] == bytes(range(128))
        # ownership is a partition of all tiles
        nt = D.tile_grid(W, H)[2]
        mine = torch.from_numpy(np.bincount(D.owned_tiles(rank, world, nt), minlength=nt))
        dist.all_reduce(mine)
        ok_part = bool((mine.numpy() == 1).all())
        out_q.put((rank, ok_img, ok_id, ok_part))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,H", [(24, 24), (37, 19), (256, 192)])
def test_tile_gather_world2(W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, W, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert len(res) == 2
    for rank, ok_img, ok_id, ok_part in res:
        assert ok_img and ok_id and ok_part, (rank, ok_img, ok_id, ok_part)


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_pack_unpack_roundtrip(nranks):
    rng = np.random.default_rng(nranks)
    img = rng.random((45, 61, 3))
    nt = D.tile_grid(61, 45)[2]
    gathered = np.concatenate([DL.pack(img, r, nranks) for r in range(nranks)])
    assert (DL.unpack(gathered, nranks, 61, 45) == img).all()
    assert sum(len(D.owned_tiles(r, nranks, nt)) for r in range(nranks)) == nt


def test_bench_launches_its_ranks():
    """`bench.py --gpus 2` started without a launcher re-executes itself under
    torch.distributed.run (one process per rank); the line reports n_gpus 2."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["ranks_ms_max"] == 2.0
