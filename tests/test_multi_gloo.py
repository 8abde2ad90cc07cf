"""CPU, world_size 2 (gloo): the multi-GPU frame path's host logic.

Each rank renders its cyclic share of 32x32 tiles (here with the FP64 oracle
standing in for the device render, so the test runs without a GPU; the same
round trip through rr_render_tiles + rr_detile on the device is
tests/test_gpu_p2p.py::test_tile_shards_gather_detile), the
tile-major shard buffers are gathered to rank 0 (dist.gather, as bench.py does
over NCCL) and de-tiled with the same index map as rr_detile / detile_kernel.
The result must be byte-identical to the single-rank frame."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

W, H, T = 72, 40, 32   # partial edge tiles on both axes


def tiles_of_shard(w, h, tw, th, shard, n):
    tiles_x, tiles_y = -(-w // tw), -(-h // th)
    return list(range(shard, tiles_x * tiles_y, n))


def render_shard(frame, w, h, tw, th, shard, n):
    """Tile-major shard buffer (rr_render_tiles layout: tile k of the shard at
    k*3*tw*th, row-major inside, partial tiles zero-padded)."""
    tiles = tiles_of_shard(w, h, tw, th, shard, n)
    tiles_x = -(-w // tw)
    buf = np.zeros((len(tiles), th, tw, 3), np.uint8)
    for k, t in enumerate(tiles):
        tx, ty = t % tiles_x, t // tiles_x
        blk = frame[ty * th:(ty + 1) * th, tx * tw:(tx + 1) * tw]
        buf[k, :blk.shape[0], :blk.shape[1]] = blk
    return buf.reshape(-1)


def detile(gathered, w, h, tw, th, n, max_k):
    """Same index map as detile_kernel (csrc/rr_kernels.cu)."""
    tiles_x = -(-w // tw)
    out = np.zeros((h, w, 3), np.uint8)
    g = gathered.reshape(n, max_k, th, tw, 3)
    for py in range(h):
        for px in range(w):
            tile = (py // th) * tiles_x + px // tw
            out[py, px] = g[tile % n, tile // n, py % th, px % tw]
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle import Oracle
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    frame, _, _, _ = Oracle().render(cfg, W, H)          # stand-in for the device frame
    max_k = len(tiles_of_shard(W, H, T, T, 0, world))
    mine = np.zeros(max_k * T * T * 3, np.uint8)
    part = render_shard(frame, W, H, T, T, rank, world)
    mine[:part.size] = part
    t = torch.from_numpy(mine)
    bufs = [torch.zeros_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, bufs, dst=0)
    if rank == 0:
        g = torch.stack(bufs).numpy()
        q.put(bool(np.array_equal(detile(g, W, H, T, T, world, max_k), frame)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tile_shard_gather_detile_roundtrip(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5)


def test_shard_tile_counts_cover_frame_once():
    for n in (1, 2, 4, 8):
        seen = sorted(t for s in range(n) for t in tiles_of_shard(1920, 1080, 32, 32, s, n))
        assert seen == list(range(60 * 34))


def test_c_abi_tile_count_matches_host_logic():
    """rr_shard_tile_count is pure host code: callable without a GPU."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2005_05386_b200", "csrc", "librray_cuda.so"))
    for n in (1, 2, 3, 8):
        for s in range(n):
            assert lib.rr_shard_tile_count(1920, 1080, 32, 32, s, n) == \
                len(tiles_of_shard(1920, 1080, 32, 32, s, n))
    assert lib.rr_shard_tile_count(10, 10, 32, 32, 2, 2) == -1     # shard out of range
    assert lib.rr_shard_tile_count(10, 10, 32, 32, 1, 2) == 0      # one tile, two shards
