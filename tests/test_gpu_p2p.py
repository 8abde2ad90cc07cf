"""GPU: the multi-process frame exchange, through the library's
own API.

* p2p: rank 0 exports its frame (rr_frame_export), every other rank imports
  it on ITS OWN context's device (rr_frame_import: cudaIpcOpenMemHandle with
  lazy peer access, peer access enabled where supported), proves the mapping
  with a device-side store (rr_frame_probe), and rr_render_shard's epilogue
  stores its tiles straight into it; on a multi-GPU node those stores travel
  over NVLink/NVSwitch.  Run on one GPU (both processes on device 0: the same
  IPC mapping and disjoint writes, the kernels never wait on each other) and,
  when the box has two or more GPUs, with rank r on device r.
* tiles: the fallback path — rr_render_tiles per rank, a gloo gather of the
  tile-major shard buffers to rank 0 and rr_detile (bench.py's NCCL gather).

The assembled frame must be byte-identical to a single-process render
(acceptance.cpp:243-253's worker-count determinism, as GPU counts)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu
W, H, T = 200, 120, 32


def _worker(rank, world, port, q, mode, spread):
    try:
        _work(rank, world, port, q, mode, spread)
    except BaseException:
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise


def _work(rank, world, port, q, mode, spread):
    import faulthandler
    import sys
    faulthandler.enable()
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    dev = rank if spread else 0
    torch.cuda.set_device(dev)
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_shadows_1080p.json"))
    r = Renderer(dev)
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    frame = torch.zeros((H, W, 3), dtype=torch.uint8, device="cuda") if rank == 0 else None
    torch.cuda.synchronize()
    if mode == "p2p":
        payload = [r.frame_export(frame) if rank == 0 else None]
        dist.broadcast_object_list(payload, src=0)
        target = frame.data_ptr() if rank == 0 else r.frame_import(payload[0])
        r.frame_probe(target, rank, 100 + rank)        # device-side store through the mapping
        dist.barrier()
        if rank == 0:
            probe = frame.view(-1)[:world].cpu().tolist()
            q.put(("probe", 0, probe == [100 + k for k in range(world)], probe))
        dist.barrier()
        r.render_shard(cam, cfg.integrator, W, H, T, T, rank, world, target)
        torch.cuda.synchronize()
        dist.barrier()
    else:
        max_k = r.shard_tile_count(W, H, T, T, 0, world)
        tiles = torch.zeros(max_k * T * T * 3, dtype=torch.uint8, device="cuda")
        r.render_tiles(cam, cfg.integrator, W, H, T, T, rank, world, tiles)
        torch.cuda.synchronize()
        bufs = [torch.zeros(tiles.numel(), dtype=torch.uint8) for _ in range(world)] if rank == 0 else None
        dist.gather(tiles.cpu(), bufs, dst=0)
        if rank == 0:
            gathered = torch.stack(bufs).cuda()
            r.detile(gathered, W, H, T, T, world, frame)
            torch.cuda.synchronize()
    if rank == 0:
        full, _ = r.render(cam, cfg.integrator, W, H)
        got = frame.cpu().numpy()
        diff = np.argwhere((got != full).any(axis=2))
        info = ""
        if len(diff):   # which shard owns the differing pixels (tile i -> shard i mod world)
            tiles_x = (W + T - 1) // T
            owners = sorted({int(((y // T) * tiles_x + x // T) % world) for y, x in diff})
            zero = int((got[diff[:, 0], diff[:, 1]] == 0).all(axis=1).sum())
            info = f"{len(diff)} px differ, owners {owners}, {zero} still zero, first {diff[0].tolist()}"
        q.put(("result", 0, not len(diff), info))
    # teardown order: consumers drop their mappings before the producer frees
    # the allocation and exits
    if mode == "p2p" and rank != 0:
        r.frame_close(target)
    dist.barrier()
    r.close()
    del frame
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, mode, spread=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode, spread)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    msgs = []
    try:   # read before join (a queue polled after join can look empty)
        while not any(m[0] == "result" for m in msgs):
            msgs.append(q.get(timeout=300))
            if msgs[-1][0] == "error":
                break
    except queue.Empty:
        pass
    for p in procs:
        p.join(300)
    errors = [m for m in msgs if m[0] == "error"]
    assert not errors, errors
    assert all(p.exitcode == 0 for p in procs), ([p.exitcode for p in procs], msgs)
    for m in msgs:
        if m[0] == "probe":
            assert m[2], m
    res = [m for m in msgs if m[0] == "result"]
    assert len(res) == 1 and res[0][2], res


@pytest.mark.parametrize("world", [2, 3])
def test_shards_write_into_exported_frame(world):
    _run(world, "p2p")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (rank r on device r)")
def test_shards_write_into_peer_device_frame():
    _run(2, "p2p", spread=True)


def test_tile_shards_gather_detile():
    _run(2, "tiles")


def test_frame_export_import_same_process():
    """A same-process import returns the exporter's address (UVA); close is a
    no-op; a probe through it lands."""
    from paper_2005_05386_b200.render import Renderer
    r = Renderer(0)
    buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    sub = buf[1024:]
    torch.cuda.synchronize()
    h = r.frame_export(sub)
    p = r.frame_import(h)
    assert p == sub.data_ptr()
    r.frame_probe(p, 5, 42)
    assert int(buf[1029].item()) == 42
    r.frame_close(p)
    r.close()


def test_frame_export_rejects_host_memory():
    """Exporting memory that is not device memory fails with a clean status
    (no crash, no mapping)."""
    import numpy as np
    from paper_2005_05386_b200.errors import Error
    from paper_2005_05386_b200.render import Renderer
    r = Renderer(0)
    host = np.zeros(4096, np.uint8)
    with pytest.raises(Error):
        r.frame_export(host.ctypes.data, host.nbytes)
    r.close()
