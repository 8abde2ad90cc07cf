"""GPU: the fused render + exchange path (rr_render_shard).  Each rank writes
its tiles straight into rank 0's frame through a CUDA-IPC mapping (on a
multi-GPU node the stores travel over NVLink/NVSwitch; here both processes
share one B200, which exercises the same IPC mapping and disjoint writes —
the kernels never wait on each other).  The assembled frame must be
byte-identical to a single-process render."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu
W, H, T = 200, 120, 32


def _worker(rank, world, port, q):
    try:
        _work(rank, world, port, q)
    except BaseException:
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise


def _work(rank, world, port, q):
    import faulthandler
    import sys
    faulthandler.enable()
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from torch.multiprocessing.reductions import reduce_tensor
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    torch.cuda.set_device(0)
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_shadows_1080p.json"))
    r = Renderer(0)
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    if rank == 0:
        frame = torch.zeros((H, W, 3), dtype=torch.uint8, device="cuda")
        # the memset runs on torch's stream; the library renders on its own
        # non-blocking stream: finish the initialisation before any shard writes
        torch.cuda.synchronize()
        payload = [reduce_tensor(frame)]
    else:
        payload = [None]
    dist.broadcast_object_list(payload, src=0)
    if rank != 0:
        fn, args = payload[0]
        frame = fn(*args)                       # IPC-mapped view of rank 0's frame
    r.render_shard(cam, cfg.integrator, W, H, T, T, rank, world, frame)
    torch.cuda.synchronize()
    dist.barrier()
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
    # teardown order: consumers drop their IPC mappings before the producer
    # frees the allocation and exits
    if rank != 0:
        del frame
        torch.cuda.synchronize()
    dist.barrier()
    r.close()
    if rank == 0:
        del frame
        torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_write_into_shared_frame():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
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
    res = [m for m in msgs if m[0] == "result"]
    assert len(res) == 1 and res[0][2], res
