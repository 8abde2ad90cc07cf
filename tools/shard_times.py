#!/usr/bin/env python3
"""Device time of one shard of an N-way tile split on one GPU (the per-GPU
work of the multi-GPU run, exchange excluded): rr_render_tiles(shard, N),
CUDA events, L2 flushed.
python tools/shard_times.py [config] [--frames K] [--tile T] [--all] [option=value ...]
(--all times every shard; default the first and the last)"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    cfgs = [a for a in sys.argv[1:] if a.endswith(".json")]
    path = cfgs[0] if cfgs else os.path.join(ROOT, "configs", "c3_bumps16_1080p.json")
    frames = int(sys.argv[sys.argv.index("--frames") + 1]) if "--frames" in sys.argv else 10
    cfg = load_config(path)
    cfg.scene.lights = []
    T = int(sys.argv[sys.argv.index("--tile") + 1]) if "--tile" in sys.argv else 32
    w, h = cfg.output.width, cfg.output.height
    r = Renderer(0)
    for o in [a for a in sys.argv if "=" in a]:     # rr_options, e.g. order_units=0
        k, v = o.split("=", 1)
        r.set_options(**{k: int(v)})
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()       # a real stream: NULL would select the context's own
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    base = None
    for n in (1, 2, 4, 8):
        worst = 0.0
        for shard in (range(n) if "--all" in sys.argv else sorted({0, n - 1})):
            k = r.shard_tile_count(w, h, T, T, shard, n)
            tiles = torch.zeros(k * T * T * 3, dtype=torch.uint8, device="cuda")
            ts = []
            for i in range(frames + 2):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                r.render_tiles(cam, cfg.integrator, w, h, T, T, shard, n, tiles, stream=sp)
                b.record(stream)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(a.elapsed_time(b))
            worst = max(worst, statistics.median(ts))
        base = base or worst
        print(f"{os.path.basename(path)} T={T} N={n}: slowest shard {worst:.3f} ms  "
              f"ideal {base / n:.3f} ms  efficiency {base / n / worst:.3f}", flush=True)


if __name__ == "__main__":
    main()
