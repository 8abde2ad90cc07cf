#!/usr/bin/env python3
"""Render a few frames of one config through rr_render_device, for ncu
captures (`ncu -k regex:march_kernel -c N python tools/prof_frame.py CFG`)
and quick CUDA-event timing (`--time`).

python tools/prof_frame.py configs/c3_bumps16_1080p.json [--frames 1] [--time]
                           [--opt key=value ...] [--size WxH]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--frames", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=0)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--size", default="")
    ap.add_argument("--opt", action="append", default=[])
    a = ap.parse_args()

    import torch
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer

    r = Renderer(0)
    if a.opt:
        r.set_options(**{k: int(v) for k, v in (o.split("=", 1) for o in a.opt)})
    for path in a.configs:
        cfg = load_config(path)
        w, h = cfg.output.width, cfg.output.height
        if a.size:
            w, h = (int(x) for x in a.size.split("x"))
        r.set_config(cfg)
        cam = r.build_camera(cfg.camera)
        rgb = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
        flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        for _ in range(a.warmup):
            r.render_device(cam, cfg.integrator, w, h, rgb)
        ts = []
        st = None
        for _ in range(a.frames):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = r.render_device(cam, cfg.integrator, w, h, rgb, with_stats=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        if a.time:
            ts.sort()
            print(f"{os.path.basename(path)} {w}x{h}: median {ts[len(ts)//2]:.3f} ms "
                  f"min {ts[0]:.3f} kernel={r.last_kernel} steps={st['total_steps']} "
                  f"integrated={st.get('integrated_steps')} bump_evals={st.get('bump_evals')} "
                  f"digest={hashlib.sha1(rgb.cpu().numpy().tobytes()).hexdigest()[:12]}")
    r.close()


if __name__ == "__main__":
    main()
