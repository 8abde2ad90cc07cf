"""`python -m paper_2005_05386_b200` — the rray CLI render path on B200.

Mirrors /root/reference/proj/tools/rray_main.cpp:
  render CONFIG [-o PATH] [--h H] [--size WxH] [--print-config]
      -> PPM image + `<stem>.report.txt` sidecar (rray_main.cpp:53-83),
         one summary line on stdout, exit codes 0 ok / 1 config / 2 numeric /
         3 I/O (rray_main.cpp:185-194).
plus the B200 extension
  animate CONFIG --frames N [...]
      -> BASELINE configs[4] driver: time-varying Gaussian bumps
         c_j(t) = c_j + A (sin(w t + phi_j), cos(w t + phi_j), 0),
         phi_j = 2 pi j / N_bumps, t = frame / fps; every frame is a static
         reference-schema scene (uploaded per frame), rendered on the GPU.
and, off the render hot path, on the same device code
  geodesic CONFIG --start x,y,z --dir x,y,z [-o CSV] [--h H]
      -> trace_geodesic polyline as CSV (rray_main.cpp:86-116) from rr_trace
  verify [--seed N]
      -> the property suites restated on the device arithmetic
         (verify.py; rray_main.cpp:118-131), exit 0 iff all pass, else 2.
"""
from __future__ import annotations

import argparse
import copy
import math
import os
import sys
import time

from . import config as cfgmod
from .errors import ConfigError, Error, IoError, NumericError, ValidationError


def _size(s: str):
    try:
        w, h = s.lower().split("x")
        w, h = int(w), int(h)
    except ValueError:
        raise ValidationError(f"--size expects WxH, got '{s}'") from None
    if w < 1 or h < 1:
        raise ValidationError(f"--size expects WxH, got '{s}'")
    return w, h


def report_path(output_path: str) -> str:
    """rray_main.cpp:47-51."""
    stem, dot, _ = output_path.rpartition(".")
    return (stem if dot else output_path) + ".report.txt"


def _load(args) -> cfgmod.RunConfig:
    cfg = cfgmod.load_config(args.config)
    if getattr(args, "output", None):
        cfg.output.path = args.output
    if getattr(args, "h", 0.0) and args.h > 0.0:
        cfg.integrator.h = args.h
    if getattr(args, "size", None):
        cfg.output.width, cfg.output.height = _size(args.size)
    return cfg


def cmd_render(cfg: cfgmod.RunConfig, device: int = 0) -> int:
    """rray_main.cpp:53-83 on the GPU (one launch per frame; lit frames two)."""
    from .render import Image, Renderer, write_ppm
    t0 = time.perf_counter()
    r = Renderer(device)
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    rgb, st = r.render(cam, cfg.integrator, cfg.output.width, cfg.output.height)
    wall = time.perf_counter() - t0
    kernel = r.last_kernel
    r.close()
    write_ppm(Image(cfg.output.width, cfg.output.height, rgb), cfg.output.path)
    rays = cfg.output.width * cfg.output.height
    avg = st["total_steps"] / rays
    rpath = report_path(cfg.output.path)
    try:
        with open(rpath, "w") as f:
            f.write(f"image: {cfg.output.path}\n"
                    f"wall_seconds: {wall}\n"
                    f"rays: {rays}\n"
                    f"avg_steps_per_ray: {avg}\n"
                    f"pixel_errors: {st['pixel_errors']}\n"
                    f"kernel: cuda ({kernel})\n"
                    f"device_ms: {st['device_ms']}\n"
                    f"shadow_steps: {st['shadow_steps']}\n"
                    f"config:\n{cfgmod.serialize_config(cfg)}")
    except OSError:
        raise IoError(f"cannot open report '{rpath}' for writing") from None
    print(f"{cfg.output.path}: {cfg.output.width}x{cfg.output.height}, {wall:g} s, "
          f"{avg:g} steps/ray, {st['pixel_errors']} pixel errors")
    return 0


def _vec3(s: str, flag: str):
    """rray_main.cpp:38-45."""
    parts = s.split(",")
    try:
        if len(parts) != 3:
            raise ValueError
        return [float(x) for x in parts]
    except ValueError:
        raise ValidationError(f"{flag} expects x,y,z, got '{s}'") from None


def cmd_geodesic(cfg: cfgmod.RunConfig, start, direction, out_path: str, device: int = 0) -> int:
    """rray_main.cpp:86-116: one geodesic polyline as CSV, traced on the device."""
    import numpy as np
    from .render import Renderer
    try:
        f = open(out_path, "w")
    except OSError:
        raise IoError(f"cannot open '{out_path}' for writing") from None
    with f:
        f.write("t,x,y,z,vx,vy,vz\n")
        row = lambda t, st: f.write(",".join(f"{v:.17g}" for v in (t, *st)) + "\n")
        r = Renderer(device)
        try:
            r.set_config(cfg)
            g = r.metric_tensor(np.array(start, np.float64))
            d = np.array(direction, np.float64)
            ln = float(np.sqrt(d @ g @ d))
            if ln == 0.0:
                row(0.0, [*start, *direction])
                print("warning: zero direction, wrote the start state only", file=sys.stderr)
                return 0
            s0 = np.concatenate([np.array(start, np.float64), d / ln])
            states, counts, fail = r.trace(cfg.integrator, s0[None, :], use_bounds=True)
        finally:
            r.close()
        if fail[0] >= 0:
            raise NumericError("trace_geodesic: metric evaluation failed (|det J| <= 1e-14) "
                               f"at step {int(fail[0])}")
        h = cfg.integrator.h
        for i in range(int(counts[0])):
            row(i * h, states[0, i])
    print(f"{out_path}: {int(counts[0])} states, h = {h:g}")
    return 0


ANIMATION_CULL_GRID = 192   # culling-grid resolution for per-frame scene changes


def animated_config(cfg: cfgmod.RunConfig, frame: int, fps: float, omega: float,
                    amp: float) -> cfgmod.RunConfig:
    """Frame `frame` of the BASELINE configs[4] bump animation (static scene)."""
    out = copy.deepcopy(cfg)
    if not isinstance(out.metric, cfgmod.GraphMetric):
        raise ValidationError("animate: metric must be a graph of Gaussian bumps")
    leaves = []

    def walk(f):
        if isinstance(f, cfgmod.GaussianField):
            leaves.append(f)
        elif isinstance(f, cfgmod.SumField):
            for t in f.terms:
                walk(t)
    walk(out.metric.field)
    t = frame / fps
    n = max(1, len(leaves))
    for j, g in enumerate(leaves):
        phi = 2.0 * math.pi * j / n
        c = g.params.center
        g.params.center = [c[0] + amp * math.sin(omega * t + phi),
                           c[1] + amp * math.cos(omega * t + phi), c[2]]
    return out


def cmd_animate(cfg: cfgmod.RunConfig, frames: int, fps: float, omega: float, amp: float,
                pattern: str | None, device: int = 0) -> int:
    from .render import Image, Renderer, write_ppm
    r = Renderer(device)
    # every frame is a new scene, so the culling grid is rebuilt per frame:
    # 192^3 rebuilds in ~0.1 ms, the static-frame default 256^3 in ~1.9 ms
    # (profiles/r2z_grid_ab.log)
    r.set_options(cull_grid=ANIMATION_CULL_GRID)
    cam = None
    w, h = cfg.output.width, cfg.output.height
    t0 = time.perf_counter()
    total_steps = 0
    for k in range(frames):
        fc = animated_config(cfg, k, fps, omega, amp)
        r.set_config(fc)                      # per-frame scene upload (+ culling grid)
        if cam is None:
            cam = r.build_camera(fc.camera)
        rgb, st = r.render(cam, fc.integrator, w, h)
        total_steps += st["total_steps"]
        if pattern:
            write_ppm(Image(w, h, rgb), pattern % k)
    wall = time.perf_counter() - t0
    r.close()
    print(f"animate: {frames} frames {w}x{h}, {wall:g} s, {frames / wall:.2f} fps, "
          f"{total_steps / wall:.4g} steps/s")
    return 0


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="rray-b200",
                                description="B200 ray tracer for designed Riemannian metrics on R^3")
    sub = p.add_subparsers(dest="cmd", required=True)
    pr = sub.add_parser("render", help="render a scene to a PPM image")
    pr.add_argument("config")
    pr.add_argument("-o", "--output")
    pr.add_argument("--h", type=float, default=0.0)
    pr.add_argument("--size")
    pr.add_argument("--print-config", action="store_true")
    pr.add_argument("--device", type=int, default=int(os.environ.get("RRAY_CUDA_DEVICE", "0")))
    pa = sub.add_parser("animate", help="render a time-varying bump animation (configs[4])")
    pa.add_argument("config")
    pa.add_argument("--frames", type=int, default=8)
    pa.add_argument("--fps", type=float, default=30.0)
    pa.add_argument("--omega", type=float, default=2.0)
    pa.add_argument("--amp", type=float, default=0.3)
    pa.add_argument("-o", "--output", help="printf pattern for frames, e.g. frame_%%04d.ppm")
    pa.add_argument("--size")
    pa.add_argument("--h", type=float, default=0.0)
    pa.add_argument("--device", type=int, default=0)
    pg = sub.add_parser("geodesic", help="export one geodesic polyline as CSV")
    pg.add_argument("config")
    pg.add_argument("--start", required=True)
    pg.add_argument("--dir", required=True)
    pg.add_argument("-o", "--output", default="geodesic.csv")
    pg.add_argument("--h", type=float, default=0.0)
    pg.add_argument("--print-config", action="store_true")
    pg.add_argument("--device", type=int, default=0)
    pv = sub.add_parser("verify", help="run the numerical property suites (on the device)")
    pv.add_argument("--seed", type=int, default=42)
    pv.add_argument("--device", type=int, default=0)
    args = p.parse_args(argv)
    try:
        if args.cmd == "verify":
            from .verify import cmd_verify
            return cmd_verify(args.seed, args.device)
        if args.cmd == "geodesic":
            out_path = args.output
            args.output = None                    # -o is the CSV, not output.path
            cfg = _load(args)
            if args.print_config:
                sys.stdout.write(cfgmod.serialize_config(cfg))
                return 0
            return cmd_geodesic(cfg, _vec3(args.start, "--start"), _vec3(args.dir, "--dir"),
                                out_path, args.device)
        if args.cmd == "render":
            cfg = _load(args)
            if args.print_config:
                sys.stdout.write(cfgmod.serialize_config(cfg))
                return 0
            return cmd_render(cfg, args.device)
        cfg = _load(args)
        return cmd_animate(cfg, args.frames, args.fps, args.omega, args.amp, args.output,
                           args.device)
    except ConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except IoError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except NumericError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
