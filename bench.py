#!/usr/bin/env python3
"""Benchmark of the per-pixel geodesic tracing hot path on B200.

Workload (BASELINE.json configs[2], primary rays): 1920x1080, graph metric of
16 accumulated Gaussian bumps (SURVEY.md Appendix B literal values), sphere +
sphere + floor scene, RK4 h=0.05, max 400 steps (configs/c3_bumps16_1080p.json).
A "step" of this benchmark is one whole frame: raygen -> metric -> RK4 ->
intersection -> shading for all 2,073,600 pixels.

  value  = geodesic RK4 steps/s, steps counted exactly as the reference's
           RenderStats.total_steps (sum of PixelOutcome.steps), device-timed
           with CUDA events around each frame's launch, inputs resident.
  e2e    = the same metric through the public API with host buffers: scene
           upload + camera + rr_render (frame D2H into pinned host memory).
  fps    = frames per second of `value`'s timing.

python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Under torchrun (N>1) every rank renders a cyclic share of 32x32 tiles and its
shade epilogue stores them straight into rank 0's frame (CUDA IPC over
NVLink; one 4-byte NCCL all-reduce per frame as the completion barrier), with
an NCCL gather + de-tile fallback.  The roofline is per GPU (rank 0's shard).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = os.path.join(ROOT, "configs", "c3_bumps16_1080p.json")
SHADOW_CONFIG = os.path.join(ROOT, "configs", "c3_bumps16_shadows_1080p.json")
WORKLOAD = "c3_bumps16_1080p"
METRIC = "geodesic RK4 steps/s (1920x1080, 16 Gaussian bumps, RK4 h=0.05)"
UNIT = "steps/s"
TILE = 32
# SURVEY App. A algorithmic FLOP accounting (FMA = 2): per Gaussian term per
# accel evaluation 36, fixed per accel evaluation 13, RK4 combination 78,
# chord test of the sphere+sphere+floor scene 58 per step.
FLOP_BUMP, FLOP_ACCEL, FLOP_RK4, FLOP_ISECT = 36, 13, 78, 58
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 at max clock


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", default=CONFIG)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-shadows", action="store_true")
    p.add_argument("--no-parity", action="store_true",
                   help="skip the untimed full-frame parity checks against the reference / oracle")
    p.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                   help="gloo: host-synchronised collectives (dry runs of the N>1 path on fewer GPUs)")
    p.add_argument("--no-extras", action="store_true",
                   help="skip the secondary workloads (C1, C2, C4+mesh, C5 4K, C3 rk23)")
    p.add_argument("--cpu-row-step", type=int, default=0, help="reference row subsample (0=auto)")
    p.add_argument("--opt", action="append", default=[],
                   help="renderer option key=value (rr_options field), e.g. cull_grid=64")
    return p.parse_args()


# ---- clocks sampling (B200_PROFILING.md clocks line) ---------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- reference CPU path (oracle/_ref = the reference compiled from its sources) ---
def reference_sample(cfg, row_step: int):
    from oracle import Reference
    ref = Reference()
    w, h = cfg.output.width, cfg.output.height
    cores = ref.hardware_concurrency()
    if row_step <= 0:
        # calibrate to ~10 s of work: time every 135th row first
        _, st = ref.render_rows(cfg, w, h, 0, 135, kernel="avx2", workers=cores)
        per_row = st["wall_seconds"] / max(1, len(range(0, h, 135)))
        row_step = max(1, min(h, int(math.ceil(h * per_row / 10.0))))
    _, st = ref.render_rows(cfg, w, h, 0, row_step, kernel="avx2", workers=cores)
    rows = len(range(0, h, row_step))
    return {
        "steps_per_s": st["total_steps"] / st["wall_seconds"],
        "wall_s": st["wall_seconds"],
        "rows": rows,
        "row_step": row_step,
        "cores": st["workers"],
        "fps_extrapolated": (rows / h) / st["wall_seconds"],
        "sample": f"every {row_step}th row ({rows} of {h} rows, {rows * w} rays) of the same frame, "
                  f"reference render() row work items, KernelKind::Avx2, {st['workers']} threads",
    }


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals, walls, info = [], [], None
    for i in range(args.warmup + args.steps):
        info = reference_sample(cfg, args.cpu_row_step if i else args.cpu_row_step)
        if args.cpu_row_step <= 0:
            args.cpu_row_step = info["row_step"]
        if i >= args.warmup:
            vals.append(info["steps_per_s"])
            walls.append(info["wall_s"])
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(walls), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "width": cfg.output.width, "height": cfg.output.height,
                   "bumps": 16, "scheme": cfg.integrator.scheme, "h": cfg.integrator.h,
                   "max_steps": cfg.integrator.max_steps, "shadows": False},
        "fps": info["fps_extrapolated"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "reference",
                         "sample": info["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- own arm ----------------------------------------------------------------------
def algorithmic_flops(stats, scheme):
    """SURVEY App. A per integrated step: RK4 combination + 4 fixed accel
    terms + 36 per evaluated bump, and the chord test.  A straight jump
    through metric-free space (jump_steps) is charged its chord test only:
    no RK4 or metric work runs for it."""
    evals_per_step = 4 if scheme == "rk4" else 1
    comb = FLOP_RK4 if scheme == "rk4" else 12
    steps = stats["integrated_steps"]
    rk = steps - stats.get("jump_steps", 0) - stats.get("shadow_jump_steps", 0)
    return (stats["bump_evals"] * FLOP_BUMP + rk * (evals_per_step * FLOP_ACCEL + comb) +
            steps * FLOP_ISECT)


def simt(stats):
    """Lane efficiency of the persistent warp loop: integrated ray-steps per
    lane slot (32 x warp loop iterations), per pass."""
    out = {}
    prim = stats["integrated_steps"] - stats["shadow_integrated_steps"]
    if stats["lane_slots"]:
        out["primary"] = prim / stats["lane_slots"]
    if stats["shadow_lane_slots"]:
        out["shadow"] = stats["shadow_integrated_steps"] / stats["shadow_lane_slots"]
    return out


def rk4_steps(st):
    """Integrated steps that ran the integrator (straight jumps excluded)."""
    return st["integrated_steps"] - st["jump_steps"] - st["shadow_jump_steps"]


def spill_report():
    """ptxas -v registers / spill bytes of the dominant kernels
    (paper_2005_05386_b200/csrc/ptxas.log, written by the build)."""
    import re
    path = os.path.join(ROOT, "paper_2005_05386_b200", "csrc", "ptxas.log")
    want = {"march2_kernel<bumps16> (C3 frame)": "march2_kernelILi1ELi16ELi0ELb0EE",
            "march2_kernel<bumps16> lit hit records (C3 + lights)": "march2_kernelILi1ELi16ELi1ELb0EE",
            "march2_kernel<bumps16> lit shadows (C3 + lights)": "march2_kernelILi1ELi16ELi2ELb0EE",
            "march2_kernel<bumps16,rk23>": "march2_kernelILi4ELi16ELi0ELb0EE",
            "march2_kernel<twist> (C4)": "march2_kernelILi3ELi0ELi0ELb0EE",
            "march_kernel<diffeo,mesh> (C4 + mesh, static twist)": "march_kernelILi3ELi1ELi1ELi0ELb1EE",
            "march2_kernel<chain,mesh> (C4 bend + mesh, static fold)": "march2_kernelILi5ELi306ELi0ELb1EE"}
    out = {}
    try:
        lines = open(path).read().split("\n")
    except OSError:
        return None
    cur = None
    for i, ln in enumerate(lines):
        m = re.search(r"Compiling entry function '(\S+)'", ln)
        if m:
            cur = m.group(1)
            continue
        for label, key in want.items():
            if cur and key in cur and "Used" in ln and "registers" in ln:
                regs = int(re.search(r"Used (\d+) registers", ln).group(1))
                sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", lines[i - 1])
                out[label] = {"registers": regs, "spill_stores": int(sp.group(1)) if sp else 0,
                              "spill_loads": int(sp.group(2)) if sp else 0}
    return out


def e2e_frames(r, cfg, w, h, n, steps_of):
    """The metric end to end through the public host API: per frame the scene
    upload (unchanged scene: parameter-block compare, no re-upload), camera
    build and rr_render into PINNED host memory (the kernel's 16-B stores
    travel straight into it), stats read back."""
    import torch
    host = torch.empty((h, w, 3), dtype=torch.uint8).pin_memory()
    r.set_config(cfg)
    r.render(r.build_camera(cfg.camera), cfg.integrator, w, h, out=host)   # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r.set_config(cfg)                              # scene upload (params + cull grid)
        cam_e = r.build_camera(cfg.camera)
        _, est = r.render(cam_e, cfg.integrator, w, h, out=host)  # frame -> pinned host + stats
    e2e_s = (time.perf_counter() - t0) / n
    # per frame host->device: the kernel parameter blocks (scene program +
    # camera); device->host: the frame + the stats block
    info = r.lib.rr_build_info().decode()
    param_bytes = int(info.split("param_bytes=")[1].split()[0]) if "param_bytes=" in info else 0
    return {"value": steps_of(est) / e2e_s, "unit": UNIT, "h2d_bytes_per_step": param_bytes,
            "d2h_bytes_per_step": 3 * w * h + 8 * 11, "fps": 1.0 / e2e_s,
            "output": "kernel stores into pinned host memory (UVA)"}


def cpu_sample(kind, cfg, w, h, target_s=4.0, kernel="avx2", workers=0):
    """A bounded CPU sample of a workload (~target_s of host time): every k-th
    row of the same frame, k calibrated on a sparse pass.  kind "reference":
    the reference's own render() row work item (oracle/_ref); kind "oracle":
    the FP64 oracle extension (oracle/rro.c) for paths the reference lacks
    (shadow geodesics, meshes, rk23).  steps/s counts reference-equivalent
    steps (primary + shadow)."""
    try:
        from oracle import Oracle, Reference
        if kind == "reference":
            lib = Reference()

            def run(step):
                _, st = lib.render_rows(cfg, w, h, 0, step, kernel=kernel, workers=workers)
                return st["wall_seconds"], st["total_steps"], st["workers"]
        else:
            lib = Oracle()

            def run(step):
                _, _, st = lib.render_rows(cfg, w, h, 0, step, threads=workers)
                return st["wall_seconds"], st["total_steps"] + st["shadow_steps"], workers or lib.threads
        step0 = max(1, h // 64)
        wall, _, _ = run(step0)
        per_row = wall / len(range(0, h, step0))
        step = max(1, min(h, math.ceil(h * per_row / target_s)))
        # at least 4 rows per thread: the row is the work item, and a sample
        # of fewer rows than threads would under-report the CPU's throughput
        threads = workers or os.cpu_count() or 1
        step = max(1, min(step, h // (4 * threads)))
        wall, steps, cores = run(step)
        rows = len(range(0, h, step))
        label = (f"reference render() row work items, KernelKind::{kernel.capitalize()}"
                 if kind == "reference" else
                 "FP64 oracle extension (oracle/rro.c; the reference has no counterpart)")
        return {"value": steps / wall, "unit": UNIT, "cores": cores,
                "kind": "reference" if kind == "reference" else "port",
                "sample": f"every {step}th row ({rows} of {h} rows, {rows * w} rays) of the same "
                          f"frame, {label}, {cores} threads",
                "fps_extrapolated": (rows / h) / wall, "wall_s": wall}
    except Exception as e:   # checker build absent on this box
        return {"value": None, "unit": UNIT, "cores": 0, "kind": kind, "sample": f"unavailable: {e}"}


def frame_parity(r, cfg, w, h, kind, row_step=1):
    """Untimed per-pixel parity of the benchmarked frame: the production frame
    kernel with its PixelOutcome sink (rr_render_outcomes) against the
    reference's own MarchFn (kind "reference", AVX2, all host threads) or the
    FP64 oracle (kind "oracle": the shadow extension), every row_step-th row;
    flags (GRAZING / LIMIT / SHADOW exemptions) computed by the oracle for the
    differing pixels (oracle.parity.check_frame)."""
    t0 = time.perf_counter()
    try:
        import numpy as np
        from oracle import Oracle, Reference
        from oracle.parity import check_frame
        r.set_config(cfg)
        cam = r.build_camera(cfg.camera)
        rgb, out, _ = r.render_outcomes(cam, cfg.integrator, w, h)
        kern = r.last_kernel
        orc = Oracle()
        if kind == "reference":
            ref_rgb, ref_out, _ = Reference().render_rows(cfg, w, h, 0, row_step, kernel="avx2",
                                                          with_outcomes=True)
        else:
            ref_rgb, ref_out, _ = orc.render_rows(cfg, w, h, 0, row_step)
        rows = np.arange(0, h, row_step)
        g_out = out.reshape(h, w)[::row_step].reshape(-1)
        g_rgb = rgb[::row_step]

        def flag_fn(idx):
            pix = rows[idx // w].astype(np.int64) * w + idx % w
            return orc.flags_pixels(cfg, w, h, pix, ref_out[idx])

        rep, _, cand = check_frame(g_out, ref_out, g_rgb, ref_rgb, flag_fn)
        return {"ok": rep.ok, "pixels": rep.n, "rows": f"every {row_step} of {h}",
                "against": ("reference MarchFn (oracle/_ref, KernelKind::Avx2)" if kind == "reference"
                            else "FP64 oracle extension (oracle/rro.c)"),
                "kernel": kern + " + PixelOutcome sink",
                "status_mm": rep.status_mismatch, "prim_mm": rep.prim_mismatch,
                "endpoint_max": rep.endpoint_max_rel, "endpoint_p99": rep.endpoint_p99_rel,
                "endpoint_fail": rep.endpoint_fail, "rgb_max": rep.rgb_max, "rgb_fail": rep.rgb_fail,
                "magenta": [rep.magenta_gpu, rep.magenta_ref], "exempt": rep.exempt,
                "flagged_candidates": cand, "host_s": time.perf_counter() - t0}
    except Exception as e:
        return {"ok": None, "unavailable": f"{type(e).__name__}: {e}"}


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except OSError:
        return {}


def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2005_05386_b200.render import Renderer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    gloo = args.dist_backend == "gloo"
    cdev = "cpu" if gloo else "cuda"     # device of the collectives' tensors
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w, h = cfg.output.width, cfg.output.height
    integ = cfg.integrator
    r = Renderer(local)
    if args.opt:
        r.set_options(**{k: type(r.options()[k])(v) for k, v in (o.split("=", 1) for o in args.opt)})
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    # a dedicated (non-NULL) stream: NULL selects the context's own stream in the C-ABI
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def device_time(fn, n, warm):
        """CUDA-event times (ms) of n calls of fn on the bench stream, L2
        flushed (untimed) before each."""
        for _ in range(warm):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(n)]
        torch.cuda.synchronize()
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    frame = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
    exchange = None
    if world > 1:
        # Fused render + exchange (default): rank 0 shares its frame through a
        # CUDA-IPC handle; every rank's shade epilogue stores its tiles straight
        # into it over NVLink/NVSwitch; one tiny NCCL all-reduce per frame is
        # the completion barrier.  Fallback: tile buffers + one NCCL gather +
        # detile on rank 0.
        exchange = "p2p-epilogue"
        target = frame.data_ptr()
        ok = 1
        try:
            # library-owned mapping (rr_frame_export / rr_frame_import on this
            # rank's own device, peer access enabled where supported)
            payload = [r.frame_export(frame) if rank == 0 else None]
            dist.broadcast_object_list(payload, src=0)
            if rank != 0:
                target = r.frame_import(payload[0])
            torch.cuda.synchronize()
            dist.barrier()
            r.frame_probe(target, rank, rank + 1)     # device-side store through the mapping
        except Exception:
            ok = 0
        dist.barrier()
        if rank == 0 and ok:
            ok = int(frame.view(-1)[:world].cpu().tolist() == list(range(1, world + 1)))
        okt = torch.tensor([ok], device=cdev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if int(okt.item()) == 0:
            exchange = "nccl-gather"
        done = torch.zeros(1, device=cdev)
        max_k = r.shard_tile_count(w, h, TILE, TILE, 0, world)
        tiles = torch.zeros(max_k * TILE * TILE * 3, dtype=torch.uint8, device="cuda")
        gathered = torch.empty((world, tiles.numel()), dtype=torch.uint8, device="cuda") if rank == 0 else None

    def one_frame():
        if world == 1:
            r.render_device(cam, integ, w, h, frame, stream=sp)
        elif exchange == "p2p-epilogue":
            r.render_shard(cam, integ, w, h, TILE, TILE, rank, world, target, stream=sp)
            if gloo:
                torch.cuda.synchronize()
            dist.all_reduce(done)     # completion barrier: rank 0's frame is whole after it
        else:
            r.render_tiles(cam, integ, w, h, TILE, TILE, rank, world, tiles, stream=sp)
            if gloo:
                torch.cuda.synchronize()
                g_cpu = [torch.empty_like(tiles, device="cpu") for _ in range(world)] if rank == 0 else None
                dist.gather(tiles.cpu(), g_cpu, dst=0)
                if rank == 0:
                    gathered.copy_(torch.stack(g_cpu))
            else:
                dist.gather(tiles, list(gathered.unbind(0)) if rank == 0 else None, dst=0)
            if rank == 0:
                r.detile(gathered, w, h, TILE, TILE, world, frame, stream=sp)

    for _ in range(args.warmup):
        one_frame()
    torch.cuda.synchronize()

    # ---- device-timed region: K frames, L2 flushed between frames (untimed)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            one_frame()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    times_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(times_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # ---- per-frame work accounting (deterministic; one extra stats frame)
    if world == 1:
        st = r.render_device(cam, integ, w, h, frame, stream=sp, with_stats=True)
    else:
        st = r.render_tiles(cam, integ, w, h, TILE, TILE, rank, world, tiles, stream=sp,
                            with_stats=True)
        st_local = dict(st)
        keys = ["total_steps", "integrated_steps", "bump_evals", "pixel_errors", "lane_slots",
                "jump_steps", "shadow_jump_steps", "shadow_integrated_steps", "shadow_lane_slots"]
        t = torch.tensor([st[k] for k in keys], dtype=torch.float64, device=cdev)
        dist.all_reduce(t)
        st.update({k: int(v) for k, v in zip(keys, t.tolist())})
    steps_per_frame = st["total_steps"]
    value = steps_per_frame * args.steps / (total_ms * 1e-3)
    fps = args.steps / (total_ms * 1e-3)

    # roofline of the march kernel (the dominant kernel): algorithmic FLOP per
    # launch / mean launch time, per GPU (N > 1: this rank's shard and its own
    # launch time against its own GPU's peak)
    kernel_ms = statistics.mean(times_ms)
    flop_launch = algorithmic_flops(st if world == 1 else st_local, integ.scheme)
    peak = r.fp32_peak_tflops()
    achieved = flop_launch / (kernel_ms * 1e-3) / 1e12
    traffic = load_traffic().get(r.last_kernel)

    # ---- dispatch-order ablation (single GPU): the timed frames dispatch ray-
    #      pair units expensive-first using the previous frame's per-unit costs
    #      (rr_options.order_units, temporal coherence; outputs unaffected);
    #      the same frame with the plain tile order, for comparison
    unit_order = None
    if world == 1:
        r.set_options(order_units=0)
        off_ms = statistics.mean(device_time(lambda: r.render_device(cam, integ, w, h, frame, stream=sp),
                                             max(3, args.steps // 2), 1))
        r.set_options(order_units=1)
        r.set_config(cfg)
        unit_order = {"timed_frames": "expensive-first (previous frame's unit costs)",
                      "ms_per_frame_plain_order": off_ms}

    # ---- EXTENSION: the north-star frame — the same 1080p frame with shadow
    #      geodesics to 2 point lights (BASELINE configs[2] as specified), one
    #      hit-record launch + shadow launch, device-timed the same way, with its own roofline,
    #      e2e, CPU baseline (FP64 oracle extension) and parity
    shadows = None
    single = world == 1
    if single and not args.no_shadows:
        from paper_2005_05386_b200.config import load_config
        scfg = load_config(SHADOW_CONFIG)
        r.set_config(scfg)
        scam = r.build_camera(scfg.camera)
        sms = device_time(lambda: r.render_device(scam, scfg.integrator, w, h, frame, stream=sp),
                          args.steps, max(2, args.warmup))
        sst = r.render_device(scam, scfg.integrator, w, h, frame, stream=sp, with_stats=True)
        s_ms = statistics.mean(sms)
        s_flop = algorithmic_flops(sst, integ.scheme)
        s_ach = s_flop / (s_ms * 1e-3) / 1e12
        shadows = {"workload": "c3_bumps16_shadows_1080p", "lights": len(scfg.scene.lights),
                   "ms_per_frame": s_ms, "fps": 1e3 / s_ms,
                   "primary_steps": sst["total_steps"], "shadow_steps": sst["shadow_steps"],
                   "integrated_steps": sst["integrated_steps"],
                   "steps_per_s": (sst["total_steps"] + sst["shadow_steps"]) / (s_ms * 1e-3),
                   "rk4_steps_per_s": rk4_steps(sst) / (s_ms * 1e-3),
                   "roofline": {"bound": "fp32", "achieved": s_ach, "peak": peak, "unit": "TFLOP/s",
                                "frac": s_ach / peak, "frac_nominal": s_ach / NOMINAL_FP32_TFLOPS,
                                "traffic": load_traffic().get(r.last_kernel + "+lights"),
                                "flop_per_launch": s_flop,
                                "kernel": r.last_kernel + " (lit: hit-record + shadow launches)"},
                   "simt_efficiency": simt(sst),
                   "launches_per_frame": sst["kernel_launches"],
                   "e2e": e2e_frames(r, scfg, w, h, max(3, args.steps),
                                     lambda st: st["total_steps"] + st["shadow_steps"])}
        if not args.no_cpu_baseline:
            shadows["cpu_baseline"] = cpu_sample("oracle", scfg, w, h)
        if not args.no_parity:
            shadows["parity"] = frame_parity(r, scfg, w, h, "oracle", row_step=4)
        r.set_config(cfg)

    # ---- the other BASELINE.json configs, device-timed the same way (secondary)
    extras = None
    if single and not args.no_extras:
        from paper_2005_05386_b200.config import load_config
        extras = {}
        for name, cpu_kind in (("c1_gauss1_512", "reference"), ("c2_flat_1080p", "reference"),
                               ("c4_twist_1080p", "reference"), ("c4_twist_mesh_1080p", "oracle"),
                               ("c4_twist_bend_mesh_1080p", "oracle"),
                               ("c5_bumps16_4k", "reference"), ("c3_bumps16_rk23_1080p", "oracle")):
            ecfg = load_config(os.path.join(ROOT, "configs", name + ".json"))
            ew, eh = ecfg.output.width, ecfg.output.height
            ebuf = torch.empty((eh, ew, 3), dtype=torch.uint8, device="cuda")
            r.set_config(ecfg)
            ecam = r.build_camera(ecfg.camera)
            # median of 5 frames after 3 warm-ups (the first warm-up records the
            # unit costs the dispatch order of the next frames uses)
            ems = statistics.median(device_time(
                lambda: r.render_device(ecam, ecfg.integrator, ew, eh, ebuf, stream=sp), 5, 3))
            est = r.render_device(ecam, ecfg.integrator, ew, eh, ebuf, stream=sp, with_stats=True)
            ent = {"size": f"{ew}x{eh}", "scheme": ecfg.integrator.scheme,
                   "h": ecfg.integrator.h, "max_steps": ecfg.integrator.max_steps,
                   "ms_per_frame": ems, "fps": 1e3 / ems, "timing": "median of 5 frames, 3 warm-up, L2 flushed",
                   "steps_per_s": est["total_steps"] / (ems * 1e-3),
                   "integrated_steps_per_s": est["integrated_steps"] / (ems * 1e-3),
                   "avg_steps_per_ray": est["total_steps"] / (ew * eh),
                   "simt_efficiency": simt(est),
                   "kernel": r.last_kernel}
            mkind = type(ecfg.metric).__name__          # EuclideanMetric / GraphMetric / DiffeoMetric
            if mkind == "EuclideanMetric":
                # Euclidean rays jump straight to their exit/hit: the reference-
                # equivalent steps/s is mostly skipped work, not throughput
                ent["note"] = ("steps_per_s counts reference-equivalent steps; Gamma = 0 rays "
                               "jump straight to their exit or hit (integrated_steps_per_s is "
                               "the work done)")
            else:
                ent["rk4_steps_per_s"] = rk4_steps(est) / (ems * 1e-3)
                eflop = algorithmic_flops(est, ecfg.integrator.scheme)
                if mkind == "GraphMetric":
                    ent["achieved_tflops"] = eflop / (ems * 1e-3) / 1e12
                    ent["frac"] = ent["achieved_tflops"] / peak
            if not args.no_cpu_baseline:
                ent["cpu_baseline"] = cpu_sample(cpu_kind, ecfg, ew, eh)
            extras[name] = ent
            del ebuf
        # BASELINE configs[4] as an animation: every frame a NEW scene (bump
        # centres move, cli.animated_config), so each frame pays the scene
        # upload and the device culling-grid rebuild before its render.
        # Wall clock per frame (host upload work included), device-synchronised.
        from paper_2005_05386_b200.cli import ANIMATION_CULL_GRID, animated_config
        acfg = load_config(os.path.join(ROOT, "configs", "c5_bumps16_4k.json"))
        grid0 = r.options()["cull_grid"]
        r.set_options(cull_grid=ANIMATION_CULL_GRID)    # as `animate` does: the grid is rebuilt per frame
        aw, ah = acfg.output.width, acfg.output.height
        abuf = torch.empty((ah, aw, 3), dtype=torch.uint8, device="cuda")
        r.set_config(acfg)
        acam = r.build_camera(acfg.camera)
        r.render_device(acam, acfg.integrator, aw, ah, abuf, stream=sp)
        frames = [animated_config(acfg, k, 30.0, 2.0, 0.3) for k in range(1, 7)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        asteps = 0
        for fc in frames:
            r.set_config(fc)
            ast = r.render_device(acam, fc.integrator, aw, ah, abuf, stream=sp, with_stats=True)
            asteps += ast["total_steps"]
        torch.cuda.synchronize()
        ams = (time.perf_counter() - t0) * 1e3 / len(frames)
        r.set_options(cull_grid=grid0)
        extras["c5_anim_4k"] = {"size": f"{aw}x{ah}", "frames": len(frames),
                                "ms_per_frame": ams, "fps": 1e3 / ams,
                                "steps_per_s": asteps / (ams * 1e-3 * len(frames)),
                                "timing": "wall clock per frame: scene upload + device culling-grid "
                                          "rebuild + render (the render's stats D2H syncs each frame)",
                                "cull_grid": ANIMATION_CULL_GRID,
                                "kernel": r.last_kernel}
        del abuf
        r.set_config(cfg)

    # ---- e2e through the public API with host buffers (rank 0 only, N=1 path)
    e2e = e2e_frames(r, cfg, w, h, max(3, args.steps), lambda st: st["total_steps"]) if single else None

    cpu = None
    parity = None
    if rank == 0 and single:
        if not args.no_cpu_baseline:
            try:
                info = reference_sample(cfg, args.cpu_row_step)
                cpu = {"value": info["steps_per_s"], "unit": UNIT, "cores": info["cores"],
                       "kind": "reference", "sample": info["sample"],
                       "fps_extrapolated": info["fps_extrapolated"],
                       "scalar_1thread": cpu_sample("reference", cfg, w, h, target_s=3.0,
                                                    kernel="scalar", workers=1)}
            except Exception as e:   # reference build absent on this box
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {e}"}
        if not args.no_parity:
            # the headline frame, every pixel, against the reference's own
            # MarchFn (AVX2, all host threads); untimed
            parity = frame_parity(r, cfg, w, h, "reference", row_step=1)

    if rank == 0:
        n_eff = st["bump_evals"] / max(1, 4 * st["integrated_steps"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "width": w, "height": h, "bumps": 16,
                       "scheme": integ.scheme, "h": integ.h, "max_steps": integ.max_steps,
                       "shadows": False, "tile": TILE if world > 1 else None,
                       "exchange": exchange,
                       "l2": "flushed between frames (256 MB write, untimed)",
                       "parallelism": f"tiles{world}"},
            "fps": fps,
            "frame_steps": steps_per_frame,
            "avg_steps_per_ray": steps_per_frame / (w * h),
            "n_eff_bumps": n_eff,
            "rk4_steps_per_s": rk4_steps(st) * args.steps / (total_ms * 1e-3),
            "integrated_steps_per_s": st["integrated_steps"] * args.steps / (total_ms * 1e-3),
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "frac_nominal": achieved / NOMINAL_FP32_TFLOPS,
                         "traffic": traffic,
                         "peak_source": "measured FFMA microbenchmark (rr_measure_fp32_peak)",
                         "peak_nominal": NOMINAL_FP32_TFLOPS,
                         "flop_per_launch": flop_launch, "kernel": r.last_kernel},
            "spills": spill_report(),
            "e2e": e2e,
            "parity": parity,
            "unit_order": unit_order,
            "shadows": shadows,
            "workloads": extras,
            # kernels per frame counted by the library (march + the graph-replayed
            # dispatch-order sort), + rank 0's detile on the gather exchange
            "gpu_launches": args.steps * (int(st["kernel_launches"]) +
                                          (0 if world == 1 or exchange == "p2p-epilogue" else 1)),
            "simt_efficiency": simt(st),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if rank != 0 and exchange == "p2p-epilogue":
            r.frame_close(target)     # drop the IPC mapping before rank 0 frees its frame
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()
    r.close()


def main():
    args = parse_args()
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(args.config)
    cfg.scene.lights = []
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
