"""Cost of the fused lit launch per light: the C3 + lights frame rendered with
0, 1 and 2 of its lights (CUDA events, L2 flushed).  python tools/lightsplit.py"""
import os, sys, copy
sys.path.insert(0, os.getcwd())
import torch
from paper_2005_05386_b200.config import load_config
from paper_2005_05386_b200.render import Renderer
cfg = load_config("configs/c3_bumps16_shadows_1080p.json")
r = Renderer(0)
w, h = cfg.output.width, cfg.output.height
rgb = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
lights = list(cfg.scene.lights)
for sel in ([], [0], [1], [0, 1]):
    n = len(sel)
    c = copy.deepcopy(cfg); c.scene.lights = [lights[k] for k in sel]
    r.set_config(c); cam = r.build_camera(c.camera)
    for _ in range(3): r.render_device(cam, c.integrator, w, h, rgb)
    ts = []
    for _ in range(10):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); st = r.render_device(cam, c.integrator, w, h, rgb, with_stats=True); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"lights={sel}: {ts[5]:.3f} ms kernel={r.last_kernel} shadow_steps={st['shadow_steps']} shadow_int={st['shadow_integrated_steps']} evals={st['bump_evals']} "
          f"shadow_simt={st['shadow_integrated_steps'] / max(1, st['shadow_lane_slots']):.3f} "
          f"shadow_jumps={st['shadow_jump_steps']}")
