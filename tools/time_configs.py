"""Device-time a list of configs (run under gpurun):
    python tools/time_configs.py configs/a.json[:WxH] ... [--opt k=v]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2005_05386_b200.config import load_config  # noqa: E402
from paper_2005_05386_b200.render import Renderer  # noqa: E402

opts = {}
paths = []
args = sys.argv[1:]
while args:
    a = args.pop(0)
    if a == "--opt":
        k, v = args.pop(0).split("=")
        opts[k] = float(v) if "." in v else int(v)
    else:
        paths.append(a)
r = Renderer(0)
if opts:
    r.set_options(**opts)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for spec in paths:
    path, _, size = spec.partition(":")
    cfg = load_config(path)
    w, h = (int(x) for x in size.split("x")) if size else (cfg.output.width, cfg.output.height)
    buf = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    r.render_device(cam, cfg.integrator, w, h, buf, stream=s.cuda_stream)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        r.render_device(cam, cfg.integrator, w, h, buf, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = r.render_device(cam, cfg.integrator, w, h, buf, stream=s.cuda_stream, with_stats=True)
    print(f"{os.path.basename(path):34s} {w}x{h} {statistics.median(ts):9.3f} ms  steps/ray "
          f"{st['total_steps'] / (w * h):7.1f} integrated {st['integrated_steps']:.3e} "
          f"{r.last_kernel}", flush=True)
