"""Parity vs work of the bump-culling radius (run on the GPU box).

For each radius R (in sigmas) renders C3/C5-shaped frames through the CUDA
path and compares them with the FP64 oracle under the north-star contract.
Prints endpoint error statistics, status/prim flips and N_eff."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402
from oracle.parity import compare_outcomes, compare_rgb  # noqa: E402
from paper_2005_05386_b200.config import load_config  # noqa: E402
from paper_2005_05386_b200.render import Renderer  # noqa: E402

w, h = int(sys.argv[1]) if len(sys.argv) > 1 else 320, int(sys.argv[2]) if len(sys.argv) > 2 else 180
orc = Oracle()
r = Renderer(0)
radii = [float(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else \
    [3.0, 4.0, 5.0, 5.5, 6.0, 6.5, 7.0, 8.0, 0.0]
names = sys.argv[4].split(",") if len(sys.argv) > 4 else ["c3_bumps16_1080p", "c1_gauss1_512"]
for name in names:
    cfg = load_config(os.path.join(ROOT, "configs", name + ".json"))
    if "shadows" not in name:
        cfg.scene.lights = []
    t0 = time.time()
    ref_rgb, ref_out, _, flags = orc.render(cfg, w, h, with_flags=True)
    rays = orc.primary_rays(orc.camera(cfg), w, h)
    print(f"{name} {w}x{h}: oracle {time.time() - t0:.1f}s, exempt {(flags & 5 != 0).sum()}", flush=True)
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    for R in radii:
        mode = int(os.environ.get("CULL_MODE", "1"))   # 1 uniform radius, 2 equal-error radii
        r.set_options(cull=mode if R > 0 else 0, cull_radius_sigma=R if R > 0 else 7.0)
        rgb, st = r.render(cam, cfg.integrator, w, h)
        out = r.march(cfg.integrator, rays)
        rep = compare_outcomes(out, ref_out, flags)
        rep = compare_rgb(rgb, ref_rgb, flags, rep)
        neff = st["bump_evals"] / max(1, 4 * st["integrated_steps"])
        print(json.dumps({"cfg": name, "R": R, "ok": rep.ok, "neff": round(neff, 3),
                          "endpoint_max": rep.endpoint_max_rel, "endpoint_p99": rep.endpoint_p99_rel,
                          "status_mm": rep.status_mismatch, "prim_mm": rep.prim_mismatch,
                          "endpoint_fail": rep.endpoint_fail, "rgb_fail": rep.rgb_fail,
                          "rgb_max": rep.rgb_max}), flush=True)
