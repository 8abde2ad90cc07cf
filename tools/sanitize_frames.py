#!/usr/bin/env python3
"""Small frames of every kernel family for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per gpurun call):

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_frames.py

compute-sanitizer is closed on the GPU pool, so the substitute is the
RR_CHECKS=1 build (device bounds checks on every frame / hit-record /
visibility / outcome / flag index, and a pre-poisoned visibility buffer that
the last-light shading must never read unpublished):

  tools/build_variants.sh checks "-DRR_CHECKS=1"
  RRAY_CUDA_LIB=build/exp/librray_checks.so python tools/sanitize_frames.py

whose frame digests must equal the default build's.

Covers the lit ray-pair launches (hit records, last-finisher shading,
shared-memory staging), the unlit ray-pair frame with the outcome sink, the
twist ray-pair kernel, the static chain fold with meshes, the one-ray mesh
and Euclidean kernels (per-warp stat sums), tile shards and rr_march."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer

    r = Renderer(0)
    cases = [("c3_bumps16_shadows_1080p", 96, 54), ("c3_bumps16_1080p", 100, 60),
             ("c4_twist_1080p", 64, 36), ("c4_twist_mesh_1080p", 64, 36),
             ("c3_bumps16_rk23_1080p", 64, 36), ("c2_flat_1080p", 64, 36),
             ("c4_twist_bend_mesh_1080p", 64, 36), ("c1_gauss1_512", 64, 64)]
    if "--full" in sys.argv:   # the benchmarked frames at full size (lit, unlit, C4 + mesh, 4K)
        cases += [("c3_bumps16_shadows_1080p", 1920, 1080), ("c3_bumps16_1080p", 1920, 1080),
                  ("c4_twist_mesh_1080p", 1920, 1080), ("c5_bumps16_4k", 3840, 2160)]
    for name, w, h in cases:
        cfg = load_config(os.path.join(ROOT, "configs", name + ".json"))
        r.set_config(cfg)
        cam = r.build_camera(cfg.camera)
        rgb, out, st = r.render_outcomes(cam, cfg.integrator, w, h)
        rgb2, _ = r.render(cam, cfg.integrator, w, h)
        assert np.array_equal(rgb, rgb2), name
        n = r.shard_tile_count(w, h, 32, 32, 1, 2)
        tiles = torch.zeros(max(1, n) * 32 * 32 * 3, dtype=torch.uint8, device="cuda")
        r.render_tiles(cam, cfg.integrator, w, h, 32, 32, 1, 2, tiles)
        torch.cuda.synchronize()
        import hashlib
        digest = hashlib.sha1(rgb.tobytes() + tiles.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"{name} {w}x{h}: kernel={r.last_kernel} steps={st['total_steps']} frame+tiles sha1 {digest}",
              flush=True)
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    r.set_config(cfg)
    rays = np.zeros(77, dtype=[("position", "<f8", (3,)), ("direction", "<f8", (3,))])
    rays["position"] = (0.0, 0.0, 0.2)
    rays["direction"][:, 0] = 1.0
    rays["direction"][:, 2] = np.linspace(-0.3, 0.3, 77)
    rays["direction"] /= np.linalg.norm(rays["direction"], axis=1)[:, None]
    out = r.march(cfg.integrator, rays)
    print(f"rr_march 77 rays: kernel={r.last_kernel} hits={(out['status'] == 1).sum()}")
    r.close()


if __name__ == "__main__":
    main()
