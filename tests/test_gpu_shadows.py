"""GPU: shadow geodesics + point lights (EXTENSION).

No reference counterpart exists; the FP64 definition is the
oracle's shadow_march/shade_lit (oracle/rro.c, include/rray_cuda.h).  The CUDA
hit pass + shadow pass must match it under the same contract as the primary
path, with pixels whose light visibility flips under +-1e-4 rad shadow-ray
perturbations flagged SHADOW (penumbra edges are hard edges)."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

LIGHTS = [{"position": [2.0, 3.0, 4.0], "intensity": 0.6},
          {"position": [7.0, -4.0, 3.0], "intensity": 0.5}]


def _cfg(name, lights=LIGHTS, **integ):
    from paper_2005_05386_b200.config import parse_config
    d = json.load(open(os.path.join(ROOT, "configs", name + ".json")))
    d["scene"]["lights"] = lights
    d["scene"]["ambient"] = 0.2
    d["integrator"].update(integ)
    return parse_config(json.dumps(d))


@pytest.fixture(scope="module")
def renderer():
    from paper_2005_05386_b200.render import Renderer
    r = Renderer(0)
    yield r
    r.close()


CASES = [("c3_bumps16_shadows_1080p", {}, 160, 90),
         ("c1_gauss1_512", {"h": 0.02, "max_steps": 1000}, 96, 96),
         ("c4_twist_1080p", {"h": 0.02, "max_steps": 1000}, 96, 54),
         ("c2_flat_1080p", {}, 128, 72)]


@pytest.mark.parametrize("name,integ,w,h", CASES)
def test_shadow_frame_parity_vs_oracle(renderer, oracle_lib, name, integ, w, h):
    from oracle.parity import compare_rgb
    cfg = _cfg(name, **integ)
    ref_rgb, _, ref_st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rep = compare_rgb(rgb, ref_rgb, flags)
    assert rep.ok, rep.summary()
    # ray-pair Gaussian-bump RK4 frames fuse the hit and shadow work into one
    # launch; the other kernels use a hit-record launch + a shadow launch
    assert st["kernel_launches"] - st["sort_kernels"] == 2      # hit-record launch + shadow launch
    # shadow work is counted and close to the oracle's
    assert abs(st["shadow_steps"] - ref_st["shadow_steps"]) <= 0.02 * max(1, ref_st["shadow_steps"])


def test_shadows_change_the_image_and_stay_deterministic(renderer):
    import torch
    cfg = _cfg("c3_bumps16_shadows_1080p")
    flat = _cfg("c3_bumps16_shadows_1080p", lights=[])
    w, h, t = 160, 96, 32
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    lit, _ = renderer.render(cam, cfg.integrator, w, h)
    again, _ = renderer.render(cam, cfg.integrator, w, h)
    assert np.array_equal(lit, again)
    for n in (2, 3):
        max_k = renderer.shard_tile_count(w, h, t, t, 0, n)
        g = torch.zeros((n, max_k * t * t * 3), dtype=torch.uint8, device="cuda")
        for s in range(n):
            renderer.render_tiles(cam, cfg.integrator, w, h, t, t, s, n, g[s])
        frame = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
        renderer.detile(g, w, h, t, t, n, frame)
        torch.cuda.synchronize()
        assert np.array_equal(frame.cpu().numpy(), lit)
    renderer.set_config(flat)
    plain, st = renderer.render(cam, flat.integrator, w, h)
    assert st["kernel_launches"] - st["sort_kernels"] == 1 and st["shadow_steps"] == 0
    assert (lit.astype(int) - plain.astype(int)).any()


def test_larger_frame_parity_with_shadows(renderer, oracle_lib):
    """C3 with both lights at 384x216 (83k primary rays + shadow geodesics)."""
    from oracle.parity import compare_outcomes, compare_rgb
    cfg = _cfg("c3_bumps16_shadows_1080p")
    w, h = 384, 216
    ref_rgb, ref_out, ref_st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
    out = renderer.march(cfg.integrator, rays)
    rep = compare_outcomes(out, ref_out, flags)
    rep = compare_rgb(rgb, ref_rgb, flags, rep)
    assert rep.ok, rep.summary()
    assert rep.exempt < 0.01 * w * h and rep.endpoint_max_rel < 1e-4
    print("C3 384x216 parity:", rep.summary())


@pytest.mark.parametrize("lights", [
    LIGHTS[:1],                                                    # nl == 1: no visibility bytes
    LIGHTS + [{"position": [4.0, 0.0, 6.0], "intensity": 0.3},    # 5 lights: the unit's last
              {"position": [1.0, -3.0, 2.0], "intensity": 0.2},   # finisher sums 4 published
              {"position": [8.0, 2.0, 1.5], "intensity": 0.25}],  # visibility bytes
    [{"position": [4.0, 0.0, -3.0], "intensity": 0.9}],            # below the floor: all blocked
])
def test_light_count_parity_lit_launches(renderer, oracle_lib, lights):
    """The lit ray-pair frame (a hit-record launch, then one work item per
    (pixel unit, light), the unit's last light to finish shades) against the
    oracle's shade_lit for 1, 5 and an occluded light, plus byte-identity
    across repeated frames."""
    from oracle.parity import compare_rgb
    cfg = _cfg("c3_bumps16_shadows_1080p", lights=lights)
    w, h = 160, 90
    ref_rgb, _, ref_st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rep = compare_rgb(rgb, ref_rgb, flags)
    assert rep.ok, rep.summary()
    assert st["kernel_launches"] - st["sort_kernels"] == 2 and renderer.last_kernel.startswith("march2_kernel")
    assert abs(st["shadow_steps"] - ref_st["shadow_steps"]) <= 0.02 * max(1, ref_st["shadow_steps"])
    for _ in range(2):
        again, _ = renderer.render(cam, cfg.integrator, w, h)
        assert np.array_equal(again, rgb)
