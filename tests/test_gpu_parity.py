"""GPU parity: the CUDA path (C-ABI librray_cuda.so) against the reference.

Golden vectors (tests/golden/*.npz) were dumped from the reference itself;
larger frames are checked live against the FP64 oracle (bit-identical to the
reference, tests/test_oracle.py).  Tolerances are BASELINE.json's north star:
identical status/prim except GRAZING/LIMIT rays, endpoints within 1e-4
relative, RGB within 1/255 except wrapped channels, equal magenta counts.
"""
import json
import os

import numpy as np
import pytest

from conftest import ROOT, golden_cases, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def renderer():
    from paper_2005_05386_b200.render import Renderer
    r = Renderer(0)
    yield r
    r.close()


def _camera(r, cfg, cam_cfg):
    if cam_cfg is not cfg:
        r.set_config(cam_cfg)
        cam = r.build_camera(cam_cfg.camera)
        r.set_config(cfg)
        return cam
    r.set_config(cfg)
    return r.build_camera(cfg.camera)


@pytest.mark.parametrize("name", golden_cases())
def test_march_matches_reference_golden(renderer, name):
    from oracle.parity import compare_outcomes
    cfg, cam_cfg, z = load_golden(name)
    renderer.set_config(cfg)
    out = renderer.march(cfg.integrator, z["rays"])
    rep = compare_outcomes(out, z["outcomes"], z["flags"])
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)
    assert renderer.last_kernel.startswith("march")


@pytest.mark.parametrize("name", golden_cases())
def test_render_matches_reference_golden(renderer, name):
    from oracle.parity import compare_rgb
    cfg, cam_cfg, z = load_golden(name)
    cam = _camera(renderer, cfg, cam_cfg if str(z["camera_config"]) != str(z["config"]) else cfg)
    w, h = int(z["w"]), int(z["h"])
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rep = compare_rgb(rgb, z["rgb"], z["flags"])
    assert rep.ok, rep.summary()
    assert st["pixel_errors"] == int(z["pixel_errors"])
    # reference step accounting (RenderStats.total_steps) within FP32 noise
    ref_steps = int(z["total_steps"])
    assert abs(st["total_steps"] - ref_steps) <= max(2, 0.01 * ref_steps)
    assert st["integrated_steps"] >= 0 and st["rays"] == w * h


@pytest.mark.parametrize("cfg_name,w,h", [("c1_gauss1_512", 160, 120),
                                          ("c3_bumps16_1080p", 192, 108),
                                          ("c4_twist_1080p", 128, 72)])
def test_frame_parity_vs_oracle(renderer, oracle_lib, cfg_name, w, h):
    from oracle.parity import compare_outcomes, compare_rgb
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", cfg_name + ".json"))
    cfg.scene.lights = []
    ref_rgb, ref_out, ref_st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rep = compare_rgb(rgb, ref_rgb, flags)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
    out = renderer.march(cfg.integrator, rays)
    rep = compare_outcomes(out, ref_out, flags, rep)
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)
    assert abs(st["total_steps"] - ref_st["total_steps"]) <= 0.01 * ref_st["total_steps"]


def test_culling_is_parity_neutral(renderer, oracle_lib):
    """Per-warp bump culling (the default uniform 5.5 sigma radius, cull=1, and
    the equal-error radii, cull=2) must stay inside the parity contract,
    change the image by at most rounding, and the equal-error radii must
    evaluate fewer bumps than the uniform radius, which evaluates fewer than
    no culling (cull=0)."""
    from oracle.parity import compare_outcomes, compare_rgb
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    w, h = 128, 72
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    saved = renderer.options()
    ref_rgb, ref_out, _, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
    res = {}
    try:
        for mode in (2, 1, 0):
            renderer.set_options(cull=mode)
            rgb, st = renderer.render(cam, cfg.integrator, w, h)
            out = renderer.march(cfg.integrator, rays)
            rep = compare_rgb(rgb, ref_rgb, flags, compare_outcomes(out, ref_out, flags))
            assert rep.ok, f"cull={mode}: " + rep.summary()
            assert rep.endpoint_max_rel < 2e-5, f"cull={mode}: {rep.endpoint_max_rel}"
            res[mode] = st["bump_evals"]
    finally:
        renderer.set_options(**saved)
    assert res[2] < res[1] < res[0]


def test_render_is_deterministic_and_tiling_invariant(renderer):
    """Bytes independent of repeat and of the shard count (acceptance.cpp:243-253
    at 1/2/4/8 workers -> 1/2/4/8 shards here)."""
    import torch
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    w, h, tw, th = 200, 120, 32, 32
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    full, _ = renderer.render(cam, cfg.integrator, w, h)
    again, _ = renderer.render(cam, cfg.integrator, w, h)
    assert np.array_equal(full, again)
    for n in (1, 2, 4, 8):
        max_k = renderer.shard_tile_count(w, h, tw, th, 0, n)
        gathered = torch.zeros((n, max_k * tw * th * 3), dtype=torch.uint8, device="cuda")
        for s in range(n):
            renderer.render_tiles(cam, cfg.integrator, w, h, tw, th, s, n, gathered[s])
        frame = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
        renderer.detile(gathered, w, h, tw, th, n, frame)
        torch.cuda.synchronize()
        assert np.array_equal(frame.cpu().numpy(), full), f"{n} shards"


def test_null_deformations_match_euclidean_bytes(renderer):
    """Zero-amplitude graph and identity diffeo render the Euclidean bytes
    (acceptance.cpp:205-221)."""
    from paper_2005_05386_b200.config import parse_config
    base = {"scene": {"primitives": [{"kind": "grid_planes", "spacing": 1.0, "half_width": 0.03}]},
            "camera": {"position": [0.5, 0.4, 0.6], "look_dir": [1.0, 0.12, 0.07]},
            "integrator": {"h": 0.01, "max_steps": 2000, "scheme": "euler"}}
    imgs = []
    for metric in ({"kind": "euclidean"},
                   {"kind": "graph", "field": {"kind": "gaussian", "amplitude": 0.0,
                                               "center": [0, 0, 0], "sigma": [1, 1, 1]}},
                   {"kind": "diffeo", "map": {"kind": "identity"}}):
        cfg = parse_config(json.dumps(dict(base, metric=metric)))
        renderer.set_config(cfg)
        cam = renderer.build_camera(cfg.camera)
        imgs.append(renderer.render(cam, cfg.integrator, 96, 72)[0])
    assert np.array_equal(imgs[0], imgs[1]) and np.array_equal(imgs[0], imgs[2])


def test_errors_map_to_reference_exit_codes(renderer):
    from paper_2005_05386_b200.config import IntegratorConfig
    from paper_2005_05386_b200.errors import ValidationError
    cfg, _, z = load_golden("c1_gauss1_512")
    renderer.set_config(cfg)
    with pytest.raises(ValidationError):
        renderer.march(IntegratorConfig(h=-1.0), z["rays"][:4])
    with pytest.raises(ValidationError):
        renderer.march(IntegratorConfig(max_steps=0), z["rays"][:4])
    assert len(renderer.march(cfg.integrator, z["rays"][:0])) == 0


def test_march_tail_and_odd_batch_sizes(renderer):
    from oracle.parity import compare_outcomes
    cfg, _, z = load_golden("c3_bumps16_1080p")
    renderer.set_config(cfg)
    for n in (1, 31, 33, 100):
        out = renderer.march(cfg.integrator, z["rays"][:n])
        rep = compare_outcomes(out, z["outcomes"][:n], z["flags"][:n])
        assert rep.ok, (n, rep.summary())


@pytest.mark.parametrize("skip", [0, 1])
def test_straight_jumps_match_stepping(renderer, skip):
    """Empty-space skipping / Euclidean straight jumps against the golden
    reference outcomes, with skipping off (every step integrated) and on."""
    from oracle.parity import compare_outcomes
    for name in ("ref_grid_euclid", "c2_flat_1080p", "c3_bumps16_1080p", "graph_grid_spheres"):
        cfg, _, z = load_golden(name)
        renderer.set_options(skip=skip)
        renderer.set_config(cfg)
        out = renderer.march(cfg.integrator, z["rays"])
        rep = compare_outcomes(out, z["outcomes"], z["flags"])
        assert rep.ok, (name, skip, rep.summary())
        assert (out["steps"] == z["outcomes"]["steps"]).mean() > 0.97, name
    renderer.set_options(skip=1)
