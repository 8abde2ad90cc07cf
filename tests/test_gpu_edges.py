"""GPU: edge cases of the march contract (kernel_impl.hpp:22-94, scene.cpp)
against the FP64 oracle: empty scene, camera inside a primitive (inside-start
s = 0), max_steps = 1, a step longer than the scene, non-default culling
options, and a frame larger than one wave of the persistent grid."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def renderer():
    from paper_2005_05386_b200.render import Renderer
    r = Renderer(0)
    yield r
    r.close()


def cfg_of(name, **edits):
    from paper_2005_05386_b200.config import parse_config
    d = json.load(open(os.path.join(ROOT, "configs", name + ".json")))
    for k, v in edits.items():
        sec, _, key = k.partition("__")
        if key:
            d[sec][key] = v
        else:
            d[sec] = v
    return parse_config(json.dumps(d))


def check(renderer, oracle_lib, cfg, w, h, opts=None):
    from oracle.parity import compare_outcomes, compare_rgb
    ref_rgb, ref_out, ref_st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    saved = renderer.options()
    if opts:
        renderer.set_options(**opts)
    try:
        renderer.set_config(cfg)
        cam = renderer.build_camera(cfg.camera)
        rgb, st = renderer.render(cam, cfg.integrator, w, h)
        rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
        out = renderer.march(cfg.integrator, rays)
    finally:
        if opts:
            renderer.set_options(**saved)
    rep = compare_outcomes(out, ref_out, flags)
    rep = compare_rgb(rgb, ref_rgb, flags, rep)
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)
    return out, ref_out, st, ref_st


def test_empty_scene_all_misses(renderer, oracle_lib):
    cfg = cfg_of("c3_bumps16_1080p", scene__primitives=[])
    out, ref, st, rst = check(renderer, oracle_lib, cfg, 64, 36)
    assert (out["status"] == 0).all() and (ref["status"] == 0).all()
    assert abs(st["total_steps"] - rst["total_steps"]) <= 0.01 * rst["total_steps"]


def test_camera_inside_sphere_hits_at_zero(renderer, oracle_lib):
    prims = [{"kind": "sphere", "center": [0, 0, 0.2], "radius": 0.5},
             {"kind": "half_space", "normal": [0, 0, 1], "offset": -1.0}]
    cfg = cfg_of("c1_gauss1_512", scene__primitives=prims)
    out, ref, _, _ = check(renderer, oracle_lib, cfg, 32, 24)
    assert (ref["prim"] == 0).all() and (ref["t"] == 0.0).all() and (out["steps"] == 1).all()


@pytest.mark.parametrize("integ", [{"h": 0.05, "max_steps": 1, "scheme": "rk4"},
                                   {"h": 5.0, "max_steps": 10, "scheme": "rk4"},
                                   {"h": 0.02, "max_steps": 37, "scheme": "euler"}])
def test_extreme_integrator_settings(renderer, oracle_lib, integ):
    cfg = cfg_of("c3_bumps16_1080p", integrator=integ)
    check(renderer, oracle_lib, cfg, 64, 36)


@pytest.mark.parametrize("opts", [{"cull": 0}, {"cull_grid": 16}, {"cull_grid": 128},
                                  {"cull_grid": 192}, {"cull_radius_sigma": 8.0}, {"skip": 0}])
def test_culling_options_keep_parity(renderer, oracle_lib, opts):
    cfg = cfg_of("c3_bumps16_1080p")
    check(renderer, oracle_lib, cfg, 96, 54, opts)


def test_large_frame_accounting(renderer):
    """4K frame (259k warp units, many waves of the persistent grid): every
    pixel written once, stats cover every ray, deterministic."""
    cfg = cfg_of("c5_bumps16_4k")
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    a, st = renderer.render(cam, cfg.integrator, 3840, 2160)
    b, _ = renderer.render(cam, cfg.integrator, 3840, 2160)
    assert st["rays"] == 3840 * 2160 and np.array_equal(a, b)
    assert 150 < st["total_steps"] / st["rays"] < 200     # ~170 reference steps/ray


def test_pinned_host_output_is_written_by_the_kernel():
    """rr_render stores straight into page-locked caller memory (UVA) and
    gives the same bytes as the pageable (device buffer + copy) route."""
    import torch
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    cfg.scene.lights = []
    r = Renderer(0)
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    w, h = 321, 179
    pageable, st0 = r.render(cam, cfg.integrator, w, h)
    pinned = torch.full((h, w, 3), 7, dtype=torch.uint8).pin_memory()
    _, st1 = r.render(cam, cfg.integrator, w, h, out=pinned)
    assert np.array_equal(pinned.numpy(), pageable)
    assert st0["total_steps"] == st1["total_steps"]
    from paper_2005_05386_b200.config import Light
    cfg.scene.lights = [Light([2.0, 3.0, 4.0], 0.6)]
    r.set_config(cfg)
    lit, _ = r.render(cam, cfg.integrator, w, h)
    _, _ = r.render(cam, cfg.integrator, w, h, out=pinned)
    assert np.array_equal(pinned.numpy(), lit)
    r.close()


def test_option_validation(renderer):
    """Out-of-range options fail with a config error and leave the context's
    options unchanged (the culling grid is capped at 256^3)."""
    from paper_2005_05386_b200.errors import Error
    before = renderer.options()
    assert before["cull_grid"] == 256                     # the static-frame default
    for bad in ({"cull_grid": 257}, {"cull_grid": -1}, {"cull": 3}):
        with pytest.raises(Error):
            renderer.set_options(**bad)
        assert renderer.options() == before
