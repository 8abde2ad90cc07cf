"""GPU: adaptive Bogacki-Shampine 3(2) integrator (EXTENSION, integrator.scheme
"rk23").

No reference counterpart (SPEC.md:393 lists adaptive stepping as a non-goal);
the FP64 definition is oracle/rro.c rk23_core.  The FP32 device march makes
its own accept/reject decisions, so step sequences may drift from the
oracle's by a few attempts; the contract is the primary one (identical prims
except GRAZING, endpoints 1e-4 relative, RGB within 1) plus step totals
within 2%."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _cfg(name, lights=None, **integ):
    from paper_2005_05386_b200.config import parse_config
    d = json.load(open(os.path.join(ROOT, "configs", name + ".json")))
    d["scene"]["lights"] = lights or []
    d["integrator"].update({"scheme": "rk23", "tol": 1e-6})
    d["integrator"].update(integ)
    return parse_config(json.dumps(d))


@pytest.fixture(scope="module")
def renderer():
    from paper_2005_05386_b200.render import Renderer
    r = Renderer(0)
    yield r
    r.close()


CASES = [("c3_bumps16_1080p", {}, 192, 108),
         ("c1_gauss1_512", {"h": 0.02, "max_steps": 1000}, 128, 96),
         ("c4_twist_1080p", {"h": 0.02, "max_steps": 1000}, 96, 54),
         ("c2_flat_1080p", {}, 128, 72),
         ("c3_bumps16_1080p", {"tol": 1e-4}, 128, 72)]


@pytest.mark.parametrize("name,integ,w,h", CASES)
def test_rk23_frame_parity_vs_oracle(renderer, oracle_lib, name, integ, w, h):
    from oracle.parity import compare_outcomes, compare_rgb
    cfg = _cfg(name, **integ)
    ref_rgb, ref_out, ref_st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
    out = renderer.march(cfg.integrator, rays)
    rep = compare_rgb(rgb, ref_rgb, flags)
    rep = compare_outcomes(out, ref_out, flags, rep)
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)
    assert abs(st["total_steps"] - ref_st["total_steps"]) <= 0.02 * ref_st["total_steps"]


def test_rk23_takes_fewer_evaluations_than_rk4(renderer):
    """Same image content at fewer metric evaluations: 3 per attempt vs 4
    (straight jumps off, so both count every integrated step)."""
    w, h = 192, 108
    renderer.set_options(skip=0)
    a = _cfg("c3_bumps16_1080p")
    b = _cfg("c3_bumps16_1080p", scheme="rk4")
    renderer.set_config(a)
    cam = renderer.build_camera(a.camera)
    rgb23, st23 = renderer.render(cam, a.integrator, w, h)
    renderer.set_config(b)
    rgb4, st4 = renderer.render(cam, b.integrator, w, h)
    assert 3 * st23["integrated_steps"] < 4 * st4["integrated_steps"]
    renderer.set_options(skip=1)
    assert np.mean(np.abs(rgb23.astype(int) - rgb4.astype(int)) <= 1) > 0.99


def test_rk23_shadows_parity(renderer, oracle_lib):
    from oracle.parity import compare_rgb
    lights = [{"position": [2.0, 3.0, 4.0], "intensity": 0.6},
              {"position": [7.0, -4.0, 3.0], "intensity": 0.5}]
    cfg = _cfg("c3_bumps16_shadows_1080p", lights=lights)
    w, h = 160, 90
    ref_rgb, _, ref_st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rep = compare_rgb(rgb, ref_rgb, flags)
    assert rep.ok, rep.summary()
    assert abs(st["shadow_steps"] - ref_st["shadow_steps"]) <= 0.03 * max(1, ref_st["shadow_steps"])


def test_rk23_mesh_parity(renderer, oracle_lib):
    from oracle.parity import compare_outcomes
    from paper_2005_05386_b200.config import parse_config
    d = json.load(open(os.path.join(ROOT, "configs", "c4_twist_mesh_1080p.json")))
    d["scene"]["primitives"][-1]["generator"].update(nu=40, nv=24)
    d["integrator"].update({"h": 0.02, "max_steps": 1000, "scheme": "rk23", "tol": 1e-6})
    cfg = parse_config(json.dumps(d))
    w, h = 96, 54
    ref_rgb, ref_out, _, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    assert (ref_out["prim"] == 3).sum() > 10
    renderer.set_config(cfg)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
    out = renderer.march(cfg.integrator, rays)
    rep = compare_outcomes(out, ref_out, flags)
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)


def test_rk23_rejects_bad_tolerance(renderer):
    from paper_2005_05386_b200.errors import ConfigError
    cfg = _cfg("c2_flat_1080p")
    cfg.integrator.tol = 0.0
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    with pytest.raises(ConfigError):
        renderer.render(cam, cfg.integrator, 32, 32)
