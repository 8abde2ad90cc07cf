"""GPU: triangle-mesh primitive with the device BVH (EXTENSION, SURVEY §8
a16/f2) against the FP64 oracle (whose BVH is checked against brute force in
tests/test_oracle_mesh.py)."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def mesh_cfg(nu, nv, metric=None, lights=None, **integ):
    from paper_2005_05386_b200.config import parse_config
    d = json.load(open(os.path.join(ROOT, "configs", "c4_twist_mesh_1080p.json")))
    d["scene"]["primitives"][-1]["generator"].update(nu=nu, nv=nv)
    if metric is not None:
        d["metric"] = metric
    if lights:
        d["scene"]["lights"] = lights
    d["integrator"].update(integ)
    return parse_config(json.dumps(d))


@pytest.fixture(scope="module")
def renderer():
    from paper_2005_05386_b200.render import Renderer
    r = Renderer(0)
    yield r
    r.close()


@pytest.mark.parametrize("nu,nv,metric,integ,w,h", [
    (40, 24, {"kind": "euclidean"}, {"h": 0.02, "max_steps": 1000}, 96, 54),
    (40, 24, None, {"h": 0.02, "max_steps": 1000}, 96, 54),
    (250, 200, None, {"h": 0.02, "max_steps": 1000}, 64, 36),          # the 100k-triangle mesh
    (40, 24, {"kind": "graph", "field": {"kind": "gaussian", "amplitude": 0.6,
                                          "center": [4.5, 1.0, 0.3], "sigma": [0.8, 0.8, 0.8]}},
     {"h": 0.02, "max_steps": 1000}, 96, 54),
])
def test_mesh_parity_vs_oracle(renderer, oracle_lib, nu, nv, metric, integ, w, h):
    from oracle.parity import compare_outcomes, compare_rgb
    cfg = mesh_cfg(nu, nv, metric, **integ)
    ref_rgb, ref_out, _, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    assert (ref_out["prim"] == 3).sum() > 10           # the mesh is in view
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, st = renderer.render(cam, cfg.integrator, w, h)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
    out = renderer.march(cfg.integrator, rays)
    rep = compare_outcomes(out, ref_out, flags)
    rep = compare_rgb(rgb, ref_rgb, flags, rep)
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)


def test_mesh_with_shadows(renderer, oracle_lib):
    from oracle.parity import compare_rgb
    cfg = mesh_cfg(40, 24, {"kind": "euclidean"}, [{"position": [3.0, 4.0, 5.0], "intensity": 0.8}],
                   h=0.02, max_steps=1000)
    w, h = 96, 54
    ref_rgb, _, _, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, _ = renderer.render(cam, cfg.integrator, w, h)
    assert compare_rgb(rgb, ref_rgb, flags).ok


@pytest.mark.parametrize("metric", [
    {"kind": "diffeo", "map": {"kind": "bend", "curvature": 0.12}},
    {"kind": "diffeo", "map": {"kind": "compose", "maps": [{"kind": "twist"},
                                                           {"kind": "bend", "curvature": 0.08}]}},
])
def test_bend_deformation_parity(renderer, oracle_lib, metric):
    """EXTENSION: Barr bend (north star "twist/bend deformation") vs the FP64 oracle."""
    from oracle.parity import compare_outcomes, compare_rgb
    cfg = mesh_cfg(40, 24, metric, h=0.02, max_steps=1000)
    w, h = 96, 54
    ref_rgb, ref_out, _, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, _ = renderer.render(cam, cfg.integrator, w, h)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), w, h)
    out = renderer.march(cfg.integrator, rays)
    rep = compare_outcomes(out, ref_out, flags)
    rep = compare_rgb(rgb, ref_rgb, flags, rep)
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)
