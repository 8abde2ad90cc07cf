"""GPU: the reference-shaped module API (render.hpp:14-50, camera.hpp:15-30):
build_camera(metric, position, look_dir, up_hint, fov) and render(metric,
scene, cam, integrator, w, h) -> RenderResult, as a caller written against the
reference uses them; the frame equals the context API's and the stats carry
the reference fields."""
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c3_bumps16_1080p.json", "c4_twist_1080p.json"])
def test_module_render_matches_context_render(name):
    from paper_2005_05386_b200 import render as R
    from paper_2005_05386_b200.config import fov_radians, load_config
    cfg = load_config(os.path.join(ROOT, "configs", name))
    w, h = 256, 144
    c = cfg.camera
    cam = R.build_camera(cfg.metric, c.position, c.look_dir, c.up_hint, fov_radians(c))
    res = R.render(cfg.metric, cfg.scene, cam, cfg.integrator, w, h)
    assert isinstance(res.stats, R.RenderStats)
    assert res.stats.rays == w * h and res.stats.total_steps > 0
    assert res.stats.pixel_errors == 0
    assert res.image.data.shape == (h, w, 3)
    r = R.Renderer(0)
    r.set_config(cfg)
    img, st = r.render(r.build_camera(cfg.camera), cfg.integrator, w, h)
    r.close()
    assert np.array_equal(res.image.data, img)
    assert res.stats.total_steps == st["total_steps"]
