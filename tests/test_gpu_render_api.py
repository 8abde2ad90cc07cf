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


def _cfg(name):
    from paper_2005_05386_b200.config import load_config
    return load_config(os.path.join(ROOT, "configs", name))


def test_march_fn_thunk_matches_context_march():
    """march_fn(KernelKind.Cuda) is the MarchFn mirror (kernel.hpp:47): it
    writes out[0..n) and leaves the rest untouched."""
    from paper_2005_05386_b200 import abi
    from paper_2005_05386_b200 import render as R
    from oracle import Oracle
    cfg = _cfg("c3_bumps16_1080p.json")
    o = Oracle()
    rays = o.primary_rays(o.camera(cfg), 48, 27)
    out = np.zeros(len(rays), abi.OUTCOME_DTYPE)
    out["steps"] = -7
    n = len(rays) - 5
    R.march_fn(R.KernelKind.Cuda)(R.MarchContext(cfg.metric, cfg.scene, cfg.integrator), rays, out, n)
    r = R.Renderer(0)
    r.set_config(cfg)
    want = r.march(cfg.integrator, rays[:n])
    r.close()
    assert np.array_equal(out[:n], want)
    assert (out["steps"][n:] == -7).all()


def test_march_device_matches_march():
    import torch
    from paper_2005_05386_b200 import abi
    from paper_2005_05386_b200.render import Renderer
    from oracle import Oracle
    cfg = _cfg("c4_twist_1080p.json")
    o = Oracle()
    rays = o.primary_rays(o.camera(cfg), 40, 24)
    r = Renderer(0)
    r.set_config(cfg)
    host = r.march(cfg.integrator, rays)
    d_rays = torch.from_numpy(rays.view(np.uint8).copy()).cuda()
    d_out = torch.zeros(len(rays) * abi.OUTCOME_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    r.march_device(cfg.integrator, d_rays, d_out, len(rays))
    torch.cuda.synchronize()
    dev = d_out.cpu().numpy().view(abi.OUTCOME_DTYPE)
    r.close()
    assert np.array_equal(dev, host)


def test_pixel_direction_matches_oracle():
    """camera.cpp:22-29 in FP64 on the host: byte-equal to the oracle's (and
    so to the reference's, test_oracle.py) primary rays."""
    from paper_2005_05386_b200 import render as R
    from oracle import Oracle
    cfg = _cfg("c4_twist_1080p.json")
    o = Oracle()
    cam_o = o.camera(cfg)
    c = cfg.camera
    from paper_2005_05386_b200.config import fov_radians
    cam = R.build_camera(cfg.metric, c.position, c.look_dir, c.up_hint, fov_radians(c))
    w, h = 37, 21
    rays = o.primary_rays(cam_o, w, h)
    for px, py in [(0, 0), (w - 1, 0), (0, h - 1), (18, 10), (w - 1, h - 1)]:
        d = R.pixel_direction(cam, px, py, w, h)
        assert tuple(d) == tuple(rays[py * w + px]["direction"])


@pytest.mark.parametrize("name", ["c3_bumps16_1080p.json", "c4_twist_1080p.json"])
def test_device_accel_and_fp64_metric_helpers(name):
    """rr_accel (device flow_accel, FP32) against the FP64 oracle, and
    against -Gamma(v, v) from the library's FP64 finite-difference
    Christoffel symbols (metric.cpp:88-133); g(p) symmetric positive definite."""
    from paper_2005_05386_b200.render import Renderer
    from oracle import Oracle
    cfg = _cfg(name)
    o = Oracle()
    r = Renderer(0)
    r.set_config(cfg)
    rng = np.random.default_rng(3)
    pos = rng.uniform([1, -3, -1], [7, 3, 2], (16, 3))
    vel = rng.normal(size=(16, 3))
    acc, val = r.accel(pos, vel)
    for i in range(len(pos)):
        a_o, _ = o.flow_accel(cfg, pos[i], vel[i])
        scale = max(1.0, float(np.abs(a_o).max()))
        assert np.allclose(acc[i], a_o, atol=2e-5 * scale, rtol=0), (i, acc[i], a_o)
        g = r.metric_tensor(pos[i])
        assert np.allclose(g, g.T) and np.linalg.eigvalsh(g).min() > 0
        gam = r.christoffel_fd(pos[i])
        a_fd = -np.einsum("mij,i,j->m", gam, vel[i], vel[i])
        assert np.allclose(a_fd, a_o, atol=1e-5 * scale, rtol=0), (i, a_fd, a_o)
    assert (val > 0).all()
    from paper_2005_05386_b200.config import DiffeoMetric
    if isinstance(cfg.metric, DiffeoMetric):
        img = r.diffeo_image(pos[0])
        assert img.shape == (3,) and np.isfinite(img).all()
    r.close()
