"""GPU: expensive-first dispatch (rr_options.order_units).

A ray-pair launch records its units' costs; the next launch with the same unit
layout sorts them on the device (a CUDA graph of the iota + CUB radix-sort
kernels, captured once) and dispatches the units in that order.  The order
must never change a pixel (a unit's result depends only on its own rays), and
the library must count the sort's kernels in rr_stats.kernel_launches (the
bench's gpu_launches claim)."""
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
W, H = 384, 216


def _frames(cfg_name, order, n=3, size=(W, H)):
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    cfg = load_config(os.path.join(ROOT, "configs", cfg_name))
    r = Renderer(0)
    r.set_options(order_units=order)
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    out = []
    for _ in range(n):
        img, st = r.render(cam, cfg.integrator, *size)
        out.append((np.asarray(img).copy(), st))
    r.close()
    return out


@pytest.mark.parametrize("cfg", ["c3_bumps16_1080p.json", "c3_bumps16_shadows_1080p.json"])
def test_order_never_changes_pixels_and_is_counted(cfg):
    plain = _frames(cfg, 0)
    ordered = _frames(cfg, 1)
    ref = plain[0][0]
    for img, _ in plain + ordered:
        assert np.array_equal(img, ref)
    # march launches: one (unlit) or a hit-record + a shadow launch (lit)
    marches = 2 if "shadows" in cfg else 1
    # no recorded costs yet: the march alone; unordered frames never sort
    assert ordered[0][1]['kernel_launches'] == marches and ordered[0][1]['sort_kernels'] == 0
    assert all(st['kernel_launches'] == marches and st['sort_kernels'] == 0 for _, st in plain)
    # later frames replay the sort graph(s): lit frames sort the shadow items too
    sorts = [st['kernel_launches'] - marches for _, st in ordered[1:]]
    assert sorts[0] >= 1 and sorts[0] == sorts[1]
    assert all(st['sort_kernels'] == k for (_, st), k in zip(ordered[1:], sorts))
    if "shadows" in cfg:
        unlit = _frames("c3_bumps16_1080p.json", 1, n=2)
        assert sorts[0] > unlit[1][1]['sort_kernels']
    assert ordered[1][1]['total_steps'] == plain[1][1]['total_steps']


def test_new_layout_starts_unordered():
    """Costs recorded for one frame size are not applied to another."""
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    r = Renderer(0)
    r.set_config(cfg)
    cam = r.build_camera(cfg.camera)
    _, a = r.render(cam, cfg.integrator, W, H)
    _, b = r.render(cam, cfg.integrator, W, H)
    img_c, c = r.render(cam, cfg.integrator, W // 2, H // 2)
    img_d, d = r.render(cam, cfg.integrator, W // 2, H // 2)
    r.close()
    assert a['kernel_launches'] == 1 and b['kernel_launches'] > 1
    assert c['kernel_launches'] == 1 and d['kernel_launches'] > 1
    assert np.array_equal(np.asarray(img_c), np.asarray(img_d))
