"""GPU: per-pixel outcome parity of the PRODUCTION frame kernels, at the
benchmarked resolutions and settings.

rr_render_outcomes runs the same frame launch rr_render does (the ray-pair
march2_kernel for Gaussian-bump RK4 frames — unlit, or the lit launches —
and march_kernel for the diffeo/mesh frames) with a PixelOutcome sink, so
hit primitive, endpoint, t and steps of every pixel of the benchmarked frame
are compared with the reference (oracle/_ref, the reference compiled from its
own sources) or the FP64 oracle (bit-identical to it, tests/test_oracle.py;
the only definition of the shadow/mesh extensions).  Contract (BASELINE.json
north star, oracle/parity.py): status and prim identical except GRAZING /
LIMIT rays, endpoints within 1e-4 relative, RGB within 1/255 except WRAP
channels and SHADOW pixels, equal magenta counts.  Flags are computed by the
oracle for the pixels that differ (check_frame): they only ever exempt.

The full-size cases take ~15-40 s of host time each on the GPU box's cores
(reference AVX2 / FP64 oracle, all threads).
"""
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


def _load(name, **integ):
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", name + ".json"))
    for k, v in integ.items():
        setattr(cfg.integrator, k, v)
    return cfg


def _gpu_frame(renderer, cfg, w, h):
    renderer.set_config(cfg)
    cam = renderer.build_camera(cfg.camera)
    rgb, out, st = renderer.render_outcomes(cam, cfg.integrator, w, h)
    return rgb, out, st, renderer.last_kernel


def _rows(a, w, h, row0, step):
    """Row subsample (row0, row0+step, ...) of a row-major per-pixel array."""
    return a.reshape(h, w, *a.shape[1:])[row0::step].reshape(-1, *a.shape[1:])


def _log(name, rep, cand, kern):
    """RR_PARITY_LOG=path: append the report (evidence for profiles/)."""
    path = os.environ.get("RR_PARITY_LOG")
    if path:
        import json
        with open(path, "a") as f:
            f.write(json.dumps({"case": name, "kernel": kern, "ok": rep.ok, "summary": rep.summary(),
                                "flagged_candidates": cand}) + "\n")


def _check_vs_oracle(oracle_lib, cfg, w, h, rgb, out, row0=0, step=1):
    from oracle.parity import check_frame
    ref_rgb, ref_out, ref_st = oracle_lib.render_rows(cfg, w, h, row0, step)
    rows = np.arange(row0, h, step)
    g_out = _rows(out, w, h, row0, step)
    g_rgb = rgb[row0::step]

    def flag_fn(idx):
        pix = rows[idx // w].astype(np.int64) * w + idx % w
        return oracle_lib.flags_pixels(cfg, w, h, pix, ref_out[idx])

    rep, flags, cand = check_frame(g_out, ref_out, g_rgb, ref_rgb, flag_fn)
    return rep, cand, ref_st


# ---- the ray-pair kernel's outcomes through the MarchFn entry ---------------

@pytest.mark.parametrize("name", golden_cases())
def test_rr_march_outcomes_vs_reference_goldens(renderer, name):
    """rr_march (MarchFn, kernel.hpp:47): a Gaussian-bump RK4 scene runs the
    ray-pair kernel (64-ray units), everything else march_kernel; outcomes
    vs the reference goldens."""
    from oracle.parity import compare_outcomes
    cfg, _, z = load_golden(name)
    renderer.set_config(cfg)
    out = renderer.march(cfg.integrator, z["rays"])
    rep = compare_outcomes(out, z["outcomes"], z["flags"])
    assert rep.ok, rep.summary() + " " + "; ".join(rep.details)
    if name in ("c1_gauss1_512", "c3_bumps16_1080p", "c5_bumps16_4k"):
        assert renderer.last_kernel.startswith("march2_kernel"), renderer.last_kernel


def test_outcome_sink_does_not_change_the_frame(renderer):
    """The sink is a branch in the production kernels: frames rendered with
    and without it are byte-identical (unlit ray-pair, lit ray-pair,
    one-ray diffeo + mesh)."""
    for name, w, h in (("c3_bumps16_1080p", 320, 180), ("c3_bumps16_shadows_1080p", 320, 180),
                       ("c4_twist_mesh_1080p", 192, 108)):
        cfg = _load(name)
        rgb_o, out, st_o, kern = _gpu_frame(renderer, cfg, w, h)
        cam = renderer.build_camera(cfg.camera)
        rgb, st = renderer.render(cam, cfg.integrator, w, h)
        assert np.array_equal(rgb, rgb_o), name
        assert st["total_steps"] == st_o["total_steps"] == int(out["steps"].sum()), name
        if name.startswith("c3"):
            assert kern.startswith("march2_kernel"), kern


@pytest.mark.parametrize("name,w,h", [("c1_gauss1_512", 160, 120), ("c3_bumps16_1080p", 192, 108),
                                      ("c3_bumps16_shadows_1080p", 192, 108),
                                      ("c5_bumps16_4k", 240, 135)])
def test_march2_frame_outcomes_vs_oracle(renderer, oracle_lib, name, w, h):
    cfg = _load(name)
    rgb, out, st, kern = _gpu_frame(renderer, cfg, w, h)
    assert kern.startswith("march2_kernel"), kern
    rep, cand, _ = _check_vs_oracle(oracle_lib, cfg, w, h, rgb, out)
    _log(f"{name} {w}x{h}", rep, cand, kern)
    assert rep.ok, f"{name}: {rep.summary()} candidates={cand}"
    assert (out["status"] == 1).sum() > 0.3 * w * h


# ---- the benchmarked frames, at their benchmarked settings ------------------

def test_c3_1080p_full_frame_vs_reference(renderer, oracle_lib, reference_lib):
    """The headline frame: 1920x1080, 16 bumps, RK4 h=0.05 / 400, every pixel,
    against the reference's own MarchFn (KernelKind::Avx2, all host threads)."""
    from oracle.parity import check_frame
    cfg = _load("c3_bumps16_1080p")
    w, h = 1920, 1080
    rgb, out, st, kern = _gpu_frame(renderer, cfg, w, h)
    assert kern == "march2_kernel<bumps16>"
    ref_rgb, ref_out, _ = reference_lib.render_rows(cfg, w, h, 0, 1, kernel="avx2",
                                                   with_outcomes=True)
    rep, _, cand = check_frame(out, ref_out, rgb, ref_rgb,
                               lambda idx: oracle_lib.flags_pixels(cfg, w, h, idx, ref_out[idx]))
    _log("c3_bumps16_1080p 1920x1080 full frame vs reference", rep, cand, kern)
    assert rep.ok, f"{rep.summary()} candidates={cand}"
    assert rep.n == w * h
    assert abs(st["total_steps"] - int(ref_out["steps"].sum())) <= 1e-3 * st["total_steps"]


def test_c3_lit_1080p_full_frame_vs_oracle(renderer, oracle_lib):
    """The north-star frame: C3 + shadow geodesics to 2 point lights (hit-record
    + shadow launches), every pixel, against the FP64 oracle extension."""
    cfg = _load("c3_bumps16_shadows_1080p")
    w, h = 1920, 1080
    rgb, out, st, kern = _gpu_frame(renderer, cfg, w, h)
    assert kern == "march2_kernel<bumps16>" and st["kernel_launches"] - st["sort_kernels"] == 2
    rep, cand, ref_st = _check_vs_oracle(oracle_lib, cfg, w, h, rgb, out)
    _log("c3_bumps16_shadows_1080p 1920x1080 full frame vs oracle", rep, cand, kern)
    assert rep.ok, f"{rep.summary()} candidates={cand}"
    assert rep.n == w * h
    assert abs(st["shadow_steps"] - ref_st["shadow_steps"]) <= 5e-3 * ref_st["shadow_steps"]


def test_c4_twist_mesh_benchmarked_settings_vs_oracle(renderer, oracle_lib):
    """C4 as benchmarked: twist pull-back + 100k-triangle mesh, 1920x1080,
    RK4 h=0.01, max 2000 (configs/c4_twist_mesh_1080p.json), every 2nd row."""
    cfg = _load("c4_twist_mesh_1080p")
    assert cfg.integrator.h == 0.01 and cfg.integrator.max_steps == 2000
    w, h = 1920, 1080
    rgb, out, st, kern = _gpu_frame(renderer, cfg, w, h)
    assert kern in ("march_kernel<diffeo,mesh>", "march2_kernel<twist,mesh>"), kern
    rep, cand, _ = _check_vs_oracle(oracle_lib, cfg, w, h, rgb, out, 0, 2)
    _log("c4_twist_mesh_1080p 1920x1080 h=0.01 every 2nd row vs oracle", rep, cand, kern)
    assert rep.ok, f"{rep.summary()} candidates={cand}"
    assert (out["prim"] == 3).sum() > 0.01 * w * h        # the mesh is in view (~2% of the frame)


def test_c5_4k_row_subsample_vs_oracle(renderer, oracle_lib):
    """C5 as benchmarked: 3840x2160, 16 bumps, RK4 h=0.05 / 256; the GPU renders
    the whole 4K frame, every 4th row is compared."""
    cfg = _load("c5_bumps16_4k")
    w, h = 3840, 2160
    rgb, out, st, kern = _gpu_frame(renderer, cfg, w, h)
    assert kern == "march2_kernel<bumps16>"
    rep, cand, _ = _check_vs_oracle(oracle_lib, cfg, w, h, rgb, out, 1, 4)
    _log("c5_bumps16_4k 3840x2160 every 4th row vs oracle", rep, cand, kern)
    assert rep.ok, f"{rep.summary()} candidates={cand}"
