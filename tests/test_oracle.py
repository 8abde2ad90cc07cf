"""CPU: the FP64 oracle (oracle/rro.c) is pinned bit-for-bit to the reference.

Golden vectors in tests/golden were dumped from the reference itself
(oracle/_ref, tests/golden/make_golden.py); these tests need no GPU and no
/root/reference."""
import numpy as np
import pytest

from conftest import golden_cases, load_golden, outcomes_identical
from paper_2005_05386_b200 import abi


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_reference_outcomes_bitwise(oracle_lib, name):
    cfg, _, z = load_golden(name)
    out = oracle_lib.march(cfg, z["rays"])
    assert outcomes_identical(out, z["outcomes"])


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_render_matches_reference_rgb_bytes(oracle_lib, name):
    cfg, cam_cfg, z = load_golden(name)
    w, h = int(z["w"]), int(z["h"])
    rgb, out, st, _ = oracle_lib.render(cfg, w, h, camera_cfg=cam_cfg)
    assert np.array_equal(rgb, z["rgb"])
    assert st["total_steps"] == int(z["total_steps"])
    assert st["pixel_errors"] == int(z["pixel_errors"])


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_primary_rays_match_reference(oracle_lib, name):
    _, cam_cfg, z = load_golden(name)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cam_cfg), int(z["w"]), int(z["h"]))
    assert rays.tobytes() == z["rays"].tobytes()


def test_oracle_reproduces_reference_goldens_256(oracle_lib):
    """tests/make_goldens.cpp goldens: twist and quadric via the renderer,
    grid_euclid via the independent straight-line tracer (byte-identical to
    the Euclidean render, acceptance.cpp:145-157)."""
    from paper_2005_05386_b200.config import parse_config
    import os
    from conftest import GOLDEN
    g = np.load(os.path.join(GOLDEN, "reference_goldens.npz"))
    for cfg_name, ppm in [("grid_euclid", "grid_euclid_256"), ("twist", "twist_256"),
                          ("quadric_graph", "quadric_graph_256")]:
        text = str(g["config_" + cfg_name])
        if cfg_name == "grid_euclid":
            text = text  # the oracle grid config of reference_tracer.cpp:185-209 equals it
        cfg = parse_config(text)
        rgb, _, _, _ = oracle_lib.render(cfg, 256, 256)
        blob = g["ppm_" + ppm].tobytes()
        header = b"P6\n256 256\n255\n"
        assert blob[:len(header)] == header
        assert rgb.tobytes() == blob[len(header):], ppm


KATS = [
    # (metric json, pos, vel, expected accel) -- test_geodesics.cpp:33-38
    ({"kind": "graph", "field": {"kind": "polynomial", "terms": [
        {"coef": 1.0, "powers": [2, 0, 0]}, {"coef": 1.0, "powers": [0, 2, 0]},
        {"coef": -1.0, "powers": [0, 0, 2]}]}}, [1, 0, 0], [0, 1, 0], [-0.8, 0, 0]),
    ({"kind": "euclidean"}, [0.3, -1.0, 2.0], [0.5, 0.25, -1.0], [0, 0, 0]),
]


@pytest.mark.parametrize("metric,pos,vel,want", KATS)
def test_accel_known_answers(oracle_lib, metric, pos, vel, want):
    from paper_2005_05386_b200.config import parse_config
    import json
    cfg = parse_config(json.dumps({"metric": metric}))
    acc, val = oracle_lib.flow_accel(cfg, pos, vel)
    assert np.allclose(acc, want, rtol=0, atol=1e-15)
    assert val == 1.0


def test_single_twist_closed_form_matches_oracle(oracle_lib):
    """The GPU's single-twist fast path (csrc/rr_kernels.cu accel_diffeo)
    uses a = (z'(2y' + z'x), z'(z'y - 2x'), 0): -J^-1 D^2phi[v, v] of the
    twist (diffeo.hpp:143-173) with the rotation cancelled.  Pin the identity
    against the oracle's general FP64 jet fold at random states."""
    from paper_2005_05386_b200.config import parse_config
    import json
    cfg = parse_config(json.dumps({"metric": {"kind": "diffeo", "map": {"kind": "twist"}}}))
    rng = np.random.default_rng(7)
    for _ in range(200):
        p = rng.uniform(-10, 10, 3)
        v = rng.normal(size=3)
        acc, val = oracle_lib.flow_accel(cfg, p, v)
        want = [v[2] * (v[2] * p[0] + 2 * v[1]), v[2] * (v[2] * p[1] - 2 * v[0]), 0.0]
        assert np.allclose(acc, want, rtol=1e-12, atol=1e-12)
        assert val > 1e-14


def test_euler_step_known_answer(oracle_lib):
    """test_geodesics.cpp:57-65"""
    from paper_2005_05386_b200.config import parse_config
    import json
    cfg = parse_config(json.dumps({"metric": KATS[0][0], "integrator": {"scheme": "euler"}}))
    out, _ = oracle_lib.step(cfg, [1, 0, 0, 0, 1, 0], 0.01)
    assert np.allclose(out, [1.0, 0.01, 0.0, -0.008, 1.0, 0.0], rtol=1e-14, atol=1e-16)


SCENE_KATS = [
    # test_scene.cpp:26-34, :65-74, :76-89
    ({"primitives": [{"kind": "sphere", "center": [1, 0, 0], "radius": 0.5}],
      "bounds": {"min": [-100] * 3, "max": [100] * 3}}, [0, 0, 0], [2, 0, 0], (0.5, 0.25, 0)),
    ({"primitives": [{"kind": "half_space", "normal": [0, 0, 1], "offset": -1.0}],
      "bounds": {"min": [-100] * 3, "max": [100] * 3}}, [0, 0, -1.5], [0, 0, -2], (0.0, 0.0, 0)),
    ({"primitives": [{"kind": "sphere", "center": [3, 0, 0], "radius": 0.5},
                     {"kind": "sphere", "center": [1.5, 0, 0], "radius": 0.5}],
      "bounds": {"min": [-100] * 3, "max": [100] * 3}}, [0, 0, 0], [4, 0, 0], (1.0, 0.25, 1)),
    ({"primitives": [{"kind": "grid_planes", "spacing": 0.25, "half_width": 0.01}],
      "bounds": {"min": [-10] * 3, "max": [10] * 3}}, [0.02, 0.1, 0.1], [1.02, 0.1, 0.1], (0.24, 0.22, 0)),
]


@pytest.mark.parametrize("scene,a,b,want", SCENE_KATS)
def test_intersection_known_answers(oracle_lib, scene, a, b, want):
    from paper_2005_05386_b200.config import parse_config
    import json
    cfg = parse_config(json.dumps({"metric": {"kind": "euclidean"}, "scene": scene}))
    hit = oracle_lib.intersect(cfg, a, b)
    assert hit is not None
    pt, s, prim = hit
    assert abs(pt[0] - want[0]) < 1e-12 and abs(s - want[1]) < 1e-12 and prim == want[2]


def test_oracle_against_live_reference(oracle_lib, reference_lib):
    """When oracle/_ref is built, re-check a fresh random-camera case live."""
    from paper_2005_05386_b200.config import parse_config, reference_json
    import json
    rng = np.random.default_rng(7)
    for _ in range(3):
        d = {"metric": {"kind": "graph", "field": {"kind": "sum", "terms": [
                {"kind": "gaussian", "amplitude": float(rng.uniform(-1, 1)),
                 "center": [float(x) for x in rng.uniform([1, -2, -0.5], [6, 2, 1.5])],
                 "sigma": [float(x) for x in rng.uniform(0.4, 0.9, 3)]} for _ in range(3)]}},
             "scene": {"primitives": [{"kind": "sphere", "center": [4, 0, 0.3], "radius": 1.0},
                                      {"kind": "half_space", "normal": [0, 0, 1], "offset": -1.0}]},
             "camera": {"position": [0, 0, 0.2], "look_dir": [1, float(rng.uniform(-.2, .2)), 0]},
             "integrator": {"h": 0.05, "max_steps": 300, "scheme": "rk4"}}
        cfg = parse_config(json.dumps(d))
        rays = reference_lib.primary_rays(reference_json(cfg), 24, 16)
        ref = reference_lib.march(reference_json(cfg), rays, "scalar")
        assert outcomes_identical(oracle_lib.march(cfg, rays), ref)


def test_oracle_row_subsample_and_pixel_flags_match_full_frame(oracle_lib):
    """rro_render_rows / rro_flags_pixels (the full-size parity machinery)
    reproduce the whole-frame rro_render / rro_flags bytes, lights included."""
    import os
    from conftest import ROOT
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_shadows_1080p.json"))
    w, h = 64, 36
    rgb, out, st, flags = oracle_lib.render(cfg, w, h, with_flags=True)
    r_rgb, r_out, r_st = oracle_lib.render_rows(cfg, w, h, 1, 3)
    rows = list(range(1, h, 3))
    assert np.array_equal(r_rgb, rgb[rows])
    assert outcomes_identical(r_out, out.reshape(h, w)[rows].reshape(-1))
    assert r_st["rays"] == len(rows) * w and r_st["wall_seconds"] > 0
    pix = np.arange(0, w * h, 7, dtype=np.int64)
    f = oracle_lib.flags_pixels(cfg, w, h, pix, out[pix])
    assert np.array_equal(f, flags[pix])


def test_check_frame_flags_only_failing_pixels(oracle_lib):
    """oracle.parity.check_frame: identical outcomes need no flags; a broken
    pixel is reported unless the oracle flags it."""
    import os
    from conftest import ROOT
    from oracle.parity import check_frame
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c1_gauss1_512.json"))
    w, h = 48, 32
    rgb, out, _, _ = oracle_lib.render(cfg, w, h)
    calls = []

    def flag_fn(idx):
        calls.append(len(idx))
        return oracle_lib.flags_pixels(cfg, w, h, idx, out[idx])

    rep, _, cand = check_frame(out, out, rgb, rgb, flag_fn)
    assert rep.ok and cand == 0 and not calls
    bad = out.copy()
    i = int(np.nonzero(out["status"] == 1)[0][0])
    bad["point"][i] += 1.0
    rep, _, cand = check_frame(bad, out, rgb, rgb, flag_fn)
    assert cand == 1 and calls == [1] and rep.endpoint_fail == 1 and not rep.ok


def test_reference_row_outcomes_match_oracle(reference_lib, oracle_lib):
    """refc_render_rows' outcome records (the reference's own MarchFn per row)
    are bit-identical to the oracle's row subsample."""
    import os
    from conftest import ROOT
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    w, h = 96, 54
    rgb, out, st = reference_lib.render_rows(cfg, w, h, 2, 5, kernel="avx2", workers=4,
                                             with_outcomes=True)
    o_rgb, o_out, _ = oracle_lib.render_rows(cfg, w, h, 2, 5)
    assert outcomes_identical(out, o_out)
    assert np.array_equal(rgb, o_rgb)
