"""CPU: the config parser accepts/rejects exactly what the reference parser
does (config.cpp) and produces the same fully-defaulted document; the CLI
keeps rray's flags and exit codes (rray_main.cpp)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from paper_2005_05386_b200.config import config_to_dict, parse_config, serialize_config
from paper_2005_05386_b200.errors import ConfigError, ParseError

G = {"kind": "gaussian", "amplitude": 1.0, "center": [1, 2, 3], "sigma": [0.5, 0.6, 0.7]}
BASE = {"metric": {"kind": "graph", "field": G}}


def doc(**over):
    d = json.loads(json.dumps(BASE))
    for k, v in over.items():
        d[k] = v
    return json.dumps(d)


VALID = [
    '{"metric": {"kind": "euclidean"}}',
    doc(),
    doc(scene={}),
    doc(scene={"bounds": {"min": [-5, -5, -5], "max": [5, 5, 5]}}),
    doc(scene={"primitives": []}),
    doc(scene={"primitives": [{"kind": "grid_planes"}]}),
    doc(scene={"primitives": [{"kind": "grid_planes", "spacing": 0.5, "half_width": 0.1,
                               "bounds": {"min": [-1, -1, -1], "max": [1, 1, 1]}}]}),
    doc(scene={"primitives": [{"kind": "sphere", "center": [1, 1, 1], "radius": 2}]}),
    doc(scene={"primitives": [{"kind": "half_space", "normal": [0, 0, 2], "offset": -1}]}),
    doc(camera={"fov_deg": 90, "position": [1, 2, 3]}),
    doc(integrator={"h": 0.5, "max_steps": 3, "scheme": "rk4"}),
    doc(output={"path": "a.ppm", "width": 7, "height": 9}),
    json.dumps({"metric": {"kind": "graph", "field": {"kind": "sum", "terms": [
        G, {"kind": "polynomial", "terms": [{"coef": 2, "powers": [1, 2, 1]}]},
        {"kind": "sum", "terms": []}]}}}),
    json.dumps({"metric": {"kind": "diffeo", "map": {"kind": "compose", "maps": [
        {"kind": "twist"}, {"kind": "identity"},
        {"kind": "affine", "matrix": [[1, 2, 3], [4, 5, 6], [7, 8, 10]]},
        {"kind": "local_bump", "amplitude": 0.3, "center": [0, 0, 0], "sigma": [1, 1, 1],
         "direction": [0, 1, 0]}]}}}),
]

INVALID = [
    "{not json",
    "[]",
    "{}",
    '{"metric": {"kind": "euclidean"}, "extra": 1}',
    '{"metric": {"kind": "nope"}}',
    '{"metric": {"kind": "euclidean", "field": 1}}',
    '{"metric": {"kind": "graph"}}',
    doc(scene={"primitives": [{"kind": "sphere", "center": [9.5, 0, 0], "radius": 1}]}),
    doc(scene={"primitives": [{"kind": "sphere", "center": [0, 0, 0], "radius": 0}]}),
    doc(scene={"primitives": [{"kind": "grid_planes", "spacing": 0.1, "half_width": 0.05}]}),
    doc(scene={"primitives": [{"kind": "grid_planes", "half_width": 0}]}),
    doc(scene={"primitives": [{"kind": "grid_planes", "bounds": {"min": [-20, 0, 0], "max": [1, 1, 1]}}]}),
    doc(scene={"primitives": [{"kind": "half_space", "normal": [0, 0, 0], "offset": 1}]}),
    doc(scene={"primitives": [{"kind": "cone"}]}),
    doc(scene={"bounds": {"min": [1, 1, 1], "max": [1, 2, 2]}}),
    doc(scene={"fog_density": -1}),
    doc(camera={"fov_deg": 180}),
    doc(camera={"look_dir": [0, 0, 1], "up_hint": [0, 0, 2]}),
    doc(camera={"position": [1, 2]}),
    doc(integrator={"h": 0}),
    doc(integrator={"max_steps": 0}),
    doc(integrator={"max_steps": 2.5}),
    doc(integrator={"scheme": "rk45"}),
    doc(output={"width": 0}),
    doc(output={"format": "png"}),
    doc(output={"path": ""}),
    json.dumps({"metric": {"kind": "graph", "field": dict(G, sigma=[1, 0, 1])}}),
    json.dumps({"metric": {"kind": "graph", "field": dict(G, amplitude="1")}}),
    json.dumps({"metric": {"kind": "graph", "field": dict(G, amplitude=True)}}),
    json.dumps({"metric": {"kind": "graph", "field": {"kind": "polynomial", "terms": [
        {"coef": 1, "powers": [2, 2, 1]}]}}}),
    json.dumps({"metric": {"kind": "graph", "field": {"kind": "polynomial", "terms": [
        {"coef": 1, "powers": [1, 0, -1]}]}}}),
    json.dumps({"metric": {"kind": "graph", "field": {"kind": "polynomial", "terms": [
        {"coef": 1, "powers": [1.0, 0, 0]}]}}}),
    json.dumps({"metric": {"kind": "diffeo", "map": {"kind": "compose", "maps": []}}}),
    json.dumps({"metric": {"kind": "diffeo", "map": {"kind": "affine", "matrix": [[1, 0], [0, 1]]}}}),
    json.dumps({"metric": {"kind": "diffeo", "map": {"kind": "local_bump", "amplitude": 1,
                                                     "center": [0, 0, 0], "sigma": [1, 1, 1]}}}),
    doc(scene={"lights": []}),     # EXT key: the reference rejects it (allow_ext=False here)
]


@pytest.mark.parametrize("text", VALID)
def test_valid_documents_match_reference(reference_lib, text):
    rc, ref_doc = reference_lib.parse(text)
    assert rc == 0, ref_doc
    ours = config_to_dict(parse_config(text, allow_ext=False))
    assert json.loads(ref_doc) == json.loads(json.dumps(ours))


@pytest.mark.parametrize("text", INVALID)
def test_invalid_documents_rejected_like_reference(reference_lib, text):
    rc, msg = reference_lib.parse(text)
    assert rc == 1, "reference accepted it"
    with pytest.raises(ConfigError) as e:
        parse_config(text, allow_ext=False)
    if isinstance(e.value, ParseError):
        assert "config:" in str(e.value)
    else:   # same key path in the message
        assert str(e.value).split(":")[0] == msg.split(":")[0]


def test_round_trip_is_identity():
    for text in VALID:
        cfg = parse_config(text)
        assert parse_config(serialize_config(cfg)) == cfg


def test_extension_keys_accepted_by_default():
    cfg = parse_config(doc(scene={"lights": [{"position": [1, 2, 3]}], "ambient": 0.3}))
    assert cfg.scene.lights[0].intensity == 1.0 and cfg.scene.ambient == 0.3


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2005_05386_b200", *args], cwd=ROOT,
                          capture_output=True, text=True)


def test_cli_print_config_and_exit_codes(tmp_path):
    cfgp = os.path.join(ROOT, "configs", "c1_gauss1_512.json")
    r = _cli("render", cfgp, "--print-config", "--size", "33x22", "--h", "0.5", "-o", "x.ppm")
    assert r.returncode == 0
    d = json.loads(r.stdout)
    assert d["output"]["width"] == 33 and d["output"]["height"] == 22
    assert d["integrator"]["h"] == 0.5 and d["output"]["path"] == "x.ppm"
    assert _cli("render", cfgp, "--size", "bad", "--print-config").returncode == 1
    assert _cli("render", str(tmp_path / "missing.json")).returncode == 3
    bad = tmp_path / "bad.json"
    bad.write_text('{"metric": {"kind": "x"}}')
    assert _cli("render", str(bad)).returncode == 1
    # geodesic: argument errors are config errors (rray_main.cpp:38-45) before any device work
    assert _cli("geodesic", cfgp, "--start", "1,2", "--dir", "1,0,0").returncode == 1
    assert _cli("geodesic", cfgp, "--start", "0,0,0", "--dir", "1,0,0", "--print-config").returncode == 0


def test_animation_moves_bump_centres():
    from paper_2005_05386_b200.cli import animated_config
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c5_bumps16_4k.json"))
    f0 = animated_config(cfg, 0, 30.0, 2.0, 0.3)
    f5 = animated_config(cfg, 5, 30.0, 2.0, 0.3)
    c = cfg.metric.field.terms[3].params.center
    c0 = f0.metric.field.terms[3].params.center
    c5 = f5.metric.field.terms[3].params.center
    assert c0 != c5 and abs(c5[2] - c[2]) == 0.0
    assert abs(((c0[0] - c[0]) ** 2 + (c0[1] - c[1]) ** 2) ** 0.5 - 0.3) < 1e-12
