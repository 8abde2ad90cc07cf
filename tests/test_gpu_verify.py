"""GPU: the off-path tools on the device — `verify` property suites
(verify.cpp:274-401 restated, paper_2005_05386_b200/verify.py) and the
`geodesic` polyline export (rray_main.cpp:86-116) against the FP64 oracle's
own RK4/Euler steps (oracle/rro.c rro_step)."""
import os
import subprocess
import sys

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


def test_verify_suites_pass(renderer):
    from paper_2005_05386_b200.verify import run_all_checks
    res = run_all_checks(renderer, 42)
    assert len(res) == 6 + 4 + 2 + 3
    bad = [f"{r.name}: {r.detail}" for r in res if not r.passed]
    assert not bad, bad


def test_verify_cli_exit_code():
    r = subprocess.run([sys.executable, "-m", "paper_2005_05386_b200", "verify", "--seed", "7"],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().splitlines()[-1] == "15/15 suites passed (seed 7)"


@pytest.mark.parametrize("metric,scheme", [
    ({"kind": "graph", "field": {"kind": "gaussian", "amplitude": 1.0, "center": [0.3, -0.2, 0.1],
                                 "sigma": [0.8, 0.7, 0.9]}}, "rk4"),
    ({"kind": "diffeo", "map": {"kind": "twist"}}, "euler"),
    ({"kind": "diffeo", "map": {"kind": "compose", "maps": [
        {"kind": "local_bump", "amplitude": 0.3, "center": [0.4, 0, -0.2], "sigma": [0.8, 0.9, 0.7],
         "direction": [0.5, 0.3, -0.6]}, {"kind": "twist"}]}}, "rk4"),
    ({"kind": "graph", "field": {"kind": "polynomial", "terms": [
        {"coef": 0.3, "powers": [2, 0, 0]}, {"coef": -0.2, "powers": [1, 1, 1]}]}}, "rk4"),
])
def test_trace_matches_oracle_steps(renderer, oracle_lib, metric, scheme):
    """Device polylines vs the FP64 oracle's flow steps (rro_step), state by state."""
    from paper_2005_05386_b200 import config as cfgmod
    from paper_2005_05386_b200.config import IntegratorConfig
    scene = cfgmod.Scene()
    m = cfgmod._parse_metric(metric, "metric")
    renderer.set_scene(m, scene)
    integ = IntegratorConfig(h=0.01, max_steps=300, scheme=scheme)
    start = np.array([0.4, -0.2, 0.3, 0.8, 0.5, 0.33])
    states, counts, fail = renderer.trace(integ, start[None, :], use_bounds=False)
    assert fail[0] == -1 and counts[0] == 301
    cfg = cfgmod.RunConfig()
    cfg.metric, cfg.integrator = m, integ
    ref = [start]
    s = start.copy()
    for _ in range(300):
        s, _val = oracle_lib.step(cfg, s, 0.01)
        ref.append(s)
    ref = np.array(ref)
    err = np.abs(states[0] - ref).max(axis=1) / np.maximum(1.0, np.abs(ref).max(axis=1))
    assert err.max() < 2e-5, err.max()


def test_trace_stops_after_leaving_bounds(renderer):
    from paper_2005_05386_b200 import config as cfgmod
    from paper_2005_05386_b200.config import IntegratorConfig
    scene = cfgmod.Scene()
    scene.bounds = cfgmod.Aabb([-1.0, -1.0, -1.0], [1.0, 1.0, 1.0])
    renderer.set_scene(cfgmod.EuclideanMetric(), scene)
    integ = IntegratorConfig(h=0.1, max_steps=100, scheme="euler")
    states, counts, fail = renderer.trace(integ, np.array([[0.0, 0, 0, 1, 0, 0]]), use_bounds=True)
    # x = 0.1 i leaves [-1, 1] at i = 11 (the exiting state is kept): 12 states
    assert counts[0] == 12 and fail[0] == -1
    assert abs(states[0, 11, 0] - 1.1) < 1e-6
    states, counts, _ = renderer.trace(integ, np.array([[0.0, 0, 0, 1, 0, 0]]), use_bounds=False)
    assert counts[0] == 101


def test_geodesic_cli_writes_csv(tmp_path):
    out = tmp_path / "g.csv"
    cfgp = os.path.join(ROOT, "configs", "c4_twist_1080p.json")
    r = subprocess.run([sys.executable, "-m", "paper_2005_05386_b200", "geodesic", cfgp,
                        "--start", "0,0,0.2", "--dir", "1,0.2,0", "-o", str(out), "--h", "0.05"],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "t,x,y,z,vx,vy,vz"
    rows = np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])
    assert rows[0, 0] == 0.0 and np.allclose(rows[0, 1:4], [0, 0, 0.2])
    assert np.allclose(np.diff(rows[:, 0]), 0.05)
    assert f"{len(rows)} states, h = 0.05" in r.stdout
