"""GPU: `python -m paper_2005_05386_b200 render/animate` (rray_main.cpp render
path on B200): PPM + report sidecar, parity with the reference frame."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu


def test_cli_render_writes_ppm_and_report(tmp_path):
    from oracle.parity import compare_rgb
    from paper_2005_05386_b200.render import read_ppm
    cfg, _, z = load_golden("ref_twist")
    cfgp = tmp_path / "twist.json"
    cfgp.write_text(str(z["config"]))
    out = tmp_path / "twist.ppm"
    r = subprocess.run([sys.executable, "-m", "paper_2005_05386_b200", "render", str(cfgp), "-o",
                        str(out), "--size", f"{int(z['w'])}x{int(z['h'])}"], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    img = read_ppm(str(out))
    assert compare_rgb(img.data, z["rgb"], z["flags"]).ok
    rep = (tmp_path / "twist.report.txt").read_text()
    assert "kernel: cuda (march_kernel<diffeo>)" in rep and "pixel_errors: 0" in rep
    assert "steps/ray" in r.stdout


def test_cli_animate_frames(tmp_path):
    cfgp = os.path.join(ROOT, "configs", "c5_bumps16_4k.json")
    pat = str(tmp_path / "f_%02d.ppm")
    r = subprocess.run([sys.executable, "-m", "paper_2005_05386_b200", "animate", cfgp, "--frames",
                        "3", "--size", "160x90", "-o", pat], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    frames = [open(pat % k, "rb").read() for k in range(3)]
    assert frames[0] != frames[1] != frames[2]
    assert "fps" in r.stdout


def test_cli_geodesic_csv(tmp_path):
    """`geodesic` (rray_main.cpp:86-116): t,x,y,z,vx,vy,vz rows from the
    device trace_geodesic, starting at the given point with unit g-speed."""
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    cfgp = os.path.join(ROOT, "configs", "c3_bumps16_1080p.json")
    out = tmp_path / "g.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2005_05386_b200", "geodesic", cfgp, "--start",
                        "0,0,0.5", "--dir", "1,0.2,0", "-o", str(out), "--h", "0.05"], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "t,x,y,z,vx,vy,vz"
    rows = np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])
    assert len(rows) > 10 and np.allclose(rows[0, 1:4], [0, 0, 0.5])
    assert np.allclose(np.diff(rows[:, 0]), 0.05)
    cfg = load_config(cfgp)
    cfg.integrator.h = 0.05
    rr = Renderer(0)
    rr.set_config(cfg)
    g = rr.metric_tensor(np.array([0, 0, 0.5]))
    d = np.array([1, 0.2, 0])
    assert abs(rows[0, 4:] @ g @ rows[0, 4:] - 1.0) < 1e-12      # unit g-speed start
    states, counts, _ = rr.trace(cfg.integrator, np.concatenate([[0, 0, 0.5], d / np.sqrt(d @ g @ d)]))
    rr.close()
    assert int(counts[0]) == len(rows)
    assert np.array_equal(states[0, :len(rows)], rows[:, 1:])
