"""CPU: the oracle's mesh primitive (EXTENSION).  Its BVH only prunes: results
must equal a brute-force scan of every triangle; hit points lie on the mesh."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT, outcomes_identical
from paper_2005_05386_b200.config import parse_config


def mesh_cfg(nu=24, nv=12, metric=None, **integ):
    d = json.load(open(os.path.join(ROOT, "configs", "c4_twist_mesh_1080p.json")))
    d["scene"]["primitives"][-1]["generator"].update(nu=nu, nv=nv)
    if metric is not None:
        d["metric"] = metric
    d["integrator"].update(integ or {"h": 0.04, "max_steps": 400})
    return parse_config(json.dumps(d))


@pytest.mark.parametrize("metric", [None, {"kind": "euclidean"}])
def test_mesh_bvh_equals_bruteforce(oracle_lib, metric):
    cfg = mesh_cfg(metric=metric)
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), 32, 18)
    oracle_lib.set_mesh_bruteforce(False)
    a = oracle_lib.march(cfg, rays)
    oracle_lib.set_mesh_bruteforce(True)
    try:
        b = oracle_lib.march(cfg, rays)
    finally:
        oracle_lib.set_mesh_bruteforce(False)
    assert outcomes_identical(a, b)
    assert (a["prim"] == 3).sum() > 10      # the mesh is visible


def test_mesh_hit_points_on_triangles(oracle_lib):
    from paper_2005_05386_b200.config import Mesh
    cfg = mesh_cfg(metric={"kind": "euclidean"})
    mesh = [p for p in cfg.scene.primitives if isinstance(p, Mesh)][0]
    rays = oracle_lib.primary_rays(oracle_lib.camera(cfg), 32, 18)
    out = oracle_lib.march(cfg, rays)
    hits = out[out["prim"] == 3]
    v = mesh.vertices[mesh.triangles]            # (m, 3, 3)
    n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    for p in hits["point"][:50]:
        dist = np.abs(((p - v[:, 0]) * n).sum(1))
        assert dist.min() < 1e-9


def test_bend_pullback_geodesics_are_straight(oracle_lib):
    """EXTENSION bend: Phi maps geodesics of g = J^T J to straight lines (the
    reference's pull-back straightness property, verify.cpp:233-261)."""
    cfg = parse_config(json.dumps({"metric": {"kind": "diffeo", "map": {"kind": "bend",
                                                                        "curvature": 0.15}},
                                   "integrator": {"scheme": "rk4"}}))
    k = 0.15

    def phi(p):
        c = 1 / k
        th = k * p[0]
        return np.array([-np.sin(th) * (p[1] - c), np.cos(th) * (p[1] - c) + c, p[2]])
    st = [0.5, 0.4, 0.6, 0.8, 0.3, 0.2]
    pts = [phi(np.array(st[:3]))]
    for _ in range(200):
        st, val = oracle_lib.step(cfg, st, 0.01)
        assert val > 1e-14
        pts.append(phi(np.array(st[:3])))
    P = np.array(pts)
    d = (P[-1] - P[0]) / np.linalg.norm(P[-1] - P[0])
    dev = np.linalg.norm((P - P[0]) - np.outer((P - P[0]) @ d, d), axis=1).max()
    assert dev < 1e-10
