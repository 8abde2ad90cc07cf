"""Device-side property suites: `python -m paper_2005_05386_b200 verify`.

Restates the reference's `rray verify` (src/verify/verify.cpp:274-401,
tools/rray_main.cpp:118-131) against the B200 build's arithmetic — the
suites that exercise what the device computes (the flow acceleration and
the Euler/RK4 steps), on the reference's own designed fields
(verify.cpp:47-84, 178-198):

  metrics/christoffel-oracle/<family>   device Gamma vs the FP64 finite-
                                        difference oracle (metric.cpp:88-133)
  geodesics/euler-order/<family>        Euler endpoint error ratios ~2
  geodesics/energy-rk4                  RK4 energy drift
  geodesics/energy-euler-halving        Euler drift ratio ~0.5
  geodesics/pullback-straightness/<map> Phi-images of diffeo geodesics are
                                        straight lines (Euler ratios ~0.5, RK4)

The device Gamma is recovered from `rr_accel` (a = -Gamma(y, y)) by
polarisation: Gamma_ii = -a(e_i), Gamma_ij = -(a(e_i+e_j) - a(e_i) - a(e_j))/2.
Polylines come from `rr_trace` (trace_geodesic on the device); g and Phi
are the FP64 host mirrors (`rr_metric_tensor`, `rr_diffeo_image`).

FP32 tolerances.  The reference's thresholds that sit below FP32 resolution
are restated for FP32 and marked "(fp32 tol ...)" in the detail: Gamma 1e-5
absolute becomes 1e-5 relative to max(1, |Gamma|); RK4 energy drift and RK4
straightness 1e-8 become 1e-5 ("RK4 < 1e-8 is not attainable in
FP32").  The order/halving ratio windows are the reference's own.  The FP64
field-library identities (fields/derivatives, sym-inverse round trip, det
identities, twist volume) check the reference's FP64 field calculus, which
has no device counterpart, and are not restated.  Sample points use numpy's
PCG64 with the given seed over [-2, 2]^3 (verify.cpp:17-23 uses mt19937_64:
the seed is deterministic, the points differ).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

from . import config as cfgmod

K_START = np.array([0.4, -0.2, 0.3])           # verify.cpp:86-87
K_START_DIR = np.array([1.0, 0.6, 0.45])


@dataclass
class CheckResult:                             # verify.hpp CheckResult
    name: str
    passed: bool
    detail: str


def _gauss(a, c, s):
    return {"kind": "gaussian", "amplitude": a, "center": list(c), "sigma": list(s)}


def _bump(a, c, s, d):
    return {"kind": "local_bump", "amplitude": a, "center": list(c), "sigma": list(s),
            "direction": list(d)}


QUADRIC = {"kind": "polynomial", "terms": [{"coef": 1.0, "powers": [2, 0, 0]},
                                           {"coef": 1.0, "powers": [0, 2, 0]},
                                           {"coef": -1.0, "powers": [0, 0, 2]}]}   # scalar_field.hpp:82-84
GAUSSIAN = _gauss(1.0, (0.3, -0.2, 0.1), (0.8, 0.7, 0.9))                          # verify.cpp:49-51
TWO_GAUSSIANS = {"kind": "sum", "terms": [_gauss(0.8, (-0.6, 0.4, 0.0), (0.7, 0.9, 0.8)),
                                          _gauss(-0.5, (0.5, -0.3, 0.6), (1.1, 0.6, 0.7))]}
BUMP_A = _bump(0.3, (0.4, 0.0, -0.2), (0.8, 0.9, 0.7), (0.5, 0.3, -0.6))            # verify.cpp:58-68
BUMP_B = _bump(-0.25, (-0.3, 0.2, 0.3), (0.9, 0.7, 0.8), (-0.4, 0.6, 0.3))
TWIST = {"kind": "twist"}


def _graph(f):
    return {"kind": "graph", "field": f}


def _diffeo(m):
    return {"kind": "diffeo", "map": m}


ORACLE_FAMILIES = [                                                                 # verify.cpp:178-189
    ("graph-quadric", _graph(QUADRIC)),
    ("graph-gaussian", _graph(GAUSSIAN)),
    ("graph-two-gaussians", _graph(TWO_GAUSSIANS)),
    ("diffeo-twist", _diffeo(TWIST)),
    ("diffeo-bump", _diffeo(BUMP_A)),
    ("diffeo-compose-bumps", _diffeo({"kind": "compose", "maps": [BUMP_A, BUMP_B]})),
]
CURVED_FAMILIES = [ORACLE_FAMILIES[i] for i in (0, 1, 3, 4)]                        # verify.cpp:191-198
STRAIGHTNESS_MAPS = [("twist", TWIST), ("local-bump", BUMP_A),
                     ("compose-2", {"kind": "compose", "maps": [BUMP_A, BUMP_B]})]  # verify.cpp:381-385


def _fmt(x: float) -> str:
    return f"{x:.3e}"


class _Suite:
    def __init__(self, renderer):
        self.r = renderer
        # a scene is required by the context; verify never intersects it
        self.scene = cfgmod.Scene()
        self.scene.bounds = cfgmod.Aabb([-1e3] * 3, [1e3] * 3)

    def use(self, metric_json):
        self.r.set_scene(cfgmod._parse_metric(metric_json, "metric"), self.scene)

    # -- device Gamma by polarisation ----------------------------------------
    def device_gamma(self, pts: np.ndarray) -> np.ndarray:
        e = np.eye(3)
        dirs = [e[0], e[1], e[2], e[0] + e[1], e[0] + e[2], e[1] + e[2]]
        n = len(pts)
        pos = np.repeat(pts, len(dirs), axis=0)
        vel = np.tile(np.array(dirs), (n, 1))
        acc, _ = self.r.accel(pos, vel)
        acc = acc.reshape(n, len(dirs), 3)
        gam = np.zeros((n, 3, 3, 3))                  # [point, m, i, j]
        for i in range(3):
            gam[:, :, i, i] = -acc[:, i, :]
        for q, (i, j) in enumerate(((0, 1), (0, 2), (1, 2))):
            off = -(acc[:, 3 + q, :] - acc[:, i, :] - acc[:, j, :]) / 2.0
            gam[:, :, i, j] = off
            gam[:, :, j, i] = off
        return gam

    def unit_speed_start(self) -> np.ndarray:         # verify.cpp:89-93
        g = self.r.metric_tensor(K_START)
        n = np.sqrt(K_START_DIR @ g @ K_START_DIR)
        return np.concatenate([K_START, K_START_DIR / n])

    def polyline(self, start, scheme: str, h: float, steps: int) -> np.ndarray:
        integ = cfgmod.IntegratorConfig(h=h, max_steps=steps, scheme=scheme)
        states, counts, fail = self.r.trace(integ, start[None, :], use_bounds=False)
        if fail[0] >= 0:
            from .errors import NumericError
            raise NumericError(f"trace_geodesic: metric evaluation failed (|det J| <= 1e-14) "
                               f"at step {int(fail[0])}")
        return states[0, :counts[0]]

    def energy_drift(self, scheme: str, h: float, steps: int) -> float:   # verify.cpp:229-249
        line = self.polyline(self.unit_speed_start(), scheme, h, steps)
        e = np.array([s[3:] @ self.r.metric_tensor(s[:3]) @ s[3:] for s in line])
        return float(np.max(np.abs(e[1:] - e[0]) / e[0]))


def run_all_checks(renderer, seed: int = 42) -> List[CheckResult]:
    """verify.cpp:274-401 restated on the device (see the module docstring)."""
    s = _Suite(renderer)
    out: List[CheckResult] = []
    add = lambda name, ok, detail: out.append(CheckResult(name, bool(ok), detail))
    pts = np.random.default_rng(seed).uniform(-2.0, 2.0, size=(100, 3))

    # metrics/christoffel-oracle (verify.cpp:140-148, 329-333)
    for name, m in ORACLE_FAMILIES:
        s.use(m)
        dev = s.device_gamma(pts)
        worst = 0.0
        for k, p in enumerate(pts):
            fd = renderer.christoffel_fd(p)
            worst = max(worst, float(np.max(np.abs(dev[k] - fd)) / max(1.0, np.max(np.abs(fd)))))
        add("metrics/christoffel-oracle/" + name, worst < 1e-5,
            f"max rel err {_fmt(worst)} (fp32 tol 1e-5 x max(1,|Gamma|); ref 1e-5 abs in fp64)")

    # geodesics/euler-order (verify.cpp:200-216, 355-366)
    for name, m in CURVED_FAMILIES:
        s.use(m)
        start = s.unit_speed_start()
        errs = []
        for h in (1e-2, 5e-3, 2.5e-3):
            steps = int(round(0.64 / h))
            xe = s.polyline(start, "euler", h, steps)[-1, :3]
            xr = s.polyline(start, "rk4", h / 64.0, steps * 64)[-1, :3]
            errs.append(float(np.linalg.norm(xe - xr)))
        ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
        add("geodesics/euler-order/" + name, all(1.7 < r < 2.3 for r in ratios),
            "ratios " + " ".join(_fmt(r) for r in ratios) + " (expect ~2)")

    # geodesics/energy-rk4 and energy-euler-halving (verify.cpp:368-389)
    ok, detail = True, ""
    for name, m in ORACLE_FAMILIES:
        s.use(m)
        d = s.energy_drift("rk4", 1e-3, 1000)
        ok = ok and d < 1e-5
        detail += f"{name} {_fmt(d)}  "
    add("geodesics/energy-rk4", ok, detail + "(fp32 tol 1e-5; ref 1e-8 in fp64)")
    ok, detail = True, ""
    for name, m in CURVED_FAMILIES:
        s.use(m)
        r = s.energy_drift("euler", 1e-3, 1000) / s.energy_drift("euler", 2e-3, 500)
        ok = ok and 0.4 < r < 0.6
        detail += f"{name} {_fmt(r)}  "
    add("geodesics/energy-euler-halving", ok, detail + "(expect ~0.5)")

    # geodesics/pullback-straightness (verify.cpp:251-280, 391-399)
    for name, mp in STRAIGHTNESS_MAPS:
        s.use(_diffeo(mp))
        start = s.unit_speed_start()
        q0 = renderer.diffeo_image(start[:3])
        eps = 1e-6                                     # w = J v (FP64 central difference)
        w = (renderer.diffeo_image(start[:3] + eps * start[3:]) -
             renderer.diffeo_image(start[:3] - eps * start[3:])) / (2 * eps)

        def deviation(scheme, h):
            steps = int(round(1.0 / h))
            line = s.polyline(start, scheme, h, steps)
            return max(float(np.linalg.norm(renderer.diffeo_image(st[:3]) - (q0 + i * h * w)))
                       for i, st in enumerate(line))

        eul = [deviation("euler", h) for h in (1e-2, 5e-3, 2.5e-3)]
        rk4 = deviation("rk4", 1e-2)
        ratios = [eul[i + 1] / eul[i] for i in range(len(eul) - 1)]
        add("geodesics/pullback-straightness/" + name,
            all(0.4 < r < 0.6 for r in ratios) and rk4 < 1e-5,
            "euler ratios " + " ".join(_fmt(r) for r in ratios) +
            f", rk4 {_fmt(rk4)} (fp32 tol 1e-5; ref 1e-8 in fp64)")
    return out


def cmd_verify(seed: int = 42, device: int = 0) -> int:
    """rray_main.cpp:118-131: table + summary; exit 0 iff every suite passes, else 2."""
    from .render import Renderer
    r = Renderer(device)
    try:
        results = run_all_checks(r, seed)
    finally:
        r.close()
    width = max(len(x.name) for x in results)
    failures = sum(not x.passed for x in results)
    for x in results:
        print(f"{'[PASS]' if x.passed else '[FAIL]':6s} {x.name:<{width}s} {x.detail}")
    print(f"{len(results) - failures}/{len(results)} suites passed (seed {seed})")
    return 0 if failures == 0 else 2
