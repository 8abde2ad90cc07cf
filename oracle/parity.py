"""TEST INFRASTRUCTURE ONLY — the parity contract of BASELINE.json's north star.

GPU (FP32) results are compared with the FP64 oracle (which is bit-identical
to the reference, see tests/test_oracle.py):

* status and hit-primitive equal on every ray not flagged GRAZING/LIMIT;
* geodesic endpoints within 1e-4 relative on those rays' hits;
* pixel RGB within 1/255 on pixels not flagged GRAZING/LIMIT, per channel
  except channels flagged WRAP_X/Y/Z;
* magenta (failed) counts equal.

Flags come from oracle.Oracle.render(with_flags=True) (rro.c rro_flags):
GRAZING = status/prim changes under +-1e-4 rad direction perturbations,
WRAP = a hit coordinate within 1e-4 of an integer (frac() discontinuity of
render.cpp:18; WRAP_X/Y/Z name the channel), LIMIT = a hit on the last step
or an exhausted miss that one more step would turn into a hit, SHADOW = a
light's visibility flips under +-1e-4 rad shadow-ray perturbations (EXT).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import FLAG_GRAZING, FLAG_LIMIT, FLAG_SHADOW, FLAG_WRAP_X, FLAG_WRAP_Y, FLAG_WRAP_Z

ENDPOINT_RTOL = 1e-4
RGB_TOL = 1


@dataclass
class ParityReport:
    n: int = 0
    exempt: int = 0
    status_mismatch: int = 0
    prim_mismatch: int = 0
    endpoint_max_rel: float = 0.0
    endpoint_p99_rel: float = 0.0
    endpoint_fail: int = 0
    rgb_max: int = 0
    rgb_fail: int = 0
    magenta_gpu: int = 0
    magenta_ref: int = 0
    details: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return (self.status_mismatch == 0 and self.prim_mismatch == 0 and self.endpoint_fail == 0
                and self.rgb_fail == 0 and self.magenta_gpu == self.magenta_ref)

    def summary(self) -> str:
        return (f"n={self.n} exempt={self.exempt} status_mm={self.status_mismatch} "
                f"prim_mm={self.prim_mismatch} endpoint_max={self.endpoint_max_rel:.2e} "
                f"p99={self.endpoint_p99_rel:.2e} endpoint_fail={self.endpoint_fail} "
                f"rgb_max={self.rgb_max} rgb_fail={self.rgb_fail} "
                f"magenta={self.magenta_gpu}/{self.magenta_ref}")


def compare_outcomes(gpu: np.ndarray, ref: np.ndarray, flags: np.ndarray | None = None,
                     rep: ParityReport | None = None) -> ParityReport:
    rep = rep or ParityReport()
    n = len(ref)
    flags = np.zeros(n, np.uint8) if flags is None else flags
    exempt = (flags & (FLAG_GRAZING | FLAG_LIMIT)) != 0
    keep = ~exempt
    rep.n = n
    rep.exempt = int(exempt.sum())
    st_mm = (gpu["status"] != ref["status"]) & keep
    rep.status_mismatch = int(st_mm.sum())
    hit = (ref["status"] == 1) & (gpu["status"] == 1) & keep
    rep.prim_mismatch = int(((gpu["prim"] != ref["prim"]) & hit).sum())
    if hit.any():
        d = np.linalg.norm(gpu["point"][hit] - ref["point"][hit], axis=1)
        nrm = np.maximum(np.linalg.norm(ref["point"][hit], axis=1), 1e-300)
        rel = d / nrm
        rep.endpoint_max_rel = float(rel.max())
        rep.endpoint_p99_rel = float(np.percentile(rel, 99))
        rep.endpoint_fail = int((rel > ENDPOINT_RTOL).sum())
    rep.magenta_gpu = int((gpu["status"] == 2).sum())
    rep.magenta_ref = int((ref["status"] == 2).sum())
    bad = np.nonzero(st_mm)[0][:5]
    for i in bad:
        rep.details.append(f"ray {i}: gpu status {gpu['status'][i]} prim {gpu['prim'][i]} steps "
                           f"{gpu['steps'][i]} vs ref {ref['status'][i]} {ref['prim'][i]} {ref['steps'][i]}")
    return rep


def compare_rgb(gpu_rgb: np.ndarray, ref_rgb: np.ndarray, flags: np.ndarray | None = None,
                rep: ParityReport | None = None) -> ParityReport:
    rep = rep or ParityReport()
    g = gpu_rgb.reshape(-1, 3).astype(np.int32)
    r = ref_rgb.reshape(-1, 3).astype(np.int32)
    flags = np.zeros(len(r), np.uint8) if flags is None else flags
    keep = (flags & (FLAG_GRAZING | FLAG_LIMIT | FLAG_SHADOW)) == 0
    diff = np.abs(g - r)
    # a channel whose coordinate sits on an integer wraps frac() (render.cpp:18)
    for ch, bit in enumerate((FLAG_WRAP_X, FLAG_WRAP_Y, FLAG_WRAP_Z)):
        diff[(flags & bit) != 0, ch] = 0
    diff = diff.max(axis=1)
    rep.rgb_max = int(diff[keep].max()) if keep.any() else 0
    rep.rgb_fail = int((diff[keep] > RGB_TOL).sum())
    magenta = lambda a: int(((a[:, 0] == 255) & (a[:, 1] == 0) & (a[:, 2] == 255)).sum())
    rep.magenta_gpu = magenta(g)
    rep.magenta_ref = magenta(r)
    return rep
