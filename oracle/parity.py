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

from . import (FLAG_GRAZING, FLAG_LIMIT, FLAG_SHADOW, FLAG_WRAP, FLAG_WRAP_X, FLAG_WRAP_Y,
               FLAG_WRAP_Z)

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


# ---- full-size frames --------------------------------------------------------
# Flags only ever EXEMPT a difference, so a full-size check needs the
# (expensive, 4-12 extra FP64 marches per pixel) GRAZING / LIMIT / SHADOW
# flags of the pixels whose GPU result differs from the oracle's, and nothing
# else: WRAP (a coordinate test on the FP64 outcome) is computed everywhere,
# the candidates are the pixels that fail any rule with WRAP alone, and the
# oracle flags exactly those (rro_flags_pixels).  The report is then the
# ordinary compare_outcomes / compare_rgb report over the whole frame.

def wrap_flags(ref: np.ndarray, eps: float = 1e-4) -> np.ndarray:
    """rro.c near_integer per hit coordinate (render.cpp:18's frac wrap)."""
    f = np.zeros(len(ref), np.uint8)
    hit = ref["status"] == 1
    for k, bit in enumerate((FLAG_WRAP_X, FLAG_WRAP_Y, FLAG_WRAP_Z)):
        c = ref["point"][:, k]
        near = np.abs(c - np.rint(c)) < eps
        f |= np.where(hit & near, np.uint8(bit | FLAG_WRAP), np.uint8(0))
    return f


def failing_pixels(gpu: np.ndarray, ref: np.ndarray, gpu_rgb, ref_rgb, flags) -> np.ndarray:
    """Pixels that break a parity rule under `flags` (the per-pixel version of
    compare_outcomes + compare_rgb)."""
    keep = (flags & (FLAG_GRAZING | FLAG_LIMIT)) == 0
    bad = (gpu["status"] != ref["status"]) & keep
    hit = (ref["status"] == 1) & (gpu["status"] == 1) & keep
    bad |= (gpu["prim"] != ref["prim"]) & hit
    d = np.linalg.norm(gpu["point"] - ref["point"], axis=1)
    nrm = np.maximum(np.linalg.norm(ref["point"], axis=1), 1e-300)
    bad |= hit & (d / nrm > ENDPOINT_RTOL)
    if gpu_rgb is not None:
        g = gpu_rgb.reshape(-1, 3).astype(np.int32)
        r = ref_rgb.reshape(-1, 3).astype(np.int32)
        diff = np.abs(g - r)
        for ch, bit in enumerate((FLAG_WRAP_X, FLAG_WRAP_Y, FLAG_WRAP_Z)):
            diff[(flags & bit) != 0, ch] = 0
        keep_rgb = (flags & (FLAG_GRAZING | FLAG_LIMIT | FLAG_SHADOW)) == 0
        bad |= (diff.max(axis=1) > RGB_TOL) & keep_rgb
    return bad


def check_frame(gpu_out: np.ndarray, ref_out: np.ndarray, gpu_rgb, ref_rgb, flag_fn):
    """Full-frame (or row-subsample) parity.  flag_fn(idx) -> the oracle's
    flags of the listed pixels (indices into the arrays given here).
    Returns (ParityReport, flags, candidates)."""
    flags = wrap_flags(ref_out)
    cand = np.nonzero(failing_pixels(gpu_out, ref_out, gpu_rgb, ref_rgb, flags))[0]
    if len(cand):
        flags[cand] |= flag_fn(cand)
    rep = compare_outcomes(gpu_out, ref_out, flags)
    if gpu_rgb is not None:
        rep = compare_rgb(gpu_rgb, ref_rgb, flags, rep)
    return rep, flags, int(len(cand))
