"""TEST INFRASTRUCTURE ONLY — Python bindings of the parity checkers.

* ``Oracle``    — liboracle.so, the FP64 C restatement of the reference path
                  (oracle/rro.c), built by ``make -C oracle``.
* ``Reference`` — oracle/_ref/librray_ref.so, the UNMODIFIED reference sources
                  compiled from /root/reference by ``make -C oracle ref`` plus
                  the C wrapper oracle/ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
--impl reference legs) may import this package, and only as the checker or
the timed CPU baseline — never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2005_05386_b200 import abi
from paper_2005_05386_b200.config import MetricDesc, RunConfig, SceneDesc, fov_radians, reference_json

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librray_ref.so")

FLAG_GRAZING, FLAG_WRAP, FLAG_LIMIT = 1, 2, 4
FLAG_WRAP_X, FLAG_WRAP_Y, FLAG_WRAP_Z = 8, 16, 32
FLAG_SHADOW = 64


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class Oracle:
    """FP64 restatement of the reference path over C-ABI descriptors."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        P = C.c_void_p
        D3 = C.POINTER(C.c_double)
        lib.rro_last_error.restype = C.c_char_p
        lib.rro_flow_accel.argtypes = [C.POINTER(abi.rr_metric_desc), D3, D3, D3, D3]
        lib.rro_step.argtypes = [C.POINTER(abi.rr_metric_desc), D3, C.c_double, C.c_int, D3, D3]
        lib.rro_intersect.argtypes = [C.POINTER(abi.rr_scene_desc), D3, D3, D3, D3, C.POINTER(C.c_int)]
        lib.rro_intersect.restype = C.c_int
        lib.rro_march.argtypes = [C.POINTER(abi.rr_metric_desc), C.POINTER(abi.rr_scene_desc),
                                  C.POINTER(abi.rr_integrator), P, P, C.c_size_t, C.c_int]
        lib.rro_build_camera.argtypes = [C.POINTER(abi.rr_metric_desc), D3, D3, D3, C.c_double,
                                         C.POINTER(abi.rr_camera)]
        lib.rro_build_camera.restype = C.c_int
        lib.rro_pixel_direction.argtypes = [C.POINTER(abi.rr_camera), C.c_int, C.c_int, C.c_int,
                                            C.c_int, D3]
        lib.rro_render.argtypes = [C.POINTER(abi.rr_metric_desc), C.POINTER(abi.rr_scene_desc),
                                   C.POINTER(abi.rr_camera), C.POINTER(abi.rr_integrator),
                                   C.c_int, C.c_int, P, P, C.POINTER(abi.rr_stats), C.c_int]
        lib.rro_flags.argtypes = [C.POINTER(abi.rr_metric_desc), C.POINTER(abi.rr_scene_desc),
                                  C.POINTER(abi.rr_camera), C.POINTER(abi.rr_integrator),
                                  C.c_int, C.c_int, P, C.c_double, C.c_double, P, C.c_int]
        lib.rro_render_rows.argtypes = [C.POINTER(abi.rr_metric_desc), C.POINTER(abi.rr_scene_desc),
                                        C.POINTER(abi.rr_camera), C.POINTER(abi.rr_integrator),
                                        C.c_int, C.c_int, C.c_int, C.c_int, P, P,
                                        C.POINTER(abi.rr_stats), C.c_int]
        lib.rro_flags_pixels.argtypes = [C.POINTER(abi.rr_metric_desc), C.POINTER(abi.rr_scene_desc),
                                         C.POINTER(abi.rr_camera), C.POINTER(abi.rr_integrator),
                                         C.c_int, C.c_int, P, P, C.c_size_t, C.c_double, C.c_double,
                                         P, C.c_int]
        lib.rro_set_mesh_bruteforce.argtypes = [C.c_int]
        self.lib = lib
        self.threads = os.cpu_count() or 1

    def set_mesh_bruteforce(self, on: bool):
        self.lib.rro_set_mesh_bruteforce(1 if on else 0)

    @staticmethod
    def _d3(v):
        return (C.c_double * 3)(*[float(x) for x in v])

    def camera(self, cfg: RunConfig) -> abi.rr_camera:
        md = MetricDesc(cfg.metric)
        cam = abi.rr_camera()
        c = cfg.camera
        rc = self.lib.rro_build_camera(C.byref(md.desc), self._d3(c.position), self._d3(c.look_dir),
                                       self._d3(c.up_hint), fov_radians(c), C.byref(cam))
        if rc:
            raise RuntimeError(self.lib.rro_last_error().decode())
        return cam

    def primary_rays(self, cam: abi.rr_camera, w: int, h: int) -> np.ndarray:
        rays = np.zeros(w * h, abi.RAY_DTYPE)
        d = (C.c_double * 3)()
        for py in range(h):
            for px in range(w):
                self.lib.rro_pixel_direction(C.byref(cam), px, py, w, h, d)
                rays[py * w + px] = ((cam.position.x, cam.position.y, cam.position.z), tuple(d))
        return rays

    def march(self, cfg: RunConfig, rays: np.ndarray) -> np.ndarray:
        md, sd = MetricDesc(cfg.metric), SceneDesc(cfg.scene)
        integ = cfg.integrator.to_abi()
        rays = np.ascontiguousarray(rays, abi.RAY_DTYPE)
        out = np.zeros(len(rays), abi.OUTCOME_DTYPE)
        self.lib.rro_march(C.byref(md.desc), C.byref(sd.desc), C.byref(integ), _ptr(rays),
                           _ptr(out), len(rays), self.threads)
        return out

    def render(self, cfg: RunConfig, w: int = 0, h: int = 0, with_flags: bool = False,
               perturb: float = 1e-4, wrap_eps: float = 1e-4, camera_cfg: RunConfig = None):
        """-> (rgb[h,w,3] u8, outcomes[h*w], stats dict, flags[h*w] or None)."""
        w = w or cfg.output.width
        h = h or cfg.output.height
        md, sd = MetricDesc(cfg.metric), SceneDesc(cfg.scene)
        integ = cfg.integrator.to_abi()
        cam = self.camera(camera_cfg if camera_cfg is not None else cfg)
        rgb = np.zeros((h, w, 3), np.uint8)
        out = np.zeros(w * h, abi.OUTCOME_DTYPE)
        st = abi.rr_stats()
        self.lib.rro_render(C.byref(md.desc), C.byref(sd.desc), C.byref(cam), C.byref(integ), w, h,
                            _ptr(rgb), _ptr(out), C.byref(st), self.threads)
        flags = None
        if with_flags:
            flags = np.zeros(w * h, np.uint8)
            self.lib.rro_flags(C.byref(md.desc), C.byref(sd.desc), C.byref(cam), C.byref(integ),
                               w, h, _ptr(out), perturb, wrap_eps, _ptr(flags), self.threads)
        return rgb, out, st.as_dict(), flags

    def render_rows(self, cfg: RunConfig, w: int, h: int, row0: int, row_step: int,
                    camera_cfg: RunConfig = None, threads: int = 0):
        """Rows row0, row0+row_step, ... of the w x h frame (lights included)
        -> (rgb[rows,w,3], outcomes[rows*w], stats with wall_seconds)."""
        md, sd = MetricDesc(cfg.metric), SceneDesc(cfg.scene)
        integ = cfg.integrator.to_abi()
        cam = self.camera(camera_cfg if camera_cfg is not None else cfg)
        rows = len(range(row0, h, row_step))
        rgb = np.zeros((rows, w, 3), np.uint8)
        out = np.zeros(rows * w, abi.OUTCOME_DTYPE)
        st = abi.rr_stats()
        self.lib.rro_render_rows(C.byref(md.desc), C.byref(sd.desc), C.byref(cam), C.byref(integ),
                                 w, h, row0, row_step, _ptr(rgb), _ptr(out), C.byref(st),
                                 threads or self.threads)
        return rgb, out, st.as_dict()

    def flags_pixels(self, cfg: RunConfig, w: int, h: int, pix, outcomes, perturb: float = 1e-4,
                     wrap_eps: float = 1e-4, camera_cfg: RunConfig = None) -> np.ndarray:
        """rro_flags for the listed pixels only (row-major indices of the w x h
        frame; outcomes = their FP64 outcomes)."""
        md, sd = MetricDesc(cfg.metric), SceneDesc(cfg.scene)
        integ = cfg.integrator.to_abi()
        cam = self.camera(camera_cfg if camera_cfg is not None else cfg)
        pix = np.ascontiguousarray(pix, np.int64)
        outcomes = np.ascontiguousarray(outcomes, abi.OUTCOME_DTYPE)
        flags = np.zeros(len(pix), np.uint8)
        if len(pix):
            self.lib.rro_flags_pixels(C.byref(md.desc), C.byref(sd.desc), C.byref(cam),
                                      C.byref(integ), w, h, _ptr(pix), _ptr(outcomes), len(pix),
                                      perturb, wrap_eps, _ptr(flags), self.threads)
        return flags

    def flow_accel(self, cfg: RunConfig, pos, vel):
        md = MetricDesc(cfg.metric)
        acc = (C.c_double * 3)()
        val = C.c_double()
        self.lib.rro_flow_accel(C.byref(md.desc), self._d3(pos), self._d3(vel), acc, C.byref(val))
        return list(acc), val.value

    def step(self, cfg: RunConfig, state6, h: float):
        md = MetricDesc(cfg.metric)
        s = (C.c_double * 6)(*[float(x) for x in state6])
        out = (C.c_double * 6)()
        val = C.c_double()
        self.lib.rro_step(C.byref(md.desc), s, h, cfg.integrator.scheme_id, out, C.byref(val))
        return list(out), val.value

    def intersect(self, cfg: RunConfig, a, b):
        sd = SceneDesc(cfg.scene)
        pt = (C.c_double * 3)()
        s = C.c_double()
        prim = C.c_int()
        hit = self.lib.rro_intersect(C.byref(sd.desc), self._d3(a), self._d3(b), pt, C.byref(s),
                                     C.byref(prim))
        return (list(pt), s.value, prim.value) if hit else None


class refc_stats(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("rays", C.c_longlong),
                ("total_steps", C.c_longlong), ("pixel_errors", C.c_longlong),
                ("workers", C.c_int), ("pad_", C.c_int)]


KERNELS = {"auto": 0, "scalar": 1, "generic": 2, "avx2": 3}


class Reference:
    """The unmodified reference library (oracle/_ref), driven by config JSON."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        lib = C.CDLL(path)
        P = C.c_void_p
        D = C.POINTER(C.c_double)
        lib.refc_last_error.restype = C.c_char_p
        lib.refc_render.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, P,
                                    C.POINTER(refc_stats), C.c_char_p]
        lib.refc_render_rows.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, P, P, C.POINTER(refc_stats)]
        lib.refc_camera.argtypes = [C.c_char_p, D]
        lib.refc_primary_rays.argtypes = [C.c_char_p, C.c_int, C.c_int, P]
        lib.refc_march.argtypes = [C.c_char_p, C.c_int, P, P, C.c_size_t]
        lib.refc_flow_accel.argtypes = [C.c_char_p, D, D, D, D]
        lib.refc_step.argtypes = [C.c_char_p, D, C.c_double, D, D]
        lib.refc_intersect.argtypes = [C.c_char_p, D, D, D, D, C.POINTER(C.c_int)]
        lib.refc_shade.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_double, P]
        lib.refc_shade.restype = None
        lib.refc_parse.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        self.lib = lib

    def hardware_concurrency(self) -> int:
        return int(self.lib.refc_hardware_concurrency())

    def _check(self, rc: int):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.lib.refc_last_error().decode()}")

    @staticmethod
    def _json(cfg_or_text) -> bytes:
        if isinstance(cfg_or_text, RunConfig):
            return reference_json(cfg_or_text).encode()
        return cfg_or_text.encode() if isinstance(cfg_or_text, str) else cfg_or_text

    def render(self, cfg, kernel="auto", workers=0, w=0, h=0, camera_cfg=None):
        j = self._json(cfg)
        cj = self._json(camera_cfg) if camera_cfg is not None else None
        if isinstance(cfg, RunConfig):
            w = w or cfg.output.width
            h = h or cfg.output.height
        rgb = np.zeros((h, w, 3), np.uint8)
        st = refc_stats()
        self._check(self.lib.refc_render(j, KERNELS[kernel], workers, w, h, _ptr(rgb), C.byref(st), cj))
        return rgb, {n: getattr(st, n) for n, _ in refc_stats._fields_}

    def render_rows(self, cfg, w, h, row0, row_step, kernel="auto", workers=0,
                    with_outcomes=False):
        """Rows row0, row0+row_step, ... of the w x h frame through the
        reference's row work item -> (rgb[rows,w,3], stats) or, with
        with_outcomes, (rgb, outcomes[rows*w], stats)."""
        rows = len(range(row0, h, row_step))
        rgb = np.zeros((rows, w, 3), np.uint8)
        out = np.zeros(rows * w, abi.OUTCOME_DTYPE) if with_outcomes else None
        st = refc_stats()
        self._check(self.lib.refc_render_rows(self._json(cfg), KERNELS[kernel], workers, w, h, row0,
                                              row_step, _ptr(rgb),
                                              _ptr(out) if out is not None else None, C.byref(st)))
        stats = {n: getattr(st, n) for n, _ in refc_stats._fields_}
        return (rgb, out, stats) if with_outcomes else (rgb, stats)

    def camera(self, cfg):
        out = (C.c_double * 19)()
        self._check(self.lib.refc_camera(self._json(cfg), out))
        return list(out)

    def primary_rays(self, cfg, w, h):
        rays = np.zeros(w * h, abi.RAY_DTYPE)
        self._check(self.lib.refc_primary_rays(self._json(cfg), w, h, _ptr(rays)))
        return rays

    def march(self, cfg, rays, kernel="scalar"):
        rays = np.ascontiguousarray(rays, abi.RAY_DTYPE)
        out = np.zeros(len(rays), abi.OUTCOME_DTYPE)
        self._check(self.lib.refc_march(self._json(cfg), KERNELS[kernel], _ptr(rays), _ptr(out),
                                        len(rays)))
        return out

    def flow_accel(self, cfg, pos, vel):
        acc = (C.c_double * 3)()
        val = C.c_double()
        self._check(self.lib.refc_flow_accel(self._json(cfg), (C.c_double * 3)(*pos),
                                             (C.c_double * 3)(*vel), acc, C.byref(val)))
        return list(acc), val.value

    def step(self, cfg, state6, h):
        out = (C.c_double * 6)()
        val = C.c_double()
        self._check(self.lib.refc_step(self._json(cfg), (C.c_double * 6)(*state6), h, out,
                                       C.byref(val)))
        return list(out), val.value

    def intersect(self, cfg, a, b):
        pt = (C.c_double * 3)()
        s = C.c_double()
        prim = C.c_int()
        rc = self.lib.refc_intersect(self._json(cfg), (C.c_double * 3)(*a), (C.c_double * 3)(*b),
                                     pt, C.byref(s), C.byref(prim))
        if rc > 1:
            self._check(rc - 1)
        return (list(pt), s.value, prim.value) if rc == 1 else None

    def shade(self, hit, point, t, kappa):
        rgb = np.zeros(3, np.uint8)
        self.lib.refc_shade(int(hit), point[0], point[1], point[2], t, kappa, _ptr(rgb))
        return rgb

    def parse(self, text: str) -> str:
        buf = C.create_string_buffer(1 << 20)
        rc = self.lib.refc_parse(text.encode(), buf, len(buf))
        if rc:
            return rc, self.lib.refc_last_error().decode()
        return 0, buf.value.decode()
