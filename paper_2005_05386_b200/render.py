"""Host-side mirror of the reference render API over the CUDA C-ABI.

Names and argument meaning follow /root/reference/proj/include/rray/render/
(render.hpp:14-50, kernel.hpp:24-59, camera.hpp:15-30, image.hpp:9-43) so
code written against the reference reads the same:

    cam = build_camera(metric, position, look_dir, up_hint, fov)
    res = render(metric, scene, cam, integrator, width, height)   # RenderResult
    march = march_fn(KernelKind.Cuda); march(ctx, rays, out, n)

Every call goes through ``csrc/librray_cuda.so`` (sm_100a).  There is no CPU
fallback: a missing library or a non-B200 device raises DeviceError.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
import time
from dataclasses import dataclass, field, fields
from typing import Optional

import numpy as np

from . import abi
from .config import (CameraSpec, IntegratorConfig, MetricDesc, RunConfig, Scene, SceneDesc,
                     fov_radians)
from .errors import DeviceError, IoError, raise_for_status

LIB_PATH = os.environ.get("RRAY_CUDA_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "csrc", "librray_cuda.so")
_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads and binds librray_cuda.so; raises DeviceError when it is absent."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
            _lib = abi.bind(C.CDLL(path))
        return _lib


def _sym(s) -> np.ndarray:
    """{xx, xy, xz, yy, yz, zz} -> symmetric 3x3."""
    return np.array([[s[0], s[1], s[2]], [s[1], s[3], s[4]], [s[2], s[4], s[5]]], np.float64)


def _addr(a) -> C.c_void_p:
    """Device/host address of a numpy array, torch tensor or int."""
    if a is None:
        return C.c_void_p(0)
    if isinstance(a, int):
        return C.c_void_p(a)
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())   # torch.Tensor


class Renderer:
    """One CUDA context (rr_ctx) on one device; thread-safe."""

    def __init__(self, device: int = 0, options: Optional[dict] = None):
        self.lib = load_library()
        ctx = C.c_void_p()
        rc = self.lib.rr_create(C.byref(ctx), int(device))
        if rc:
            raise_for_status(rc, self.lib.rr_last_error(None).decode() or f"rr_create({device}) failed")
        self.ctx = ctx
        self.device = device
        self._keep = None
        if options:
            self.set_options(**options)

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if self.ctx:
            self.lib.rr_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc:
            raise_for_status(rc, self.lib.rr_last_error(self.ctx).decode())

    @property
    def last_kernel(self) -> str:
        return self.lib.rr_last_kernel(self.ctx).decode()

    # -- configuration ----------------------------------------------------
    def options(self) -> dict:
        o = abi.rr_options()
        self._check(self.lib.rr_get_options(self.ctx, C.byref(o)))
        return {n: getattr(o, n) for n, _ in abi.rr_options._fields_ if n != "pad_"}

    def set_options(self, **kw):
        o = abi.rr_options()
        self._check(self.lib.rr_get_options(self.ctx, C.byref(o)))
        for k, v in kw.items():
            setattr(o, k, v)
        self._check(self.lib.rr_set_options(self.ctx, C.byref(o)))

    def set_scene(self, metric, scene: Scene):
        md, sd = MetricDesc(metric), SceneDesc(scene)
        self._check(self.lib.rr_set_scene(self.ctx, C.byref(md.desc), C.byref(sd.desc)))
        self._keep = (md, sd)

    def set_config(self, cfg: RunConfig):
        self.set_scene(cfg.metric, cfg.scene)

    def build_camera(self, spec: CameraSpec, fov: Optional[float] = None) -> abi.rr_camera:
        cam = abi.rr_camera()
        self._check(self.lib.rr_build_camera(
            self.ctx, C.byref(abi.rr_vec3.of(spec.position)), C.byref(abi.rr_vec3.of(spec.look_dir)),
            C.byref(abi.rr_vec3.of(spec.up_hint)), fov_radians(spec) if fov is None else fov,
            C.byref(cam)))
        return cam

    # -- work -------------------------------------------------------------
    def march(self, integ: IntegratorConfig, rays: np.ndarray) -> np.ndarray:
        rays = np.ascontiguousarray(rays, abi.RAY_DTYPE)
        out = np.zeros(len(rays), abi.OUTCOME_DTYPE)
        it = integ.to_abi()
        self._check(self.lib.rr_march(self.ctx, C.byref(it), _addr(rays), _addr(out), len(rays)))
        return out

    def march_device(self, integ: IntegratorConfig, d_rays, d_out, n: int, stream=None):
        it = integ.to_abi()
        self._check(self.lib.rr_march_device(self.ctx, C.byref(it), _addr(d_rays), _addr(d_out), n,
                                             _addr(stream)))

    def render(self, cam: abi.rr_camera, integ: IntegratorConfig, width: int, height: int,
               out=None):
        """Whole frame into host memory (numpy or pinned torch) -> (rgb, stats)."""
        if out is None:
            out = np.zeros((height, width, 3), np.uint8)
        st = abi.rr_stats()
        it = integ.to_abi()
        self._check(self.lib.rr_render(self.ctx, C.byref(cam), C.byref(it), width, height,
                                       _addr(out), C.byref(st)))
        return out, st.as_dict()

    def render_outcomes(self, cam: abi.rr_camera, integ: IntegratorConfig, width: int,
                        height: int, rgb=True):
        """The frame kernel with its PixelOutcome sink -> (rgb or None,
        outcomes[h*w] row-major, stats): per-pixel parity of the frame path."""
        out = np.zeros(width * height, abi.OUTCOME_DTYPE)
        img = np.zeros((height, width, 3), np.uint8) if rgb else None
        st = abi.rr_stats()
        it = integ.to_abi()
        self._check(self.lib.rr_render_outcomes(self.ctx, C.byref(cam), C.byref(it), width, height,
                                                _addr(img), _addr(out), C.byref(st)))
        return img, out, st.as_dict()

    def render_device(self, cam, integ: IntegratorConfig, width: int, height: int, d_rgb,
                      stream=None, with_stats: bool = False):
        st = abi.rr_stats() if with_stats else None
        it = integ.to_abi()
        self._check(self.lib.rr_render_device(self.ctx, C.byref(cam), C.byref(it), width, height,
                                              _addr(d_rgb), C.byref(st) if st is not None else None,
                                              _addr(stream)))
        return st.as_dict() if st is not None else None

    def shard_tile_count(self, width, height, tile_w, tile_h, shard, n_shards) -> int:
        return int(self.lib.rr_shard_tile_count(width, height, tile_w, tile_h, shard, n_shards))

    def render_tiles(self, cam, integ: IntegratorConfig, width, height, tile_w, tile_h, shard,
                     n_shards, d_tiles, stream=None, with_stats: bool = False):
        st = abi.rr_stats() if with_stats else None
        it = integ.to_abi()
        self._check(self.lib.rr_render_tiles(self.ctx, C.byref(cam), C.byref(it), width, height,
                                             tile_w, tile_h, shard, n_shards, _addr(d_tiles),
                                             C.byref(st) if st is not None else None,
                                             _addr(stream)))
        return st.as_dict() if st is not None else None

    def render_shard(self, cam, integ: IntegratorConfig, width, height, tile_w, tile_h, shard,
                     n_shards, d_frame, stream=None, with_stats: bool = False):
        """This shard's tiles written straight into a (possibly peer-mapped) frame."""
        st = abi.rr_stats() if with_stats else None
        it = integ.to_abi()
        self._check(self.lib.rr_render_shard(self.ctx, C.byref(cam), C.byref(it), width, height,
                                             tile_w, tile_h, shard, n_shards, _addr(d_frame),
                                             C.byref(st) if st is not None else None,
                                             _addr(stream)))
        return st.as_dict() if st is not None else None

    # -- cross-process frame exchange ------------------------
    def frame_export(self, d_frame, nbytes: int = 0) -> bytes:
        """Handle (bytes, picklable) of a device frame buffer (torch tensor or
        address) for rr_frame_import in another process."""
        if not nbytes and hasattr(d_frame, "numel"):
            nbytes = d_frame.numel() * d_frame.element_size()
        h = abi.rr_frame_handle()
        self._check(self.lib.rr_frame_export(self.ctx, _addr(d_frame), nbytes, C.byref(h)))
        return bytes(h)

    def frame_import(self, handle: bytes) -> int:
        """Maps an exported frame on this context's device -> device address."""
        h = abi.rr_frame_handle.from_buffer_copy(handle)
        p = C.c_void_p()
        self._check(self.lib.rr_frame_import(self.ctx, C.byref(h), C.byref(p)))
        return int(p.value)

    def frame_close(self, d_frame):
        self._check(self.lib.rr_frame_close(self.ctx, _addr(d_frame)))

    def frame_probe(self, d_frame, offset: int, value: int):
        self._check(self.lib.rr_frame_probe(self.ctx, _addr(d_frame), offset, value))

    def detile(self, d_gathered, width, height, tile_w, tile_h, n_shards, d_rgb, stream=None):
        self._check(self.lib.rr_detile(self.ctx, _addr(d_gathered), width, height, tile_w, tile_h,
                                       n_shards, _addr(d_rgb), _addr(stream)))

    # -- off the render path: geodesic export + device verify --------------
    def trace(self, integ: IntegratorConfig, starts: np.ndarray, use_bounds: bool = True):
        """trace_geodesic (integrate.cpp:40-54) on the device for each start
        (n x 6 doubles {x, y, z, vx, vy, vz}) -> (states n x (max_steps+1) x 6,
        counts n, fail_step n)."""
        starts = np.ascontiguousarray(np.asarray(starts, np.float64).reshape(-1, 6))
        n = len(starts)
        states = np.zeros((n, integ.max_steps + 1, 6), np.float64)
        counts = np.zeros(n, np.int32)
        fail = np.zeros(n, np.int32)
        it = integ.to_abi()
        self._check(self.lib.rr_trace(self.ctx, C.byref(it), _addr(starts), n, int(use_bounds),
                                      _addr(states), _addr(counts), _addr(fail)))
        return states, counts, fail

    def accel(self, pos: np.ndarray, vel: np.ndarray):
        """Device flow_accel (integrate.hpp:46-53): (-Gamma(vel, vel), validity)."""
        pos = np.ascontiguousarray(np.asarray(pos, np.float64).reshape(-1, 3))
        vel = np.ascontiguousarray(np.asarray(vel, np.float64).reshape(-1, 3))
        acc = np.zeros_like(pos)
        val = np.zeros(len(pos), np.float64)
        self._check(self.lib.rr_accel(self.ctx, _addr(pos), _addr(vel), len(pos), _addr(acc),
                                      _addr(val)))
        return acc, val

    def metric_tensor(self, p) -> np.ndarray:
        """FP64 g(p) as a 3x3 matrix (metric.cpp:12-15, :40-42)."""
        p = np.ascontiguousarray(p, np.float64)
        g = np.zeros(6, np.float64)
        self._check(self.lib.rr_metric_tensor(self.ctx, _addr(p), _addr(g)))
        return _sym(g)

    def christoffel_fd(self, p, h_fd: float = 1e-4) -> np.ndarray:
        """FP64 finite-difference Gamma[m, i, j] (metric.cpp:88-133)."""
        p = np.ascontiguousarray(p, np.float64)
        gam = np.zeros(18, np.float64)
        self._check(self.lib.rr_christoffel_fd(self.ctx, _addr(p), h_fd, _addr(gam)))
        return np.stack([_sym(gam[6 * m:6 * m + 6]) for m in range(3)])

    def diffeo_image(self, p) -> np.ndarray:
        p = np.ascontiguousarray(p, np.float64)
        out = np.zeros(3, np.float64)
        self._check(self.lib.rr_diffeo_image(self.ctx, _addr(p), _addr(out)))
        return out

    def fp32_peak_tflops(self) -> float:
        v = C.c_double()
        self._check(self.lib.rr_measure_fp32_peak(self.ctx, C.byref(v)))
        return v.value


# ---- reference-API mirror (render.hpp / kernel.hpp / camera.hpp) -------------

class KernelKind(enum.Enum):          # kernel.hpp:24 + Cuda
    Auto = 0
    Scalar = 1
    Generic = 2
    Avx2 = 3
    Cuda = 4


def kernel_from_env() -> KernelKind:  # kernel_dispatch.cpp:66-76 (+ "cuda")
    from .errors import ValidationError
    v = os.environ.get("RRAY_KERNEL")
    if v is None or v in ("", "auto"):
        return KernelKind.Auto
    table = {"scalar": KernelKind.Scalar, "generic": KernelKind.Generic,
             "avx2": KernelKind.Avx2, "cuda": KernelKind.Cuda}
    if v not in table:
        raise ValidationError(f"RRAY_KERNEL must be one of scalar|generic|avx2|cuda|auto, got '{v}'")
    return table[v]


def resolve_kernel(kind: KernelKind) -> KernelKind:
    """This build ships only the CUDA backend: Auto resolves to Cuda."""
    return KernelKind.Cuda if kind == KernelKind.Auto else kind


@dataclass
class RenderStats:                    # render.hpp:24-33 (+ device extensions)
    wall_seconds: float = 0.0
    rays: int = 0
    total_steps: int = 0
    pixel_errors: int = 0
    device_ms: float = 0.0
    integrated_steps: int = 0
    bump_evals: int = 0
    shadow_steps: int = 0
    kernel_launches: int = 0
    lane_slots: int = 0
    shadow_lane_slots: int = 0
    jump_steps: int = 0
    shadow_jump_steps: int = 0
    shadow_integrated_steps: int = 0
    sort_kernels: int = 0

    @classmethod
    def from_dict(cls, st: dict) -> "RenderStats":
        names = {f.name for f in fields(cls)}
        return cls(**{k: v for k, v in st.items() if k in names})

    def avg_steps_per_ray(self) -> float:
        return self.total_steps / self.rays if self.rays > 0 else 0.0


@dataclass
class RenderOptions:                  # render.hpp:35-38
    workers: int = 0                  # accepted for API parity; the device schedules itself
    kernel: KernelKind = KernelKind.Auto
    device: int = 0


@dataclass
class Image:                          # image.hpp:9-38
    width: int
    height: int
    data: np.ndarray = field(repr=False)   # (h, w, 3) uint8, row-major RGB8

    def get(self, px, py):
        return tuple(int(x) for x in self.data[py, px])


@dataclass
class RenderResult:
    image: Image
    stats: RenderStats


@dataclass
class Camera:                         # camera.hpp:15-23
    raw: abi.rr_camera
    metric: object = None

    @property
    def frame(self):
        return [self.raw.frame[i].tolist() for i in range(3)]

    @property
    def position(self):
        return self.raw.position.tolist()


_renderers = {}
_renderers_lock = threading.Lock()


def _renderer(device: int) -> Renderer:
    with _renderers_lock:
        r = _renderers.get(device)
        if r is None:
            r = _renderers[device] = Renderer(device)
        return r


def build_camera(metric, position, look_dir, up_hint, fov: float, device: int = 0) -> Camera:
    """camera.cpp:9-20 (FP64 Gram-Schmidt against g(position))."""
    r = _renderer(device)
    with _renderers_lock:
        r.set_scene(metric, Scene(primitives=[]))
        cam = r.build_camera(CameraSpec(list(position), list(look_dir), list(up_hint)), fov=fov)
    return Camera(cam, metric)


def pixel_direction(cam: Camera, px: int, py: int, width: int, height: int):
    """camera.cpp:22-29."""
    lib = load_library()
    out = abi.rr_vec3()
    rc = lib.rr_pixel_direction(C.byref(cam.raw), px, py, width, height, C.byref(out))
    raise_for_status(rc, "rr_pixel_direction: invalid arguments")
    return out.tolist()


def render(metric, scene: Scene, cam: Camera, integ: IntegratorConfig, width: int, height: int,
           opt: RenderOptions = RenderOptions()) -> RenderResult:
    """render.cpp:43-111 on the GPU: raygen + march + shade fused in one launch (lit
    frames: a hit-record launch + a shadow / shade launch)."""
    kind = opt.kernel if opt.kernel != KernelKind.Auto else kernel_from_env()
    if resolve_kernel(kind) != KernelKind.Cuda:
        from .errors import ValidationError
        raise ValidationError(f"kernel '{kind.name.lower()}' is not available in this build (cuda only)")
    t0 = time.perf_counter()
    r = _renderer(opt.device)
    with _renderers_lock:
        r.set_scene(metric, scene)
        rgb, st = r.render(cam.raw, integ, width, height)
    st["wall_seconds"] = time.perf_counter() - t0
    st["rays"] = width * height
    return RenderResult(Image(width, height, rgb), RenderStats.from_dict(st))


@dataclass
class MarchContext:                   # kernel.hpp:41-45
    metric: object
    scene: Scene
    integ: IntegratorConfig
    device: int = 0


def march_fn(kind: KernelKind):
    """kernel_dispatch.cpp:40-54: MarchFn(ctx, rays, out, n) for the CUDA kernel."""
    if resolve_kernel(kind) != KernelKind.Cuda:
        from .errors import ValidationError
        raise ValidationError(f"kernel '{kind.name.lower()}' is not available in this build (cuda only)")

    def march(ctx: MarchContext, rays: np.ndarray, out: np.ndarray, n: int):
        r = _renderer(ctx.device)
        with _renderers_lock:
            r.set_scene(ctx.metric, ctx.scene)
            res = r.march(ctx.integ, rays[:n])
        out[:n] = res
    return march


def kernel_name(kind: KernelKind) -> str:
    return kind.name.lower()


# ---- image I/O (image.cpp:11-46) ----------------------------------------------

def ppm_bytes(img: Image) -> bytes:
    return f"P6\n{img.width} {img.height}\n255\n".encode() + np.ascontiguousarray(img.data).tobytes()


def write_ppm(img: Image, path: str):
    try:
        with open(path, "wb") as f:
            f.write(ppm_bytes(img))
    except OSError:
        raise IoError(f"cannot open '{path}' for writing") from None


def read_ppm(path: str) -> Image:
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError:
        raise IoError(f"cannot open '{path}' for reading") from None
    parts = blob.split(maxsplit=4)
    if len(parts) < 5 or parts[0] != b"P6" or parts[3] != b"255":
        raise IoError(f"'{path}' is not an 8-bit P6 PPM")
    w, h = int(parts[1]), int(parts[2])
    header_len = len(b" ".join(parts[:4])) + 1
    data = np.frombuffer(blob[header_len:header_len + 3 * w * h], np.uint8)
    if data.size != 3 * w * h:
        raise IoError(f"'{path}' truncated")
    return Image(w, h, data.reshape(h, w, 3).copy())
