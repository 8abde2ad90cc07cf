"""Run configuration: the reference's JSON schema, parsed and validated the same way.

Mirrors /root/reference/proj/src/config/config.cpp (parse_config :437-456,
serialize_config :466-483): every document the reference accepts parses to the
same values here, every document it rejects is rejected with a
ValidationError/ParseError naming the same key.  One superset key is accepted
(EXTENSION, SPEC.md:491,494 lists it as a reference non-goal):

    scene.lights: [{"position": [x,y,z], "intensity": I}]   point lights for
                   shadow geodesics; absent/empty = reference shading.
    scene.ambient: ambient term of the lit shading (default 0.2).
    metric.map (any level) = {"kind": "bend", "curvature": k}   Barr bend about z.
    integrator.scheme = "rk23", integrator.tol   adaptive Bogacki-Shampine 3(2).
    scene.primitives[i] = {"kind": "mesh", "vertices": [...], "triangles": [...]}
                   or {"kind": "mesh", "generator": {"kind": "torus", ...}}
                   triangle meshes (BVH-accelerated on the GPU).

``metric_desc`` / ``scene_desc`` flatten the parsed trees into the C-ABI
descriptors of include/rray_cuda.h.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Union

from . import abi
from .errors import ParseError, ValidationError

Vec3 = List[float]


# ---- data model (field/diffeo/metric/scene types of the reference) --------

@dataclass
class GaussianParams:                 # scalar_field.hpp:16-22
    amplitude: float = 0.0
    center: Vec3 = field(default_factory=lambda: [0.0, 0.0, 0.0])
    sigma: Vec3 = field(default_factory=lambda: [1.0, 1.0, 1.0])


@dataclass
class PolyTerm:                       # scalar_field.hpp:25-30
    coef: float = 0.0
    powers: List[int] = field(default_factory=lambda: [0, 0, 0])


@dataclass
class GaussianField:
    params: GaussianParams


@dataclass
class PolynomialField:
    terms: List[PolyTerm]


@dataclass
class SumField:
    terms: list


ScalarField = Union[GaussianField, PolynomialField, SumField]


@dataclass
class IdentityMap:
    pass


@dataclass
class AffineMap:                      # diffeo.hpp:61-72
    matrix: List[List[float]] = field(default_factory=lambda: [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    offset: Vec3 = field(default_factory=lambda: [0.0, 0.0, 0.0])


@dataclass
class TwistMap:
    pass


@dataclass
class BendMap:                        # EXTENSION: Barr bend, angle = curvature * x
    curvature: float = 0.1


@dataclass
class LocalBumpMap:                   # diffeo.hpp:80-86
    bump: GaussianParams
    direction: Vec3


@dataclass
class ComposeMap:                     # maps[0] is the outermost map (diffeo.hpp:88-93)
    maps: list


Diffeo = Union[IdentityMap, AffineMap, TwistMap, LocalBumpMap, ComposeMap, BendMap]


@dataclass
class EuclideanMetric:
    pass


@dataclass
class GraphMetric:
    field: ScalarField


@dataclass
class DiffeoMetric:
    map: Diffeo


Metric = Union[EuclideanMetric, GraphMetric, DiffeoMetric]


@dataclass
class Aabb:                           # aabb.hpp:7-22
    min: Vec3 = field(default_factory=lambda: [-10.0, -10.0, -10.0])
    max: Vec3 = field(default_factory=lambda: [10.0, 10.0, 10.0])

    def contains_point(self, p) -> bool:
        return all(self.min[i] <= p[i] <= self.max[i] for i in range(3))

    def contains(self, inner: "Aabb") -> bool:
        return self.contains_point(inner.min) and self.contains_point(inner.max)


@dataclass
class GridPlanes:                     # scene.hpp:20-26
    spacing: float = 1.0
    half_width: float = 0.02
    bounds: Aabb = field(default_factory=Aabb)


@dataclass
class Sphere:                         # scene.hpp:28-33
    center: Vec3 = field(default_factory=lambda: [0.0, 0.0, 0.0])
    radius: float = 1.0


@dataclass
class HalfSpace:                      # scene.hpp:35-41
    normal: Vec3 = field(default_factory=lambda: [0.0, 0.0, 1.0])
    offset: float = 0.0


@dataclass
class Mesh:                           # EXTENSION: triangle mesh primitive
    vertices: object = None           # numpy (n, 3) float64
    triangles: object = None          # numpy (m, 3) int32
    generator: Optional[dict] = None  # the procedural spec it came from, if any

    def __eq__(self, o):
        import numpy as np
        return (isinstance(o, Mesh) and self.generator == o.generator and
                np.array_equal(self.vertices, o.vertices) and
                np.array_equal(self.triangles, o.triangles))


def torus_mesh(center, major, minor, nu, nv, wobble=0.0):
    """Deterministic torus around the z axis: nu*nv*2 triangles.  `wobble`
    modulates the tube radius by (1 + wobble sin(5u) sin(3v))."""
    import numpy as np
    u = 2.0 * np.pi * np.arange(nu) / nu
    v = 2.0 * np.pi * np.arange(nv) / nv
    U, V = np.meshgrid(u, v, indexing="ij")
    r = minor * (1.0 + wobble * np.sin(5.0 * U) * np.sin(3.0 * V))
    x = (major + r * np.cos(V)) * np.cos(U) + center[0]
    y = (major + r * np.cos(V)) * np.sin(U) + center[1]
    z = r * np.sin(V) + center[2]
    verts = np.stack([x, y, z], -1).reshape(-1, 3)
    i = np.arange(nu)[:, None]
    j = np.arange(nv)[None, :]
    a = i * nv + j
    b = ((i + 1) % nu) * nv + j
    c_ = ((i + 1) % nu) * nv + (j + 1) % nv
    d = i * nv + (j + 1) % nv
    t1 = np.stack([a, b, c_], -1).reshape(-1, 3)
    t2 = np.stack([a, c_, d], -1).reshape(-1, 3)
    tris = np.stack([t1, t2], 1).reshape(-1, 3).astype(np.int32)
    return verts.astype(np.float64), tris


@dataclass
class Light:                          # EXTENSION
    position: Vec3
    intensity: float = 1.0


@dataclass
class Scene:                          # scene.hpp:45-51 (+ lights EXT)
    primitives: list = field(default_factory=list)
    bounds: Aabb = field(default_factory=Aabb)
    fog_density: float = 0.05
    lights: List[Light] = field(default_factory=list)
    ambient: float = 0.2              # EXTENSION: used only when lights are present


@dataclass
class CameraSpec:                     # config.hpp:18-25
    position: Vec3 = field(default_factory=lambda: [0.5, 0.5, 0.5])
    look_dir: Vec3 = field(default_factory=lambda: [1.0, 0.0, 0.0])
    up_hint: Vec3 = field(default_factory=lambda: [0.0, 0.0, 1.0])
    fov_deg: float = 60.0


@dataclass
class IntegratorConfig:               # integrate.hpp:30-36 (+ rk23/tol EXTENSION)
    h: float = 1e-2
    max_steps: int = 2000
    scheme: str = "euler"
    tol: float = 1e-6

    @property
    def scheme_id(self) -> int:
        return {"euler": abi.RR_SCHEME_EULER, "rk4": abi.RR_SCHEME_RK4,
                "rk23": abi.RR_SCHEME_RK23}[self.scheme]

    def to_abi(self) -> abi.rr_integrator:
        return abi.rr_integrator(float(self.h), int(self.max_steps), self.scheme_id,
                                 float(self.tol))


@dataclass
class OutputSpec:                     # config.hpp:27-34
    path: str = "render.ppm"
    width: int = 512
    height: int = 512
    format: str = "ppm"


@dataclass
class RunConfig:                      # config.hpp:36-44
    metric: Metric = field(default_factory=EuclideanMetric)
    scene: Scene = field(default_factory=Scene)
    camera: CameraSpec = field(default_factory=CameraSpec)
    integrator: IntegratorConfig = field(default_factory=IntegratorConfig)
    output: OutputSpec = field(default_factory=OutputSpec)


# ---- parsing (config.cpp:14-431) -------------------------------------------

def _fail(path: str, msg: str):
    raise ValidationError(f"{path}: {msg}")


def _check_keys(o, path, allowed):
    if not isinstance(o, dict):
        _fail(path, "must be an object")
    for k in o:
        if k not in allowed:
            _fail(path, f"unexpected key '{k}'")


def _is_number(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _is_integer(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _as_double(v, path) -> float:
    if not _is_number(v):
        _fail(path, "must be a number")
    return float(v)


def _get_double(o, path, key) -> float:
    if key not in o:
        _fail(f"{path}.{key}", "required")
    return _as_double(o[key], f"{path}.{key}")


def _get_double_or(o, path, key, default) -> float:
    return _as_double(o[key], f"{path}.{key}") if key in o else default


def _get_int_or(o, path, key, default) -> int:
    if key not in o:
        return default
    if not _is_integer(o[key]):
        _fail(f"{path}.{key}", "must be an integer")
    return int(o[key])


def _get_string_or(o, path, key, default) -> str:
    if key not in o:
        return default
    if not isinstance(o[key], str):
        _fail(f"{path}.{key}", "must be a string")
    return o[key]


def _as_vec3(v, path) -> Vec3:
    if not isinstance(v, list) or len(v) != 3:
        _fail(path, "must be an array of 3 numbers")
    return [_as_double(v[0], path + "[0]"), _as_double(v[1], path + "[1]"),
            _as_double(v[2], path + "[2]")]


def _get_vec3(o, path, key) -> Vec3:
    if key not in o:
        _fail(f"{path}.{key}", "required")
    return _as_vec3(o[key], f"{path}.{key}")


def _get_vec3_or(o, path, key, default) -> Vec3:
    return _as_vec3(o[key], f"{path}.{key}") if key in o else list(default)


def _norm(v) -> float:
    return math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])


def _cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def _parse_gaussian_params(o, path) -> GaussianParams:           # :144-152
    g = GaussianParams()
    g.amplitude = _get_double(o, path, "amplitude")
    g.center = _get_vec3(o, path, "center")
    g.sigma = _get_vec3(o, path, "sigma")
    if not (g.sigma[0] > 0.0 and g.sigma[1] > 0.0 and g.sigma[2] > 0.0):
        _fail(path + ".sigma", "all spreads must be > 0")
    return g


def _parse_field(o, path) -> ScalarField:                        # :154-196
    kind = _get_string_or(o, path, "kind", "")
    if kind == "gaussian":
        _check_keys(o, path, {"kind", "amplitude", "center", "sigma"})
        return GaussianField(_parse_gaussian_params(o, path))
    if kind == "polynomial":
        _check_keys(o, path, {"kind", "terms"})
        terms = o.get("terms")
        if not isinstance(terms, list):
            _fail(path + ".terms", "required array")
        ts = []
        for i, t in enumerate(terms):
            tp = f"{path}.terms[{i}]"
            _check_keys(t, tp, {"coef", "powers"})
            pt = PolyTerm()
            pt.coef = _get_double(t, tp, "coef")
            pw = t.get("powers")
            if not isinstance(pw, list) or len(pw) != 3:
                _fail(tp + ".powers", "must be an array of 3 integers")
            total = 0
            pt.powers = [0, 0, 0]
            for k in range(3):
                if not _is_integer(pw[k]):
                    _fail(tp + ".powers", "must be integers")
                pt.powers[k] = int(pw[k])
                if pt.powers[k] < 0:
                    _fail(tp + ".powers", "must be >= 0")
                total += pt.powers[k]
            if total > 4:
                _fail(tp + ".powers", "total degree must be <= 4")
            ts.append(pt)
        return PolynomialField(ts)
    if kind == "sum":
        _check_keys(o, path, {"kind", "terms"})
        terms = o.get("terms")
        if not isinstance(terms, list):
            _fail(path + ".terms", "required array")
        return SumField([_parse_field(t, f"{path}.terms[{i}]") for i, t in enumerate(terms)])
    _fail(path + ".kind", f"must be one of gaussian|polynomial|sum, got '{kind}'")


def _parse_diffeo(o, path, allow_ext: bool = True) -> Diffeo:     # :198-244
    kind = _get_string_or(o, path, "kind", "")
    if kind == "bend" and allow_ext:                                # EXTENSION
        _check_keys(o, path, {"kind", "curvature"})
        b = BendMap(_get_double(o, path, "curvature"))
        if not (b.curvature != 0.0 and math.isfinite(b.curvature)):
            _fail(path + ".curvature", "must be nonzero")
        return b
    if kind == "identity":
        _check_keys(o, path, {"kind"})
        return IdentityMap()
    if kind == "affine":
        _check_keys(o, path, {"kind", "matrix", "offset"})
        mj = o.get("matrix")
        if not isinstance(mj, list) or len(mj) != 3:
            _fail(path + ".matrix", "must be an array of 3 rows of 3 numbers")
        a = AffineMap()
        a.matrix = [[0.0] * 3 for _ in range(3)]
        for i in range(3):
            row = mj[i]
            if not isinstance(row, list) or len(row) != 3:
                _fail(path + ".matrix", "must be an array of 3 rows of 3 numbers")
            for j in range(3):
                a.matrix[i][j] = _as_double(row[j], f"{path}.matrix[{i}]")
        a.offset = _get_vec3_or(o, path, "offset", [0.0, 0.0, 0.0])
        return a
    if kind == "twist":
        _check_keys(o, path, {"kind"})
        return TwistMap()
    if kind == "local_bump":
        _check_keys(o, path, {"kind", "amplitude", "center", "sigma", "direction"})
        bump = _parse_gaussian_params(o, path)
        return LocalBumpMap(bump, _get_vec3(o, path, "direction"))
    if kind == "compose":
        _check_keys(o, path, {"kind", "maps"})
        maps = o.get("maps")
        if not isinstance(maps, list) or not maps:
            _fail(path + ".maps", "required non-empty array")
        return ComposeMap([_parse_diffeo(m, f"{path}.maps[{i}]", allow_ext) for i, m in enumerate(maps)])
    _fail(path + ".kind",
          f"must be one of identity|affine|twist|local_bump|compose, got '{kind}'")


def _parse_metric(o, path, allow_ext: bool = True) -> Metric:     # :246-265
    kind = _get_string_or(o, path, "kind", "") if isinstance(o, dict) else ""
    if not isinstance(o, dict):
        _fail(path, "must be an object")
    if kind == "euclidean":
        _check_keys(o, path, {"kind"})
        return EuclideanMetric()
    if kind == "graph":
        _check_keys(o, path, {"kind", "field"})
        if "field" not in o:
            _fail(path + ".field", "required")
        return GraphMetric(_parse_field(o["field"], path + ".field"))
    if kind == "diffeo":
        _check_keys(o, path, {"kind", "map"})
        if "map" not in o:
            _fail(path + ".map", "required")
        return DiffeoMetric(_parse_diffeo(o["map"], path + ".map", allow_ext))
    _fail(path + ".kind", f"must be one of euclidean|graph|diffeo, got '{kind}'")


def _parse_aabb(o, path) -> Aabb:                                 # :267-275
    _check_keys(o, path, {"min", "max"})
    b = Aabb(_get_vec3(o, path, "min"), _get_vec3(o, path, "max"))
    if not (b.min[0] < b.max[0] and b.min[1] < b.max[1] and b.min[2] < b.max[2]):
        _fail(path, "min must be strictly below max componentwise")
    return b


def _parse_scene(o, path, allow_ext: bool) -> Scene:              # :277-338
    s = Scene()
    s.bounds = Aabb()
    if o is not None:
        keys = {"primitives", "bounds", "fog_density"} | ({"lights", "ambient"} if allow_ext else set())
        _check_keys(o, path, keys)
        if "bounds" in o:
            s.bounds = _parse_aabb(o["bounds"], path + ".bounds")
        s.fog_density = _get_double_or(o, path, "fog_density", 0.05)
        if not (s.fog_density >= 0.0):
            _fail(path + ".fog_density", "must be >= 0")
        if allow_ext and "lights" in o:
            s.lights = _parse_lights(o["lights"], path + ".lights")
        if allow_ext:
            s.ambient = _get_double_or(o, path, "ambient", 0.2)
            if not (s.ambient >= 0.0):
                _fail(path + ".ambient", "must be >= 0")
    prims = o.get("primitives") if o is not None else None
    if o is None or "primitives" not in o:
        s.primitives.append(GridPlanes(1.0, 0.02, Aabb(list(s.bounds.min), list(s.bounds.max))))
        return s
    if not isinstance(prims, list):
        _fail(path + ".primitives", "must be an array")
    for i, p in enumerate(prims):
        pp = f"{path}.primitives[{i}]"
        kind = _get_string_or(p, pp, "kind", "") if isinstance(p, dict) else ""
        if not isinstance(p, dict):
            _fail(pp, "must be an object")
        if kind == "grid_planes":
            _check_keys(p, pp, {"kind", "spacing", "half_width", "bounds"})
            g = GridPlanes()
            g.spacing = _get_double_or(p, pp, "spacing", 1.0)
            g.half_width = _get_double_or(p, pp, "half_width", 0.02)
            g.bounds = Aabb(list(s.bounds.min), list(s.bounds.max))
            if "bounds" in p:
                g.bounds = _parse_aabb(p["bounds"], pp + ".bounds")
            if not (g.half_width > 0.0):
                _fail(pp + ".half_width", "must be > 0")
            if not (g.spacing > 2.0 * g.half_width):
                _fail(pp + ".spacing", "must be > 2 * half_width")
            if not s.bounds.contains(g.bounds):
                _fail(pp + ".bounds", "must lie inside scene.bounds")
            s.primitives.append(g)
        elif kind == "sphere":
            _check_keys(p, pp, {"kind", "center", "radius"})
            sp = Sphere(_get_vec3(p, pp, "center"), _get_double(p, pp, "radius"))
            if not (sp.radius > 0.0):
                _fail(pp + ".radius", "must be > 0")
            r = sp.radius
            box = Aabb([c - r for c in sp.center], [c + r for c in sp.center])
            if not s.bounds.contains(box):
                _fail(pp, "sphere must lie inside scene.bounds")
            s.primitives.append(sp)
        elif kind == "half_space":
            _check_keys(p, pp, {"kind", "normal", "offset"})
            hs = HalfSpace(_get_vec3(p, pp, "normal"), _get_double(p, pp, "offset"))
            if not (_norm(hs.normal) > 0.0):
                _fail(pp + ".normal", "must be nonzero")
            s.primitives.append(hs)
        elif kind == "mesh" and allow_ext:
            s.primitives.append(_parse_mesh(p, pp))
        else:
            _fail(pp + ".kind", f"must be one of grid_planes|sphere|half_space, got '{kind}'")
    return s


def _parse_mesh(p, pp) -> Mesh:                                  # EXTENSION
    import numpy as np
    _check_keys(p, pp, {"kind", "vertices", "triangles", "generator"})
    if "generator" in p:
        g = p["generator"]
        _check_keys(g, pp + ".generator", {"kind", "center", "major", "minor", "nu", "nv", "wobble"})
        if _get_string_or(g, pp + ".generator", "kind", "") != "torus":
            _fail(pp + ".generator.kind", "must be 'torus'")
        nu = _get_int_or(g, pp + ".generator", "nu", 64)
        nv = _get_int_or(g, pp + ".generator", "nv", 32)
        if nu < 3 or nv < 3:
            _fail(pp + ".generator", "nu, nv must be >= 3")
        spec = {"kind": "torus", "center": _get_vec3(g, pp + ".generator", "center"),
                "major": _get_double(g, pp + ".generator", "major"),
                "minor": _get_double(g, pp + ".generator", "minor"), "nu": nu, "nv": nv,
                "wobble": _get_double_or(g, pp + ".generator", "wobble", 0.0)}
        if not (spec["major"] > spec["minor"] > 0.0):
            _fail(pp + ".generator", "need major > minor > 0")
        v, t = torus_mesh(spec["center"], spec["major"], spec["minor"], nu, nv, spec["wobble"])
        return Mesh(v, t, spec)
    vs, ts = p.get("vertices"), p.get("triangles")
    if not isinstance(vs, list) or not isinstance(ts, list) or not ts:
        _fail(pp, "mesh needs 'vertices' and non-empty 'triangles' (or a 'generator')")
    v = np.array([_as_vec3(x, f"{pp}.vertices[{i}]") for i, x in enumerate(vs)], np.float64).reshape(-1, 3)
    tl = []
    for i, t in enumerate(ts):
        if not isinstance(t, list) or len(t) != 3 or not all(_is_integer(k) for k in t):
            _fail(f"{pp}.triangles[{i}]", "must be 3 vertex indices")
        if not all(0 <= k < len(v) for k in t):
            _fail(f"{pp}.triangles[{i}]", "vertex index out of range")
        tl.append(t)
    return Mesh(v, np.array(tl, np.int32), None)


def _parse_lights(o, path) -> List[Light]:                        # EXTENSION
    if not isinstance(o, list):
        _fail(path, "must be an array")
    out = []
    for i, l in enumerate(o):
        lp = f"{path}[{i}]"
        _check_keys(l, lp, {"position", "intensity"})
        light = Light(_get_vec3(l, lp, "position"), _get_double_or(l, lp, "intensity", 1.0))
        if not (light.intensity >= 0.0):
            _fail(lp + ".intensity", "must be >= 0")
        out.append(light)
    return out


def _parse_camera(o, path) -> CameraSpec:                         # :340-352
    c = CameraSpec()
    if o is None:
        return c
    _check_keys(o, path, {"position", "look_dir", "up_hint", "fov_deg"})
    c.position = _get_vec3_or(o, path, "position", c.position)
    c.look_dir = _get_vec3_or(o, path, "look_dir", c.look_dir)
    c.up_hint = _get_vec3_or(o, path, "up_hint", c.up_hint)
    c.fov_deg = _get_double_or(o, path, "fov_deg", c.fov_deg)
    if not (0.0 < c.fov_deg < 180.0):
        _fail(path + ".fov_deg", "must be in (0, 180)")
    if not (_norm(_cross(c.look_dir, c.up_hint)) > 1e-12):
        _fail(path, "look_dir and up_hint must be linearly independent")
    return c


def _parse_integrator(o, path, allow_ext: bool = True) -> IntegratorConfig:  # :354-370
    c = IntegratorConfig()
    if o is None:
        return c
    _check_keys(o, path, {"h", "max_steps", "scheme"} | ({"tol"} if allow_ext else set()))
    c.h = _get_double_or(o, path, "h", c.h)
    if not (c.h > 0.0):
        _fail(path + ".h", "must be > 0")
    c.max_steps = _get_int_or(o, path, "max_steps", c.max_steps)
    if c.max_steps < 1:
        _fail(path + ".max_steps", "must be >= 1")
    scheme = _get_string_or(o, path, "scheme", "euler")
    if scheme not in ("euler", "rk4") and not (allow_ext and scheme == "rk23"):
        _fail(path + ".scheme", f"must be euler|rk4, got '{scheme}'")
    c.scheme = scheme
    if allow_ext:
        c.tol = _get_double_or(o, path, "tol", 1e-6)
        if not (c.tol > 0.0):
            _fail(path + ".tol", "must be > 0")
    return c


def _parse_output(o, path) -> OutputSpec:                         # :372-386
    out = OutputSpec()
    if o is None:
        return out
    _check_keys(o, path, {"path", "width", "height", "format"})
    out.path = _get_string_or(o, path, "path", out.path)
    if not out.path:
        _fail(path + ".path", "must be non-empty")
    out.width = _get_int_or(o, path, "width", out.width)
    out.height = _get_int_or(o, path, "height", out.height)
    if out.width < 1 or out.height < 1:
        _fail(path + ".width/height", "must be >= 1")
    out.format = _get_string_or(o, path, "format", out.format)
    if out.format != "ppm":
        _fail(path + ".format", f"only 'ppm' is supported by this build, got '{out.format}'")
    return out


def _reject_constant(name):
    raise ValueError(f"invalid literal {name}")


def parse_config(text: str, allow_ext: bool = True) -> RunConfig:  # :437-456
    try:
        root = json.loads(text, parse_constant=_reject_constant)
    except ValueError as e:
        raise ParseError(f"config: {e}") from None
    _check_keys(root, "config", {"metric", "scene", "camera", "integrator", "output"})
    if "metric" not in root:
        _fail("config.metric", "required")
    cfg = RunConfig()
    cfg.metric = _parse_metric(root["metric"], "metric", allow_ext)
    cfg.scene = _parse_scene(root.get("scene"), "scene", allow_ext)
    cfg.camera = _parse_camera(root.get("camera"), "camera")
    cfg.integrator = _parse_integrator(root.get("integrator"), "integrator", allow_ext)
    cfg.output = _parse_output(root.get("output"), "output")
    return cfg


def load_config(path: str, allow_ext: bool = True) -> RunConfig:  # :458-464
    from .errors import IoError
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise IoError(f"cannot open config '{path}'") from None
    return parse_config(text, allow_ext)


# ---- serialization (config.cpp:388-483) -------------------------------------

def _field_json(f):
    if isinstance(f, GaussianField):
        return {"kind": "gaussian", "amplitude": f.params.amplitude,
                "center": list(f.params.center), "sigma": list(f.params.sigma)}
    if isinstance(f, PolynomialField):
        return {"kind": "polynomial",
                "terms": [{"coef": t.coef, "powers": list(t.powers)} for t in f.terms]}
    return {"kind": "sum", "terms": [_field_json(t) for t in f.terms]}


def _diffeo_json(d):
    if isinstance(d, IdentityMap):
        return {"kind": "identity"}
    if isinstance(d, AffineMap):
        return {"kind": "affine", "matrix": [list(r) for r in d.matrix], "offset": list(d.offset)}
    if isinstance(d, TwistMap):
        return {"kind": "twist"}
    if isinstance(d, BendMap):
        return {"kind": "bend", "curvature": d.curvature}
    if isinstance(d, LocalBumpMap):
        return {"kind": "local_bump", "amplitude": d.bump.amplitude, "center": list(d.bump.center),
                "sigma": list(d.bump.sigma), "direction": list(d.direction)}
    return {"kind": "compose", "maps": [_diffeo_json(m) for m in d.maps]}


def _metric_json(m):
    if isinstance(m, EuclideanMetric):
        return {"kind": "euclidean"}
    if isinstance(m, GraphMetric):
        return {"kind": "graph", "field": _field_json(m.field)}
    return {"kind": "diffeo", "map": _diffeo_json(m.map)}


def _aabb_json(b):
    return {"min": list(b.min), "max": list(b.max)}


def _prim_json(p):
    if isinstance(p, Mesh):
        if p.generator is not None:
            return {"kind": "mesh", "generator": dict(p.generator)}
        return {"kind": "mesh", "vertices": p.vertices.tolist(), "triangles": p.triangles.tolist()}
    if isinstance(p, GridPlanes):
        return {"kind": "grid_planes", "spacing": p.spacing, "half_width": p.half_width,
                "bounds": _aabb_json(p.bounds)}
    if isinstance(p, Sphere):
        return {"kind": "sphere", "center": list(p.center), "radius": p.radius}
    return {"kind": "half_space", "normal": list(p.normal), "offset": p.offset}


def config_to_dict(cfg: RunConfig, include_ext: bool = True) -> dict:
    prims = [p for p in cfg.scene.primitives if include_ext or not isinstance(p, Mesh)]
    scene = {"primitives": [_prim_json(p) for p in prims],
             "bounds": _aabb_json(cfg.scene.bounds), "fog_density": cfg.scene.fog_density}
    if include_ext and cfg.scene.lights:
        scene["lights"] = [{"position": list(l.position), "intensity": l.intensity}
                           for l in cfg.scene.lights]
        scene["ambient"] = cfg.scene.ambient
    return {
        "metric": _metric_json(cfg.metric),
        "scene": scene,
        "camera": {"position": list(cfg.camera.position), "look_dir": list(cfg.camera.look_dir),
                   "up_hint": list(cfg.camera.up_hint), "fov_deg": cfg.camera.fov_deg},
        "integrator": dict({"h": cfg.integrator.h, "max_steps": cfg.integrator.max_steps,
                            "scheme": cfg.integrator.scheme},
                           **({"tol": cfg.integrator.tol}
                              if include_ext and cfg.integrator.scheme == "rk23" else {})),
        "output": {"path": cfg.output.path, "width": cfg.output.width,
                   "height": cfg.output.height, "format": cfg.output.format},
    }


def serialize_config(cfg: RunConfig, include_ext: bool = True) -> str:
    """Fully defaulted, round-trippable 2-space JSON (sorted keys, as nlohmann)."""
    return json.dumps(config_to_dict(cfg, include_ext), indent=2, sort_keys=True) + "\n"


def reference_json(cfg: RunConfig) -> str:
    """The document with EXTENSION keys stripped (what the reference parser accepts)."""
    return serialize_config(cfg, include_ext=False)


# ---- flattening into C-ABI descriptors --------------------------------------

class MetricDesc:
    """Owns the node arrays behind an ``rr_metric_desc``."""

    def __init__(self, metric: Metric):
        self.field_nodes: list = []
        self.poly_terms: list = []
        self.diffeo_nodes: list = []
        self.children: list = []
        kind, root = abi.RR_METRIC_EUCLIDEAN, 0
        if isinstance(metric, GraphMetric):
            kind, root = abi.RR_METRIC_GRAPH, self._add_field(metric.field)
        elif isinstance(metric, DiffeoMetric):
            kind, root = abi.RR_METRIC_DIFFEO, self._add_diffeo(metric.map)
        self._fn = (abi.rr_field_node * max(1, len(self.field_nodes)))(*self.field_nodes)
        self._pt = (abi.rr_poly_term * max(1, len(self.poly_terms)))(*self.poly_terms)
        self._dn = (abi.rr_diffeo_node * max(1, len(self.diffeo_nodes)))(*self.diffeo_nodes)
        self._ch = (C.c_int32 * max(1, len(self.children)))(*self.children)
        self.desc = abi.rr_metric_desc(
            kind, root, len(self.field_nodes), len(self.poly_terms), len(self.diffeo_nodes),
            len(self.children), self._fn, self._pt, self._dn, self._ch)

    @staticmethod
    def _gauss(g: GaussianParams) -> abi.rr_gaussian:
        return abi.rr_gaussian(float(g.amplitude), abi.rr_vec3.of(g.center), abi.rr_vec3.of(g.sigma))

    def _add_field(self, f) -> int:
        idx = len(self.field_nodes)
        node = abi.rr_field_node()
        self.field_nodes.append(node)
        if isinstance(f, GaussianField):
            node.kind = abi.RR_FIELD_GAUSSIAN
            node.gaussian = self._gauss(f.params)
        elif isinstance(f, PolynomialField):
            node.kind, node.first, node.count = abi.RR_FIELD_POLYNOMIAL, len(self.poly_terms), len(f.terms)
            for t in f.terms:
                pt = abi.rr_poly_term()
                pt.coef = float(t.coef)
                pt.powers[:] = [int(x) for x in t.powers]
                self.poly_terms.append(pt)
        else:
            base = len(self.children)
            self.children.extend([0] * len(f.terms))
            node.kind, node.first, node.count = abi.RR_FIELD_SUM, base, len(f.terms)
            for i, t in enumerate(f.terms):
                self.children[base + i] = self._add_field(t)
        self.field_nodes[idx] = node
        return idx

    def _add_diffeo(self, d) -> int:
        idx = len(self.diffeo_nodes)
        node = abi.rr_diffeo_node()
        self.diffeo_nodes.append(node)
        if isinstance(d, IdentityMap):
            node.kind = abi.RR_DIFFEO_IDENTITY
        elif isinstance(d, AffineMap):
            node.kind = abi.RR_DIFFEO_AFFINE
            for i in range(3):
                for j in range(3):
                    node.matrix[i][j] = float(d.matrix[i][j])
            node.offset = abi.rr_vec3.of(d.offset)
        elif isinstance(d, TwistMap):
            node.kind = abi.RR_DIFFEO_TWIST
        elif isinstance(d, BendMap):
            node.kind = abi.RR_DIFFEO_BEND
            node.curvature = float(d.curvature)
        elif isinstance(d, LocalBumpMap):
            node.kind = abi.RR_DIFFEO_LOCAL_BUMP
            node.bump = self._gauss(d.bump)
            node.direction = abi.rr_vec3.of(d.direction)
        else:
            base = len(self.children)
            self.children.extend([0] * len(d.maps))
            node.kind, node.first, node.count = abi.RR_DIFFEO_COMPOSE, base, len(d.maps)
            for i, m in enumerate(d.maps):
                self.children[base + i] = self._add_diffeo(m)
        self.diffeo_nodes[idx] = node
        return idx


class SceneDesc:
    """Owns the primitive/light arrays behind an ``rr_scene_desc``."""

    def __init__(self, scene: Scene, with_lights: bool = True):
        import numpy as np
        prims = []
        self._mesh_arrays = []
        for p in scene.primitives:
            q = abi.rr_primitive()
            if isinstance(p, Mesh):
                v = np.ascontiguousarray(p.vertices, np.float64)
                t = np.ascontiguousarray(p.triangles, np.int32)
                self._mesh_arrays += [v, t]
                q.kind = abi.RR_PRIM_MESH
                q.n_vertices, q.n_triangles = len(v), len(t)
                q.vertices = v.ctypes.data_as(C.POINTER(C.c_double))
                q.triangles = t.ctypes.data_as(C.POINTER(C.c_int32))
            elif isinstance(p, GridPlanes):
                q.kind = abi.RR_PRIM_GRID_PLANES
                q.spacing, q.half_width = float(p.spacing), float(p.half_width)
                q.bounds = abi.rr_aabb(abi.rr_vec3.of(p.bounds.min), abi.rr_vec3.of(p.bounds.max))
            elif isinstance(p, Sphere):
                q.kind = abi.RR_PRIM_SPHERE
                q.center, q.radius = abi.rr_vec3.of(p.center), float(p.radius)
            else:
                q.kind = abi.RR_PRIM_HALF_SPACE
                q.normal, q.offset = abi.rr_vec3.of(p.normal), float(p.offset)
            prims.append(q)
        lights = [abi.rr_light(abi.rr_vec3.of(l.position), float(l.intensity))
                  for l in (scene.lights if with_lights else [])]
        self._pr = (abi.rr_primitive * max(1, len(prims)))(*prims)
        self._li = (abi.rr_light * max(1, len(lights)))(*lights)
        self.desc = abi.rr_scene_desc(
            len(prims), len(lights), self._pr, self._li,
            abi.rr_aabb(abi.rr_vec3.of(scene.bounds.min), abi.rr_vec3.of(scene.bounds.max)),
            float(scene.fog_density), float(scene.ambient))


def fov_radians(cam: CameraSpec) -> float:
    """cfg.camera.fov_deg * M_PI / 180.0 (rray_main.cpp:56)."""
    return cam.fov_deg * math.pi / 180.0
