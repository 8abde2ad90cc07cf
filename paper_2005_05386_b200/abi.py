"""ctypes mirror of include/rray_cuda.h (the C-ABI boundary).

Struct layouts are byte-identical to the C header; ``tests/test_abi.py``
checks sizes/offsets against the compiled library.  numpy dtypes are given for
the bulk records (``RAY_DTYPE`` == render::RayStart, ``OUTCOME_DTYPE`` ==
render::PixelOutcome, /root/reference/proj/include/rray/render/kernel.hpp:26-39).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

# status codes (rray_main.cpp:185-194) + device extension
RR_OK, RR_ERR_CONFIG, RR_ERR_NUMERIC, RR_ERR_IO, RR_ERR_DEVICE = 0, 1, 2, 3, 4

RR_FIELD_GAUSSIAN, RR_FIELD_POLYNOMIAL, RR_FIELD_SUM = 0, 1, 2
(RR_DIFFEO_IDENTITY, RR_DIFFEO_AFFINE, RR_DIFFEO_TWIST, RR_DIFFEO_LOCAL_BUMP,
 RR_DIFFEO_COMPOSE, RR_DIFFEO_BEND) = 0, 1, 2, 3, 4, 5
RR_METRIC_EUCLIDEAN, RR_METRIC_GRAPH, RR_METRIC_DIFFEO = 0, 1, 2
RR_PRIM_GRID_PLANES, RR_PRIM_SPHERE, RR_PRIM_HALF_SPACE, RR_PRIM_MESH = 0, 1, 2, 3
RR_SCHEME_EULER, RR_SCHEME_RK4, RR_SCHEME_RK23 = 0, 1, 2
RR_MISS, RR_HIT, RR_FAILED = 0, 1, 2


class rr_vec3(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]

    @classmethod
    def of(cls, v):
        return cls(float(v[0]), float(v[1]), float(v[2]))

    def tolist(self):
        return [self.x, self.y, self.z]


class rr_aabb(C.Structure):
    _fields_ = [("min", rr_vec3), ("max", rr_vec3)]


class rr_gaussian(C.Structure):
    _fields_ = [("amplitude", C.c_double), ("center", rr_vec3), ("sigma", rr_vec3)]


class rr_poly_term(C.Structure):
    _fields_ = [("coef", C.c_double), ("powers", C.c_int32 * 3), ("pad_", C.c_int32)]


class rr_field_node(C.Structure):
    _fields_ = [("kind", C.c_int32), ("first", C.c_int32), ("count", C.c_int32),
                ("pad_", C.c_int32), ("gaussian", rr_gaussian)]


class rr_diffeo_node(C.Structure):
    _fields_ = [("kind", C.c_int32), ("first", C.c_int32), ("count", C.c_int32),
                ("pad_", C.c_int32), ("matrix", (C.c_double * 3) * 3), ("offset", rr_vec3),
                ("bump", rr_gaussian), ("direction", rr_vec3), ("curvature", C.c_double)]


class rr_metric_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("root", C.c_int32), ("n_field_nodes", C.c_int32),
                ("n_poly_terms", C.c_int32), ("n_diffeo_nodes", C.c_int32),
                ("n_children", C.c_int32),
                ("field_nodes", C.POINTER(rr_field_node)),
                ("poly_terms", C.POINTER(rr_poly_term)),
                ("diffeo_nodes", C.POINTER(rr_diffeo_node)),
                ("children", C.POINTER(C.c_int32))]


class rr_primitive(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("spacing", C.c_double),
                ("half_width", C.c_double), ("bounds", rr_aabb), ("center", rr_vec3),
                ("radius", C.c_double), ("normal", rr_vec3), ("offset", C.c_double),
                ("n_vertices", C.c_int32), ("n_triangles", C.c_int32),
                ("vertices", C.POINTER(C.c_double)), ("triangles", C.POINTER(C.c_int32))]


class rr_light(C.Structure):
    _fields_ = [("position", rr_vec3), ("intensity", C.c_double)]


class rr_scene_desc(C.Structure):
    _fields_ = [("n_primitives", C.c_int32), ("n_lights", C.c_int32),
                ("primitives", C.POINTER(rr_primitive)), ("lights", C.POINTER(rr_light)),
                ("bounds", rr_aabb), ("fog_density", C.c_double), ("ambient", C.c_double)]


class rr_integrator(C.Structure):
    _fields_ = [("h", C.c_double), ("max_steps", C.c_int32), ("scheme", C.c_int32),
                ("tol", C.c_double)]


class rr_ray_start(C.Structure):
    _fields_ = [("position", rr_vec3), ("direction", rr_vec3)]


class rr_pixel_outcome(C.Structure):
    _fields_ = [("status", C.c_uint8), ("prim", C.c_int32), ("point", rr_vec3),
                ("t", C.c_double), ("steps", C.c_int32)]


class rr_camera(C.Structure):
    _fields_ = [("position", rr_vec3), ("look_dir", rr_vec3), ("up_hint", rr_vec3),
                ("fov", C.c_double), ("frame", rr_vec3 * 3), ("g", C.c_double * 6)]


class rr_stats(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("rays", C.c_int64),
                ("total_steps", C.c_int64), ("pixel_errors", C.c_int64),
                ("device_ms", C.c_double), ("integrated_steps", C.c_int64),
                ("bump_evals", C.c_int64), ("shadow_steps", C.c_int64),
                ("kernel_launches", C.c_int64), ("lane_slots", C.c_int64),
                ("shadow_lane_slots", C.c_int64), ("jump_steps", C.c_int64),
                ("shadow_jump_steps", C.c_int64), ("shadow_integrated_steps", C.c_int64),
                ("sort_kernels", C.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class rr_options(C.Structure):
    _fields_ = [("cull", C.c_int32), ("cull_grid", C.c_int32),
                ("cull_radius_sigma", C.c_double), ("block_x", C.c_int32),
                ("block_y", C.c_int32), ("persistent", C.c_int32), ("skip", C.c_int32),
                ("order_units", C.c_int32)]


class rr_frame_handle(C.Structure):
    _fields_ = [("ipc", C.c_ubyte * 64), ("offset", C.c_uint64), ("bytes", C.c_uint64),
                ("ptr", C.c_uint64), ("device", C.c_int32), ("pid", C.c_int32)]


RAY_DTYPE = np.dtype([("position", "<f8", (3,)), ("direction", "<f8", (3,))])
OUTCOME_DTYPE = np.dtype({
    "names": ["status", "prim", "point", "t", "steps"],
    "formats": ["u1", "<i4", ("<f8", (3,)), "<f8", "<i4"],
    "offsets": [0, 4, 8, 32, 40],
    "itemsize": 48,
})

# Expected C sizes (checked against the header in tests/test_abi.py).
EXPECTED_SIZES = {
    "rr_vec3": 24, "rr_aabb": 48, "rr_gaussian": 56, "rr_poly_term": 24,
    "rr_field_node": 72, "rr_diffeo_node": 200, "rr_metric_desc": 56,
    "rr_primitive": 160, "rr_light": 32, "rr_scene_desc": 88, "rr_integrator": 24,
    "rr_ray_start": 48, "rr_pixel_outcome": 48, "rr_camera": 200, "rr_stats": 120,
    "rr_options": 40, "rr_frame_handle": 96,
}

STRUCTS = {
    "rr_vec3": rr_vec3, "rr_aabb": rr_aabb, "rr_gaussian": rr_gaussian,
    "rr_poly_term": rr_poly_term, "rr_field_node": rr_field_node,
    "rr_diffeo_node": rr_diffeo_node, "rr_metric_desc": rr_metric_desc,
    "rr_primitive": rr_primitive, "rr_light": rr_light, "rr_scene_desc": rr_scene_desc,
    "rr_integrator": rr_integrator, "rr_ray_start": rr_ray_start,
    "rr_pixel_outcome": rr_pixel_outcome, "rr_camera": rr_camera, "rr_stats": rr_stats,
    "rr_options": rr_options, "rr_frame_handle": rr_frame_handle,
}

# Every symbol include/rray_cuda.h declares, with its ctypes signature.
_P = C.c_void_p
SIGNATURES = {
    "rr_abi_version": (C.c_int, []),
    "rr_build_info": (C.c_char_p, []),
    "rr_create": (C.c_int, [C.POINTER(_P), C.c_int]),
    "rr_destroy": (None, [_P]),
    "rr_last_error": (C.c_char_p, [_P]),
    "rr_set_options": (C.c_int, [_P, C.POINTER(rr_options)]),
    "rr_get_options": (C.c_int, [_P, C.POINTER(rr_options)]),
    "rr_set_scene": (C.c_int, [_P, C.POINTER(rr_metric_desc), C.POINTER(rr_scene_desc)]),
    "rr_build_camera": (C.c_int, [_P, C.POINTER(rr_vec3), C.POINTER(rr_vec3),
                                  C.POINTER(rr_vec3), C.c_double, C.POINTER(rr_camera)]),
    "rr_pixel_direction": (C.c_int, [C.POINTER(rr_camera), C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.POINTER(rr_vec3)]),
    "rr_march": (C.c_int, [_P, C.POINTER(rr_integrator), _P, _P, C.c_size_t]),
    "rr_march_device": (C.c_int, [_P, C.POINTER(rr_integrator), _P, _P, C.c_size_t, _P]),
    "rr_render": (C.c_int, [_P, C.POINTER(rr_camera), C.POINTER(rr_integrator), C.c_int,
                            C.c_int, _P, C.POINTER(rr_stats)]),
    "rr_render_device": (C.c_int, [_P, C.POINTER(rr_camera), C.POINTER(rr_integrator),
                                   C.c_int, C.c_int, _P, C.POINTER(rr_stats), _P]),
    "rr_render_outcomes": (C.c_int, [_P, C.POINTER(rr_camera), C.POINTER(rr_integrator),
                                     C.c_int, C.c_int, _P, _P, C.POINTER(rr_stats)]),
    "rr_last_kernel": (C.c_char_p, [_P]),
    "rr_shard_tile_count": (C.c_int, [C.c_int] * 6),
    "rr_render_tiles": (C.c_int, [_P, C.POINTER(rr_camera), C.POINTER(rr_integrator),
                                  C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P,
                                  C.POINTER(rr_stats), _P]),
    "rr_render_shard": (C.c_int, [_P, C.POINTER(rr_camera), C.POINTER(rr_integrator),
                                  C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P,
                                  C.POINTER(rr_stats), _P]),
    "rr_detile": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P]),
    "rr_frame_export": (C.c_int, [_P, _P, C.c_size_t, C.POINTER(rr_frame_handle)]),
    "rr_frame_import": (C.c_int, [_P, C.POINTER(rr_frame_handle), C.POINTER(_P)]),
    "rr_frame_close": (C.c_int, [_P, _P]),
    "rr_frame_probe": (C.c_int, [_P, _P, C.c_size_t, C.c_uint8]),
    "rr_measure_fp32_peak": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "rr_trace": (C.c_int, [_P, C.POINTER(rr_integrator), _P, C.c_size_t, C.c_int, _P, _P, _P]),
    "rr_accel": (C.c_int, [_P, _P, _P, C.c_size_t, _P, _P]),
    "rr_metric_tensor": (C.c_int, [_P, _P, _P]),
    "rr_christoffel_fd": (C.c_int, [_P, _P, C.c_double, _P]),
    "rr_diffeo_image": (C.c_int, [_P, _P, _P]),
}


def bind(lib: C.CDLL) -> C.CDLL:
    """Attach argtypes/restype for every ABI symbol (raises if one is missing)."""
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
