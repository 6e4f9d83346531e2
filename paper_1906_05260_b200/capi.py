"""ctypes mirror of include/vrod_capi.h — the C-ABI drop-in boundary.

The header restates the reference's C++ core API (`proj/core/include/vrod/`)
as plain C. This module only declares the structs and signatures and marshals a Python
`Scene` (paper_1906_05260_b200.scene) into a `vrod_scene*` of a given library handle.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

VROD_OK = 0
VROD_INVALID_ARGUMENT = 1
VROD_OUT_OF_RANGE = 2
VROD_SIMULATION_ERROR = 3
VROD_RUNTIME_ERROR = 4
VROD_DEVICE_ERROR = 5

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


class Material(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("stretch_x", "stretch_y", "stretch_z", "bend_x", "bend_y", "bend_z", "volume", "density")]


class Settings(C.Structure):
    _fields_ = [("dt", C.c_double), ("iterations", C.c_int32), ("substeps", C.c_int32),
                ("beta", C.c_double), ("gravity", C.c_double * 3),
                ("dichotomous_iterations", C.c_int32), ("shape_match_period", C.c_int32),
                ("contact_stiffness", C.c_double), ("velocity_damping", C.c_double),
                ("deterministic", C.c_int32), ("scale_mode", C.c_int32)]


class Pill(C.Structure):
    _fields_ = [("c0", C.c_double * 3), ("c1", C.c_double * 3), ("r0", C.c_double), ("r1", C.c_double),
                ("rod", C.c_int32), ("element", C.c_int32), ("group", C.c_int32), ("self_collide", C.c_int32)]


PILL_DTYPE = np.dtype([("c0", "<f8", 3), ("c1", "<f8", 3), ("r0", "<f8"), ("r1", "<f8"),
                       ("rod", "<i4"), ("element", "<i4"), ("group", "<i4"), ("self_collide", "<i4")])
assert PILL_DTYPE.itemsize == C.sizeof(Pill)


# PillTransform (skinning.h:19-25): center xyz, scale, rotation wxyz — 8 doubles.
TRANSFORM_DTYPE = np.dtype([("center", "<f8", 3), ("scale", "<f8"), ("rotation", "<f8", 4)])


class StepReport(C.Structure):
    _fields_ = [("step", C.c_int32), ("contact_count", C.c_int32), ("broad_pairs", C.c_int32),
                ("skipped_singular", C.c_int32), ("dof_count", C.c_int32), ("pad_", C.c_int32),
                ("time", C.c_double), ("residuals", C.c_double * 8), ("max_penetration", C.c_double),
                ("predict_ms", C.c_double), ("broad_ms", C.c_double), ("narrow_ms", C.c_double),
                ("solve_ms", C.c_double), ("finalize_ms", C.c_double), ("total_ms", C.c_double)]


class RodDesc(C.Structure):
    _fields_ = [("vertex_count", C.c_int32), ("material", C.c_int32), ("collision_group", C.c_int32),
                ("self_collide", C.c_int32),
                ("rest_centers", _dp), ("rest_scales", _dp), ("radii", _dp), ("lengths", _dp),
                ("initial_lengths", _dp), ("rest_frames", _dp), ("darboux", _dp), ("tangent_dots", _dp),
                ("scale_grads", _dp), ("scale_laplacians", _dp),
                ("centers", _dp), ("scales", _dp), ("frames", _dp), ("center_vel", _dp), ("scale_vel", _dp),
                ("angular_vel", _dp), ("pinned", _u8p), ("bone_count", C.c_int32), ("pad_", C.c_int32),
                ("bones", _ip), ("bone_weights", _dp)]


class RestPoseOut(C.Structure):
    _fields_ = [(n, _dp) for n in ("rest_scales", "radii", "lengths", "initial_lengths", "rest_frames",
                                   "darboux", "tangent_dots", "scale_grads", "scale_laplacians")]


class SolverInfo(C.Structure):
    _fields_ = [("rod_count", C.c_int32), ("total_vertices", C.c_int32), ("total_elements", C.c_int32),
                ("dof_count", C.c_int32), ("step_index", C.c_int32), ("bundle_count", C.c_int32),
                ("elastic_blocks", C.c_int32), ("pad_", C.c_int32), ("time", C.c_double)]


_SIGNATURES = {
    "vrod_last_error": (C.c_char_p, []),
    "vrod_backend_name": (C.c_char_p, []),
    "vrod_capi_version": (C.c_int32, []),
    "vrod_default_material": (None, [C.POINTER(Material)]),
    "vrod_default_settings": (None, [C.POINTER(Settings)]),
    "vrod_make_rest_pose": (C.c_int, [C.c_int32, _dp, C.c_int32, _dp, C.c_int32, _dp, C.POINTER(RestPoseOut)]),
    "vrod_scene_create": (C.c_int, [C.POINTER(C.c_void_p)]),
    "vrod_scene_destroy": (None, [C.c_void_p]),
    "vrod_scene_set_settings": (C.c_int, [C.c_void_p, C.POINTER(Settings)]),
    "vrod_scene_add_material": (C.c_int, [C.c_void_p, C.POINTER(Material)]),
    "vrod_scene_add_rod": (C.c_int, [C.c_void_p, C.POINTER(RodDesc)]),
    "vrod_scene_add_plane": (C.c_int, [C.c_void_p, _dp, C.c_double]),
    "vrod_scene_add_bone": (C.c_int, [C.c_void_p, C.c_int32, _dp, _dp, _dp]),
    "vrod_scene_add_kinematic_pill": (C.c_int, [C.c_void_p, C.POINTER(Pill), C.c_int32]),
    "vrod_scene_add_bundle": (C.c_int, [C.c_void_p, C.c_int32, _ip, _ip]),
    "vrod_scene_add_pin_motion": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, _dp, _dp, C.c_double, C.c_double]),
    "vrod_scene_add_soft_pin": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, _dp, C.c_double]),
    "vrod_scene_add_activation": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_double,
                                            C.c_int32, C.c_int32]),
    "vrod_scene_validate": (C.c_int, [C.c_void_p]),
    "vrod_solver_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "vrod_solver_destroy": (None, [C.c_void_p]),
    "vrod_solver_step": (C.c_int, [C.c_void_p, C.POINTER(StepReport)]),
    "vrod_solver_probe_convergence": (C.c_int, [C.c_void_p, C.c_int32, _dp]),
    "vrod_solver_get_info": (C.c_int, [C.c_void_p, C.POINTER(SolverInfo)]),
    "vrod_solver_get_rod_sizes": (C.c_int, [C.c_void_p, _ip]),
    "vrod_solver_get_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp]),
    "vrod_solver_set_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp]),
    "vrod_solver_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "vrod_solver_get_rest": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp]),
    "vrod_solver_set_loads": (C.c_int, [C.c_void_p, _dp, _u8p, _dp, _u8p, _dp, _u8p]),
    "vrod_solver_energy": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "vrod_solver_get_inverse_weights": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "vrod_solver_get_weights": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "vrod_solver_get_contacts": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _ip, _ip, _dp, _dp]),
    "vrod_solver_current_pills": (C.c_int, [C.c_void_p, C.c_int64, _i64p, C.c_void_p]),
    "vrod_batch_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "vrod_solver_scene_count": (C.c_int, [C.c_void_p, _ip]),
    "vrod_solver_scene_reports": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "vrod_pill_project": (C.c_int, [C.c_int64, _dp, C.c_void_p, _dp, _dp, _u8p]),
    "vrod_deepest_penetration": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, _dp, _dp, _dp, _dp]),
    "vrod_broad_phase": (C.c_int, [C.c_int64, C.c_void_p, C.c_int64, _i64p, _ip]),
    "vrod_find_contacts": (C.c_int, [C.c_int64, C.c_void_p, C.c_int64, _ip, C.c_int32, C.c_int64, _u64p, _dp,
                                     C.c_int64, _i64p, _ip, _ip, _dp, _dp, _dp]),
    "vrod_pair_key": (C.c_uint64, [C.POINTER(Pill), C.POINTER(Pill)]),
    "vrod_solver_pill_transforms": (C.c_int, [C.c_void_p, C.c_int64, _i64p, C.c_void_p]),
    "vrod_solver_rest_pill_transforms": (C.c_int, [C.c_void_p, C.c_int64, _i64p, C.c_void_p]),
    "vrod_solver_rest_pills": (C.c_int, [C.c_void_p, C.c_int64, _i64p, C.c_void_p]),
    "vrod_skin_bind": (C.c_int, [C.c_int32, _dp, C.c_int32, _ip, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                 C.c_double, C.POINTER(C.c_void_p)]),
    "vrod_skin_destroy": (None, [C.c_void_p]),
    "vrod_skin_smooth": (C.c_int, [C.c_void_p, C.c_int32]),
    "vrod_skin_get_binding": (C.c_int, [C.c_void_p, _ip, _ip, _dp, _ip, _ip]),
    "vrod_skin_deform": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, _dp]),
    "vrod_skin_deform_solver": (C.c_int, [C.c_void_p, C.c_void_p, _dp]),
    "vrod_solver_shape_match": (C.c_int, [C.c_void_p, C.c_int32, _ip, _dp]),
    "vrod_extract_rotation": (C.c_int, [C.c_int64, _dp, _dp, C.c_int32, C.c_double, _dp]),
    "vrod_solver_jacobi_sweep": (C.c_int, [C.c_void_p, C.c_double, C.c_double, _ip, _ip]),
    "vrod_solver_elastic_residuals": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _dp]),
}

# Optional entry points (product-only extensions; absent from the oracle libraries).
_OPTIONAL = {}


def bind(lib: C.CDLL) -> C.CDLL:
    """Attach argtypes/restype for every C-ABI symbol; raises if one is missing."""
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError if the library does not export it
        fn.restype = res
        fn.argtypes = args
    for name, (res, args) in _OPTIONAL.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.restype = res
            fn.argtypes = args
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def ptr(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C-ABI must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))
