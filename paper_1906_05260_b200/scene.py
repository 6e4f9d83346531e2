"""Host-side mirror of the reference's scene model (`proj/core/include/vrod/{rod,scene}.h`).

Plain data, same names and defaults as the reference structs, so a user of
`vrod::Scene` / `vrod::Rod` builds the same thing here:

    MaterialParams   rod.h:13-24          SolverSettings  scene.h:25-39
    RodRestPose      rod.h:30-46          RodState        rod.h:50-60
    Rod              rod.h:64-74          Scene           scene.h:109-126
    HalfPlane, Pill  collision.h:16-30    Bone, KinematicPill, PinMotion, SoftPin, Activation  scene.h:41-92

Vectors are numpy float64 arrays: Vec3 -> (3,), Quat -> (4,) in (w, x, y, z) order.
`marshal_scene` converts a Scene into a `vrod_scene*` of any library exporting
include/vrod_capi.h.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import capi

INF = math.inf


# ---- errors (types.h:25-28, 67-77) -------------------------------------------------------------

class VrodError(Exception):
    """Base of the errors raised through the C-ABI."""


class InvalidArgument(VrodError, ValueError):
    """std::invalid_argument raised by `require` (types.h:67-69)."""


class OutOfRange(VrodError, IndexError):
    """std::out_of_range raised by `require_index` (types.h:71-77)."""


class SimulationError(VrodError, RuntimeError):
    """vrod::SimulationError: non-finite state during a step (types.h:25-28)."""


class DeviceError(VrodError, RuntimeError):
    """CUDA failure inside the product library."""


_ERRORS = {capi.VROD_INVALID_ARGUMENT: InvalidArgument, capi.VROD_OUT_OF_RANGE: OutOfRange,
           capi.VROD_SIMULATION_ERROR: SimulationError, capi.VROD_RUNTIME_ERROR: VrodError,
           capi.VROD_DEVICE_ERROR: DeviceError}


def check(lib, rc: int) -> None:
    if rc != capi.VROD_OK:
        raise _ERRORS.get(rc, VrodError)(lib.vrod_last_error().decode())


# ---- plain data --------------------------------------------------------------------------------

@dataclass
class MaterialParams:
    stretch_x: float = 1e4
    stretch_y: float = 1e4
    stretch_z: float = 1e4
    bend_x: float = 1e3
    bend_y: float = 1e3
    bend_z: float = 0.0
    volume: float = 1e6
    density: float = 1000.0


SCALE_SIMULATED = 0
SCALE_POST_STEP_LENGTH_RATIO = 1


@dataclass
class SolverSettings:
    dt: float = 1.0 / 60.0
    iterations: int = 20
    substeps: int = 1
    beta: float = 0.75
    gravity: tuple = (0.0, 0.0, -9.81)
    dichotomous_iterations: int = 10
    shape_match_period: int = 2
    contact_stiffness: float = INF
    velocity_damping: float = 0.0
    deterministic: bool = False
    scale_mode: int = SCALE_SIMULATED


@dataclass
class RodRestPose:
    centers: np.ndarray          # (n,3)
    scales: np.ndarray           # (n,)
    radii: np.ndarray            # (n,)
    lengths: np.ndarray          # (m,)
    initial_lengths: np.ndarray  # (m,)
    frames: np.ndarray           # (m,4) wxyz
    darboux: np.ndarray          # (m-1,3)
    tangent_dots: np.ndarray     # (m,)
    scale_grads: np.ndarray      # (m,)
    scale_laplacians: np.ndarray  # (m-1,)

    def vertex_count(self) -> int:
        return int(self.centers.shape[0])

    def element_count(self) -> int:
        return int(self.frames.shape[0])

    def copy(self) -> "RodRestPose":
        return RodRestPose(**{k: np.array(v, copy=True) for k, v in self.__dict__.items()})


@dataclass
class RodState:
    centers: np.ndarray
    scales: np.ndarray
    frames: np.ndarray
    center_vel: np.ndarray
    scale_vel: np.ndarray
    angular_vel: np.ndarray

    def copy(self) -> "RodState":
        return RodState(**{k: np.array(v, copy=True) for k, v in self.__dict__.items()})


@dataclass
class Rod:
    rest: RodRestPose
    state: RodState
    material: int = 0
    pinned: np.ndarray | None = None  # (n,) uint8
    collision_group: int = -1
    self_collide: bool = False
    bones: Sequence[int] = ()
    bone_weights: np.ndarray | None = None  # (n, len(bones))

    def __post_init__(self):
        if self.pinned is None:
            self.pinned = np.zeros(self.rest.vertex_count(), dtype=np.uint8)


@dataclass
class HalfPlane:
    normal: tuple = (0.0, 0.0, 1.0)
    offset: float = 0.0


@dataclass
class RigidKeyframe:
    t: float = 0.0
    position: tuple = (0.0, 0.0, 0.0)
    rotation: tuple = (1.0, 0.0, 0.0, 0.0)


@dataclass
class Bone:
    keys: list = field(default_factory=list)


@dataclass
class Pill:
    c0: tuple = (0.0, 0.0, 0.0)
    c1: tuple = (0.0, 0.0, 0.0)
    r0: float = 0.0
    r1: float = 0.0
    rod: int = -1
    element: int = -1
    group: int = -1
    self_collide: bool = False

    def to_c(self) -> capi.Pill:
        return capi.Pill((C.c_double * 3)(*self.c0), (C.c_double * 3)(*self.c1), self.r0, self.r1,
                         self.rod, self.element, self.group, int(self.self_collide))


@dataclass
class KinematicPill:
    pill: Pill
    bone: int = -1


@dataclass
class PinMotion:
    rod: int = 0
    vertex: int = 0
    start: tuple = (0.0, 0.0, 0.0)
    target: tuple = (0.0, 0.0, 0.0)
    t0: float = 0.0
    t1: float = 0.0


@dataclass
class SoftPin:
    rod: int = 0
    vertex: int = 0
    target: tuple = (0.0, 0.0, 0.0)
    stiffness: float = INF


@dataclass
class Activation:
    rod: int = 0
    factor: float = 0.2
    t_start: float = 0.0
    t_end: float = 1.0
    first_element: int = 0
    last_element: int = -1


@dataclass
class Probe:  # scene.h:95-100 — per-step logging of one vertex (metrics.py ProbeWriter)
    name: str = ""
    rod: int = 0
    vertex: int = 0


@dataclass
class SkinSetup:  # scene.h:102-107 — surface mesh skinned to the rods' pills
    vertices: list = field(default_factory=list)   # (x, y, z) per vertex
    triangles: list = field(default_factory=list)  # (a, b, c) vertex ids
    max_influences: int = 8
    epsilon: float = 1e-4
    smooth_iterations: int = 0


@dataclass
class Scene:
    rods: list = field(default_factory=list)
    materials: list = field(default_factory=list)
    planes: list = field(default_factory=list)
    kinematic_pills: list = field(default_factory=list)
    bones: list = field(default_factory=list)
    bundles: list = field(default_factory=list)  # list of list[(rod, vertex)]
    pin_motions: list = field(default_factory=list)
    soft_pins: list = field(default_factory=list)
    activations: list = field(default_factory=list)
    settings: SolverSettings = field(default_factory=SolverSettings)
    probes: list = field(default_factory=list)  # caller-side (metrics), not sent to the solver
    skin: SkinSetup | None = None               # caller-side (the CLI binds it), not sent to the solver

    def vertex_count(self) -> int:
        return sum(r.rest.vertex_count() for r in self.rods)

    def element_count(self) -> int:
        return sum(r.rest.element_count() for r in self.rods)


# ---- rest pose (rod.h:88-93) -------------------------------------------------------------------

def _f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        out = out.reshape(shape)
    return out


def make_rest_pose(lib, centers, radii, scales=None) -> RodRestPose:
    """make_rest_pose(centers, radii, scales) — rod.h:88-90, computed by `lib`'s host code."""
    c = _f64(centers, (-1, 3))
    n = c.shape[0]
    r = _f64(np.atleast_1d(radii))
    s = None if scales is None else _f64(np.atleast_1d(scales))
    m = max(n - 1, 0)
    out = dict(scales=np.zeros(n), radii=np.zeros(n), lengths=np.zeros(m), initial_lengths=np.zeros(m),
               frames=np.zeros((m, 4)), darboux=np.zeros((max(m - 1, 0), 3)), tangent_dots=np.zeros(m),
               scale_grads=np.zeros(m), scale_laplacians=np.zeros(max(m - 1, 0)))
    po = capi.RestPoseOut(capi.ptr(out["scales"]), capi.ptr(out["radii"]), capi.ptr(out["lengths"]),
                          capi.ptr(out["initial_lengths"]), capi.ptr(out["frames"]), capi.ptr(out["darboux"]),
                          capi.ptr(out["tangent_dots"]), capi.ptr(out["scale_grads"]),
                          capi.ptr(out["scale_laplacians"]))
    check(lib, lib.vrod_make_rest_pose(n, capi.ptr(c), r.size, capi.ptr(r), 0 if s is None else s.size,
                                       capi.ptr(s), C.byref(po)))
    return RodRestPose(centers=c.copy(), **out)


def make_rest_state(rest: RodRestPose) -> RodState:
    """make_rest_state, rod.h:93 / rod.cpp:114-123."""
    n, m = rest.vertex_count(), rest.element_count()
    return RodState(centers=rest.centers.copy(), scales=rest.scales.copy(), frames=rest.frames.copy(),
                    center_vel=np.zeros((n, 3)), scale_vel=np.zeros(n), angular_vel=np.zeros((m, 3)))


def straight_rod(lib, origin, direction, length: float, elements: int, radius: float, material: int = 0) -> Rod:
    """scenarios.cpp:14-28 pattern: evenly spaced straight rod at rest."""
    d = np.asarray(direction, dtype=np.float64)
    d = d / math.sqrt(float(d @ d))
    o = np.asarray(origin, dtype=np.float64)
    centers = np.array([o + (length * v / elements) * d for v in range(elements + 1)])
    rest = make_rest_pose(lib, centers, [radius])
    return Rod(rest=rest, state=make_rest_state(rest), material=material)


# ---- marshalling into a vrod_scene* ------------------------------------------------------------

def settings_to_c(s: SolverSettings) -> capi.Settings:
    return capi.Settings(s.dt, s.iterations, s.substeps, s.beta, (C.c_double * 3)(*s.gravity),
                         s.dichotomous_iterations, s.shape_match_period, s.contact_stiffness,
                         s.velocity_damping, int(bool(s.deterministic)), int(s.scale_mode))


def _check_sizes(rod: Rod, r: int) -> None:
    """The array-size checks of RodRestPose::validate (rod.cpp:15-28) and Scene::validate
    (scene.cpp:71-80) that a pointer-based C-ABI cannot see, with the reference's messages."""
    rest, st = rod.rest, rod.state
    n = rest.vertex_count()
    m = int(np.asarray(rest.frames).reshape(-1, 4).shape[0])
    sizes = lambda a: int(np.asarray(a).shape[0]) if np.ndim(a) else 1  # noqa: E731
    if n < 2:
        raise InvalidArgument("rest pose: need at least 2 vertices")
    if m != n - 1:
        raise InvalidArgument("rest pose: frame count must be vertex count - 1")
    for a, what in ((rest.scales, "scales"), (rest.radii, "radii")):
        if sizes(a) != n:
            raise InvalidArgument(f"rest pose: {what} size mismatch")
    for a, what in ((rest.lengths, "lengths"), (rest.initial_lengths, "initial lengths"),
                    (rest.tangent_dots, "tangent dots"), (rest.scale_grads, "scale grads")):
        if sizes(a) != m:
            raise InvalidArgument(f"rest pose: {what} size mismatch")
    if sizes(rest.darboux) != max(0, m - 1):
        raise InvalidArgument("rest pose: darboux size mismatch")
    if sizes(rest.scale_laplacians) != max(0, m - 1):
        raise InvalidArgument("rest pose: scale laplacians size mismatch")
    if sizes(rod.pinned) != n:
        raise InvalidArgument(f"rod {r} pinned flags size")
    if sizes(st.centers) != n or sizes(st.scales) != n or sizes(st.center_vel) != n or sizes(st.scale_vel) != n:
        raise InvalidArgument(f"rod {r} state size")
    if sizes(st.frames) != m or sizes(st.angular_vel) != m:
        raise InvalidArgument(f"rod {r} frame count")
    if len(rod.bones):
        rows = rod.bone_weights
        if rows is None or len(rows) != n:
            raise InvalidArgument(f"rod {r} bone weights per vertex")
        if any(len(row) != len(rod.bones) for row in rows):
            raise InvalidArgument(f"rod {r} bone weight row size")


def _rod_desc(rod: Rod, keep: list) -> capi.RodDesc:
    def arr(a, shape=None):
        x = _f64(a, shape)
        keep.append(x)
        return capi.ptr(x)

    n = rod.rest.vertex_count()
    pinned = np.ascontiguousarray(np.asarray(rod.pinned, dtype=np.uint8))
    keep.append(pinned)
    d = capi.RodDesc()
    d.vertex_count = n
    d.material = rod.material
    d.collision_group = rod.collision_group
    d.self_collide = int(bool(rod.self_collide))
    r = rod.rest
    d.rest_centers, d.rest_scales, d.radii = arr(r.centers), arr(r.scales), arr(r.radii)
    d.lengths, d.initial_lengths, d.rest_frames = arr(r.lengths), arr(r.initial_lengths), arr(r.frames)
    d.darboux, d.tangent_dots = arr(r.darboux), arr(r.tangent_dots)
    d.scale_grads, d.scale_laplacians = arr(r.scale_grads), arr(r.scale_laplacians)
    s = rod.state
    d.centers, d.scales, d.frames = arr(s.centers), arr(s.scales), arr(s.frames)
    d.center_vel, d.scale_vel, d.angular_vel = arr(s.center_vel), arr(s.scale_vel), arr(s.angular_vel)
    d.pinned = capi.ptr(pinned, C.c_uint8)
    d.bone_count = len(rod.bones)
    if rod.bones:
        b = np.ascontiguousarray(np.asarray(rod.bones, dtype=np.int32))
        keep.append(b)
        d.bones = capi.ptr(b, C.c_int32)
        d.bone_weights = arr(rod.bone_weights)
    return d


def marshal_scene(lib, scene: Scene) -> C.c_void_p:
    """Build a vrod_scene* in `lib` (caller owns it: lib.vrod_scene_destroy)."""
    h = C.c_void_p()
    check(lib, lib.vrod_scene_create(C.byref(h)))
    try:
        st = settings_to_c(scene.settings)
        check(lib, lib.vrod_scene_set_settings(h, C.byref(st)))
        for m in scene.materials:
            cm = capi.Material(m.stretch_x, m.stretch_y, m.stretch_z, m.bend_x, m.bend_y, m.bend_z, m.volume,
                               m.density)
            check(lib, lib.vrod_scene_add_material(h, C.byref(cm)))
        for r, rod in enumerate(scene.rods):
            _check_sizes(rod, r)
            keep: list = []
            d = _rod_desc(rod, keep)
            check(lib, lib.vrod_scene_add_rod(h, C.byref(d)))
        for p in scene.planes:
            nrm = _f64(p.normal)
            check(lib, lib.vrod_scene_add_plane(h, capi.ptr(nrm), float(p.offset)))
        for b in scene.bones:
            k = len(b.keys)
            t = _f64([kf.t for kf in b.keys])
            pos = _f64([kf.position for kf in b.keys]).reshape(-1)
            rot = _f64([kf.rotation for kf in b.keys]).reshape(-1)
            check(lib, lib.vrod_scene_add_bone(h, k, capi.ptr(t), capi.ptr(pos), capi.ptr(rot)))
        for kp in scene.kinematic_pills:
            cp = kp.pill.to_c()
            check(lib, lib.vrod_scene_add_kinematic_pill(h, C.byref(cp), kp.bone))
        for members in scene.bundles:
            rods = np.ascontiguousarray([m[0] for m in members], dtype=np.int32)
            verts = np.ascontiguousarray([m[1] for m in members], dtype=np.int32)
            check(lib, lib.vrod_scene_add_bundle(h, len(members), capi.ptr(rods, C.c_int32),
                                                 capi.ptr(verts, C.c_int32)))
        for pm in scene.pin_motions:
            a, b = _f64(pm.start), _f64(pm.target)
            check(lib, lib.vrod_scene_add_pin_motion(h, pm.rod, pm.vertex, capi.ptr(a), capi.ptr(b), pm.t0, pm.t1))
        for sp in scene.soft_pins:
            t = _f64(sp.target)
            check(lib, lib.vrod_scene_add_soft_pin(h, sp.rod, sp.vertex, capi.ptr(t), sp.stiffness))
        for a in scene.activations:
            check(lib, lib.vrod_scene_add_activation(h, a.rod, a.factor, a.t_start, a.t_end, a.first_element,
                                                     a.last_element))
    except BaseException:
        lib.vrod_scene_destroy(h)
        raise
    return h


def validate(lib, scene: Scene) -> None:
    """Scene::validate (scene.cpp:63-157) through `lib`; raises InvalidArgument / OutOfRange."""
    h = marshal_scene(lib, scene)
    try:
        check(lib, lib.vrod_scene_validate(h))
    finally:
        lib.vrod_scene_destroy(h)
