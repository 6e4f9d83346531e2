"""B200-native VIPER rod-solver substep (arXiv 1906.05260) behind the reference's core API.

    from paper_1906_05260_b200 import Solver, Scene, Rod, MaterialParams, make_rest_pose
    solver = Solver(scene)          # vrod::Solver(Scene)            solver.h:60
    report = solver.step()          # vrod::Solver::step()           solver.cpp:363-388

The compute path is libvrod_b200.so (hand-written sm_100a CUDA + host C++ behind the C-ABI
in include/vrod_capi.h). There is no CPU fallback: if the library is missing, importing the
solver raises.
"""
from __future__ import annotations

from . import capi, workloads
from ._lib import LIB_PATH, library
from .handle import Skin as _SkinHandle
from .handle import StepReport, SolverHandle
from .scene import (Activation, Bone, DeviceError, HalfPlane, InvalidArgument, KinematicPill, MaterialParams,
                    OutOfRange, Pill, PinMotion, RigidKeyframe, Rod, RodRestPose, RodState, Scene,
                    SimulationError, SoftPin, SolverSettings, VrodError, make_rest_state)
from . import scene as _scene


class Solver(SolverHandle):
    """vrod::Solver on the B200 (solver.h:54-115)."""

    def __init__(self, scene: Scene):
        super().__init__(library(), scene)


class BatchSolver(SolverHandle):
    """Independent scenes stepped together in one device world (BASELINE C5): every scene's
    results equal that scene alone; `scene_reports()` gives each scene's StepReport."""

    def __init__(self, scenes: list[Scene]):
        super().__init__(library(), None, _batch=list(scenes))


class Skin(_SkinHandle):
    """bind_skin / smooth_binding / deform_mesh (skinning.h) on the B200. Bind a mesh to a
    solver's rest pills with `Skin.for_solver(solver, vertices, triangles)`, then every frame
    `deform_solver(solver)` deforms it from the live state on the device."""

    def __init__(self, vertices, triangles, rest_pills, rest_transforms, max_influences: int = 8,
                 epsilon: float = 1e-4):
        super().__init__(library(), vertices, triangles, rest_pills, rest_transforms, max_influences, epsilon)

    @classmethod
    def for_solver(cls, solver: SolverHandle, vertices, triangles=None, max_influences: int = 8,
                   epsilon: float = 1e-4, smooth_iterations: int = 0) -> "Skin":
        """The CLI's binding flow (vrod_main.cpp:52-63)."""
        sk = cls(vertices, triangles, solver.rest_pills(), solver.rest_pill_transforms(), max_influences, epsilon)
        if smooth_iterations:
            sk.smooth(smooth_iterations)
        return sk


def make_rest_pose(centers, radii, scales=None) -> RodRestPose:
    """make_rest_pose (rod.h:88-90), computed by the product's host code."""
    return _scene.make_rest_pose(library(), centers, radii, scales)


def straight_rod(origin, direction, length, elements, radius, material=0) -> Rod:
    return _scene.straight_rod(library(), origin, direction, length, elements, radius, material)


def validate(scene: Scene) -> None:
    """Scene::validate (scene.cpp:63-157)."""
    _scene.validate(library(), scene)


__all__ = ["Solver", "BatchSolver", "Skin", "Scene", "Rod", "RodRestPose", "RodState", "MaterialParams", "SolverSettings", "HalfPlane",
           "Pill", "KinematicPill", "Bone", "RigidKeyframe", "PinMotion", "SoftPin", "Activation", "StepReport",
           "make_rest_pose", "make_rest_state", "straight_rod", "validate", "VrodError", "InvalidArgument",
           "OutOfRange", "SimulationError", "DeviceError", "library", "LIB_PATH", "capi", "workloads"]
