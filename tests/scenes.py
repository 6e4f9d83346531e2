"""Small scenes that exercise every branch of the substep, for parity tests.

Patterns follow the reference's built-in scenarios (proj/core/src/scenarios.cpp) and the
fixtures of its unit tests (proj/tests/test_util.h), restated with the Python scene API.
Each builder takes the library whose make_rest_pose computes rest poses.
"""
from __future__ import annotations

import math

import numpy as np

from paper_1906_05260_b200 import workloads
from paper_1906_05260_b200.scene import (Activation, Bone, HalfPlane, KinematicPill, MaterialParams, Pill,
                                         PinMotion, RigidKeyframe, Rod, Scene, SoftPin, SolverSettings,
                                         make_rest_pose, make_rest_state, straight_rod)


def volume_dominant() -> MaterialParams:  # scenarios.cpp:32-39
    return MaterialParams(volume=1e8)


def curved_rod(lib, n: int = 6) -> Rod:  # test_util.h:52-66
    i = np.arange(n)
    centers = np.stack([0.3 * np.sin(0.9 * i), 0.2 * np.cos(1.3 * i), 0.45 * i], axis=1)
    radii = 0.04 + 0.015 * ((i * 7) % 3)
    scales = 0.8 + 0.1 * (i % 4)
    rest = make_rest_pose(lib, centers, radii, scales)
    return Rod(rest=rest, state=make_rest_state(rest))


def floor(lib) -> Scene:  # scenario_floor, scenarios.cpp:129-140
    s = Scene(materials=[MaterialParams()], planes=[HalfPlane((0.0, 0.0, 1.0), 0.0)])
    s.rods.append(straight_rod(lib, (-0.5, 0.0, 0.2), (1, 0, 0), 1.0, 20, 0.05))
    s.settings = SolverSettings(velocity_damping=0.1, substeps=4)
    return s


def stretch(lib) -> Scene:  # scenario_stretch, scenarios.cpp:71-88
    s = Scene(materials=[volume_dominant()])
    rod = straight_rod(lib, (0, 0, 0), (0, 0, 1), 1.0, 20, 0.05)
    rod.pinned[0] = rod.pinned[-1] = 1
    s.rods.append(rod)
    s.pin_motions += [PinMotion(0, 0, (0, 0, 0), (0, 0, -0.5), 0.0, 1.0),
                      PinMotion(0, 20, (0, 0, 1), (0, 0, 1.5), 0.0, 1.0)]
    s.settings = SolverSettings(gravity=(0.0, 0.0, 0.0), velocity_damping=0.1, substeps=4)
    return s


def activation(lib) -> Scene:  # scenario_activation, scenarios.cpp:142-160
    s = Scene(materials=[volume_dominant()])
    s.rods.append(straight_rod(lib, (0, 0, 0), (0, 0, 1), 1.0, 20, 0.05))
    s.activations.append(Activation(rod=0, factor=0.2, t_start=0.0, t_end=0.5))
    s.settings = SolverSettings(gravity=(0.0, 0.0, 0.0), velocity_damping=0.1, substeps=4)
    return s


def bergou(lib, classic: bool) -> Scene:  # scenario_bergou(_baseline), scenarios.cpp:164-192
    s = Scene(materials=[volume_dominant()])
    rod = straight_rod(lib, (0, 0, 0), (0, 0, 1), 1.0, 20, 0.05)
    rod.pinned[0] = rod.pinned[-1] = 1
    rod.state.scales[0] = rod.state.scales[1] = 1.2
    s.rods.append(rod)
    s.settings = SolverSettings(gravity=(0.0, 0.0, 0.0), substeps=4, scale_mode=1 if classic else 0)
    return s


def band(lib) -> Scene:  # scenario_band (skin omitted: out of scope), scenarios.cpp:194-232
    mat = MaterialParams(stretch_x=1e6, stretch_y=1e6, stretch_z=1e6, bend_x=1e5, bend_y=1e5, volume=1e8)
    s = Scene(materials=[mat])
    elements = 12
    for i in range(3):
        ang = 2.0 * math.pi * i / 3.0 + math.pi / 2.0
        rod = straight_rod(lib, (0.05 * math.cos(ang), 0.05 * math.sin(ang), 0.0), (0, 0, -1), 0.6, elements, 0.03)
        rod.pinned[0] = 1
        rod.collision_group = 1
        rod.state.center_vel[elements // 2:, 0] = 0.5
        s.rods.append(rod)
    for v in range(elements + 1):
        s.bundles.append([(0, v), (1, v), (2, v)])
    s.settings = SolverSettings(velocity_damping=0.02, substeps=4)
    return s


def pile(lib, pallets: int = 1) -> Scene:  # scenario_bench, scenarios.cpp:234-282
    mat = MaterialParams(stretch_x=1e6, stretch_y=1e6, stretch_z=1e6, bend_x=1e4, bend_y=1e4, volume=1e7,
                         density=100.0)
    s = Scene(materials=[mat], planes=[HalfPlane((0.0, 0.0, 1.0), 0.0)])
    radius, length, spacing, elements = 0.05, 1.8, 0.16, 10
    for p in range(pallets):
        ox = 3.0 * p
        for col in range(15):
            s.rods.append(straight_rod(lib, (ox - 0.5 * length, spacing * (col - 7.0), radius), (1, 0, 0), length,
                                       elements, radius))
        for col in range(12):
            s.rods.append(straight_rod(lib, (ox + spacing * (col - 5.5), -0.5 * length, 3.0 * radius), (0, 1, 0),
                                       length, elements, radius))
    s.settings = SolverSettings(velocity_damping=0.01, substeps=4, iterations=10)
    return s


def crossing(lib) -> Scene:  # test_solver.cpp:341-379 (two crossing rods, plane, contacts)
    s = Scene(materials=[MaterialParams()], planes=[HalfPlane((0.0, 0.0, 1.0), -0.2)])
    t = np.arange(5) / 4.0
    b_c = np.stack([-0.5 + t, 0.02 * t, np.zeros(5)], axis=1)
    a_c = np.stack([np.full(5, 0.01), -0.5 + t, np.full(5, 0.12)], axis=1)
    for c in (a_c, b_c):
        rest = make_rest_pose(lib, c, [0.05])
        s.rods.append(Rod(rest=rest, state=make_rest_state(rest)))
    s.settings = SolverSettings(deterministic=True)
    return s


def kitchen_sink(lib) -> Scene:
    """Soft pins, a bone-posed and a static kinematic pill, self-collision, two materials,
    perturbed curved rods with velocities, partial activation, damping, 2 substeps."""
    s = Scene(materials=[MaterialParams(), MaterialParams(stretch_x=0.0, stretch_y=2e4, bend_x=0.0, volume=0.0,
                                                          density=500.0)])
    rng = np.random.default_rng(7)
    for k in range(3):
        rod = curved_rod(lib, 7)
        rod.rest.centers = rod.rest.centers + np.array([0.05 * k, 0.0, 0.0])
        rod.state = make_rest_state(rod.rest)
        rod.state.centers += rng.uniform(-0.02, 0.02, rod.state.centers.shape)
        rod.state.center_vel += rng.uniform(-0.3, 0.3, rod.state.center_vel.shape)
        rod.state.scale_vel += rng.uniform(-0.2, 0.2, rod.state.scale_vel.shape)
        rod.state.angular_vel += rng.uniform(-1.0, 1.0, rod.state.angular_vel.shape)
        rod.material = k % 2
        s.rods.append(rod)
    # a coiled self-colliding rod
    th = np.linspace(0, 4 * math.pi, 25)
    coil = np.stack([0.12 * np.cos(th) + 1.0, 0.12 * np.sin(th), 0.02 * th], axis=1)
    rest = make_rest_pose(lib, coil, [0.035])
    rod = Rod(rest=rest, state=make_rest_state(rest), self_collide=True)
    rod.pinned[0] = 1
    s.rods.append(rod)
    s.soft_pins.append(SoftPin(0, 3, (0.0, 0.1, 1.2), 50.0))
    s.soft_pins.append(SoftPin(1, 0, (0.05, 0.2, 0.0), math.inf))
    s.bones.append(Bone([RigidKeyframe(0.0, (0.2, 0.0, 0.3), (1.0, 0.0, 0.0, 0.0)),
                         RigidKeyframe(0.2, (0.0, 0.1, 0.6), (math.cos(0.4), 0.0, math.sin(0.4), 0.0))]))
    s.kinematic_pills.append(KinematicPill(Pill((0.0, -0.3, 0.0), (0.0, 0.3, 0.0), 0.06, 0.08), bone=0))
    s.kinematic_pills.append(KinematicPill(Pill((1.0, 0.0, 0.1), (1.0, 0.0, 0.5), 0.05, 0.05)))
    s.activations.append(Activation(rod=2, factor=0.3, t_start=0.0, t_end=0.1, first_element=1, last_element=3))
    s.planes.append(HalfPlane((0.0, 0.0, 1.0), -0.05))
    s.settings = SolverSettings(substeps=2, iterations=12, velocity_damping=0.05, shape_match_period=3)
    s.bundles.append([(0, 2), (1, 2), (2, 2)])
    s.bundles.append([(0, 5), (1, 6), (2, 6)])
    return s


def _axis_quat(axis, angle):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    return (math.cos(0.5 * angle), *(math.sin(0.5 * angle) * a))


def lbs_rig(lib) -> Scene:
    """Bone-rigged rods: the linear-blend warm start `warm_start_lbs`
    (solver.cpp:75-100) moves every unpinned vertex by its bones' slerped relative transform
    between t_prev and t_new (Bone::position_at / rotation_at, scene.cpp:22-48) before the sweeps.
    Two keyframed bones with several spans each (the slerp and the linear position blend are both
    exercised); a two-bone rod with weights blending linearly from root to tip, a one-bone rod, a
    three-weight rod crossing the others (contacts), an unrigged rod, a bone-posed kinematic pill,
    gravity, two substeps."""
    s = Scene(materials=[MaterialParams(stretch_x=1e5, stretch_y=1e5, stretch_z=1e5, bend_x=1e4, bend_y=1e4,
                                        volume=1e7)])
    s.bones.append(Bone([RigidKeyframe(0.0, (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0)),
                         RigidKeyframe(0.08, (0.02, 0.0, 0.01), _axis_quat((0, 0, 1), 0.15)),
                         RigidKeyframe(0.2, (0.01, 0.03, -0.01), _axis_quat((1, 1, 0), 0.2)),
                         RigidKeyframe(0.5, (-0.02, 0.01, 0.0), _axis_quat((0, 1, 1), -0.15))]))
    s.bones.append(Bone([RigidKeyframe(0.02, (0.0, 0.0, 0.6), (1.0, 0.0, 0.0, 0.0)),
                         RigidKeyframe(0.15, (0.0, -0.03, 0.63), _axis_quat((1, 0, 0), 0.2)),
                         RigidKeyframe(0.4, (0.03, 0.0, 0.62), _axis_quat((0.3, -1, 0.2), 0.3))]))
    n = 13
    # two bones, weights root -> tip
    rod = straight_rod(lib, (0.0, 0.0, 0.0), (0, 0, 1), 0.6, n - 1, 0.03)
    w1 = np.arange(n) / (n - 1)
    rod.bones = [0, 1]
    rod.bone_weights = np.stack([1.0 - w1, w1], axis=1)
    rod.pinned[0] = 1
    s.rods.append(rod)
    # one bone
    rod = straight_rod(lib, (0.07, 0.0, 0.0), (0, 0, 1), 0.6, n - 1, 0.03)
    rod.bones = [1]
    rod.bone_weights = np.ones((n, 1))
    s.rods.append(rod)
    # three weights (bone 0 twice: duplicate bone entries are allowed), crossing the others
    rod = straight_rod(lib, (-0.3, 0.035, 0.3), (1, 0, 0), 0.6, n - 1, 0.025)
    u = np.arange(n) / (n - 1)
    rod.bones = [0, 1, 0]
    w0, w1 = 0.5 * (1.0 - u), 0.25 + 0.5 * u * (1.0 - u)
    rod.bone_weights = np.stack([w0, w1, 1.0 - w0 - w1], axis=1)
    s.rods.append(rod)
    # unrigged
    s.rods.append(straight_rod(lib, (0.035, -0.3, 0.45), (0, 1, 0), 0.6, n - 1, 0.025))
    s.kinematic_pills.append(KinematicPill(Pill((-0.05, 0.0, 0.2), (0.05, 0.0, 0.2), 0.03, 0.03), bone=0))
    s.settings = SolverSettings(substeps=2, iterations=10, velocity_damping=0.02)
    return s


def mini_muscle(lib) -> Scene:
    """C3 pattern at 1/8 scale: 4 muscles x 8 rods x 10 vertices."""
    return workloads.c3_muscle_bundle(lib, rods_per_muscle=8, vertices=10)


def mini_forest(lib) -> Scene:
    """C4 pattern at small scale: 6 x 5 rods x 12 vertices."""
    return workloads.c4_rod_forest(lib, nx=6, ny=5, vertices=12)


SCENES = {
    "floor": floor,
    "stretch": stretch,
    "activation": activation,
    "bergou": lambda lib: bergou(lib, False),
    "bergou_baseline": lambda lib: bergou(lib, True),
    "band": band,
    "pile": pile,
    "crossing": crossing,
    "kitchen_sink": kitchen_sink,
    "lbs_rig": lbs_rig,
    "mini_muscle": mini_muscle,
    "mini_forest": mini_forest,
    "C1": workloads.c1_single_rod,
}


def pile_noplane(lib) -> Scene:
    s = pile(lib)
    s.planes.clear()
    return s


def pile_nogravity(lib) -> Scene:
    s = pile(lib)
    s.settings.gravity = (0.0, 0.0, 0.0)
    return s


def pile_bottom_only(lib) -> Scene:
    s = pile(lib)
    s.rods = s.rods[:15]
    return s


DEBUG_SCENES = {"pile_noplane": pile_noplane, "pile_nogravity": pile_nogravity, "pile_bottom_only": pile_bottom_only}
