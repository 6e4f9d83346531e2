"""Synthetic workloads C1-C5 of BASELINE.json (concrete definitions: SURVEY.md §8(d)).

All generators are deterministic (numpy Generator seeded per config). They build plain
`Scene`s; the rest pose comes from `make_rest_pose` of the library handed in (the product or,
in tests, an oracle) — the same arrays then feed every backend.
"""
from __future__ import annotations

import math

import numpy as np

from .scene import (Activation, MaterialParams, PinMotion, Rod, RodRestPose, Scene, SolverSettings,
                    make_rest_pose, make_rest_state)


def _translated(rest: RodRestPose, offset) -> RodRestPose:
    """Rest pose of a translated copy. Every derived quantity of make_rest_pose depends on center
    differences only; for the axis-aligned templates used here those are bitwise unchanged."""
    r = rest.copy()
    r.centers = r.centers + np.asarray(offset, dtype=np.float64)
    return r


def _vertical_template(lib, n: int, element: float, radius: float) -> RodRestPose:
    centers = np.zeros((n, 3))
    centers[:, 2] = element * np.arange(n)
    return make_rest_pose(lib, centers, [radius])


def c1_single_rod(lib) -> Scene:
    """C1: one 100-vertex rod along +x, pinned at vertex 0, gravity, I=10."""
    n = 100
    centers = np.zeros((n, 3))
    centers[:, 0] = np.arange(n) / (n - 1)  # length 1.0
    rest = make_rest_pose(lib, centers, [0.02])
    rod = Rod(rest=rest, state=make_rest_state(rest))
    rod.pinned[0] = 1
    s = Scene(rods=[rod], materials=[MaterialParams()])
    s.settings = SolverSettings(iterations=10)
    return s


def _volume_dominant() -> MaterialParams:  # scenarios.cpp:32-39
    return MaterialParams(stretch_x=1e4, stretch_y=1e4, stretch_z=1e4, bend_x=1e3, bend_y=1e3, volume=1e8,
                          density=1000.0)


def c2_stretch_grid(lib, rods_per_side: int = 8, vertices: int = 256) -> Scene:
    """C2: 64 rods x 256 vertices along +z on an 8x8 grid (1 m pitch), both ends pinned and pulled
    apart to 2x over 1 s (scenario_stretch pattern, scenarios.cpp:71-88), collision group 0 for
    all (no pairs), volume-dominant material, g = 0, damping 0.1, dt = 1/240, I = 20."""
    element = 0.01
    L = element * (vertices - 1)
    tmpl = _vertical_template(lib, vertices, element, 0.01)
    s = Scene(materials=[_volume_dominant()])
    for i in range(rods_per_side):
        for j in range(rods_per_side):
            rest = _translated(tmpl, (float(i), float(j), 0.0))
            rod = Rod(rest=rest, state=make_rest_state(rest), collision_group=0)
            rod.pinned[0] = 1
            rod.pinned[-1] = 1
            r = len(s.rods)
            s.rods.append(rod)
            s.pin_motions.append(PinMotion(r, 0, tuple(rest.centers[0]), (float(i), float(j), -0.5 * L), 0.0, 1.0))
            s.pin_motions.append(PinMotion(r, vertices - 1, tuple(rest.centers[-1]), (float(i), float(j), 1.5 * L),
                                           0.0, 1.0))
    s.settings = SolverSettings(dt=1.0 / 240.0, iterations=20, substeps=1, gravity=(0.0, 0.0, 0.0),
                                velocity_damping=0.1)
    return s


def _hex_points(count: int, pitch: float) -> np.ndarray:
    """The `count` triangular-lattice points nearest the origin, ties broken by angle."""
    pts = []
    k = int(math.ceil(math.sqrt(count))) + 3
    for a in range(-k, k + 1):
        for b in range(-k, k + 1):
            x = pitch * (a + 0.5 * b)
            y = pitch * (b * math.sqrt(3.0) / 2.0)
            pts.append((round(x * x + y * y, 12), math.atan2(y, x) % (2 * math.pi), x, y))
    pts.sort()
    return np.array([(p[2], p[3]) for p in pts[:count]])


def c3_muscle_bundle(lib, muscles: int = 4, rods_per_muscle: int = 32, vertices: int = 30,
                     activate=(0, 2), gravity: bool = False) -> Scene:
    """C3: paper-scale ~26k-DOF synthetic muscle bundle: 4 muscles x 32 rods x 30
    vertices (element 0.01 m, r = 0.004 m); muscle axes at (+-d, +-d) with d set so the closest
    rods of adjacent muscles overlap by 0.02*2r (contact at t = 0); collision_group = muscle id;
    both rod ends pinned; per-muscle per-vertex shape-matching groups (scenarios.cpp:219-221);
    band material (scenarios.cpp:198-202); damping 0.02; activation 0.2 over [0, 0.5] s on
    muscles 0 and 2; default settings (dt 1/60, substeps 1, I = 20).

    Zero gravity, like the reference's stretch / activation / bergou scenarios: with gravity on,
    these thin (4 mm) rods pinned at both ends are far softer than 20 averaged-Jacobi
    iterations per 1/60 s frame can resolve and sag into a tangle (measured on the oracle:
    vertices 0.3 m below the lower pin, elements stretched 4.6x), which inflates the broad-phase
    cell and turns the workload into a transient instead of a steady frame loop.
    `gravity=True` is SURVEY §8(d)'s literal C3 (g on): see c3_muscle_bundle_gravity."""
    r = 0.004
    element = 0.01
    pitch = 0.0085
    lattice = _hex_points(rods_per_muscle, pitch)
    target = 2 * r - 0.02 * 2 * r  # center distance of the closest inter-muscle pair

    def min_sep(d):
        a = lattice + np.array([d, 0.0])
        b = lattice + np.array([-d, 0.0])
        dx = np.linalg.norm(a[:, None, :] - b[None, :, :], axis=-1).min()
        a = lattice + np.array([0.0, d])
        b = lattice + np.array([0.0, -d])
        dy = np.linalg.norm(a[:, None, :] - b[None, :, :], axis=-1).min()
        return min(dx, dy)

    lo, hi = 0.0, 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if min_sep(mid) < target:
            lo = mid
        else:
            hi = mid
    d = hi
    mat = MaterialParams(stretch_x=1e6, stretch_y=1e6, stretch_z=1e6, bend_x=1e5, bend_y=1e5, volume=1e8,
                         density=1000.0)
    tmpl = _vertical_template(lib, vertices, element, r)
    s = Scene(materials=[mat])
    axes = [(d, d), (-d, d), (-d, -d), (d, -d)][:muscles]
    for mu, (ax, ay) in enumerate(axes):
        first = len(s.rods)
        for (px, py) in lattice:
            rest = _translated(tmpl, (ax + px, ay + py, 0.0))
            rod = Rod(rest=rest, state=make_rest_state(rest), collision_group=mu)
            rod.pinned[0] = 1
            rod.pinned[-1] = 1
            s.rods.append(rod)
        for v in range(vertices):
            s.bundles.append([(first + k, v) for k in range(rods_per_muscle)])
        if mu in activate:
            for k in range(rods_per_muscle):
                s.activations.append(Activation(rod=first + k, factor=0.2, t_start=0.0, t_end=0.5))
    s.settings = SolverSettings(velocity_damping=0.02, gravity=(0.0, 0.0, -9.81) if gravity else (0.0, 0.0, 0.0))
    return s


def c3_muscle_bundle_gravity(lib) -> Scene:
    """C3 exactly as SURVEY §8(d) states it, gravity on (g = -9.81 m/s^2 along z). The muscles
    sag between their pinned tendons and press into each other: the inter-muscle contact count
    grows from 340 at t = 0 to ~1,200 after 10 frames and ~3,000 after 25 (oracle), against ~12
    in the zero-gravity steady loop — the contact-loaded variant of the headline."""
    return c3_muscle_bundle(lib, gravity=True)


def c5_scene(lib, index: int) -> Scene:
    """Scene `index` of C5, the batch of independent C3 scenes: activation on
    muscle (index mod 4) and an initial lateral velocity of amplitude 0.5 * (1 + (index mod 7)/7)
    m/s (sine profile along each rod, zero at the pinned ends, per-rod direction from a seeded
    generator). Scenes with equal (index mod 4, index mod 7) are identical: 28 distinct scenes."""
    s = c3_muscle_bundle(lib, activate=(index % 4,))
    amp = 0.5 * (1.0 + (index % 7) / 7.0)
    rng = np.random.default_rng(1000 + (index % 28))
    for rod in s.rods:
        phi = rng.uniform(0.0, 2.0 * np.pi)
        n = len(rod.state.scales)
        prof = np.sin(np.pi * np.arange(n) / (n - 1))
        rod.state.center_vel[:, 0] = amp * np.cos(phi) * prof
        rod.state.center_vel[:, 1] = amp * np.sin(phi) * prof
    return s


def c5_batch(lib, count: int, first: int = 0) -> list[Scene]:
    """Scenes first .. first+count-1 of C5 (the 28 distinct ones are built once and shared)."""
    distinct: dict[int, Scene] = {}
    out = []
    for i in range(first, first + count):
        key = i % 28
        if key not in distinct:
            distinct[key] = c5_scene(lib, i)
        out.append(distinct[key])
    return out


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [rank*n/world, (rank+1)*n/world) of n independent scenes."""
    return rank * n // world, (rank + 1) * n // world


def c4_rod_forest(lib, nx: int = 125, ny: int = 250, vertices: int = 32, seed: int = 1234,
                  pitch: float = 0.100) -> Scene:
    """C4: 1M-vertex synthetic rod forest: nx x ny vertical rods x 32 vertices
    (element 0.05 m, r = 0.05 m) on a lattice of pitch 2r = 0.100 m, so every rod starts in
    exact tangential contact with its 4 neighbours and the random sway keeps millions of pill
    contacts live; bottom vertex pinned, gravity, no groups, bench material
    (scenarios.cpp:246-251), dt = 1/240, I = 10, initial lateral velocity U[-0.5, 0.5] m/s per
    rod scaled by height fraction.

    The survey proposed a 0.098 m pitch (2% initial interpenetration). That start explodes in
    the reference algorithm itself (oracle, 8x8 rods: element lengths 67 m after 4 steps, scales
    driven to the 1e-4 floor; also with 4 substeps), so the forest starts touching instead."""
    element, r = 0.05, 0.05
    tmpl = _vertical_template(lib, vertices, element, r)
    rng = np.random.default_rng(seed)
    vel = rng.uniform(-0.5, 0.5, size=(nx * ny, 2))
    frac = np.arange(vertices) / (vertices - 1)
    mat = MaterialParams(stretch_x=1e6, stretch_y=1e6, stretch_z=1e6, bend_x=1e4, bend_y=1e4, volume=1e7,
                         density=100.0)
    s = Scene(materials=[mat])
    for i in range(nx):
        for j in range(ny):
            rest = _translated(tmpl, (pitch * i, pitch * j, 0.0))
            st = make_rest_state(rest)
            u = vel[i * ny + j]
            st.center_vel[:, 0] = u[0] * frac
            st.center_vel[:, 1] = u[1] * frac
            rod = Rod(rest=rest, state=st)
            rod.pinned[0] = 1
            s.rods.append(rod)
    s.settings = SolverSettings(dt=1.0 / 240.0, iterations=10, substeps=1)
    return s


CONFIGS = {
    "C1": c1_single_rod,
    "C2": c2_stretch_grid,
    "C3": c3_muscle_bundle,
    "C3g": c3_muscle_bundle_gravity,
    "C4": c4_rod_forest,
}


def algorithmic_bytes(V: int, E: int, I: int, coupled: bool, P: int, Nc: int) -> int:
    """B_substep of SURVEY §8(d) / BASELINE.md §4 — the roofline numerator per substep."""
    return int(160 * V + 176 * E + (64 * I * (V + E) if coupled else 0) + 24 * P + 24 * Nc * (1 + I))


# ---- skinning ---------------------------------------------------------

def sleeve_mesh(rest_pills: np.ndarray, rings: int, segments: int, margin: float = 0.3, inner: int = 0, seed: int = 7):
    """A closed-sided tube mesh (quad grid split into triangles) wrapped around the rest pills'
    bounding box along its longest axis, `margin` beyond the bounding radius, plus `inner`
    vertices placed inside random pills (they clamp to epsilon, skinning.cpp:79-81). Returns
    (vertices (n, 3), triangles (t, 3) int32)."""
    c0, c1 = np.asarray(rest_pills["c0"]), np.asarray(rest_pills["c1"])
    pts = np.concatenate([c0, c1])
    lo, hi = pts.min(0), pts.max(0)
    axis = int(np.argmax(hi - lo))
    a, b = [k for k in range(3) if k != axis]
    center = 0.5 * (lo + hi)
    radius = 0.5 * float(np.hypot(hi[a] - lo[a], hi[b] - lo[b])) + margin * max(float((hi - lo).max()), 1e-3) * 0.1 + 1e-3
    t = np.linspace(lo[axis], hi[axis], rings)
    phi = np.linspace(0.0, 2 * np.pi, segments, endpoint=False)
    V = np.zeros((rings * segments, 3))
    V[:, axis] = np.repeat(t, segments)
    V[:, a] = center[a] + radius * np.tile(np.cos(phi), rings)
    V[:, b] = center[b] + radius * np.tile(np.sin(phi), rings)
    tris = []
    for r in range(rings - 1):
        for s in range(segments):
            i0, i1 = r * segments + s, r * segments + (s + 1) % segments
            j0, j1 = i0 + segments, i1 + segments
            tris.append((i0, i1, j1))
            tris.append((i0, j1, j0))
    if inner:
        rng = np.random.default_rng(seed)
        k = rng.integers(0, len(c0), inner)
        u = rng.uniform(0.2, 0.8, inner)[:, None]
        V = np.concatenate([V, (1 - u) * c0[k] + u * c1[k]])
    return V, np.asarray(tris, dtype=np.int32).reshape(-1, 3)
