"""GPU parity: the CUDA product (through the C-ABI) against the CPU oracle on identical inputs.

Tolerances: collision primitives and contact sets are bit-exact (the collision
kernels are compiled --fmad=false and keep the reference's operation order); positions, scales
and orientations agree to a relative 1e-10 after one step and to the per-scene free-running
bound below after K steps (the sweep kernels use FMA contraction, so last-ulp differences
propagate through the stiff Jacobi iterations).
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1906_05260_b200 as pb
from paper_1906_05260_b200.handle import SolverHandle, broad_phase, deepest_penetration, find_contacts, pill_project

from scenes import SCENES
from test_oracle_pinning import random_pills

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    return pb.library()


def rel_err(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def quat_err(a, b):
    if not a.size:
        return 0.0
    return float(np.max(np.minimum(np.linalg.norm(a - b, axis=1), np.linalg.norm(a + b, axis=1))))


def compare_states(sa, sb):
    return dict(centers=rel_err(sa["centers"], sb["centers"]), scales=rel_err(sa["scales"], sb["scales"]),
                frames=quat_err(sa["frames"], sb["frames"]))


ONE_STEP_TOL = 1e-10
FREE_TOL = {"C1": 1e-8, "floor": 1e-6, "stretch": 1e-8, "activation": 1e-8, "bergou": 1e-8, "bergou_baseline": 1e-8,
            "band": 1e-6, "pile": 1e-6, "crossing": 1e-6, "kitchen_sink": 1e-6, "mini_muscle": 1e-6,
            "mini_forest": 1e-6}
FREE_STEPS = {"C1": 60, "pile": 3, "mini_forest": 5, "mini_muscle": 5}


@pytest.mark.parametrize("name", sorted(SCENES))
def test_one_step_matches_oracle(gpu, oracle, name):
    scene = SCENES[name](oracle)
    g, o = SolverHandle(gpu, scene), SolverHandle(oracle, scene)
    rg, ro = g.step(), o.step()
    e = compare_states(g.state(), o.state())
    assert max(e.values()) <= ONE_STEP_TOL, e
    assert (rg.contact_count, rg.broad_pairs) == (ro.contact_count, ro.broad_pairs)
    assert rg.skipped_singular == ro.skipped_singular
    np.testing.assert_allclose(rg.residuals, ro.residuals, rtol=1e-6, atol=1e-12)
    assert rg.max_penetration == pytest.approx(ro.max_penetration, rel=1e-6, abs=1e-12)
    cg, co = g.contacts(), o.contacts()
    for k in cg:  # contact set (pill ids) and frozen alpha/beta: bit-exact
        np.testing.assert_array_equal(cg[k], co[k], err_msg=k)


@pytest.mark.parametrize("name", sorted(SCENES))
def test_free_running_matches_oracle(gpu, oracle, name):
    scene = SCENES[name](oracle)
    g, o = SolverHandle(gpu, scene), SolverHandle(oracle, scene)
    steps = FREE_STEPS.get(name, 10)
    for _ in range(steps):
        rg, ro = g.step(), o.step()
        assert rg.contact_count == ro.contact_count
    e = compare_states(g.state(), o.state())
    assert max(e.values()) <= FREE_TOL[name], e
    assert g.time() == o.time() and g.step_index() == o.step_index()


def test_identical_input_contacts_bit_exact(gpu, oracle):
    """Same pill array in -> same broad pairs, same contacts, same alpha/beta bits out."""
    rng = np.random.default_rng(2024)
    pills = random_pills(rng, 2000, spread=3.0, rmax=0.25)
    pg, po = broad_phase(gpu, pills), broad_phase(oracle, pills)
    np.testing.assert_array_equal(pg, po)
    keys = rng.integers(0, 2**40, 100).astype(np.uint64)
    wa = rng.uniform(0, 1, 100)
    cg = find_contacts(gpu, pills, pg, 10, keys, wa)
    co = find_contacts(oracle, pills, po, 10, keys, wa)
    for k in cg:
        np.testing.assert_array_equal(cg[k], co[k], err_msg=k)
    assert len(cg["pill_a"]) > 100


def test_collision_primitives_bit_exact(gpu, oracle):
    rng = np.random.default_rng(5)
    a, b = random_pills(rng, 3000), random_pills(rng, 3000)
    a["c1"][:50] = a["c0"][:50]
    a["r0"][50:100] = 2.0
    b[100:120] = a[100:120]
    x = rng.uniform(-1.5, 1.5, (3000, 3))
    for u, v in zip(pill_project(gpu, x, b), pill_project(oracle, x, b)):
        np.testing.assert_array_equal(u, v)
    warm = rng.uniform(-0.2, 1.2, 3000)
    for it in (1, 10, 25):
        for u, v in zip(deepest_penetration(gpu, a, b, it, warm), deepest_penetration(oracle, a, b, it, warm)):
            np.testing.assert_array_equal(u, v)


def test_free_fall_predict_finalize_bitwise(gpu, oracle):
    """Predict + finalize kernels are exact: a rod with no elastic coupling (all stiffness 0
    except density) falls exactly like the oracle, bit for bit."""
    from paper_1906_05260_b200.scene import MaterialParams, Scene, SolverSettings, straight_rod
    s = Scene(materials=[MaterialParams(stretch_x=0, stretch_y=0, stretch_z=0, bend_x=0, bend_y=0, volume=0)])
    s.rods.append(straight_rod(oracle, (0, 0, 0), (0, 0, 1), 1.0, 3, 0.05))
    s.rods[0].state.center_vel[:] = [0.3, -0.2, 1.0]
    s.rods[0].state.angular_vel[:] = [0.5, 0.1, -0.7]
    s.settings = SolverSettings(substeps=2, velocity_damping=0.1)
    g, o = SolverHandle(gpu, s), SolverHandle(oracle, s)
    for _ in range(30):
        g.step()
        o.step()
    sg, so = g.state(), o.state()
    for k in sg:
        np.testing.assert_array_equal(sg[k], so[k], err_msg=k)


def test_deterministic_run_to_run(gpu, oracle):
    scene = SCENES["kitchen_sink"](oracle)
    a, b = SolverHandle(gpu, scene), SolverHandle(gpu, scene)
    for _ in range(5):
        ra, rb = a.step(), b.step()
        assert ra.max_penetration == rb.max_penetration and ra.contact_count == rb.contact_count
    sa, sb = a.state(), b.state()
    for k in sa:
        np.testing.assert_array_equal(sa[k], sb[k])


def test_errors_round_trip(gpu, oracle):
    from paper_1906_05260_b200.scene import InvalidArgument, SimulationError
    scene = SCENES["C1"](oracle)
    scene.rods[0].state.center_vel[3, 0] = np.nan
    with pytest.raises(SimulationError, match="non-finite prediction in rod 0"):
        SolverHandle(gpu, scene).step()
    scene = SCENES["C1"](oracle)
    h = SolverHandle(gpu, scene)
    fd = np.zeros((100, 3))
    fd[5, 1] = np.inf
    h.set_loads(force_density=fd)
    with pytest.raises(InvalidArgument, match="external force must be finite"):
        h.step()


def test_loads_and_queries_match(gpu, oracle):
    scene = SCENES["kitchen_sink"](oracle)
    g, o = SolverHandle(gpu, scene), SolverHandle(oracle, scene)
    rng = np.random.default_rng(1)
    V, E = g.total_vertices, g.total_elements
    loads = dict(force_density=rng.normal(0, 50, (V, 3)), torque=rng.normal(0, 1e-3, (E, 3)),
                 scale_load=rng.normal(0, 1e-3, E))
    g.set_loads(**loads)
    o.set_loads(**loads)
    for _ in range(3):
        g.step()
        o.step()
    e = compare_states(g.state(), o.state())
    assert max(e.values()) <= 1e-8, e
    assert g.kinetic_energy() == pytest.approx(o.kinetic_energy(), rel=1e-8)
    assert g.total_volume() == pytest.approx(o.total_volume(), rel=1e-10)
    assert g.total_rest_volume() == o.total_rest_volume()
    np.testing.assert_allclose(g.rest()["lengths"], o.rest()["lengths"], rtol=0, atol=0)
    np.testing.assert_allclose(g.inverse_weights()["inv_theta"], o.inverse_weights()["inv_theta"], rtol=1e-10)


def test_probe_convergence_matches(gpu, oracle):
    scene = SCENES["stretch"](oracle)
    lg = SolverHandle(gpu, scene).probe_convergence(25)
    lo = SolverHandle(oracle, scene).probe_convergence(25)
    np.testing.assert_allclose(lg, lo, rtol=1e-6, atol=1e-14)
