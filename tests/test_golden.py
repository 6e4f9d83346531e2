"""Golden fixtures made from the reference itself (tests/golden/make_golden.py, oracle/_ref).

The CPU restatement must reproduce them bit for bit (this pins the oracle where /root/reference
and oracle/_ref are absent, e.g. on the GPU box); the GPU product must reproduce the exact
scenes bit for bit and the shape-matching scenes within tolerance.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_1906_05260_b200.handle import broad_phase, deepest_penetration, find_contacts, pill_project

from golden.make_golden import GOLDEN_SCENES, golden_pills, run_scene
from scenes import SCENES

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")
SHAPE_MATCHING = {"kitchen_sink", "mini_muscle"}


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(GOLDEN))


def check_scene(lib, golden, name, exact):
    out = run_scene(lib, SCENES, name, GOLDEN_SCENES[name])
    for k, v in out.items():
        ref = golden[k]
        if k.endswith("residuals"):  # GPU: per-CTA tree sums of the RMS numerators
            np.testing.assert_allclose(v, ref, rtol=1e-12 if exact else 1e-6, atol=0 if exact else 1e-12, err_msg=k)
        elif exact or k.endswith(("counters", "contacts_pill_a", "contacts_pill_b")):
            np.testing.assert_array_equal(v, ref, err_msg=k)
        else:  # shape-matching scenes: see test_gpu_parity.BUNDLE_SCENES. Velocities are
            # (x - x_prev) / h of last-ulp rotation differences, hence the relative part.
            np.testing.assert_allclose(v, ref, rtol=1e-4, atol=1e-4, err_msg=k)


@pytest.mark.parametrize("name", sorted(GOLDEN_SCENES))
def test_oracle_reproduces_reference_golden(oracle, golden, name):
    check_scene(oracle, golden, name, exact=True)


def check_collision(lib, golden):
    a, b, x, warm, field, keys, walpha = golden_pills()
    for key, val in zip(("pp/t", "pp/d", "pp/deg"), pill_project(lib, x, b)):
        np.testing.assert_array_equal(val, golden[key], err_msg=key)
    for key, val in zip(("dp/alpha", "dp/beta", "dp/d"), deepest_penetration(lib, a, b, 10, warm)):
        np.testing.assert_array_equal(val, golden[key], err_msg=key)
    pairs = broad_phase(lib, field)
    np.testing.assert_array_equal(pairs, golden["bp/pairs"])
    for k, v in find_contacts(lib, field, pairs, 10, keys, walpha).items():
        np.testing.assert_array_equal(v, golden[f"fc/{k}"], err_msg=k)


def test_oracle_collision_golden(oracle, golden):
    check_collision(oracle, golden)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLDEN_SCENES))
def test_gpu_reproduces_reference_golden(golden, name):
    import paper_1906_05260_b200 as pb
    check_scene(pb.library(), golden, name, exact=name not in SHAPE_MATCHING)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SHAPE_MATCHING))
def test_gpu_exact_shape_mode_reproduces_reference_golden(golden, name, monkeypatch):
    """The exact-order shape-matching path (VROD_SHAPE_EXACT=1) reproduces the reference's own
    output (oracle/_ref) bit for bit on the shape-matching golden scenes too."""
    import paper_1906_05260_b200 as pb
    monkeypatch.setenv("VROD_SHAPE_EXACT", "1")
    check_scene(pb.library(), golden, name, exact=True)


@pytest.mark.gpu
def test_gpu_collision_golden(golden):
    import paper_1906_05260_b200 as pb
    check_collision(pb.library(), golden)
