"""Pin the CPU restatement oracle (oracle/vrod_oracle.cpp) before trusting it.

1. The reference's own hot-path unit tests (proj/tests/test_*.cpp) run against the reference
   sources compiled with the Eigen/doctest shims (oracle/_ref): everything passes except the
   seven cases documented in DESIGN.md §2 as reference-test defects.
2. The restatement equals that compiled reference BIT FOR BIT, through the same C-ABI, on
   scenes covering every substep branch and on the fine-grained collision functions.
3. The committed golden vectors (tests/golden, made from oracle/_ref by make_golden.py) pin it
   where /root/reference is absent (the GPU box).
"""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from paper_1906_05260_b200 import capi
from paper_1906_05260_b200.handle import SolverHandle, broad_phase, deepest_penetration, find_contacts, pill_project

from conftest import ROOT
from scenes import SCENES

KNOWN_REFERENCE_TEST_DEFECTS = {
    # code (rod.cpp:38-41) deliberately keeps tangent_dots fixed; the test expects them scaled
    "activation shortens strain lengths and refreshes derived data",
    # scene.cpp:85-89 checks the weight-row count before the bone index
    "bone skinning weights on rods are checked",
    # test_solver.cpp never compiled upstream (RestPose, unqualified helpers); these five
    # expectations do not hold for the shipped code (ulp-level constraint noise, no buckling
    # without a perturbation, slow compliant convergence, 90 steps not at equilibrium)
    "free fall reproduces the symplectic Euler recurrence exactly",
    "pinned vertices never move under gravity",
    "a scene at rest with zero gravity does not drift at all",
    "classic scale mode sets scales from the element length ratio",
    "probe_convergence logs per-sweep residuals that decrease",
}


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj"), reason="needs /root/reference")
def test_reference_unit_suite_runs_against_shimmed_reference():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/vrod_ref_tests"], check=True,
                   stdout=subprocess.DEVNULL)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "vrod_ref_tests")], capture_output=True, text=True)
    failed = set()
    for line in out.stderr.splitlines():
        if "FAILED in \"" in line:
            failed.add(line.split("FAILED in \"", 1)[1].split("\"", 1)[0])
    assert failed == KNOWN_REFERENCE_TEST_DEFECTS, out.stdout + out.stderr[-4000:]
    assert "test cases: 106 | 99 passed | 7 failed" in out.stdout


def _run(lib, scene, steps):
    h = SolverHandle(lib, scene)
    reports = [h.step() for _ in range(steps)]
    return h, reports


STEPS = {"pile": 2, "mini_forest": 3, "mini_muscle": 3, "C1": 20}


@pytest.mark.parametrize("name", sorted(SCENES))
def test_restatement_bitwise_equals_reference(ref, oracle, name):
    scene = SCENES[name](ref)
    steps = STEPS.get(name, 8)
    a, ra = _run(ref, scene, steps)
    b, rb = _run(oracle, scene, steps)
    sa, sb = a.state(), b.state()
    for k in sa:
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=f"{name}: state {k}")
    for x, y in zip(ra, rb):
        np.testing.assert_array_equal(x.residuals, y.residuals)
        assert (x.contact_count, x.broad_pairs, x.skipped_singular, x.max_penetration, x.time, x.step) == \
               (y.contact_count, y.broad_pairs, y.skipped_singular, y.max_penetration, y.time, y.step)
    ca, cb = a.contacts(), b.contacts()
    for k in ca:
        np.testing.assert_array_equal(ca[k], cb[k])
    assert a.kinetic_energy() == b.kinetic_energy()
    assert a.total_volume() == b.total_volume()
    assert a.total_rest_volume() == b.total_rest_volume()
    np.testing.assert_array_equal(a.rest()["lengths"], b.rest()["lengths"])
    np.testing.assert_array_equal(a.current_pills(), b.current_pills())


def test_probe_convergence_bitwise(ref, oracle):
    scene = SCENES["kitchen_sink"](ref)
    la = SolverHandle(ref, scene).probe_convergence(15)
    lb = SolverHandle(oracle, scene).probe_convergence(15)
    np.testing.assert_array_equal(la, lb)


def random_pills(rng, n, spread=1.0, rmax=0.3, rods=None):
    p = np.zeros(n, dtype=capi.PILL_DTYPE)
    c0 = rng.uniform(-spread, spread, (n, 3))
    p["c0"] = c0
    p["c1"] = c0 + rng.normal(0, 0.4, (n, 3))
    p["r0"] = rng.uniform(0.01, rmax, n)
    p["r1"] = rng.uniform(0.01, rmax, n)
    p["rod"] = rng.integers(-1, 6, n) if rods is None else rods
    p["element"] = rng.integers(0, 12, n)
    p["group"] = rng.integers(-1, 3, n)
    p["self_collide"] = rng.integers(0, 2, n)
    return p


def test_collision_functions_bitwise(ref, oracle):
    rng = np.random.default_rng(11)
    a, b = random_pills(rng, 400), random_pills(rng, 400)
    # degenerate cases: swallowed spheres, zero-length axes, identical pills
    a["c1"][:20] = a["c0"][:20]
    a["r0"][20:40] = 2.0
    b[40:50] = a[40:50]
    x = rng.uniform(-1.5, 1.5, (400, 3))
    for lib_out in zip(pill_project(ref, x, b), pill_project(oracle, x, b)):
        np.testing.assert_array_equal(*lib_out)
    warm = rng.uniform(-0.2, 1.2, 400)
    for it in (1, 10, 30):
        for lib_out in zip(deepest_penetration(ref, a, b, it, warm), deepest_penetration(oracle, a, b, it, warm)):
            np.testing.assert_array_equal(*lib_out)
    pills = random_pills(rng, 300, spread=2.0, rmax=0.2)
    pa, pb = broad_phase(ref, pills), broad_phase(oracle, pills)
    np.testing.assert_array_equal(pa, pb)
    keys = rng.integers(0, 2**40, 50).astype(np.uint64)
    ca = find_contacts(ref, pills, pa, 10, keys, rng.uniform(0, 1, 50))
    cb = find_contacts(oracle, pills, pb, 10, keys, rng.uniform(0, 1, 50))
    for k in ca:
        np.testing.assert_array_equal(ca[k], cb[k])
    assert len(ca["pill_a"]) > 10


def test_make_rest_pose_bitwise(ref, oracle):
    from paper_1906_05260_b200.scene import make_rest_pose
    rng = np.random.default_rng(3)
    for n in (2, 3, 9, 40):
        c = np.cumsum(rng.normal(0, 0.3, (n, 3)), axis=0)
        r = rng.uniform(0.01, 0.1, n)
        s = rng.uniform(0.5, 1.5, n)
        ra, rb = make_rest_pose(ref, c, r, s), make_rest_pose(oracle, c, r, s)
        for k in ra.__dict__:
            np.testing.assert_array_equal(getattr(ra, k), getattr(rb, k))


def test_restatement_threads_do_not_change_results():
    """The restatement's block solves run on VROD_THREADS workers (parallel.h:26-46, used by
    bench.py --impl reference); results must not depend on the thread count."""
    import hashlib
    import sys
    code = ("import ctypes as C, hashlib, sys; sys.path.insert(0, %r); sys.path.insert(0, %r);"
            "from paper_1906_05260_b200 import capi; from paper_1906_05260_b200.handle import SolverHandle;"
            "from scenes import SCENES; lib = capi.bind(C.CDLL(%r)); h = SolverHandle(lib, SCENES['mini_muscle'](lib));"
            "[h.step() for _ in range(3)]; s = h.state();"
            "print(hashlib.sha256(b''.join(s[k].tobytes() for k in sorted(s))).hexdigest())") % (
        ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so"))
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, VROD_THREADS=t)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                   check=True).stdout.strip())
    assert outs[0] == outs[1] and len(outs[0]) == 64
