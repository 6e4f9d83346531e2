"""CPU-side checks of the product library (no GPU needed): the C-ABI is complete, the host
setup path (make_rest_pose, Scene::validate, pair_key) matches the oracle bit for bit and
message for message, and the solver refuses to run without a device instead of falling back.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import capi
from paper_1906_05260_b200.handle import pair_key
from paper_1906_05260_b200.scene import (Activation, InvalidArgument, KinematicPill, MaterialParams, OutOfRange, Pill,
                                         PinMotion, SoftPin, make_rest_pose, validate)

from conftest import ROOT
from scenes import SCENES, curved_rod
from test_oracle_pinning import random_pills


def header_functions(path):
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int32_t|int|void|uint64_t)\s+(vrod_\w+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported(oracle):
    lib = C.CDLL(pb.LIB_PATH)
    for name in header_functions(os.path.join(ROOT, "include", "vrod_capi.h")):
        assert hasattr(lib, name), name
        assert hasattr(oracle, name), name
    for name in header_functions(os.path.join(ROOT, "include", "vrod_bench.h")):
        assert hasattr(lib, name), name
    assert set(capi.exported_symbols()) <= set(header_functions(os.path.join(ROOT, "include", "vrod_capi.h")))
    assert pb.library().vrod_backend_name() == b"b200-cuda"
    assert pb.library().vrod_capi_version() == oracle.vrod_capi_version()


def test_product_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pb.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_rest_pose_bitwise(oracle):
    rng = np.random.default_rng(8)
    lib = pb.library()
    for n in (2, 3, 5, 17, 64):
        c = np.cumsum(rng.normal(0, 0.2, (n, 3)), axis=0)
        for radii, scales in ((rng.uniform(0.01, 0.1, n), rng.uniform(0.5, 1.5, n)), ([0.05], None), ([0.03], [1.2])):
            a, b = make_rest_pose(lib, c, radii, scales), make_rest_pose(oracle, c, radii, scales)
            for k in a.__dict__:
                np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
    # antiparallel consecutive tangents (FromTwoVectors' degenerate branch)
    c = np.array([[0, 0, 0], [0, 0, 1], [0, 0, 0.5], [0.1, 0, 0.2]], dtype=float)
    a, b = make_rest_pose(lib, c, [0.01]), make_rest_pose(oracle, c, [0.01])
    np.testing.assert_array_equal(a.frames, b.frames)


def bad_scenes(lib):
    """(scene, expected exception) pairs covering Scene::validate (scene.cpp:63-157)."""
    out = []

    def base():
        return SCENES["C1"](lib)

    s = base(); s.materials = []; out.append(s)
    s = base(); s.materials[0].density = 0.0; out.append(s)
    s = base(); s.materials[0].stretch_x = -1.0; out.append(s)
    s = base(); s.settings.dt = 0.0; out.append(s)
    s = base(); s.settings.beta = 1.5; out.append(s)
    s = base(); s.settings.iterations = 0; out.append(s)
    s = base(); s.settings.velocity_damping = 1.0; out.append(s)
    s = base(); s.settings.gravity = (0.0, math.nan, 0.0); out.append(s)
    s = base(); s.rods[0].material = 3; out.append(s)
    s = base(); s.planes.append(type("P", (), {"normal": (0.0, 0.0, 2.0), "offset": 0.0})()); out.append(s)
    s = base(); s.bundles.append([(0, 1)]); out.append(s)
    s = base(); s.bundles.append([(0, 1), (0, 1)]); out.append(s)
    s = base(); s.bundles.append([(0, 1), (1, 1)]); out.append(s)
    s = base(); s.bundles.append([(0, 1), (0, 500)]); out.append(s)
    s = base(); s.pin_motions.append(PinMotion(0, 5, (0, 0, 0), (1, 0, 0), 0.0, 1.0)); out.append(s)
    s = base(); s.pin_motions.append(PinMotion(0, 0, (0, 0, 0), (1, 0, 0), 1.0, 0.0)); out.append(s)
    s = base(); s.soft_pins.append(SoftPin(0, 2, (0, 0, 0), 0.0)); out.append(s)
    s = base(); s.soft_pins.append(SoftPin(4, 2, (0, 0, 0), 1.0)); out.append(s)
    s = base(); s.activations.append(Activation(0, 1.0)); out.append(s)
    s = base(); s.activations.append(Activation(0, 0.2, 1.0, 0.5)); out.append(s)
    s = base(); s.activations.append(Activation(0, 0.2, first_element=200)); out.append(s)
    s = base(); s.activations.append(Activation(0, 0.2, first_element=3, last_element=2)); out.append(s)
    s = base(); s.kinematic_pills.append(KinematicPill(Pill((0, 0, 0), (1, 0, 0), 0.0, 0.1))); out.append(s)
    s = base(); s.kinematic_pills.append(KinematicPill(Pill((0, 0, 0), (1, 0, 0), 0.1, 0.1, rod=0))); out.append(s)
    s = base(); s.kinematic_pills.append(KinematicPill(Pill((0, 0, 0), (1, 0, 0), 0.1, 0.1), bone=2)); out.append(s)
    s = base(); s.rods[0].pinned = np.zeros(3, dtype=np.uint8); out.append(s)
    s = base(); s.rods[0].rest.frames[4] = [2.0, 0, 0, 0]; out.append(s)
    s = base(); s.rods[0].rest.radii[2] = -0.1; out.append(s)
    s = base(); s.rods[0].rest.lengths[2] = 0.0; out.append(s)
    s = base(); s.rods[0].bones = [0]; s.rods[0].bone_weights = np.ones((100, 1)); out.append(s)
    return out


def test_validation_messages_match_oracle(oracle):
    lib = pb.library()
    for i, scene in enumerate(bad_scenes(oracle)):
        errs = []
        for L in (lib, oracle):
            try:
                validate(L, scene)
                errs.append(None)
            except (InvalidArgument, OutOfRange) as e:
                errs.append((type(e).__name__, str(e)))
        assert errs[0] is not None, f"scene {i} accepted"
        assert errs[0] == errs[1], (i, errs)


def test_valid_scenes_accepted():
    lib = pb.library()
    for name, build in SCENES.items():
        validate(lib, build(lib))


def test_pair_key_matches(oracle):
    rng = np.random.default_rng(4)
    p = random_pills(rng, 200)
    for i in range(0, 200, 2):
        assert pair_key(pb.library(), p[i], p[i + 1]) == pair_key(oracle, p[i], p[i + 1])


def test_no_cpu_fallback_without_a_device():
    """The product never computes on the host: without a CUDA device, creating a solver fails."""
    lib = pb.library()
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = os.path.exists("/dev/nvidia0")
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(pb.DeviceError):
        pb.Solver(SCENES["C1"](lib))
