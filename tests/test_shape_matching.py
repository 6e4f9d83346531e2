"""Shape matching at the unit level (bundling.h): extract_rotation and one apply_shape_match pass
over a solver's groups, the way test_bundling.cpp drives fit_similarity / apply_shape_match.

CPU: the restatement equals the reference (oracle/_ref) bit for bit. GPU: the product agrees
within the shape-matching tolerance (warp tree reductions, FMA rotation chain).
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1906_05260_b200.handle import SolverHandle, extract_rotation

from scenes import SCENES

SHAPE_SCENES = ("band", "mini_muscle", "kitchen_sink")


def random_covariances(rng, n):
    """Near-rotation covariances (a scaled rotation plus noise) and perturbed guesses."""
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                  2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                  2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], axis=1).reshape(n, 3, 3)
    B = rng.uniform(0.5, 30, (n, 1, 1)) * R + rng.normal(0, 0.3, (n, 3, 3))
    guess = q + rng.normal(0, 0.2, (n, 4))
    guess[: n // 4] = [1, 0, 0, 0]
    return B, guess


def shape_pass(lib, name, steps=2):
    h = SolverHandle(lib, SCENES[name](lib))
    for _ in range(steps):
        h.step()
    fits = h.shape_match()
    return fits, h.state()


def similarity_recovery(lib):
    """test_bundling.cpp:93-109: a bundle moved by an exact similarity (sigma 1.3, 37 degrees
    about a tilted axis, t = (1, -2, 0.5)) is fitted back exactly."""
    scene = SCENES["band"](lib)
    h = SolverHandle(lib, scene)
    st = h.state()
    sigma, ang = 1.3, np.deg2rad(37.0)
    axis = np.array([1.0, 2.0, 2.0]) / 3.0
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    R = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K
    t = np.array([1.0, -2.0, 0.5])
    qr = np.array([np.cos(ang / 2), *(np.sin(ang / 2) * axis)])

    def qmul(a, b):
        return np.stack([a[..., 0] * b[..., 0] - np.sum(a[..., 1:] * b[..., 1:], -1),
                         *(a[..., :1] * b[..., 1:] + b[..., :1] * a[..., 1:] + np.cross(a[..., 1:], b[..., 1:])).T], -1)

    h.set_state(centers=sigma * st["centers"] @ R.T + t, scales=sigma * st["scales"],
                frames=qmul(np.broadcast_to(qr, st["frames"].shape), st["frames"]))
    return h.shape_match(), sigma, R, t


def test_restatement_extract_rotation_bitwise(ref, oracle):
    rng = np.random.default_rng(50)
    B, g = random_covariances(rng, 300)
    for it, tol in ((100, 1e-9), (3, 1e-9), (100, 1e-12)):
        np.testing.assert_array_equal(extract_rotation(ref, B, g, it, tol), extract_rotation(oracle, B, g, it, tol))


@pytest.mark.parametrize("name", SHAPE_SCENES)
def test_restatement_shape_pass_bitwise(ref, oracle, name):
    fa, sa = shape_pass(ref, name)
    fb, sb = shape_pass(oracle, name)
    np.testing.assert_array_equal(fa, fb)
    for k in sa:
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)


def test_restatement_similarity_recovery(oracle):
    fits, sigma, R, t = similarity_recovery(oracle)
    live = fits[fits[:, 13] == 0]
    assert len(live) > 0
    np.testing.assert_allclose(live[:, 0], sigma, rtol=1e-6)
    np.testing.assert_allclose(live[:, 4:13].reshape(-1, 3, 3), np.broadcast_to(R, (len(live), 3, 3)), atol=1e-6)


@pytest.mark.gpu
def test_gpu_extract_rotation(oracle):
    import paper_1906_05260_b200 as pb
    rng = np.random.default_rng(51)
    B, g = random_covariances(rng, 2000)
    for it, tol in ((100, 1e-9), (3, 1e-9)):
        qa, qb = extract_rotation(pb.library(), B, g, it, tol), extract_rotation(oracle, B, g, it, tol)
        err = np.minimum(np.abs(qa - qb).max(1), np.abs(qa + qb).max(1))
        assert err.max() < 1e-8, err.max()  # FMA chain + Taylor increment vs Eigen AngleAxis


@pytest.mark.gpu
@pytest.mark.parametrize("name", SHAPE_SCENES)
def test_gpu_shape_pass(oracle, name):
    import paper_1906_05260_b200 as pb
    fa, sa = shape_pass(pb.library(), name)
    fb, sb = shape_pass(oracle, name)
    np.testing.assert_array_equal(fa[:, 13], fb[:, 13])
    tol = 1e-6 if name == "kitchen_sink" else 1e-9  # the scenes' own free-running drift (test_gpu_parity)
    np.testing.assert_allclose(fa[:, :13], fb[:, :13], rtol=tol, atol=tol)
    for k in ("centers", "scales"):
        np.testing.assert_allclose(sa[k], sb[k], rtol=tol, atol=tol, err_msg=k)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SHAPE_SCENES)
def test_gpu_shape_pass_exact_mode_bitwise(oracle, name, monkeypatch):
    """The exact-order path (VROD_SHAPE_EXACT=1): fits, states and frames bit-identical."""
    import paper_1906_05260_b200 as pb
    monkeypatch.setenv("VROD_SHAPE_EXACT", "1")
    fa, sa = shape_pass(pb.library(), name)
    fb, sb = shape_pass(oracle, name)
    np.testing.assert_array_equal(fa, fb)
    for k in sa:
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)


@pytest.mark.gpu
def test_gpu_similarity_recovery(oracle):
    import paper_1906_05260_b200 as pb
    fa, sigma, R, t = similarity_recovery(pb.library())
    fb, *_ = similarity_recovery(oracle)
    np.testing.assert_array_equal(fa[:, 13], fb[:, 13])
    np.testing.assert_allclose(fa, fb, rtol=1e-10, atol=1e-10)

