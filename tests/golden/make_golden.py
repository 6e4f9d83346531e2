"""Generate the golden fixtures from the REFERENCE (oracle/_ref: the reference's own sources
compiled against the Eigen shim). Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

The fixtures pin the CPU restatement (and, for exact scenes, the GPU product) on the GPU box,
where /root/reference and oracle/_ref may be absent. Inputs are regenerated deterministically
by the test, so only outputs are stored.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from paper_1906_05260_b200 import capi  # noqa: E402
from paper_1906_05260_b200.handle import SolverHandle, broad_phase, deepest_penetration, find_contacts, pill_project  # noqa: E402

GOLDEN_SCENES = {"C1": 8, "pile": 2, "mini_forest": 3, "kitchen_sink": 3, "mini_muscle": 2, "crossing": 6}


def golden_pills():
    from test_oracle_pinning import random_pills
    rng = np.random.default_rng(424242)
    a, b = random_pills(rng, 256), random_pills(rng, 256)
    a["c1"][:8] = a["c0"][:8]
    a["r0"][8:16] = 2.0
    x = rng.uniform(-1.5, 1.5, (256, 3))
    warm = rng.uniform(-0.2, 1.2, 256)
    field = random_pills(rng, 400, spread=2.0, rmax=0.2)
    keys = rng.integers(0, 2**40, 20).astype(np.uint64)
    walpha = rng.uniform(0, 1, 20)
    return a, b, x, warm, field, keys, walpha


def run_scene(lib, scenes, name, steps):
    h = SolverHandle(lib, scenes[name](lib))
    reps = [h.step() for _ in range(steps)]
    out = {f"{name}/{k}": v for k, v in h.state().items()}
    out[f"{name}/residuals"] = np.array([r.residuals for r in reps])
    out[f"{name}/counters"] = np.array([[r.contact_count, r.broad_pairs, r.skipped_singular] for r in reps])
    out[f"{name}/max_penetration"] = np.array([r.max_penetration for r in reps])
    for k, v in h.contacts().items():
        out[f"{name}/contacts_{k}"] = v
    return out


def main():
    from scenes import SCENES
    lib = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libvrod_ref.so")))
    assert lib.vrod_backend_name() == b"reference-cpu"
    out = {}
    for name, steps in GOLDEN_SCENES.items():
        out.update(run_scene(lib, SCENES, name, steps))
    a, b, x, warm, field, keys, walpha = golden_pills()
    out["pp/t"], out["pp/d"], out["pp/deg"] = pill_project(lib, x, b)
    out["dp/alpha"], out["dp/beta"], out["dp/d"] = deepest_penetration(lib, a, b, 10, warm)
    pairs = broad_phase(lib, field)
    out["bp/pairs"] = pairs
    for k, v in find_contacts(lib, field, pairs, 10, keys, walpha).items():
        out[f"fc/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", len(out), "arrays")
    from test_skinning import make_skin_golden  # skinning.cpp flow on the same scenes
    skin = make_skin_golden(lib)
    np.savez_compressed(os.path.join(HERE, "skin_golden.npz"), **skin)
    print("wrote", len(skin), "skin arrays")


if __name__ == "__main__":
    main()
