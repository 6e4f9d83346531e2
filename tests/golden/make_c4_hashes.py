"""Golden SHA-256 digests of the full-size C4 rod forest (1,000,000 vertices),
generated here from the REFERENCE (oracle/_ref: the reference's own sources compiled against the
Eigen shim) and from the restatement (oracle/lib), which must agree bit for bit.

    python tests/golden/make_c4_hashes.py [--lib ref|oracle] [--steps 2]

A reference substep at this size takes minutes on the CPU (~7.7e7 broad-phase candidates searched
serially), so the GPU test (tests/test_bench_parity.py) compares hashes instead of re-running the
CPU: every output array of every substep — state, velocities, contact set with alpha/beta — and
the StepReport counters must hash to the same digests. A few sampled values per array are kept
for diagnostics when a digest differs. The scene is regenerated deterministically on the box
(numpy's seeded generator; rest poses from the oracle's make_rest_pose).
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1906_05260_b200 import capi, workloads  # noqa: E402
from paper_1906_05260_b200.handle import SolverHandle  # noqa: E402

OUT = os.path.join(HERE, "c4_hashes.json")
SAMPLE = 16


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def step_record(h: SolverHandle, rep) -> dict:
    """Digests of everything one substep produces (the reference's observable outputs)."""
    rec = {"contact_count": rep.contact_count, "broad_pairs": rep.broad_pairs,
           "skipped_singular": rep.skipped_singular, "max_penetration": rep.max_penetration.hex(),
           "residuals": [float(x) for x in rep.residuals], "time": rep.time.hex(), "step": rep.step,
           "sha256": {}, "sample": {}}
    arrays = dict(h.state())
    arrays.update({f"contacts_{k}": v for k, v in h.contacts().items()})
    for k, v in arrays.items():
        flat = np.ascontiguousarray(v).reshape(-1)
        rec["sha256"][k] = digest(flat)
        idx = np.linspace(0, max(flat.size - 1, 0), SAMPLE).astype(np.int64) if flat.size else np.zeros(0, np.int64)
        rec["sample"][k] = [float(flat[i]).hex() if flat.dtype.kind == "f" else int(flat[i]) for i in idx]
    return rec


def scene_builder(oracle):
    return workloads.c4_rod_forest(oracle)


def run(lib, oracle, steps: int) -> list[dict]:
    h = SolverHandle(lib, scene_builder(oracle))
    out = []
    for s in range(steps):
        t0 = time.time()
        rep = h.step()
        out.append(step_record(h, rep))
        print(f"step {s}: {time.time() - t0:.1f} s, contacts {rep.contact_count}, broad {rep.broad_pairs}", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="ref", choices=["ref", "oracle"])
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    oracle = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so")))
    path = os.path.join(ROOT, "oracle", "_ref", "libvrod_ref.so") if args.lib == "ref" else None
    lib = capi.bind(C.CDLL(path)) if path else oracle
    recs = run(lib, oracle, args.steps)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["workload"] = "C4 rod forest 125x250 rods x 32 vertices (workloads.c4_rod_forest defaults)"
    data[args.lib] = {"backend": lib.vrod_backend_name().decode(), "steps": recs}
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)


if __name__ == "__main__":
    main()
