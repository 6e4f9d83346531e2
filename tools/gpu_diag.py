"""Diagnostic: per-scene GPU-vs-oracle deviations (run on the GPU box)."""
from __future__ import annotations

import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1906_05260_b200 as pb  # noqa: E402
from paper_1906_05260_b200 import capi  # noqa: E402
from paper_1906_05260_b200.handle import SolverHandle  # noqa: E402
from scenes import DEBUG_SCENES, SCENES  # noqa: E402
SCENES = {**SCENES, **DEBUG_SCENES}


def main():
    orc = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so")))
    args = sys.argv[1:]
    if args and args[0] == "--fast":
        gpu = capi.bind(C.CDLL(os.path.join(ROOT, "paper_1906_05260_b200", "lib", "libvrod_b200_fast.so")))
        args = args[1:]
    else:
        gpu = pb.library()
    names = args or sorted(SCENES)
    for name in names:
        scene = SCENES[name](orc)
        try:
            g, o = SolverHandle(gpu, scene), SolverHandle(orc, scene)
            for k in range(10):
                t0 = time.time()
                rg = g.step()
                t1 = time.time()
                ro = o.step()
                sg, so = g.state(), o.state()
                dc = float(np.max(np.abs(sg["centers"] - so["centers"]))) if sg["centers"].size else 0
                ds = float(np.max(np.abs(sg["scales"] - so["scales"]))) if sg["scales"].size else 0
                fa, fb = sg["frames"], so["frames"]
                dq = float(np.max(np.minimum(np.linalg.norm(fa - fb, axis=1), np.linalg.norm(fa + fb, axis=1)))) if fa.size else 0
                print(f"{name:16s} step {k}: dc={dc:.2e} ds={ds:.2e} dq={dq:.2e} contacts {rg.contact_count}/{ro.contact_count} "
                      f"broad {rg.broad_pairs}/{ro.broad_pairs} sing {rg.skipped_singular}/{ro.skipped_singular} "
                      f"pen {rg.max_penetration:.3e}/{ro.max_penetration:.3e} res0 {rg.residuals[0]:.3e}/{ro.residuals[0]:.3e} "
                      f"gpu {1e3*(t1-t0):.2f} ms", flush=True)
        except Exception as e:  # keep going
            print(f"{name}: EXC {type(e).__name__}: {e}", flush=True)


if __name__ == "__main__":
    main()
