"""Which slots differ between the GPU (strict) and the oracle, over a grid of settings."""
import ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1906_05260_b200 import capi
from paper_1906_05260_b200.handle import SolverHandle
from scenes import DEBUG_SCENES, SCENES
orc = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so")))
gpu = capi.bind(C.CDLL(os.path.join(ROOT, "paper_1906_05260_b200", "lib", "libvrod_b200_strict.so")))
name = sys.argv[1]
for iters, subs, steps in [(10, 1, 1), (10, 1, 2), (10, 1, 4), (1, 4, 1), (2, 2, 1), (10, 4, 1)]:
    sc = {**SCENES, **DEBUG_SCENES}[name](orc)
    sc.settings.iterations = iters
    sc.settings.substeps = subs
    g, o = SolverHandle(gpu, sc), SolverHandle(orc, sc)
    for k in range(steps):
        g.step(); o.step()
        sg, so = g.state(), o.state()
        dc = np.abs(sg["centers"] - so["centers"]).max(axis=1)
        ds = np.abs(sg["scales"] - so["scales"])
        dv = np.abs(sg["center_vel"] - so["center_vel"]).max(axis=1)
        bad = np.nonzero((dc > 0) | (ds > 0))[0]
        print(f"it={iters} sub={subs} step {k}: {len(bad)} slots differ {bad[:12].tolist()} dc {dc.max():.2e} ds {ds.max():.2e} dv {dv.max():.2e}", flush=True)
