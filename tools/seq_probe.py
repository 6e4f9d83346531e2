"""Run scenes in sequence in one process (GPU strict vs oracle) to expose cross-instance leaks."""
import ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1906_05260_b200 import capi
from paper_1906_05260_b200.handle import SolverHandle
from scenes import DEBUG_SCENES, SCENES
ALL = {**SCENES, **DEBUG_SCENES}
orc = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so")))
gpu = capi.bind(C.CDLL(os.path.join(ROOT, "paper_1906_05260_b200", "lib", "libvrod_b200_strict.so")))
for name in sys.argv[1:]:
    sc = ALL[name](orc)
    g, o = SolverHandle(gpu, sc), SolverHandle(orc, sc)
    out = []
    for k in range(3):
        g.step(); o.step()
        sg, so = g.state(), o.state()
        out.append(f"{np.abs(sg['centers'] - so['centers']).max():.1e}")
    print(name, out, flush=True)
