"""Measured parity maxima of the shape-matching scenes (default latency-tuned shape path) against the
CPU oracle: one step from identical input and free-running, as tests/test_gpu_parity.py checks
them. Prints JSON."""
import ctypes as C, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import capi
from paper_1906_05260_b200.handle import SolverHandle
from scenes import SCENES
from test_bench_parity import state_err

orc = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so")))
steps = {"band": 10, "kitchen_sink": 10, "mini_muscle": 6}
out = {}
for name, k in steps.items():
    scene = SCENES[name](orc)
    g, o = SolverHandle(pb.library(), scene), SolverHandle(orc, scene)
    rec = {}
    for i in range(k):
        g.step(); o.step()
        e = state_err(g.state(), o.state())
        if i == 0:
            rec["one_step"] = e
    rec["free"] = e
    rec["steps"] = k
    out[name] = rec
print(json.dumps(out, indent=1))
