"""Where the C3 end-to-end time goes: step() alone, state() alone, and both, through the Python API."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
lib = pb.library()
s = pb.Solver(workloads.CONFIGS["C3"](lib))
for _ in range(20):
    s.step()
    s.state()
def t(f, n=200):
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e6
both = t(lambda: (s.step(), s.state()))
step = t(s.step)
state = t(s.state)
V = s.total_vertices
bufs = [np.zeros((V, 3)), np.zeros(V)]
print(f"step+state {both:.1f} us   step {step:.1f} us   state {state:.1f} us")
