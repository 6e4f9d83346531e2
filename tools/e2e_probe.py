"""Where the end-to-end C3 frame time goes: step() alone, state() alone, both."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
lib = pb.library()
s = pb.Solver(workloads.c3_muscle_bundle(lib))
for _ in range(10):
    s.step()
N = 300
t = time.perf_counter()
for _ in range(N):
    s.step()
a = (time.perf_counter() - t) / N
t = time.perf_counter()
for _ in range(N):
    s.state()
b = (time.perf_counter() - t) / N
t = time.perf_counter()
for _ in range(N):
    s.step(); s.state()
c = (time.perf_counter() - t) / N
print(f"step {a*1e3:.3f} ms  state {b*1e3:.3f} ms  both {c*1e3:.3f} ms")
