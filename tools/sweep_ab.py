"""A/B the rod-sweep variants on C4: device ms per step and per-category breakdown."""
import os, sys, ctypes as C
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
sys.path.insert(0, ROOT)
import bench
lib = bench.bind_bench(pb.library())
s = pb.Solver(workloads.c4_rod_forest(lib))
for _ in range(2):
    s.step()
ms, _ = bench.device_run(lib, s, 4, 0)
kt = bench.kernel_times(lib, s, 1)
print(os.environ.get("VROD_SWEEP_TP32", "tp64"), "ms/substep", ms / 4, {k: round(v[0], 3) for k, v in kt.items()})
