"""C4 timing probe: per-category device time of a C4 substep (kernel_times) and the graph-replayed
substep time. Usage: c4_probe.py [nx ny]"""
import ctypes as C, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
sys.argv += [] 
nx, ny = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (125, 250)
lib = pb.library()
import bench
bench.bind_bench(lib)
s = pb.Solver(workloads.c4_rod_forest(lib, nx=nx, ny=ny))
for _ in range(2):
    r = s.step()
ms, kern = bench.device_run(lib, s, 5, 0)
kt = bench.kernel_times(lib, s, 1)
print(f"C4 {nx}x{ny}: {ms / 5:.3f} ms/substep, {kern} kernels, contacts {r.contact_count}")
print({k: (round(v[0], 3), v[1]) for k, v in kt.items()})
