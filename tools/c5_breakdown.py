"""Per-category device time of a C5 batch step (1024 scenes by default) — bench.py's kernel_times."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
lib = pb.library()
s = pb.BatchSolver(workloads.c5_batch(lib, n))
s.step()
lib.vrod_bench_kernel_times.restype = C.c_int
lib.vrod_bench_kernel_times.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
ms, ln = (C.c_double * 8)(), (C.c_int64 * 8)()
assert lib.vrod_bench_kernel_times(s._h, 1, ms, ln) == 0
cats = ["predict", "collide", "ext_setup", "ext_solve", "rod_sweep", "shape", "report", "iterate"]
print(f"C5 {n} scenes: total {sum(ms):.2f} ms;", {c: (round(ms[i], 3), ln[i]) for i, c in enumerate(cats)})
