"""One C3 timing (graph replays, device-timed; the bench config): prints us/step. The library
variant comes from VROD_B200_VARIANT (see _lib.py). Usage: c3_once.py [steps]"""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
lib = pb.library()
lib.vrod_bench_run.restype = C.c_int
lib.vrod_bench_run.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
s = pb.Solver(workloads.c3_muscle_bundle(lib))
for _ in range(10):
    s.step()
ms, k = C.c_double(), C.c_int64()
assert lib.vrod_bench_run(s._h, steps, 256 << 20, C.byref(ms), C.byref(k)) == 0
print(f"{os.environ.get('VROD_B200_VARIANT', 'base'):10s} {1e3 * ms.value / steps:7.1f} us/step")
