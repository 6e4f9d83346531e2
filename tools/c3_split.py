"""C3 step time vs iteration count (graph replays, device-timed): separates the fixed per-step cost
(predict, collide, ext setup, finalize, report) from the per-iteration cost of the loop."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
lib = pb.library()
lib.vrod_bench_run.restype = C.c_int
lib.vrod_bench_run.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
for iters, period in ((20, 2), (20, 1000), (10, 2), (4, 2), (1, 1000)):
    sc = workloads.c3_muscle_bundle(lib)
    sc.settings.iterations = iters
    sc.settings.shape_match_period = period
    s = pb.Solver(sc)
    for _ in range(5):
        s.step()
    ms, k = C.c_double(), C.c_int64()
    rc = lib.vrod_bench_run(s._h, 30, 256 << 20, C.byref(ms), C.byref(k))
    assert rc == 0, lib.vrod_last_error()
    print(f"iterations {iters:2d} shape period {period:4d}: {1e3 * ms.value / 30:7.1f} us/step ({k.value} kernels)", flush=True)
