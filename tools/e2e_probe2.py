"""C3 end-to-end anatomy as bench.py times it (state_prefetch on): step()+state() per frame, vs
step() alone, vs the device-timed graph replay; plus the C-ABI get_state alone into reused buffers."""
import ctypes as C, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads, capi
lib = pb.library()
lib.vrod_bench_run.restype = C.c_int
lib.vrod_bench_run.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
s = pb.Solver(workloads.c3_muscle_bundle(lib))
s.set_option("state_prefetch", 1)
for _ in range(10):
    s.step(); s.state()
N = 300
def timed(f):
    t = time.perf_counter()
    for _ in range(N):
        f()
    return (time.perf_counter() - t) / N * 1e6
both = timed(lambda: (s.step(), s.state()))
step = timed(s.step)
st = s.state()
bufs = {k: np.empty_like(v) for k, v in st.items()}
h = s._h
def raw_state():
    lib.vrod_solver_get_state(h, capi.ptr(bufs["centers"]), capi.ptr(bufs["scales"]), capi.ptr(bufs["frames"]),
                              capi.ptr(bufs["center_vel"]), capi.ptr(bufs["scale_vel"]), capi.ptr(bufs["angular_vel"]))
s.step()
raw = timed(raw_state)
pystate = timed(s.state)
ms, k = C.c_double(), C.c_int64()
lib.vrod_bench_run(h, 200, 0, C.byref(ms), C.byref(k))
print(f"step+state {both:.1f} us | step {step:.1f} | state() {pystate:.1f} (C get_state into reused buffers {raw:.1f}) "
      f"| device replay {1e3 * ms.value / 200:.1f} us/step")
