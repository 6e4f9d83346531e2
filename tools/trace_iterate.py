"""Phase timeline of the persistent iteration kernel (CTA 0), VROD_TRACE=1: per iteration
stage X / solve blocks / gather / barrier, then shape-matching levels; per-warp phases of CTA
$VROD_TRACE_CTA in iteration 1. Usage: trace_iterate.py [C3 [warm-up steps, default 5]]"""
import ctypes as C, os, sys
os.environ["VROD_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
lib = pb.library()
s = pb.Solver(workloads.CONFIGS[name](lib))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    s.step()
lib.vrod_bench_trace.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
buf = (C.c_int64 * 1024)()
n = C.c_int32()
assert lib.vrod_bench_trace(s._h, 1024, buf, C.byref(n)) == 0
t = np.array(buf[:n.value], dtype=np.float64)
d = np.diff(t) / 1e3
print(f"{n.value} marks, total {(t[-1] - t[0]) / 1e3:.1f} us")
# layout: start, then per iteration [staged, solved, gathered, barrier] (+ one per shape level)
raw0 = (C.c_int64 * 1024)()
assert lib.vrod_bench_trace(s._h, -1024, raw0, C.byref(n)) == 0
nshape = int(raw0[598]) or 2
i, it = 1, 0
rows = []
while i + 3 < len(t):
    stage, solve, gather, bar = (t[i] - t[i - 1]) / 1e3, (t[i + 1] - t[i]) / 1e3, (t[i + 2] - t[i + 1]) / 1e3, (t[i + 3] - t[i + 2]) / 1e3
    i += 4
    shape = []
    if (it + 1) % 2 == 0 and name == "C3":
        for _ in range(nshape):
            if i < len(t):
                shape.append((t[i] - t[i - 1]) / 1e3)
                i += 1
    rows.append((stage, solve, gather, bar, shape))
    it += 1
for k, r in enumerate(rows):
    print(f"it {k:2d}: stage {r[0]:6.2f} solve {r[1]:6.2f} gather {r[2]:6.2f} barrier {r[3]:6.2f} shape {['%.2f' % x for x in r[4]]}")
a = np.array([r[:4] for r in rows])
print("mean stage/solve/gather/barrier us:", a.mean(0).round(2), " shape levels total:", round(sum(sum(r[4]) for r in rows), 1))
raw = (C.c_int64 * 1024)()
assert lib.vrod_bench_trace(s._h, -1024, raw, C.byref(n)) == 0
raw = np.array(raw[:], dtype=np.float64)
arr = raw[700:700 + 148]
arr = arr[arr > 0]
print(f"iteration 1 barrier arrivals over {len(arr)} CTAs: first..last spread {(arr.max() - arr.min()) / 1e3:.2f} us, "
      f"latest CTA {int(np.argmax(raw[700:700 + 148]))}")
order = np.argsort(arr)
print("  latest 8 CTAs (us after first):", [(int(i), round((arr[i] - arr.min()) / 1e3, 2)) for i in order[-8:]])
rel = (arr - arr.min()) / 1e3
print("  arrival percentiles (us after first): p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(rel, [10, 50, 90, 100])))
for l in range(2):
    ph = raw[600 + 8 * l: 606 + 8 * l]
    if ph[0] > 0:
        print(f"shape level/chain pos {l} group phases us: centroid {(ph[1]-ph[0])/1e3:.2f} covariance {(ph[2]-ph[1])/1e3:.2f} "
              f"rotation {(ph[3]-ph[2])/1e3:.2f} ({int(raw[606 + 8 * l])} it) scale {(ph[4]-ph[3])/1e3:.2f} apply {(ph[5]-ph[4])/1e3:.2f}"
              + (f" [covariance terms {(raw[607 + 8 * l]-ph[1])/1e3:.2f}, ordered sum {(ph[2]-raw[607 + 8 * l])/1e3:.2f}]" if raw[607 + 8 * l] > 0 else ""))
cta = int(os.environ.get("VROD_TRACE_CTA", "0"))
t0 = raw[899]
if t0 > 0:
    print(f"iteration 1, CTA {cta}: per-warp end of items / of external entries (us after staging):",
          [round((raw[900 + k] - t0) / 1e3, 2) for k in range(9)], [round((raw[916 + k] - t0) / 1e3, 2) for k in range(9)])
