import os, sys, json, time, ctypes as C
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import capi, workloads
from paper_1906_05260_b200.handle import SolverHandle
from scenes import SCENES
orc = capi.bind(C.CDLL('/root/repo/oracle/lib/libvrod_oracle.so'))
gpu = pb.library()
def err(a, b):
    out = {}
    for k in a:
        d = np.abs(a[k] - b[k]) / np.maximum(1.0, np.abs(b[k]))
        out[k] = float(d.max()) if d.size else 0.0
    return out
res = {}
for name, steps in [('kitchen_sink', 10), ('band', 10), ('mini_muscle', 10), ('C3', 10), ('C3g', 10)]:
    build = SCENES.get(name) or workloads.CONFIGS[name]
    sc = build(orc)
    o = SolverHandle(orc, sc)
    g = SolverHandle(gpu, sc)
    errs = []
    bit = True
    for k in range(steps):
        rg, ro = g.step(), o.step()
        sg, so = g.state(), o.state()
        e = err(sg, so); errs.append(max(e.values()))
        bit = bit and all(np.array_equal(sg[x], so[x]) for x in sg)
        if (rg.contact_count, rg.broad_pairs) != (ro.contact_count, ro.broad_pairs): print(name, 'contacts differ', k)
    res[name] = {'bitwise_all_steps': bit, 'max_rel_err_per_step': errs}
    print(name, os.environ.get('VROD_SHAPE_EXACT'), bit, ['%.1e' % x for x in errs], flush=True)
# timing of C3 step
lib = gpu
sc = workloads.c3_muscle_bundle(lib)
s = pb.Solver(sc)
for _ in range(20): s.step()
lib.vrod_bench_run.restype = C.c_int
lib.vrod_bench_run.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
ms = C.c_double(); kern = C.c_int64()
lib.vrod_bench_run(s._h, 100, 256 << 20, C.byref(ms), C.byref(kern))
print('C3 ms/step', ms.value / 100, 'exact' if os.environ.get('VROD_SHAPE_EXACT') == '1' else 'fast')
res['c3_ms'] = ms.value / 100
json.dump(res, open(os.environ.get('OUT', '/dev/null'), 'w'), indent=1)
