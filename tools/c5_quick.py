"""C5 quick timing: a batch of independent C3 scenes as one device world (graph replay)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
lib = bench.bind_bench(pb.library())
s = pb.BatchSolver(workloads.c5_batch(lib, n))
s.step()
ms, kern = bench.device_run(lib, s, 3, 0)
kt = bench.kernel_times(lib, s, 1)
print(f"C5 {n} scenes: {ms / 3:.3f} ms/step -> {n * 3 / (ms / 1e3):.0f} scene-substeps/s, {kern} kernels")
print({k: (round(v[0], 3), v[1]) for k, v in kt.items()})
