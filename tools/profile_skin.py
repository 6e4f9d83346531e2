"""Skinning workload for ncu: C3 solver, 1000x1000 sleeve bound to its rest pills, N fused deforms."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
lib = pb.library()
s = pb.Solver(workloads.c3_muscle_bundle(lib))
s.step()
pills, rest = s.rest_pills(), s.rest_pill_transforms()
V, T = workloads.sleeve_mesh(pills, 1000, 1000)
sk = pb.Skin(V, T, pills, rest, max_influences=8)
sk.smooth(1)
for _ in range(n):
    sk.deform_solver(s)
print("ok", V.shape)
