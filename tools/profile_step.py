"""Small fixed workload for ncu: build a config, warm up, run N graph steps."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
name, steps = sys.argv[1], int(sys.argv[2])
lib = pb.library()
s = pb.Solver(workloads.CONFIGS[name](lib))
for _ in range(3):
    s.step()
for _ in range(steps):
    r = s.step()
print(name, "ok contacts", r.contact_count, "broad", r.broad_pairs)
