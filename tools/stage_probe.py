"""Time each stage of a config on the GPU with progress output (debugging aid)."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads

def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)

name = sys.argv[1]
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = int(v)
lib = pb.library()
t0 = time.time(); scene = workloads.CONFIGS[name](lib, **kw); log("scene built", time.time() - t0)
t0 = time.time(); s = pb.Solver(scene); log("solver created", time.time() - t0, s.total_vertices)
for k in range(5):
    t0 = time.time(); r = s.step(); log("step", k, f"{1e3*(time.time()-t0):.2f} ms", "contacts", r.contact_count, "broad", r.broad_pairs)
