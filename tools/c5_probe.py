"""Time C5 batches on one GPU: setup, graph capture, steps."""
import sys, time, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
lib = pb.library()
for n in [int(x) for x in sys.argv[1:]]:
    t0 = time.time()
    scenes = workloads.c5_batch(lib, n)
    t1 = time.time()
    s = pb.BatchSolver(scenes)
    t2 = time.time()
    r = s.step()
    t3 = time.time()
    k = 3
    for _ in range(k):
        r = s.step()
    t4 = time.time()
    print(f"C5 n={n}: scenes {t1-t0:.1f}s create {t2-t1:.1f}s first step {t3-t2:.2f}s "
          f"step {1e3*(t4-t3)/k:.1f} ms -> {n*k/(t4-t3):.0f} scene-frames/s; contacts {r.contact_count}", flush=True)
    del s
