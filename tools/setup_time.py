"""Setup (hm_setup) wall time and phases.  usage: python tools/setup_time.py N d kernel [recompute|stored] [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_09707_b200 as hm  # noqa: E402
from paper_1708_09707_b200.inputs import uniform_points  # noqa: E402

n, d, kern = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
stored = len(sys.argv) > 4 and sys.argv[4] == "stored"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
P = uniform_points(n, d, 42)
for r in range(reps):
    t = time.perf_counter()
    h = hm.setup(P, hm.KernelFunction(kern), hm.HmatrixConfig(c_leaf=64, k=16, precompute_aca=stored, near_stored=stored))
    wall = time.perf_counter() - t
    st = h.stats()
    print(json.dumps({"n": n, "d": d, "rep": r, "setup_wall_s": wall, "phases_ms": h.timings(),
                      "n_dense": st["n_dense"], "n_aca": st["n_aca"], "chunks": st["n_aca_chunks"]}), flush=True)
    h.close()
