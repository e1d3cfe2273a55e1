"""One setup + products (for ncu captures).  usage: python tools/one_product.py N d kernel [recompute|stored] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_09707_b200 as hm  # noqa: E402
from paper_1708_09707_b200.inputs import symmetric, uniform_points  # noqa: E402

n, d, kern = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
stored = len(sys.argv) > 4 and sys.argv[4] == "stored"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
h = hm.setup(uniform_points(n, d, 42), hm.KernelFunction(kern),
             hm.HmatrixConfig(c_leaf=64, k=16, precompute_aca=stored, near_stored=stored))
for r in range(reps):
    h.mvp(symmetric(43 + r, n))
print("done", h.stats()["n_aca"], flush=True)
