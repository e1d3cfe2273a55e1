# compute-sanitizer driver for the ACA kernels (small cases, every size class)
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1708_09707_b200 as hm
from paper_1708_09707_b200.inputs import uniform_points, halton_points
cases = [("halton", 8192, 2, 64, False), ("uniform", 2000, 2, 64, True), ("uniform", 5000, 3, 200, True),
         ("uniform", 8192, 2, 64, False)]
for kind, n, d, cl, pre in cases:
    P = halton_points(n, d) if kind == "halton" else uniform_points(n, d, 42)
    h = hm.setup(P, hm.KernelFunction(), hm.HmatrixConfig(c_leaf=cl, k=16, precompute_aca=pre))
    z = h.mvp(np.ones(n))
    print(kind, n, d, cl, pre, h.stats()['n_aca'], float(np.linalg.norm(z)), flush=True)
