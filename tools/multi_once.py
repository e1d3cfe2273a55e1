"""One 16-RHS recompute pass (for ncu launch lists).  usage: python tools/multi_once.py N d [dmma]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1708_09707_b200 as hm  # noqa: E402
from paper_1708_09707_b200.inputs import symmetric, uniform_points  # noqa: E402

n, d = int(sys.argv[1]), int(sys.argv[2])
dmma = len(sys.argv) > 3 and sys.argv[3] == "dmma"
h = hm.setup(uniform_points(n, d, 42), hm.KernelFunction(), hm.HmatrixConfig(c_leaf=64, k=16))
X = np.stack([symmetric(43 + r, n) for r in range(16)], axis=1)
Z = h.mvp_multi(X, dmma=dmma)
print("done", float(np.linalg.norm(Z)))
