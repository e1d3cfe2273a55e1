"""Recompute-mode (matrix-free, the reference's default) product breakdown.
usage: python tools/trace_recompute.py N d kernel"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1708_09707_b200 as hm  # noqa: E402
from paper_1708_09707_b200.inputs import symmetric, uniform_points  # noqa: E402

n, d, kern = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
t = time.perf_counter()
h = hm.setup(uniform_points(n, d, 42), hm.KernelFunction(kern), hm.HmatrixConfig(c_leaf=64, k=16))
print("setup", time.perf_counter() - t, h.stats()["n_dense"], h.stats()["n_aca"], h.stats()["S_d"], flush=True)
x = symmetric(43, n)
t = time.perf_counter()
h.mvp(x)
print("mvp (first)", time.perf_counter() - t, flush=True)
h.profile_begin()
t = time.perf_counter()
h.mvp(x)
print("mvp", time.perf_counter() - t)
print({k: round(v[0], 2) for k, v in h.profile_end().items()})
