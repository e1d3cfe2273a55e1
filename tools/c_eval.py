"""Per-entry FP64 instruction counts of the kernel evaluation (c_eval).

Evaluates phi on 2^22 random point pairs in [0,1]^d (the distance distribution of the
admissible blocks' entries) with the device entry code (eval_pairs_kernel, the same
device functions the ACA and near-field kernels inline).  Run under ncu:

  ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,... -k regex:eval_pairs \
      python tools/c_eval.py
and divide the thread-instruction counts by the pair count (tools/fp64_summary.py).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_09707_b200 as hm  # noqa: E402

N = 1 << 22
for kern in ("gaussian", "matern"):
    for d in (2, 3, 4):
        rng = np.random.default_rng(1000 + d)
        y = rng.random((d, N))
        yp = rng.random((d, N))
        out = hm.eval_kernel(hm.KernelFunction(kern), y, yp)
        print(kern, d, N, float(out.sum()), flush=True)
