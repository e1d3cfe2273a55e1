"""Multi-RHS throughput (BASELINE config 5 style).

For a configuration: R right-hand sides per operator pass, exact vs DMMA near field,
device-resident X (CUDA events around K passes after W warm-ups).  Prints one JSON
line per variant: ms per pass, GFLOP/s = 2 R (S_d + S_l) / t, and the speed-up over R
single-RHS products of the same handle.
usage: python tools/bench_multi.py --n 262144 --d 4 --mode recompute --nrhs 16
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 18)
    ap.add_argument("--d", type=int, default=4)
    ap.add_argument("--kernel", default="gaussian")
    ap.add_argument("--mode", choices=["stored", "recompute"], default="recompute")
    ap.add_argument("--nrhs", type=int, default=16)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1708_09707_b200 as hm
    from paper_1708_09707_b200.inputs import symmetric, uniform_points

    n, d, R = args.n, args.d, args.nrhs
    stored = args.mode == "stored"
    t0 = time.perf_counter()
    h = hm.setup(uniform_points(n, d, 42), hm.KernelFunction(args.kernel),
                 hm.HmatrixConfig(c_leaf=64, k=16, precompute_aca=stored, near_stored=stored))
    build_s = time.perf_counter() - t0
    st = h.stats()
    f = h.aca_factors(factors=False) if not stored else None
    if stored:
        S_l = st["S_l"]
    else:
        lv = h.aca_queue
        S_l = float((f["k_eff"] * ((lv[:, 1] - lv[:, 0]) + (lv[:, 3] - lv[:, 2]))).sum())
    flops1 = 2.0 * (st["S_d"] + S_l)
    X = torch.from_numpy(np.stack([symmetric(43 + r, n) for r in range(R)])).cuda()  # rhs-major = n x R col-major
    Z = torch.empty_like(X)
    s = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.steps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    single = timed(lambda: h.mvp_device(X[0].data_ptr(), Z[0].data_ptr(), s.cuda_stream))
    variants = [("exact", False)] + ([("dmma", True)] if not stored and R % 8 == 0 else [])
    for name, dm in variants:
        ms = timed(lambda: h.mvp_multi_device(X.data_ptr(), Z.data_ptr(), R, dmma=dm, stream=s.cuda_stream))
        print(json.dumps({"workload": f"H-MVP x {R} RHS, N={n} uniform [0,1]^{d}, {args.kernel}, C_leaf=64, k=16, "
                                      f"{args.mode} near/far field", "variant": name, "nrhs": R,
                          "ms_per_pass": ms, "gflops": R * flops1 / (ms * 1e-3) / 1e9,
                          "single_rhs_ms": single, "speedup_vs_R_single": R * single / ms,
                          "S_d": st["S_d"], "S_l": S_l, "build_s": build_s}), flush=True)


if __name__ == "__main__":
    main()
