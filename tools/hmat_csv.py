#!/usr/bin/env python3
"""CSV outputs of the reference CLI (tools/hmat_cli.cpp) from the B200 engine.

Same options, same inputs (Halton points, SplitMix64 random vectors, hmat_cli.cpp:74-79)
and the same CSV columns, so reference-side scripts that read the CLI's output can read
these.  Commands (hmat_cli.cpp:117-255, 410-441):

  mvp-bench   phase,n,d,k,eta,c_leaf,time_ms_mean,time_ms_std   (setup, mvp, mvp_dense, mvp_aca)
  complexity  phase,n,d,k,eta,c_leaf,time_ms_mean,time_ms_std   (spatial, traversal, mvp per N)
  convergence kernel,d,k,e_rel_mean                             (k = 2, 4, 8, 16; no N limit:
                                                                 the exact product runs on the GPU)
  solve       one value of x per line (17 digits); iterations / residual on stderr
  batch-sweep bs,phase,n,d,k,c_leaf,time_ms_mean,time_ms_min    (bs_aca sweep: 0, 2^14..2^22 step 4x,
                                                                 phase aca; bs_dense sweep: 0,
                                                                 2^16..2^24 step 4x, phase dense;
                                                                 hmat_cli.cpp:241-283)

mvp_dense / mvp_aca come from the per-kernel event clock: the near-field kernels and the
far-field kernels (ACA factorisation included in recompute mode) of one product.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1708_09707_b200 as hm  # noqa: E402
from paper_1708_09707_b200.inputs import halton_points, symmetric  # noqa: E402


def g(v) -> str:
    """C++ ostream default formatting (6 significant digits)."""
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    return format(float(v), ".6g")


def summarize(samples):
    m = sum(samples) / len(samples)
    var = sum((s - m) ** 2 for s in samples) / len(samples)
    return m, math.sqrt(var)


def config(a, **kw):
    c = dict(eta=a.eta, c_leaf=a.c_leaf, k=a.k, bs_aca=a.bs_aca, bs_dense=a.bs_dense, precompute_aca=a.precompute,
             near_stored=a.near_stored, force_dense=a.force_dense)
    c.update(kw)
    return hm.HmatrixConfig(**c)


def split_ms(prof: dict) -> tuple[float, float]:
    near = prof.get("near_pairs", (0.0, 0))[0]
    far = sum(prof.get(k, (0.0, 0))[0] for k in ("lowrank_t", "aca", "rows_far"))
    rows = prof.get("rows", (0.0, 0))[0]
    if near == 0.0:  # rows kernel = near field (recompute / generic); far kernels separate
        return rows, far
    return near, far + rows  # symmetric near field: rows folds partials + the low-rank part


def cmd_mvp_bench(a, out):
    kern = hm.KernelFunction(a.kernel)
    raw = halton_points(a.n, a.d)
    t0 = time.perf_counter()
    h = hm.setup(raw, kern, config(a))
    setup_ms = [(time.perf_counter() - t0) * 1e3]
    if a.dump_leaves:
        # hmat_cli.cpp:213-218: dense queue then aca queue, not re-sorted
        with open(a.dump_leaves, "w") as f:
            f.write("row_lower,row_upper,col_lower,col_upper,admissible\n")
            for w, q in ((0, h.dense_queue), (1, h.aca_queue)):
                for r in q:
                    f.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{w}\n")
    x = symmetric(a.seed, a.n)
    mvp_ms, dense_ms, aca_ms = [], [], []
    for _ in range(a.trials):
        h.profile_begin()
        t = hm.MvpTimings()
        h.mvp(x, t)
        near, far = split_ms(h.profile_end())
        mvp_ms.append(t.total_ms)
        dense_ms.append(near)
        aca_ms.append(far)
    out.append("phase,n,d,k,eta,c_leaf,time_ms_mean,time_ms_std")
    for name, s in (("setup", setup_ms), ("mvp", mvp_ms), ("mvp_dense", dense_ms), ("mvp_aca", aca_ms)):
        m, sd = summarize(s)
        out.append(",".join([name, g(a.n), g(a.d), g(a.k), g(a.eta), g(a.c_leaf), g(m), g(sd)]))


def cmd_complexity(a, out):
    sizes = []
    n = 1 << 14
    while n < a.n:
        sizes.append(n)
        n <<= 1
    sizes.append(a.n)
    if len(sizes) > 1 and sizes[-2] == a.n:
        sizes.pop()
    kern = hm.KernelFunction(a.kernel)
    out.append("phase,n,d,k,eta,c_leaf,time_ms_mean,time_ms_std")
    for n in sizes:
        raw = halton_points(n, a.d)
        spatial, traversal = [], []
        for _ in range(a.trials):
            h = hm.setup(raw, kern, config(a, precompute_aca=False, near_stored=False))
            tm = h.timings()
            spatial.append(tm["morton_ms"])
            traversal.append(tm["tree_ms"])
            h.close()
        h = hm.setup(raw, kern, config(a))
        x = symmetric(a.seed, n)
        mvp = []
        for _ in range(a.trials):
            t = hm.MvpTimings()
            h.mvp(x, t)
            mvp.append(t.total_ms)
        for name, s in (("spatial", spatial), ("traversal", traversal), ("mvp", mvp)):
            m, sd = summarize(s)
            out.append(",".join([name, g(n), g(a.d), g(a.k), g(a.eta), g(a.c_leaf), g(m), g(sd)]))


def cmd_convergence(a, out):
    raw = halton_points(a.n, a.d)
    xs = [symmetric(a.seed + t, a.n) for t in range(a.trials)]
    out.append("kernel,d,k,e_rel_mean")
    for name in ("gaussian", "matern"):
        kern = hm.KernelFunction(name)
        exact = None
        for k in (2, 4, 8, 16):
            h = hm.setup(raw, kern, config(a, k=k))
            if exact is None:
                exact = [h.dense_mvp(x) for x in xs]
            mean = 0.0
            for x, ex in zip(xs, exact):
                z = h.mvp(x)
                mean += math.sqrt(float(np.sum((z - ex) ** 2)) / float(np.sum(ex * ex)))
            out.append(",".join([name, g(a.d), g(k), g(mean / a.trials)]))


def cmd_solve(a, out):
    kern = hm.KernelFunction(a.kernel)
    h = hm.setup(halton_points(a.n, a.d), kern, config(a))
    b = np.loadtxt(a.rhs, dtype=np.float64).reshape(-1) if a.rhs else symmetric(a.seed, a.n)
    r = hm.cg_solve(h, kern, b, hm.SolveConfig(sigma2=a.sigma2, tol=a.tol, max_iter=a.max_iter))
    out.extend(repr(float(v)) for v in r.x)
    print(f"iterations {r.iterations}, relative residual {r.relative_residual:g}", file=sys.stderr)


def cmd_batch_sweep(a, out):
    """hmat_cli.cpp:241-283: MvpTimings aca_ms / dense_ms of `trials` products per batch
    size (recompute mode unless --precompute).  On the device bs_aca sets the reference's
    ACA batches, chunks are runs of whole batches; bs_dense only bounds the block size."""
    kern = hm.KernelFunction(a.kernel)
    P = halton_points(a.n, a.d)
    x = symmetric(a.seed, a.n)
    out.append("bs,phase,n,d,k,c_leaf,time_ms_mean,time_ms_min")

    def measure(bs_aca, bs_dense):
        h = hm.setup(P, kern, config(a, bs_aca=bs_aca, bs_dense=bs_dense))
        aca, dense = [], []
        for _ in range(a.trials):
            t = hm.MvpTimings()
            h.mvp(x, t)
            aca.append(t.aca_ms)
            dense.append(t.dense_ms)
        h.close()
        return aca, dense

    sweep = [0] + [1 << e for e in range(14, 23, 2)]
    for bs in sweep:
        aca, _ = measure(bs, a.bs_dense)
        out.append(",".join([g(bs), "aca", g(a.n), g(a.d), g(a.k), g(a.c_leaf), g(summarize(aca)[0]), g(min(aca))]))
    sweep = [0] + [1 << e for e in range(16, 25, 2)]
    for bs in sweep:
        _, dense = measure(a.bs_aca, bs)
        out.append(",".join([g(bs), "dense", g(a.n), g(a.d), g(a.k), g(a.c_leaf), g(summarize(dense)[0]),
                             g(min(dense))]))


def main(argv=None):
    ap = argparse.ArgumentParser(description="reference-CLI-compatible CSV outputs")
    ap.add_argument("--command", required=True, choices=["mvp-bench", "complexity", "convergence", "solve",
                                                               "batch-sweep"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--kernel", default="gaussian", choices=["gaussian", "matern"])
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--eta", type=float, default=1.5)
    ap.add_argument("--c-leaf", dest="c_leaf", type=int, default=256)
    ap.add_argument("--bs-aca", dest="bs_aca", type=int, default=1 << 20)
    ap.add_argument("--bs-dense", dest="bs_dense", type=int, default=1 << 22)
    ap.add_argument("--precompute", action="store_true")
    ap.add_argument("--near-stored", dest="near_stored", action="store_true", help="(B200) keep dense leaves in HBM")
    ap.add_argument("--force-dense", dest="force_dense", action="store_true")
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--out", default="")
    ap.add_argument("--rhs", default="")
    ap.add_argument("--dump-leaves", dest="dump_leaves", default="")
    ap.add_argument("--sigma2", type=float, default=1.0)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-iter", dest="max_iter", type=int, default=500)
    a = ap.parse_args(argv)
    out: list[str] = []
    {"mvp-bench": cmd_mvp_bench, "complexity": cmd_complexity, "convergence": cmd_convergence,
     "solve": cmd_solve, "batch-sweep": cmd_batch_sweep}[a.command](a, out)
    text = "\n".join(out) + "\n"
    if a.out:
        with open(a.out, "w") as f:  # rows collected first: no partial files (hmat_cli.cpp:104-106)
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
