"""Reference CPU arm of bench.py (TEST/BASELINE INFRASTRUCTURE ONLY).

Times the UNMODIFIED reference library (oracle/_ref/libhmat_ref.so, built from
/root/reference by oracle/Makefile) on a bounded row sample of the bench workload,
with the reference's fastest product path (precompute_aca=true: factors formed
first, then the mvp() body of hmatrix.cpp:80-113 over the sampled rows).

The reference's worker pool races with more than one thread, so the
host cores are used by running one single-threaded process per core, each on a
disjoint set of leaf-level row clusters.  Throughput = sum of flops / max time.

    python -m oracle.refbench --n 1048576 --d 2 --clusters 0,17 --reps 3 --warmup 1
prints one JSON object (this worker's numbers).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def cluster_ranges(n: int, depth: int, ids):
    out = []
    for idx in ids:
        lo, hi = 0, n
        for b in range(depth - 1, -1, -1):
            mid = lo + (hi - lo + 1) // 2
            if (idx >> b) & 1:
                lo = mid
            else:
                hi = mid
        out.append((lo, hi))
    return out


def leaf_depth(n: int, c_leaf: int) -> int:
    d = 0
    while ((n - 1) >> d) + 1 > c_leaf:
        d += 1
    return d


def worker(args) -> dict:
    os.environ.setdefault("HMAT_THREADS", "1")
    import ctypes as C
    from oracle.bind import Reference
    from paper_1708_09707_b200.inputs import uniform_points, symmetric
    R = Reference()
    L = R.lib
    L.ref_mvp_rows_timed.restype = C.c_int
    L.ref_mvp_rows_timed.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    n, d = args.n, args.d
    pts = uniform_points(n, d, 42)
    t0 = time.perf_counter()
    h = R.setup(pts, kernel=args.kernel, c_leaf=args.c_leaf, k=args.k, eta=args.eta)
    t_setup = (time.perf_counter() - t0) * 1e3
    depth = leaf_depth(n, args.c_leaf)
    ids = [int(c) for c in args.clusters.split(",") if c != ""]
    ranges = np.array(cluster_ranges(n, depth, ids), dtype=np.int64).reshape(-1)
    x = symmetric(43, n)
    z = np.zeros(n)
    ta, tm, fl = C.c_double(), C.c_double(), C.c_double()
    if args.warmup:
        R._check(L.ref_mvp_rows_timed(h.h, x.ctypes.data, ranges.size // 2, ranges.ctypes.data, args.warmup,
                                      z.ctypes.data, C.byref(ta), C.byref(tm), C.byref(fl)))
    R._check(L.ref_mvp_rows_timed(h.h, x.ctypes.data, ranges.size // 2, ranges.ctypes.data, args.reps,
                                  z.ctypes.data, C.byref(ta), C.byref(tm), C.byref(fl)))
    rows = int(sum(hi - lo for lo, hi in cluster_ranges(n, depth, ids)))
    return {"flops_per_rep": fl.value, "reps": args.reps, "t_mvp_ms": tm.value, "t_aca_ms": ta.value,
            "t_setup_ms": t_setup, "rows": rows, "clusters": ids, "threads": int(L.ref_threads())}


def leaves_worker(args) -> dict:
    """Recompute-mode sample: the reference's mvp() body with ACA inside the product over
    the explicit leaf sample in args.leaves (npz written by bench.py; see
    ref_leaves_mvp_timed in ref_driver.cpp)."""
    os.environ.setdefault("HMAT_THREADS", "1")
    import ctypes as C
    from oracle.bind import Reference
    R = Reference()
    L = R.lib
    L.ref_leaves_mvp_timed.restype = C.c_int
    L.ref_leaves_mvp_timed.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_double,
                                       C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                       C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    z = np.load(args.leaves)
    coords = np.ascontiguousarray(z["coords"], dtype=np.float64)
    d, n = coords.shape
    dense = np.ascontiguousarray(z["dense"], dtype=np.int64)
    aca = np.ascontiguousarray(z["aca"], dtype=np.int64)
    x = np.ascontiguousarray(z["x"], dtype=np.float64)
    out = np.zeros(n)
    tm, fl = C.c_double(), C.c_double()
    R._check(L.ref_leaves_mvp_timed(coords.ctypes.data, n, d, int(z["kernel"]), 0.0, int(z["k"]), float(z["eta"]),
                                    dense.shape[0], dense.ctypes.data, aca.shape[0], aca.ctypes.data, x.ctypes.data,
                                    args.reps, out.ctypes.data, C.byref(tm), C.byref(fl)))
    return {"flops_per_rep": fl.value, "reps": args.reps, "t_mvp_ms": tm.value, "t_aca_ms": 0.0, "t_setup_ms": 0.0,
            "rows": int(np.unique(np.concatenate([dense[:, 0], aca[:, 0]])).size) if dense.size + aca.size else 0,
            "leaves": int(dense.shape[0] + aca.shape[0]), "threads": int(L.ref_threads())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=str, default="")
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--c-leaf", dest="c_leaf", type=int, default=64)
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--eta", type=float, default=1.5)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--clusters", type=str, default="0")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=0)
    args = ap.parse_args()
    print(json.dumps(leaves_worker(args) if args.leaves else worker(args)))


if __name__ == "__main__":
    main()
