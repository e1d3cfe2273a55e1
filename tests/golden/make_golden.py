#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs oracle/_ref/libhmat_ref.so (built by `make -C oracle` from /root/reference) single-
threaded and stores, per case, the reference's own outputs:

* Morton codes of fixed point sets (compute_morton_codes, morton.cpp:37-48) and
  morton_order permutations (morton.cpp:50-71), including clamped coordinates;
* setup(): Morton-ordered coordinates, permutation, canonical dense / aca leaf lists with
  their bounding boxes (hmatrix.cpp:38-64, tree.cpp:140-195);
* mvp(): z = H x for x = SplitMix64(7).symmetric() (hmatrix.cpp:66-123);
* batched-ACA pivots / ranks of every admissible block (aca.cpp:268-544);
* the explicit-matrix seam (aca.cpp:567-578) on exact low-rank blocks.

The fixtures pin the C restatement (tests/test_oracle_golden.py) on machines without
/root/reference (the GPU box).  Re-run after changing any case: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle.bind import Reference  # noqa: E402
from paper_1708_09707_b200.inputs import axis_major_points, halton_points, symmetric, uniform_points  # noqa: E402

# (name, n, d, c_leaf, kernel, k, eta, epsilon, points)
CASES = [
    ("u1000_d2_c32", 1000, 2, 32, 0, 16, 1.5, None, "uniform"),
    ("u777_d1_c16", 777, 1, 16, 0, 16, 1.5, None, "uniform"),
    ("u2000_d4_c48", 2000, 4, 48, 0, 16, 1.5, None, "uniform"),
    ("u4096_d3_c64_matern", 4096, 3, 64, 1, 16, 1.5, None, "uniform"),
    ("u3001_d2_c24_matern_k8", 3001, 2, 24, 1, 8, 1.5, None, "uniform"),
    ("h2048_d2_c64_k6", 2048, 2, 64, 0, 6, 1.5, None, "halton"),
    ("u1500_d2_c32_eta07_eps", 1500, 2, 32, 0, 10, 0.7, 1e-4, "uniform"),
    ("c1_u16384_d2_c64_eps", 1 << 14, 2, 64, 0, 16, 1.5, 1e-6, "uniform"),
]


def points(kind, n, d):
    return uniform_points(n, d, 42) if kind == "uniform" else halton_points(n, d)


def main():
    R = Reference()
    out = {}
    # Morton known-answer sets
    rng_sets = {
        "mort_d1": axis_major_points(300, 1, 101),
        "mort_d2": axis_major_points(512, 2, 102),
        "mort_d3": axis_major_points(300, 3, 77),
        "mort_d5": axis_major_points(512, 5, 105),
    }
    clamp = np.array([[-0.25, 1.5, 1.0, 0.0, 0.5, -0.0, 0.999999999], [0.3, -2.0, 1.0, 0.0, 0.5, 1e-300, 0.25]])
    rng_sets["mort_clamp_d2"] = clamp
    dup = np.array([[0.4, 0.4, 0.2, 0.4], [0.4, 0.4, 0.9, 0.4]])
    rng_sets["mort_dup_d2"] = dup
    for name, c in rng_sets.items():
        out[name + "_coords"] = c
        out[name + "_codes"] = R.morton_codes(c)
        sc, sp = R.morton_order(c)
        out[name + "_perm"] = sp
    for (name, n, d, c_leaf, kern, k, eta, eps, pk) in CASES:
        P = points(pk, n, d)
        h = R.setup(P, kernel=kern, c_leaf=c_leaf, k=k, eta=eta, epsilon=eps)
        coords, perm = h.points()
        out[name + "_perm"] = perm
        for which, tag in ((0, "dense"), (1, "aca")):
            lv = h.leaves(which)
            out[f"{name}_{tag}_rows"] = lv.rows.astype(np.int32)
            out[f"{name}_{tag}_boxes"] = lv.boxes
        x = symmetric(7, n)
        out[name + "_z"] = h.mvp(x)
        f = h.aca_all(factors=False)
        out[name + "_keff"] = f["k_eff"].astype(np.int8)
        out[name + "_rowpiv"] = f["row_piv"].astype(np.int32)
        out[name + "_colpiv"] = f["col_piv"].astype(np.int32)
        print(name, "dense", h.count(0), "aca", h.count(1), "|z|", float(np.linalg.norm(out[name + "_z"])))
    # explicit-matrix seam: exact low-rank blocks, zero / constant / first-column-zero blocks
    rng = np.random.default_rng(5)
    blocks = []
    for b in range(10):
        m, nn, r = rng.integers(3, 40), rng.integers(3, 40), rng.integers(1, 6)
        blocks.append(rng.uniform(-1, 1, (m, r)) @ rng.uniform(-1, 1, (r, nn)))
    blocks.append(np.zeros((5, 4)))
    blocks.append(np.ones((4, 3)))
    z3 = np.zeros((3, 3))
    z3[0, 1] = 2.0
    z3[1, 2] = 1.0
    blocks.append(z3)
    for i, bl in enumerate(blocks):
        out[f"seam_block{i}"] = bl
    for kmax, eps, eta, tag in ((4, None, 0.0, "k4"), (6, 1e-6, 0.0, "k6eps"), (3, 1e-6, 1.5, "k3eta15")):
        ke, rp, cp, us, vs = R.aca_dense(blocks, kmax, eps, eta)
        out[f"seam_{tag}_keff"] = ke
        out[f"seam_{tag}_rowpiv"] = rp
        out[f"seam_{tag}_colpiv"] = cp
        out[f"seam_{tag}_u"] = np.concatenate([u.ravel() for u in us])
        out[f"seam_{tag}_v"] = np.concatenate([v.ravel() for v in vs])
    # kernel entries incl. the K1 continued-fraction branch
    rr = np.random.default_rng(3)
    for d in (2, 3):
        y = rr.uniform(0, 3, (d, 2000))
        yp = rr.uniform(0, 3, (d, 2000))
        yp[:, :20] = y[:, :20]
        out[f"kern_d{d}_y"] = y
        out[f"kern_d{d}_yp"] = yp
        out[f"kern_d{d}_gauss"] = R.eval_kernel(0, 0.0, y, yp)
        out[f"kern_d{d}_matern"] = R.eval_kernel(1, 0.0, y, yp)
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
