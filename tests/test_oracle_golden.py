"""Pin the C restatement (oracle/) against the reference's own outputs.

tests/golden/reference_golden.npz was produced by tests/golden/make_golden.py from the
unmodified reference library (oracle/_ref, single-threaded).  Every comparison is
bitwise: Morton codes/permutations, leaf lists + boxes, batched-ACA ranks and pivots,
H-MVP output, explicit-matrix ACA factors and kernel entries.
"""
import os

import numpy as np
import pytest

from paper_1708_09707_b200.inputs import halton_points, symmetric, uniform_points

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")

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


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("name", ["mort_d1", "mort_d2", "mort_d3", "mort_d5", "mort_clamp_d2", "mort_dup_d2"])
def test_morton_codes_and_order(G, oracle, name):
    c = G[name + "_coords"]
    assert np.array_equal(oracle.morton_codes(c), G[name + "_codes"])
    _, perm = oracle.morton_order(c)
    assert np.array_equal(perm, G[name + "_perm"])


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_setup_and_mvp_bitwise(G, oracle, case):
    name, n, d, c_leaf, kern, k, eta, eps, pk = case
    P = uniform_points(n, d, 42) if pk == "uniform" else halton_points(n, d)
    h = oracle.setup(P, kernel=kern, c_leaf=c_leaf, k=k, eta=eta, epsilon=eps)
    _, perm = h.points()
    assert np.array_equal(perm, G[name + "_perm"])
    for which, tag in ((0, "dense"), (1, "aca")):
        lv = h.leaves(which)
        assert np.array_equal(lv.rows, G[f"{name}_{tag}_rows"])
        assert np.array_equal(bits(lv.boxes), bits(G[f"{name}_{tag}_boxes"]))
    f = h.aca_all(factors=False)
    assert np.array_equal(f["k_eff"], G[name + "_keff"])
    assert np.array_equal(f["row_piv"], G[name + "_rowpiv"])
    assert np.array_equal(f["col_piv"], G[name + "_colpiv"])
    z = h.mvp(symmetric(7, n))
    assert np.array_equal(bits(z), bits(G[name + "_z"]))


def test_explicit_seam(G, oracle):
    blocks = []
    i = 0
    while f"seam_block{i}" in G:
        blocks.append(G[f"seam_block{i}"])
        i += 1
    for kmax, eps, eta, tag in ((4, None, 0.0, "k4"), (6, 1e-6, 0.0, "k6eps"), (3, 1e-6, 1.5, "k3eta15")):
        ke, rp, cp, us, vs = oracle.aca_dense(blocks, kmax, eps, eta)
        assert np.array_equal(ke, G[f"seam_{tag}_keff"])
        assert np.array_equal(rp, G[f"seam_{tag}_rowpiv"])
        assert np.array_equal(cp, G[f"seam_{tag}_colpiv"])
        assert np.array_equal(bits(np.concatenate([u.ravel() for u in us])), bits(G[f"seam_{tag}_u"]))
        assert np.array_equal(bits(np.concatenate([v.ravel() for v in vs])), bits(G[f"seam_{tag}_v"]))


@pytest.mark.parametrize("d", [2, 3])
def test_kernel_entries(G, oracle, d):
    y, yp = G[f"kern_d{d}_y"], G[f"kern_d{d}_yp"]
    assert np.array_equal(bits(oracle.eval_kernel(0, 0.0, y, yp)), bits(G[f"kern_d{d}_gauss"]))
    assert np.array_equal(bits(oracle.eval_kernel(1, 0.0, y, yp)), bits(G[f"kern_d{d}_matern"]))


def test_c1_norm_anchor(G):
    """‖z‖ of config 1 (3815.9949482622451 as a left-fold sum)."""
    z = G["c1_u16384_d2_c64_eps_z"]
    acc = 0.0
    for v in z:
        acc += v * v
    assert abs(acc ** 0.5 - 3815.9949482622451) < 1e-9
