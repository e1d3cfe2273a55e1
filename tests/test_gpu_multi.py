"""Multiple right-hand sides (BASELINE config 5).

Exact mode: every column of a multi-RHS product is BITWISE equal to the single-RHS
product of that column (which is itself bitwise equal to the reference order, see
test_gpu_parity.py), in every storage mode and for passes of 1..16 columns (more
columns run in several passes).  DMMA mode (recompute near field on the FP64 tensor
cores): within 1e-12 relative l2 of the exact product per column (the per-leaf sums
are reordered; the reference bar is 1e-8).  Block CG: every column follows exactly the
single-RHS cg_solve iteration.
"""
import numpy as np
import pytest

from paper_1708_09707_b200.inputs import symmetric, uniform_points

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def rhs(n, R, seed=43):
    return np.stack([symmetric(seed + r, n) for r in range(R)], axis=1)


CASES = [
    # (n, d, c_leaf, kernel, precompute, stored)   storage path exercised
    (4096, 2, 64, "gaussian", False, False),   # recompute near + per-product ACA chunks
    (4096, 2, 64, "gaussian", True, True),     # regular geometry: symmetric near field
    (3001, 2, 48, "matern", True, True),       # irregular: full stored blocks, rank-major U
    (2500, 3, 32, "gaussian", True, False),    # stored factors, recomputed near field
    (2000, 4, 64, "gaussian", False, False),   # config-5 geometry, small
]


@pytest.mark.parametrize("n,d,c_leaf,kern,pre,stored", CASES)
@pytest.mark.parametrize("R", [1, 3, 16, 20])
def test_exact_multi_equals_single_rhs_products(gpu, n, d, c_leaf, kern, pre, stored, R):
    P = uniform_points(n, d, 42)
    h = gpu.setup(P, gpu.KernelFunction(kern),
                  gpu.HmatrixConfig(c_leaf=c_leaf, k=16, precompute_aca=pre, near_stored=stored))
    X = rhs(n, R)
    Z = h.mvp_multi(X)
    for r in range(R):
        z1 = h.mvp(X[:, r])
        assert np.array_equal(bits(Z[:, r]), bits(z1)), f"column {r}: rel {np.linalg.norm(Z[:, r] - z1) / np.linalg.norm(z1)}"


def test_exact_multi_matches_oracle(gpu, oracle):
    n = 4096
    P = uniform_points(n, 2, 42)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, k=16, precompute_aca=True, near_stored=True))
    o = oracle.setup(P, c_leaf=64, k=16)
    X = rhs(n, 5, seed=7)
    Z = h.mvp_multi(X)
    for r in range(5):
        assert np.array_equal(bits(Z[:, r]), bits(o.mvp(X[:, r])))


@pytest.mark.parametrize("n,d,R", [(4096, 2, 8), (4096, 2, 16), (3000, 4, 16), (2000, 3, 24)])
def test_dmma_near_field_within_tolerance(gpu, n, d, R):
    P = uniform_points(n, d, 42)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, k=16))
    X = rhs(n, R)
    if R % 8:
        with pytest.raises(gpu.InvalidArgument):
            h.mvp_multi(X, dmma=True)
        return
    Zd = h.mvp_multi(X, dmma=True)
    Ze = h.mvp_multi(X)
    for r in range(R):
        rel = np.linalg.norm(Zd[:, r] - Ze[:, r]) / np.linalg.norm(Ze[:, r])
        assert rel <= 1e-12, (r, rel)


def test_dmma_rejects_stored_near_field(gpu):
    P = uniform_points(2048, 2, 42)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, precompute_aca=True, near_stored=True))
    with pytest.raises(gpu.InvalidArgument):
        h.mvp_multi(rhs(2048, 8), dmma=True)


def test_block_cg_follows_single_rhs_cg(gpu, oracle):
    """Config-5 style KRR solve (A + sigma^2 I) for several right-hand sides at once."""
    n = 4096
    P = uniform_points(n, 4, 42)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, k=16))
    B = rhs(n, 4)
    B[:, 2] = 0.0  # zero right-hand side: x = 0, no iterations (solver.cpp:31-34)
    cfg = gpu.SolveConfig(sigma2=1.0, tol=1e-8, max_iter=500)
    X, it, rr = gpu.cg_solve_multi(h, B, cfg)
    for r in range(4):
        s = gpu.cg_solve(h, None, B[:, r], cfg)
        assert it[r] == s.iterations
        assert np.array_equal(bits(X[:, r]), bits(s.x))
        assert rr[r] == s.relative_residual
    assert it[2] == 0 and not np.any(X[:, 2])
    xo, ito, _ = oracle.setup(P, c_leaf=64, k=16).cg(B[:, 0], 1.0, 1e-8, 500)
    assert abs(int(it[0]) - ito) <= 1
    assert np.linalg.norm(X[:, 0] - xo) / np.linalg.norm(xo) <= 1e-9
    Xd, itd, rrd = gpu.cg_solve_multi(h, B[:, :2].repeat(4, axis=1), cfg, dmma=True)
    assert np.all(rrd <= 1e-7)
    assert np.linalg.norm(Xd[:, 0] - X[:, 0]) / np.linalg.norm(X[:, 0]) <= 1e-9


def test_config5_full_size_multi_rhs(gpu):
    """BASELINE configs[4] geometry at full size: N = 2^22 uniform points in [0,1]^4, matrix-free
    (recompute) near and far field, 16 right-hand sides per pass.  Size-independent
    properties: exact-mode columns bitwise equal to single-RHS products, DMMA columns within
    1e-12 of them."""
    n, d, R = 1 << 22, 4, 16
    P = uniform_points(n, d, 42)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, k=16))
    X = rhs(n, R)
    Ze = h.mvp_multi(X)
    for r in (0, R - 1):
        assert np.array_equal(bits(Ze[:, r]), bits(h.mvp(X[:, r])))
    Zd = h.mvp_multi(X, dmma=True)
    rel = np.linalg.norm(Zd - Ze, axis=0) / np.linalg.norm(Ze, axis=0)
    assert np.all(rel <= 1e-12), rel.max()
