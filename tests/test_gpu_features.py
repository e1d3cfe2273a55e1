"""GPU tests of the remaining reference surface and of the B200 placement features:
row-cluster ownership (world > 1) rank by rank, recompute-mode chunking, the epsilon
criterion, CG, relative_error, edge cases, error behaviour, and parity at the bench
configuration (N = 2^20) through the row-sampled oracle."""
import numpy as np
import pytest

from paper_1708_09707_b200.inputs import halton_points, symmetric, uniform_points
from paper_1708_09707_b200.partition import row_slices

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("stored", [False, True])
def test_rank_slices_concatenate_to_single_gpu_product(gpu, oracle, world, stored):
    n, d = 1 << 14, 2
    P = uniform_points(n, d, 42)
    x = symmetric(7, n)
    o = oracle.setup(P, c_leaf=64, k=16)
    _, perm = o.points()
    zm = np.empty(n)
    zm[:] = o.mvp(x)[perm]  # Morton order
    for r, (lo, hi) in enumerate(row_slices(n, world)):
        h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, k=16, precompute_aca=stored,
                                                                  near_stored=stored, rank=r, world=world))
        st = h.stats()
        assert (st["row_begin"], st["row_end"]) == (lo, hi)
        assert np.array_equal(bits(h.mvp_local(x)), bits(zm[lo:hi]))
        h.close()


def test_world_gt1_without_nccl_fails_loudly(gpu):
    P = uniform_points(4096, 2, 42)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, rank=0, world=2))
    with pytest.raises(gpu.HmError) as e:
        h.mvp(symmetric(7, 4096))
    assert e.value.status == gpu.HM_ENCCL


@pytest.mark.parametrize("chunk_rows", [64, 1000, 0])
def test_recompute_mode_chunking_is_exact(gpu, oracle, chunk_rows):
    n = 1 << 13
    P = uniform_points(n, 2, 42)
    x = symmetric(7, n)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, aca_chunk_rows=chunk_rows))
    assert np.array_equal(bits(h.mvp(x)), bits(oracle.setup(P, c_leaf=64).mvp(x)))


@pytest.mark.parametrize("kind", [0, 1])
def test_epsilon_mode_active_below_eta_one(gpu, oracle, kind):
    n = 1500
    P = uniform_points(n, 2, 42)
    x = symmetric(7, n)
    name = "matern" if kind else "gaussian"
    h = gpu.setup(P, gpu.KernelFunction(name), gpu.HmatrixConfig(c_leaf=32, k=10, eta=0.7, epsilon=1e-4))
    o = oracle.setup(P, kernel=kind, c_leaf=32, k=10, eta=0.7, epsilon=1e-4)
    fh, fo = h.aca_factors(), o.aca_all()
    assert np.array_equal(fh["k_eff"], fo["k_eff"])
    assert np.any(fh["k_eff"] < 10)  # the criterion actually stopped some blocks
    assert np.array_equal(bits(h.mvp(x)), bits(o.mvp(x)))


def test_relative_error_matches_reference(gpu, oracle):
    n = 4096
    P = uniform_points(n, 2, 42)
    x = symmetric(19, n)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64))
    o = oracle.setup(P, c_leaf=64)
    e_gpu = gpu.relative_error(h, None, x)
    e_orc = o.relative_error(x)
    assert e_gpu == pytest.approx(e_orc, rel=1e-12)
    assert np.array_equal(bits(h.dense_mvp(x)), bits(oracle_dense(oracle, P, x)))


def oracle_dense(oracle, P, x):
    h = oracle.setup(P, c_leaf=64)
    z = np.empty(P.shape[1])
    oracle._check(oracle.lib.orc_dense_mvp(h.h, x.ctypes.data, z.ctypes.data))
    return z


def test_rank_sweep_improves_error(gpu):
    n = 2048
    P = halton_points(n, 2)
    x = symmetric(23, n)
    prev = 1e9
    for k in (2, 8, 16):
        h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, k=k))
        e = gpu.relative_error(h, None, x)
        assert e < prev
        prev = e
    assert prev <= 1e-6


def test_cg_solve_matches_oracle(gpu, oracle):
    n = 4096
    P = uniform_points(n, 2, 42)
    b = symmetric(43, n)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, precompute_aca=True, near_stored=True))
    r = gpu.cg_solve(h, None, b, gpu.SolveConfig(sigma2=1.0, tol=1e-8))
    xo, ito, rro = oracle.setup(P, c_leaf=64).cg(b, 1.0, 1e-8, 500)
    assert abs(r.iterations - ito) <= 1
    assert r.relative_residual <= 1e-7
    assert np.linalg.norm(r.x - xo) / np.linalg.norm(xo) <= 1e-9


def test_cg_zero_rhs_and_validation(gpu):
    P = uniform_points(1024, 2, 42)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64))
    r = gpu.cg_solve(h, None, np.zeros(1024), gpu.SolveConfig(sigma2=1.0))
    assert r.iterations == 0 and not np.any(r.x)
    with pytest.raises(gpu.InvalidArgument):
        gpu.cg_solve(h, None, np.ones(1024), gpu.SolveConfig(tol=0.0))
    with pytest.raises(gpu.InvalidArgument):
        gpu.cg_solve(h, None, np.ones(1023), gpu.SolveConfig())


@pytest.mark.parametrize("n,d,c_leaf", [(1, 2, 64), (2, 1, 1), (3, 3, 1), (100, 2, 256), (513, 20, 16), (64, 2, 64)])
def test_edge_sizes(gpu, oracle, n, d, c_leaf):
    P = uniform_points(n, d, 9)
    x = symmetric(5, n)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=c_leaf, k=4))
    o = oracle.setup(P, c_leaf=c_leaf, k=4)
    for w in (0, 1):
        assert np.array_equal(h.leaves(w).rows, o.leaves(w).rows)
    assert np.array_equal(bits(h.mvp(x)), bits(o.mvp(x)))


def test_duplicate_and_clamped_points(gpu, oracle):
    n = 2000
    P = uniform_points(n, 2, 3)
    P[:, 500:900] = P[:, 100:500]           # duplicates
    P[:, :50] = 0.25                         # coincident cluster
    P[0, 1900:] = 1.7                        # outside [0,1]: Morton clamps, kernel uses raw values
    P[1, 1950:] = -0.3
    x = symmetric(5, n)
    for kind, name in ((0, "gaussian"), (1, "matern")):
        h = gpu.setup(P, gpu.KernelFunction(name), gpu.HmatrixConfig(c_leaf=32, k=12))
        o = oracle.setup(P, kernel=kind, c_leaf=32, k=12)
        assert np.array_equal(h.codes(), oracle.morton_codes(P))
        for w in (0, 1):
            lh, lo = h.leaves(w), o.leaves(w)
            assert np.array_equal(lh.rows, lo.rows)
            assert np.array_equal(bits(lh.boxes), bits(lo.boxes))
        assert np.array_equal(bits(h.mvp(x)), bits(o.mvp(x)))


def test_morton_primitives(gpu, oracle):
    from paper_1708_09707_b200.inputs import axis_major_points
    for d in (1, 2, 3, 5, 20):
        c = axis_major_points(3000, d, 11 + d)
        assert np.array_equal(gpu.morton_codes(c), oracle.morton_codes(c))
        sc, sp = gpu.morton_order(c, np.arange(3000) + 1000)
        oc, op = oracle.morton_order(c, np.arange(3000) + 1000)
        assert np.array_equal(sp, op) and np.array_equal(bits(sc), bits(oc))


def test_errors_map_to_reference_exception_kinds(gpu):
    P = uniform_points(256, 2, 1)
    with pytest.raises(gpu.InvalidArgument):
        gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(eta=-1.0))
    with pytest.raises(gpu.InvalidArgument):
        gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(k=0))
    with pytest.raises(gpu.InvalidArgument):
        gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=0))
    with pytest.raises(gpu.InvalidArgument):
        gpu.setup(P, gpu.KernelFunction("matern", matern_beta=3.7), gpu.HmatrixConfig())
    with pytest.raises(gpu.InvalidArgument):
        gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(bs_dense=10, c_leaf=16, force_dense=True))
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=16))
    with pytest.raises(gpu.InvalidArgument):
        h.mvp(np.zeros(255))
    bad = P.copy()
    bad[0, 3] = np.nan
    with pytest.raises(gpu.InvalidArgument):
        gpu.setup(bad, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=16))


def test_bench_config_parity_row_sampled(gpu, oracle):
    """BASELINE configs[1] geometry (N = 2^20, d = 2, C_leaf = 64, stored operator):
    tree and leaf lists bit-exact, and sampled rows of the product bitwise equal to the
    reference's order (row-sampled oracle)."""
    n, d = 1 << 20, 2
    P = uniform_points(n, d, 42)
    x = symmetric(43, n)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=64, k=16, precompute_aca=True, near_stored=True))
    o = oracle.setup(P, c_leaf=64, k=16)
    _, perm = o.points()
    _, hperm = h.points()
    assert np.array_equal(perm, hperm)
    for w in (0, 1):
        assert np.array_equal(h.leaves(w, boxes=False).rows, o.leaves(w, boxes=False).rows)
    z = h.mvp(x)
    zm = z[perm]
    ranges = [(0, 64), (262144, 262208), (700032, 700096), (n - 64, n)]
    zo = o.mvp_rows(x, ranges)
    for lo, hi in ranges:
        assert np.array_equal(bits(zm[lo:hi]), bits(zo[lo:hi]))


@pytest.mark.parametrize("n,d,c_leaf", [(64, 2, 8), (3001, 2, 48), (4096, 3, 64)])
def test_leaf_csv_dump_matches_reference(gpu, n, d, c_leaf, tmp_path):
    """dump_leaves_csv (tree.cpp:197-205): same file, byte for byte, as the reference's own
    function on the same points (oracle/_ref), header and canonical leaf order included."""
    from oracle.bind import available, reference_leaf_csv
    P = uniform_points(n, d, 79)
    h = gpu.setup(P, gpu.KernelFunction(), gpu.HmatrixConfig(c_leaf=c_leaf))
    ours = tmp_path / "ours.csv"
    h.dump_leaves_csv(str(ours))
    lines = ours.read_text().splitlines()
    assert lines[0] == "row_lower,row_upper,col_lower,col_upper,admissible"
    st = h.stats()
    assert len(lines) - 1 == st["n_dense"] + st["n_aca"]
    if available("ref"):
        ref = tmp_path / "ref.csv"
        reference_leaf_csv(P, c_leaf, 1.5, ref)
        assert ours.read_bytes() == ref.read_bytes()
    with pytest.raises(gpu.HmError):
        h.dump_leaves_csv(str(tmp_path / "no_such_dir" / "x.csv"))


@pytest.mark.parametrize("cfg", [
    # BASELINE configs[2]: N=2^22, [0,1]^3, Matern (nu = 1), matrix-free near field
    dict(n=1 << 22, d=3, kernel="matern", kind=1),
    # BASELINE configs[3] geometry: N=2^24, [0,1]^3, Gaussian, matrix-free (one GPU)
    dict(n=1 << 24, d=3, kernel="gaussian", kind=0),
], ids=["C3_2^22_d3_matern", "C4_2^24_d3_gaussian"])
def test_full_size_configs_row_sampled(gpu, oracle, cfg):
    """BASELINE configs 3 and 4 at their full N, in the reference's default recompute mode
    (ACA inside every product): sampled row clusters of the GPU product are bitwise equal
    to the reference order (row-sampled oracle)."""
    n, d = cfg["n"], cfg["d"]
    P = uniform_points(n, d, 42)
    x = symmetric(43, n)
    h = gpu.setup(P, gpu.KernelFunction(cfg["kernel"]), gpu.HmatrixConfig(c_leaf=64, k=16))
    z = h.mvp(x)
    o = oracle.setup(P, kernel=cfg["kind"], c_leaf=64, k=16)
    _, perm = o.points()
    _, hperm = h.points()
    assert np.array_equal(perm, hperm)
    zm = z[perm]
    S = n >> h.stats()["dmax_leaf"]
    ranges = [(0, S), (n // 3 // S * S, n // 3 // S * S + S), (n - S, n)]
    zo = oracle_rows = o.mvp_rows(x, ranges)
    for lo, hi in ranges:
        assert np.array_equal(bits(zm[lo:hi]), bits(oracle_rows[lo:hi])), (lo, np.max(np.abs(zm[lo:hi] - zo[lo:hi])))


def test_cli_compatible_csv_outputs(gpu, oracle, tmp_path):
    """tools/hmat_csv.py writes the reference CLI's CSV formats (hmat_cli.cpp:117-255):
    headers, one row per phase, and --dump-leaves as dense queue then aca queue."""
    import subprocess
    import sys as _sys
    from paper_1708_09707_b200.inputs import halton_points
    repo = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    tool = [_sys.executable, f"{repo}/tools/hmat_csv.py"]
    out = tmp_path / "bench.csv"
    leaves = tmp_path / "leaves.csv"
    subprocess.run(tool + ["--command", "mvp-bench", "--n", "4096", "--c-leaf", "64", "--trials", "2", "--precompute",
                           "--out", str(out), "--dump-leaves", str(leaves)], check=True)
    rows = out.read_text().splitlines()
    assert rows[0] == "phase,n,d,k,eta,c_leaf,time_ms_mean,time_ms_std"
    assert [r.split(",")[0] for r in rows[1:]] == ["setup", "mvp", "mvp_dense", "mvp_aca"]
    assert all(r.split(",")[1:6] == ["4096", "2", "16", "1.5", "64"] for r in rows[1:])
    o = oracle.setup(halton_points(4096, 2), c_leaf=64, k=16)
    want = np.concatenate([np.column_stack([o.leaves(w, boxes=False).rows, np.full(o.count(w), w)]) for w in (0, 1)])
    got = np.loadtxt(leaves, delimiter=",", skiprows=1, dtype=np.int64)
    assert np.array_equal(got, want)
    conv = subprocess.run(tool + ["--command", "convergence", "--n", "2048", "--c-leaf", "64", "--trials", "1"],
                          check=True, capture_output=True, text=True).stdout.splitlines()
    assert conv[0] == "kernel,d,k,e_rel_mean" and len(conv) == 9
    errs = [float(r.split(",")[3]) for r in conv[1:5]]
    assert errs == sorted(errs, reverse=True) and errs[-1] < 1e-6
