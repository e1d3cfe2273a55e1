import os
"""Live cross-check of the C restatement against the unmodified reference (oracle/_ref),
on randomised configurations, plus the SURVEY.md findings the parity targets rest on.
Skipped where oracle/_ref is not built."""
import numpy as np
import pytest

from paper_1708_09707_b200.inputs import axis_major_points, symmetric, uniform_points


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


CONFIGS = [
    # n, d, c_leaf, kernel, k, eta
    (50, 2, 8, 0, 4, 1.5),
    (333, 3, 20, 1, 6, 1.2),
    (1111, 2, 37, 0, 12, 2.0),
    (2500, 1, 64, 1, 16, 0.8),
    (4000, 5, 100, 0, 8, 1.5),
    (1024, 2, 1, 0, 3, 1.5),
    (700, 4, 700, 0, 16, 1.5),   # N <= C_leaf: one dense leaf
]


@pytest.mark.parametrize("cfg", CONFIGS, ids=[str(c) for c in CONFIGS])
def test_oracle_equals_reference(oracle, reference, cfg):
    n, d, c_leaf, kern, k, eta = cfg
    P = uniform_points(n, d, 1234 + n)
    ho = oracle.setup(P, kernel=kern, c_leaf=c_leaf, k=k, eta=eta)
    hr = reference.setup(P, kernel=kern, c_leaf=c_leaf, k=k, eta=eta)
    co, po = ho.points()
    cr, pr = hr.points()
    assert np.array_equal(po, pr) and np.array_equal(bits(co), bits(cr))
    for w in (0, 1):
        lo, lr = ho.leaves(w), hr.leaves(w)
        assert np.array_equal(lo.rows, lr.rows)
        assert np.array_equal(bits(lo.boxes), bits(lr.boxes))
    fo, fr = ho.aca_all(), hr.aca_all()
    assert np.array_equal(fo["k_eff"], fr["k_eff"])
    assert np.array_equal(fo["row_piv"], fr["row_piv"])
    for a, b in zip(fo["u"], fr["u"]):
        assert np.array_equal(bits(a), bits(b))
    x = symmetric(99, n)
    assert np.array_equal(bits(ho.mvp(x)), bits(hr.mvp(x)))


def test_morton_codes_random(oracle, reference):
    for d in (1, 2, 3, 5, 7, 20):
        c = axis_major_points(400, d, 7 + d)
        assert np.array_equal(oracle.morton_codes(c), reference.morton_codes(c))


def test_row_sampled_product_equals_full(oracle, reference):
    """the row-sampled reconstruction equals mvp() bitwise."""
    n = 1 << 13
    P = uniform_points(n, 2, 42)
    hr = reference.setup(P, c_leaf=64, k=16)
    ho = oracle.setup(P, c_leaf=64, k=16)
    x = symmetric(7, n)
    _, perm = hr.points()
    z = hr.mvp(x)
    zm = np.empty(n)
    zm[np.arange(n)] = z[perm]
    ranges = [(0, 64), (1024, 1088), (5000, 5100), (8128, 8192)]
    zr = reference.setup(P, c_leaf=64, k=16).mvp_rows(x, ranges)
    zo = ho.mvp_rows(x, ranges)
    for lo, hi in ranges:
        assert np.array_equal(bits(zr[lo:hi]), bits(zm[lo:hi]))
        assert np.array_equal(bits(zo[lo:hi]), bits(zm[lo:hi]))


def test_f2_single_differs_from_batched(reference):
    """aca_single stops early on a sub-threshold column, aca_batched keeps
    scanning; the parity target is the batched semantics (what mvp() uses)."""
    n = 1 << 12
    P = uniform_points(n, 2, 42)
    h = reference.setup(P, c_leaf=64, k=16)
    lv = h.leaves(1, boxes=False).rows
    coords, _ = h.points()
    # materialise a handful of small admissible blocks
    blocks = []
    for (rl, ru, cl, cu) in lv[:40]:
        if ru - rl > 128:
            continue
        yi = coords[:, rl:ru]
        yj = coords[:, cl:cu]
        r2 = ((yi[:, :, None] - yj[:, None, :]) ** 2).sum(axis=0)
        blocks.append(np.exp(-r2))
    kb, _, _, _, _ = reference.aca_dense(blocks, 16, single=False)
    ks, _, _, _, _ = reference.aca_dense(blocks, 16, single=True)
    assert np.all(kb >= ks)


def test_f3_epsilon_inert_when_eta_above_one(oracle):
    """the eps criterion uses the admissibility eta; (1-eta) < 0 makes it inert."""
    n = 1 << 12
    P = uniform_points(n, 2, 42)
    x = symmetric(7, n)
    a = oracle.setup(P, c_leaf=64, k=16, epsilon=1e-6).mvp(x)
    b = oracle.setup(P, c_leaf=64, k=16).mvp(x)
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("cfg", CONFIGS[:4], ids=[str(c) for c in CONFIGS[:4]])
def test_reference_leaf_csv_is_the_merged_canonical_list(oracle, reference, cfg, tmp_path):
    """The reference's dump_leaves_csv (tree.cpp:197-205) lists exactly the oracle's dense and
    admissible leaves merged in canonical order -- the contract hm_dump_leaves_csv follows."""
    n, d, c_leaf, kern, k, eta = cfg
    P = uniform_points(n, d, 1234 + n)
    from oracle.bind import reference_leaf_csv
    path = tmp_path / "leaves.csv"
    reference_leaf_csv(P, c_leaf, eta, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "row_lower,row_upper,col_lower,col_upper,admissible"
    got = np.array([[int(v) for v in ln.split(",")] for ln in lines[1:]], dtype=np.int64).reshape(-1, 5)
    ho = oracle.setup(P, kernel=kern, c_leaf=c_leaf, k=k, eta=eta)
    rows = np.concatenate([ho.leaves(0, boxes=False).rows, ho.leaves(1, boxes=False).rows])
    flags = np.concatenate([np.zeros(ho.count(0), np.int64), np.ones(ho.count(1), np.int64)])
    order = np.lexsort((rows[:, 3], rows[:, 2], rows[:, 1], rows[:, 0]))
    want = np.column_stack([rows[order], flags[order]])
    assert np.array_equal(got, want)


def test_reference_leaf_sample_driver_equals_reference_mvp(reference, tmp_path):
    """The recompute-mode CPU baseline (ref_leaves_mvp_timed, bench.py) runs the
    reference's own mvp() body over an explicit leaf list: with every leaf of a reference
    setup it reproduces the reference's product bitwise (Morton order)."""
    import subprocess
    import sys
    from paper_1708_09707_b200.inputs import symmetric, uniform_points
    n, d = 3000, 3
    P = uniform_points(n, d, 42)
    h = reference.setup(P, kernel=1, c_leaf=48, k=12)
    coords, perm = h.points()
    x = symmetric(5, n)
    z = h.mvp(x)
    f = tmp_path / "leaves.npz"
    np.savez(f, coords=coords, dense=h.leaves(0, boxes=False).rows, aca=h.leaves(1, boxes=False).rows,
             x=x[perm], kernel=1, k=12, eta=1.5)
    import ctypes as C
    L = reference.lib
    L.ref_leaves_mvp_timed.restype = C.c_int
    L.ref_leaves_mvp_timed.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_double,
                                       C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                       C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    dense = np.ascontiguousarray(h.leaves(0, boxes=False).rows, dtype=np.int64)
    aca = np.ascontiguousarray(h.leaves(1, boxes=False).rows, dtype=np.int64)
    xm = np.ascontiguousarray(x[perm])
    zm = np.zeros(n)
    tm, fl = C.c_double(), C.c_double()
    assert L.ref_leaves_mvp_timed(coords.ctypes.data, n, d, 1, 0.0, 12, 1.5, dense.shape[0], dense.ctypes.data,
                                  aca.shape[0], aca.ctypes.data, xm.ctypes.data, 1, zm.ctypes.data, C.byref(tm),
                                  C.byref(fl)) == 0
    assert np.array_equal(zm.view(np.uint64), z[perm].view(np.uint64))
    out = subprocess.run([sys.executable, "-m", "oracle.refbench", "--leaves", str(f), "--reps", "1"],
                         capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr


def test_reference_row_sample_driver_equals_reference_mvp(reference):
    """The stored-mode reference arm (ref_mvp_rows_timed, oracle/refbench.py) reproduces
    the reference's own product on the sampled row clusters bitwise (Morton order), with
    the O(N) permutation hoisted out of the reps and charged pro rata."""
    import ctypes as C
    from oracle.refbench import cluster_ranges, leaf_depth
    n, d, c_leaf = 4096, 2, 32
    P = uniform_points(n, d, 42)
    h = reference.setup(P, kernel=0, c_leaf=c_leaf, k=12)
    _, perm = h.points()
    x = symmetric(9, n)
    want = h.mvp(x)[perm]
    L = reference.lib
    L.ref_mvp_rows_timed.restype = C.c_int
    L.ref_mvp_rows_timed.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    ranges = np.array(cluster_ranges(n, leaf_depth(n, c_leaf), [0, 5, 77]), dtype=np.int64)
    z = np.full(n, np.nan)
    ta, tm, fl = C.c_double(), C.c_double(), C.c_double()
    assert L.ref_mvp_rows_timed(h.h, x.ctypes.data, ranges.shape[0], ranges.ctypes.data, 2, z.ctypes.data,
                                C.byref(ta), C.byref(tm), C.byref(fl)) == 0
    assert tm.value > 0.0 and fl.value > 0.0
    for lo, hi in ranges:
        assert np.array_equal(z[lo:hi].view(np.uint64), want[lo:hi].view(np.uint64))
